# Round profile refresh on the GPU box (developer tool): bench line, ncu launch list, ncu --set full summary and
# per-stage DRAM traffic of the bench workload, written to gpurun_out/ (copy the summaries to profiles/).
# usage: bash tools/prof_round.sh v4
set -x
mkdir -p gpurun_out
V=$1
python bench.py > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_$V.csv > gpurun_out/launches_$V.txt
ncu --set full --clock-control none -k regex:"lower_kernel|traverse_kernel|bucket_kernel|write_kernel|zero_kernel" -c 10 -o /tmp/full_$V python tools/fast_repro.py 4096 0 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/full_$V.ncu-rep > gpurun_out/ncu_full_batch4096_$V.txt
python tools/traffic.py /tmp/full_$V.ncu-rep gpurun_out/traffic_$V.json
ls -la gpurun_out
