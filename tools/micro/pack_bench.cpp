// Host packing throughput (gp_pack.cpp) on BB72 branch circuits, no GPU:
// pack_plan + pack_range + pack_finish + pack_head into a host image, timed
// per phase. Build: see tools/micro/Makefile (links libgreenpeas.so for the
// generator only).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/greenpeas.h"
#include "../../paper_2604_16613_b200/csrc/gp_pack.h"

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main(int argc, char **argv) {
    const int C = argc > 1 ? std::atoi(argv[1]) : 4096;
    const unsigned threads = argc > 2 ? (unsigned)std::atoi(argv[2]) : std::thread::hardware_concurrency();
    const int reps = argc > 3 ? std::atoi(argv[3]) : 5;
    const uint32_t a[3] = {3, 1, 2}, b[3] = {3, 1, 2};
    std::vector<gp_circuit *> hs(C);
    std::vector<gp_circuit_view> vs(C);
    for (int c = 0; c < C; c++) {
        hs[c] = gp_gen_bb(6, 6, a, b, 6, 1e-3, 0, 0.5, 3, 1, (uint64_t)c);
        vs[c] = gp_circuit_get_view(hs[c]);
    }
    gp::HostPool pool(threads > 1 ? threads - 1 : 0);
    gp::PackPlan pp;
    std::vector<uint8_t> img;
    uint64_t ops = 0;
    for (auto &v : vs) ops += (v.gate_offsets[v.num_layers] - v.gate_offsets[0]) + (v.noise_offsets[v.num_layers] - v.noise_offsets[0]);
    for (int r = 0; r < reps; r++) {
        const auto t0 = clk::now();
        gp::pack_plan(&pool, vs.data(), C, 0, pp);
        const auto t1 = clk::now();
        if (img.size() < pp.L.total) img.resize(pp.L.total);
        const auto t2 = clk::now();
        gp::pack_range(&pool, vs.data(), pp, img.data(), 0, C);
        const auto t3 = clk::now();
        gp::pack_finish(pp, img.data());
        gp::pack_head(pp, 8, img.data());
        const auto t4 = clk::now();
        std::printf("C=%d threads=%u image=%.1f MB ops=%.1f M  plan %.2f  range %.2f  finish+head %.2f  total %.2f ms (%.0f Mops/s)\n",
                    C, threads, pp.L.total / 1e6, ops / 1e6, ms(t0, t1), ms(t2, t3), ms(t3, t4), ms(t0, t4) - ms(t1, t2),
                    ops / 1e3 / (ms(t0, t4) - ms(t1, t2)));
    }
    for (auto h : hs) gp_circuit_free(h);
}
