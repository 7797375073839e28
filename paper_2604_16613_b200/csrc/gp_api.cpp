// gp_api.cpp -- C ABI (include/greenpeas.h) of the B200 DEM compiler.
//
// gp_compile / gp_compile_batch replace demc::compile_circuit
// (/root/reference/proj/core/src/compile.cpp:23-53). The host side does only
// what cannot run on the GPU: it validates the reference's error conditions,
// packs the flat circuit view into one pinned staging image (compact 8/16-byte
// op words), uploads it with one async copy, enqueues the device pipeline
// (gp_kernels.cu) and downloads the flat DEM into context-owned pinned memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <mutex>
#include <thread>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/greenpeas.h"
#include "gp_device.h"
#include "gp_layout.h"
#include "gp_gen.h"
#include "gp_pack.h"

using gp::BatchTotals;
using gp::CircuitMeta;
using gp::DevPlan;
using gp::DeviceHeader;
using gp::StageLayout;

namespace gp {
struct PipeState;
void pipe_destroy(PipeState *ps);
}  // namespace gp

struct gp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::function<void()> overlap;  // host work of the caller, run once while a compile's kernels run
    std::string err;
    int force_collisions = 0;
    uint32_t trav_debug = 0;
    uint32_t record_slots = 8;
    uint64_t ids_hint = 0;  // learned id capacity (grows on overflow)
    uint64_t pool_hint = 0; // learned record-pool chunks (grows on overflow)
    uint64_t items_hint = 0; // learned reduce item capacity (grows on overflow)

    uint8_t *h_stage = nullptr;
    size_t h_stage_cap = 0;
    uint8_t *d_img = nullptr;
    size_t d_img_cap = 0;
    uint8_t *d_ws = nullptr;
    size_t d_ws_cap = 0;
    uint8_t *h_out = nullptr;
    size_t h_out_cap = 0;
    uint8_t *h_map = nullptr;  // mapped pinned output of small compiles (copy_out_kernel)
    size_t h_map_cap = 0;
    DeviceHeader *h_hdr = nullptr;

    cudaEvent_t ev_start = nullptr, ev_h2d = nullptr, ev_end = nullptr;
    gp::StageEvents stage_ev{};

    gp::PackPlan pack;
    std::vector<uint32_t> out_ndet, out_nobs;

    // Last successful device plan (for gp_replay) and profiling state.
    bool has_plan = false;
    DevPlan last_plan{};
    cudaEvent_t prof[gp::kProfCount] = {};
    uint64_t prof_ns[gp::kProfCount] = {};
    uint8_t *d_flush = nullptr;
    uint64_t *d_dbg = nullptr;  // experiments only (option 99, bit 2)
    uint64_t *d_bases = nullptr;  // [8] zero bases in / scratch bases out (unpipelined compiles)
    uint8_t *d_merge = nullptr;   // gp_merge_partials: the parts' tables, concatenated
    size_t d_merge_cap = 0;
    int pipeline = -1;            // GP_OPT_PIPELINE: -1 auto, 0 off, 1 on
    // CUDA graph of the device pipeline, keyed by the launch plan's bytes: a
    // plan seen twice in a row is captured once and then relaunched as one
    // graph (repeated compiles of one circuit shape: the JIT case).
    struct {
        uint64_t key = 0, pending = 0;
        gp::DevPlan plan{};  // the plan the graph was captured from (a key hit must match it byte for byte)
        cudaGraphExec_t exec = nullptr;
        int launches = 0;
        bool used = false;  // the last compile ran as the graph (no per-stage events)
    } graph;
    gp::PipeState *pipe = nullptr;
    // Device branch generation (gp_compile_bb_branches): the spec's template
    // (host + device copies), per-branch check masks and counts.
    struct {
        gp_bb_spec spec{};
        bool valid = false;
        gp::BBTemplate t;
        uint32_t *d_tmpl = nullptr;  // xdata | zdata | zfinal | obs_off | obs_q
        size_t d_tmpl_cap = 0;
        uint64_t *d_masks = nullptr;
        size_t d_masks_cap = 0;
        uint32_t *d_counts = nullptr, *h_counts = nullptr, *d_err = nullptr, *h_err = nullptr;
        size_t counts_cap = 0;
    } bb;
    uint32_t bb_pi[5] = {};  // probability-table index per generator channel (last plan)
};

namespace {

using clk = std::chrono::steady_clock;

uint64_t ns_since(clk::time_point t0) {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
}

uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }

// One host worker pool per process, shared by every context. A compile leases
// it for its packing when it is free; when another context holds it (many
// host threads compiling at once, the demc_main.cpp:184-195 pattern) the
// caller packs on its own thread instead -- the callers already are the
// parallelism, and no context ever starts a pool of its own.
std::mutex g_pool_mu;

gp::HostPool *shared_pool() {
    static std::once_flag once;
    static std::unique_ptr<gp::HostPool> pool;
    std::call_once(once, [] {
        pool = std::make_unique<gp::HostPool>(std::max(1u, std::thread::hardware_concurrency()) - 1);
    });
    return pool.get();
}

struct PoolLease {
    gp::HostPool *pool = nullptr;
    explicit PoolLease(bool want) {
        if (want && g_pool_mu.try_lock()) pool = shared_pool();
    }
    ~PoolLease() { release(); }
    void release() {
        if (pool) g_pool_mu.unlock();
        pool = nullptr;
    }
    PoolLease(const PoolLease &) = delete;
    PoolLease &operator=(const PoolLease &) = delete;
};

gp_status fail(gp_ctx *ctx, gp_status st, const std::string &msg) {
    ctx->err = msg;
    return st;
}

}  // namespace

namespace gp {
// Host tasks [0, n) on the shared pool when it is free (else on the caller):
// the C++ drop-in's circuit flattening and demc::Dem materialisation.
// Drop-in shim (demc_shim.cpp): host work to run while the next gp_compile's
// kernels run (cleared by passing nullptr; runs at most once).
void set_compile_overlap(gp_ctx *ctx, std::function<void()> f) { ctx->overlap = std::move(f); }

void host_parallel_for(size_t n, const std::function<void(size_t)> &f) {
    PoolLease lease(n > 1);
    if (lease.pool) lease.pool->run(n, f);
    else
        for (size_t i = 0; i < n; i++) f(i);
}
}  // namespace gp

namespace {

gp_status cuda_fail(gp_ctx *ctx, cudaError_t e, const char *what) {
    return fail(ctx, GP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}


uint32_t components(uint8_t kind, uint8_t level) {  // stepg.cpp:66-103
    if (kind <= GP_NOISE_Z_ERROR) return 1;
    if (kind == GP_NOISE_DEPOLARIZE1) return level == 0 ? 2 : 3;
    return level == 0 ? 6 : level == 1 ? 10 : 15;
}

// Device workspace carve-up for a batch (capacity-checked, grown on demand).
struct WsPlan {
    size_t bytes = 0;
    uint64_t table_cap = 0, bsum_cap = 0, ids_cap = 0;
    struct Slot {
        void **dst;
        size_t bytes;
    };
};

// Output region of a compile (gp_device.h): global-offset DEM arrays plus
// the final header copy.
size_t carve_out(DevPlan &p, uint8_t *base, uint64_t e_cap, uint64_t ids_cap, uint64_t C) {
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes + 16);
        return base ? base + at : nullptr;
    };
    p.e_cap = e_cap;
    p.o_det_off = (uint32_t *)take(e_cap * 4 + 4);
    p.o_obs_off = (uint32_t *)take(e_cap * 4 + 4);
    p.o_prob = (double *)take(e_cap * 8);
    p.o_det = (uint32_t *)take(ids_cap * 4);
    p.o_obs = (uint32_t *)take(ids_cap * 4);
    p.o_edge_off = (uint64_t *)take((C + 1) * 8);
    p.hdr_out = (DeviceHeader *)take(sizeof(DeviceHeader));
    return o;
}

size_t carve(gp_ctx *ctx, DevPlan &p, const BatchTotals &t, uint8_t *base, uint32_t K, uint64_t ids_cap,
             uint64_t pool_chunks, uint64_t slabs, uint64_t items_cap, bool with_out) {
    const uint64_t S = t.sources, NB = t.buckets;
    const uint64_t nb = std::max<uint64_t>(S, NB + 1) / 2048 + 16;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes + 16);
        return base ? base + at : nullptr;
    };
    p.ell = (uint32_t *)take(t.ell * 4);
    p.leaf = (uint64_t *)take(t.leaf * 8);
    p.prob = (double *)take(S * 8);
    p.nsrc = (uint32_t *)take(t.noise * 4 + 16);
    p.noise_w = t.narrow ? (uint64_t *)take(t.noise * 8) : nullptr;  // widened by lower_kernel
    p.cnt = (uint32_t *)take(S * 4 + 4);
    p.rbits = (uint64_t *)take(S * K * 8);
    p.rtile = (uint32_t *)take(S * K * 4);
    p.K = K;
    p.pool = (uint4 *)take(pool_chunks * gp::kPoolChunk * 16);
    p.pool_chunks_cap = (uint32_t)pool_chunks;
    p.slab_words = (2 * t.max_n + 1) & ~1u;
    p.slab_stride = slabs ? t.max_l : 0;
    p.slab = (uint64_t *)take(slabs * p.slab_words * 8);
    p.slab_hdr = (uint4 *)take(slabs * 16);
    p.s_bkt = (uint32_t *)take(S * 4);
    p.s_pos = (uint32_t *)take(S * 4);
    p.force_collisions = ctx->force_collisions;
    p.bcount = (uint32_t *)take(NB * 4 + 4);
    p.boff = (uint4 *)take((NB + 1) * 16);
    // Fused items: positions are circuit regions of S slots (every source may emit).
    p.fused = p.trav.fuse_key && !p.trav.split && p.mode == gp::kModeFull;
    const uint64_t icap = p.fused ? S + 16 : items_cap;
    p.items = (DevPlan::ItemStub *)take(icap * sizeof(DevPlan::ItemStub));
    p.items_cap = icap;
    p.ecount = (uint32_t *)take(NB * 4);
    p.eids = (uint2 *)take(NB * 8);
    p.oscan = (uint4 *)take((NB + 1) * 16);
    p.e_ndno = (uint32_t *)take(icap * 4);
    p.e_item = (uint32_t *)take(icap * 4);
    p.e_prob = (double *)take(icap * 8);
    p.huge = (uint32_t *)take(NB * 4);
    if (p.fused) {
        // items moved into bucket order (contiguous runs for the bucket warps)
        // unless GP_FUSED_MOVE=0 (index lists; measured 0.45 ms slower per
        // 4,096 branches in the bucket stage)
        const char *mv = std::getenv("GP_FUSED_MOVE");
        p.fused_move = mv ? (uint32_t)std::atoi(mv) : 1;
        p.items2 = (DevPlan::ItemStub *)take(icap * sizeof(DevPlan::ItemStub));
        p.ibkt = (uint16_t *)take(S * 2);
        p.iidx = (uint32_t *)take(S * 4);
        p.ptab3 = (double *)take((size_t)t.prob_table_n * 32 + 32);
    }
    if (p.mode == gp::kModeShard) {  // compact partial table of the shard
        p.p_prob = (double *)take(S * 8);
        p.p_roff = (uint32_t *)take(S * 4 + 4);
        p.p_word = (uint32_t *)take(S * K * 4);
        p.p_bits = (uint64_t *)take(S * K * 8);
        p.p_scan = (uint4 *)take(S * 16 + 16);
    }
    p.ids_cap = ids_cap;
    p.bsum = (uint4 *)take(nb * 16);
    p.bsum_cap = nb;
    p.hdr = (DeviceHeader *)take(sizeof(DeviceHeader));
    if (with_out) {  // the output region at the end of the workspace
        const size_t bytes = carve_out(p, nullptr, items_cap, ids_cap, t.C);
        uint8_t *ob = (uint8_t *)take(bytes);
        carve_out(p, ob, items_cap, ids_cap, t.C);
    }
    return o;
}

gp_status ensure_device(gp_ctx *ctx, uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    size_t want = need + need / 4;
    cudaError_t e = cudaMalloc(buf, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(buf, need);
        want = need;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "device allocation of " + std::to_string(need) + " bytes failed");
    }
    *cap = want;
    return GP_OK;
}

gp_status ensure_host(gp_ctx *ctx, uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t want = need + need / 4 + 4096;
    if (cudaMallocHost(buf, want) != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "pinned host allocation of " + std::to_string(want) + " bytes failed");
    }
    *cap = want;
    return GP_OK;
}

// The reference's exception texts (stepg.cpp:172-174, eec.cpp:45,53).
gp_status fail_pack(gp_ctx *ctx, int err) {
    static const char *kErr[] = {"", "circuit exceeds 32-bit node index space",
                                 "detector references a measurement without a leaf",
                                 "observable references a measurement without a leaf",
                                 "circuit too wide for the device encoding"};
    return fail(ctx, err == gp::kPackTooWide ? GP_ERR_UNSUPPORTED : GP_ERR_INVALID_ARGUMENT, kErr[err]);
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return ms;
}

struct HostOut {
    uint32_t *det_off, *obs_off;
    uint64_t *edge_off;
    double *probs;
    uint32_t *det_ids, *obs_ids;
};

uint64_t plan_key(const DevPlan &p) {
    const unsigned char *b = reinterpret_cast<const unsigned char *>(&p);
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < sizeof(DevPlan); i++) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}

// Enqueues the device pipeline of plan p: directly, or as the cached graph
// when the same plan was launched just before (see gp_ctx::graph).
int launch_pipeline(gp_ctx *ctx, const DevPlan &p, cudaError_t *e) {
    auto &g = ctx->graph;
    const uint64_t key = p.dbg ? 0 : plan_key(p);
    g.used = false;
    if (key && g.exec && g.key == key && std::memcmp(&g.plan, &p, sizeof(DevPlan)) == 0) {
        *e = cudaGraphLaunch(g.exec, ctx->stream);
        cudaEventRecord(ctx->stage_ev.reduced, ctx->stream);  // stage events are not recorded inside the graph
        g.used = true;
        return g.launches;
    }
    if (!key || g.pending != key) {
        g.pending = key;
        return gp::enqueue_pipeline(p, ctx->stream, &ctx->stage_ev, nullptr, e);
    }
    cudaGraph_t graph = nullptr;
    *e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (*e != cudaSuccess) return 0;
    cudaError_t le = cudaSuccess;
    const int n = gp::enqueue_pipeline(p, ctx->stream, nullptr, nullptr, &le);
    *e = cudaStreamEndCapture(ctx->stream, &graph);
    if (*e == cudaSuccess && le != cudaSuccess) *e = le;
    if (*e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return 0;
    }
    bool updated = false;
    if (g.exec) {
        cudaGraphExecUpdateResultInfo info;
        updated = cudaGraphExecUpdate(g.exec, graph, &info) == cudaSuccess;
        if (!updated) {
            cudaGetLastError();
            cudaGraphExecDestroy(g.exec);
            g.exec = nullptr;
        }
    }
    if (!updated) *e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (*e != cudaSuccess) {
        g.exec = nullptr;
        g.key = 0;
        return 0;
    }
    g.key = key;
    g.plan = p;
    g.launches = n;
    *e = cudaGraphLaunch(g.exec, ctx->stream);
    cudaEventRecord(ctx->stage_ev.reduced, ctx->stream);
    g.used = true;
    return n;
}

// Partial table of a shard compile (gp_compile_shard), in ctx-owned pinned memory.
struct PartialOut {
    bool on_device = false;  // in: leave the table in device memory
    uint64_t n = 0, r = 0;
    double *prob = nullptr;
    uint32_t *roff = nullptr, *word = nullptr;
    uint64_t *bits = nullptr;
};

// Device-generated batch (gp_compile_bb_branches): the branches' first id.
struct BBGenReq {
    uint64_t first;
};
gp_status bbgen_draw(gp_ctx *ctx, const BBGenReq &req, size_t count, uint8_t level);
gp_status bbgen_plan(gp_ctx *ctx, size_t c0, size_t count, uint8_t level, gp::PackPlan &pp, uint32_t *pi_out);
gp_status bbgen_fill(gp_ctx *ctx, const BBGenReq &req, size_t c0, uint8_t level, const gp::PackPlan &pp,
                     const uint32_t *pi, uint8_t *img, cudaStream_t st);

gp_status run_batch(gp_ctx *ctx, const gp_circuit_view *cs, size_t count, uint8_t level, HostOut &ho,
                    DeviceHeader &hdr, gp_stats *stats, uint32_t mode = gp::kModeFull, uint32_t sh_lo = 0,
                    uint32_t sh_hi = 0xFFFFFFFFu, PartialOut *part = nullptr, const BBGenReq *gen = nullptr) {
    const auto t0 = clk::now();
    if (level > 2) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "correlation level must be 0, 1 or 2");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GP_ERR_CUDA, "cudaSetDevice failed");
    gp_status st = GP_OK;
    gp::PackPlan &pp = ctx->pack;
    // Host pool for large jobs (single large circuits pack on every core too).
    uint64_t ops = 0;
    for (size_t c = 0; !gen && c < count; c++)
        ops += (uint64_t)(cs[c].gate_offsets[cs[c].num_layers] - cs[c].gate_offsets[0]) +
               (cs[c].noise_offsets[cs[c].num_layers] - cs[c].noise_offsets[0]);
    PoolLease lease(ops >= (1u << 14));
    gp::HostPool *hpool = lease.pool;
    pp.force_wide = false;
    pp.no_narrow = false;
    cudaError_t e = cudaSuccess;
    const std::vector<CircuitMeta> &M = pp.metas;
    const size_t nchunk = gen ? 1 : count >= 1024 ? 8 : count >= 256 ? 4 : 1;
    auto slice = [&](uint64_t off, uint64_t elem, uint64_t lo, uint64_t hi) {
        if (hi > lo && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->d_img + off + lo * elem, ctx->h_stage + off + lo * elem, (hi - lo) * elem,
                                cudaMemcpyHostToDevice, ctx->stream);
    };
    if (gen) {  // device generation: plan the image from the drawn counts (no host circuits)
        cudaEventRecord(ctx->ev_start, ctx->stream);
        if ((st = bbgen_draw(ctx, *gen, count, level)) != GP_OK) return st;
        if ((st = bbgen_plan(ctx, 0, count, level, pp, ctx->bb_pi)) != GP_OK) return st;
        if ((st = ensure_host(ctx, &ctx->h_stage, &ctx->h_stage_cap, pp.L.total)) != GP_OK) return st;
        if ((st = ensure_device(ctx, &ctx->d_img, &ctx->d_img_cap, pp.L.total)) != GP_OK) return st;
    } else {
repack:  // (again with per-op probabilities when the table overflowed)
    gp::pack_plan(hpool, cs, count, level, pp);
    if (pp.err == gp::kPackIndexSpace || pp.err == gp::kPackTooWide) {
        // Circuits before the first index-space failure may still hold leaf
        // errors: the reference would have thrown on those first.
        const int leaf_err = gp::validate_leaves(cs, 0, pp.err_circuit);
        return fail_pack(ctx, leaf_err ? leaf_err : pp.err);
    }
    const StageLayout &L = pp.L;
    if ((st = ensure_host(ctx, &ctx->h_stage, &ctx->h_stage_cap, L.total)) != GP_OK) return st;
    if ((st = ensure_device(ctx, &ctx->d_img, &ctx->d_img_cap, L.total)) != GP_OK) return st;

    // Pack in circuit chunks; each chunk's slice of every section is copied
    // while the next chunk is packed (the image is circuit-major per section).
    // One chunk (one copy of the whole image) for single circuits.
    cudaEventRecord(ctx->ev_start, ctx->stream);
    for (size_t k = 0; k < nchunk; k++) {
        const size_t c0 = count * k / nchunk, c1 = count * (k + 1) / nchunk;
        if (c1 == c0) continue;
        gp::pack_range(hpool, cs, pp, ctx->h_stage, c0, c1);
        if (nchunk == 1) break;
        const CircuitMeta &a = M[c0];
        const bool last = c1 == count;
        const CircuitMeta *b = last ? nullptr : &M[c1];
        const BatchTotals &tt = pp.t;
        slice(L.lay_gate, 4, a.layer_base, last ? tt.layer_slots : b->layer_base);
        slice(L.lay_noise, 4, a.layer_base, last ? tt.layer_slots : b->layer_base);
        slice(L.gates, tt.narrow ? 4 : 8, a.gate_base, last ? tt.gates : b->gate_base);
        slice(L.noise, tt.narrow ? 4 : 8, a.noise_base, last ? tt.noise : b->noise_base);
        if (tt.wide_prob) slice(L.noise_prob, 8, a.noise_base, last ? tt.noise : b->noise_base);
        slice(L.meas_flip, 8, a.meas_base, last ? tt.meas : b->meas_base);
        slice(L.det_off, 4, a.det_base, last ? tt.det_slots : b->det_base);
        slice(L.det_meas, 4, a.det_entry_base, last ? tt.det_entries : b->det_entry_base);
        slice(L.obs_off, 4, a.obs_base, last ? tt.obs_slots : b->obs_base);
        slice(L.obs_meas, 4, a.obs_entry_base, last ? tt.obs_entries : b->obs_entry_base);
    }
    if (pp.err) return fail_pack(ctx, pp.err);
    if ((pp.need_wide.load() && !pp.force_wide) || (pp.need_wide_words.load() && !pp.no_narrow)) {
        cudaStreamSynchronize(ctx->stream);  // chunk uploads read the staging image
        if (pp.need_wide.load()) pp.force_wide = true;
        pp.no_narrow = true;
        goto repack;
    }
    gp::pack_finish(pp, ctx->h_stage);
    }  // (host packing)
    const StageLayout &L = pp.L;
    BatchTotals t = pp.t;
    if (t.sources >= 0xFFFFFFFFull || t.tiles >= 0xFFFFFFFFull || t.gates >= 0xFFFFFFFFull ||
        t.noise >= 0xFFFFFFFFull || t.meas >= 0xFFFFFFFFull || t.layer_slots >= 0xFFFFFFFFull)
        return fail(ctx, GP_ERR_UNSUPPORTED, "batch exceeds 32-bit device indexing; split it");
    gp::TravCfg tcfg;
    size_t tsmem;
    if (!gp::plan_traversal(t, ctx->device, &tcfg, &tsmem))
        return fail(ctx, GP_ERR_UNSUPPORTED, "circuit too wide for on-chip traversal state (2n words)");
    if (mode == gp::kModeShard && !tcfg.split)  // (the layer filters live in the split walk / emission)
        return fail(ctx, GP_ERR_UNSUPPORTED, "fault-range shards need the single-circuit (split) traversal");
    t.groups = 0;
    for (const CircuitMeta &m : M) t.groups += (m.W + tcfg.T - 1) / tcfg.T;
    gp::pack_head(pp, tcfg.T, ctx->h_stage);
    // One small circuit (D + O <= 64) compiles in one CTA (gp_tiny.cuh) that
    // reads its image in place from the pinned staging memory (zero copy: no
    // upload) and writes the mapped output: one launch, no copies.
    uint32_t tiny_cap = 0;
    size_t tiny_smem = 0;
    if (mode == gp::kModeFull && count == 1 && !gen && !ctx->force_collisions && t.max_W <= 1 && t.max_l >= 1 &&
        t.sources <= 8192 && !std::getenv("GP_NO_TINY")) {
        uint32_t cap = 32;
        while (cap < t.sources) cap <<= 1;
        const size_t b = gp::tiny_smem_bytes(t, M[0], cap);
        if (b <= (size_t)200 * 1024) {
            tiny_cap = cap;
            tiny_smem = b;
        }
    }
    bool uploaded = !tiny_cap;
    if (gen) {  // the head (metas, cumulative tables) and the probability table; the rest on the device
        slice(0, 1, 0, L.lay_gate);
        slice(L.prob_table, 8, 0, t.prob_table_n);
        if (e == cudaSuccess && (st = bbgen_fill(ctx, *gen, 0, level, pp, ctx->bb_pi, ctx->d_img, ctx->stream)) != GP_OK)
            return st;
        cudaMemcpyAsync(ctx->bb.h_err, ctx->bb.d_err, 4, cudaMemcpyDeviceToHost, ctx->stream);
    } else if (nchunk == 1) {
        if (uploaded) slice(0, 1, 0, pp.image_bytes());  // the whole image in one copy
    } else {
        slice(L.lay_meas, 4, 0, t.layer_slots);  // finished prefix tables
        slice(L.lay_src, 4, 0, t.layer_slots);
        slice(0, 1, 0, L.lay_gate);  // meta + cumulative tables (the image's head)
        slice(L.prob_table, 8, 0, t.prob_table_n);
    }
    lease.release();  // packing done: the pool is free for other contexts
    const uint64_t pack_ns = ns_since(t0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "upload");
    cudaEventRecord(ctx->ev_h2d, ctx->stream);

    // One CTA owning all T words of a source writes at most T records.
    uint32_t K = tcfg.direct ? std::max<uint32_t>(ctx->record_slots, tcfg.T) : ctx->record_slots;
    // Multi-CTA circuits (one word per CTA) emit through the record pool.
    uint64_t pool = 0;
    if (!tcfg.direct && !tcfg.split)
        pool = std::max<uint64_t>(ctx->pool_hint,
                                  (2 * t.sources) / gp::kPoolChunk + t.groups * tcfg.emit_warps + 16);
    // Split traversal: walker CTA g owns max_l slabs (one per boundary it may walk).
    const uint64_t slabs = tcfg.split ? t.groups * t.max_l : 0;
    uint64_t ids_cap = std::max<uint64_t>(ctx->ids_hint, 3 * t.sources + 1024);
    // Items: one per nonempty signature. All sources fit for single circuits;
    // large batches start from half (and learn the real count on overflow).
    uint64_t items_cap = std::max<uint64_t>(ctx->items_hint,
                                            t.sources <= (16u << 20) ? t.sources + 16 : t.sources / 2 + 16);
    DevPlan p{};
    int launches = 0;
    for (int attempt = 0;; attempt++) {
        p = DevPlan{};
        p.img = ctx->d_img;
        p.lay = L;
        p.tot = t;
        p.trav = tcfg;
        p.trav.debug = ctx->trav_debug;
        p.trav_smem = tsmem;
        p.mode = mode;
        p.shard_lo = sh_lo;
        p.shard_hi = sh_hi;
        const size_t need = carve(ctx, p, t, nullptr, K, ids_cap, pool, slabs, items_cap, true);
        if ((st = ensure_device(ctx, &ctx->d_ws, &ctx->d_ws_cap, need)) != GP_OK) return st;
        carve(ctx, p, t, ctx->d_ws, K, ids_cap, pool, slabs, items_cap, true);
        p.base_in = ctx->d_bases;
        p.base_out = ctx->d_bases + 4;
        // Small outputs go straight to mapped host memory (one wait, no round trip).
        {
            size_t mo = 0;
            auto mtake = [&](size_t bytes) {
                const size_t at = mo;
                mo = (size_t)align16(mo + bytes);
                return at;
            };
            const size_t m_hdr = mtake(sizeof(DeviceHeader)), m_det_off = mtake((p.e_cap + 1) * 4),
                         m_obs_off = mtake((p.e_cap + 1) * 4), m_prob = mtake(p.e_cap * 8),
                         m_det = mtake(p.ids_cap * 4), m_obs = mtake(p.ids_cap * 4), m_edge = mtake((t.C + 1) * 8);
            p.out_mapped = mode == gp::kModeFull && mo <= (size_t(128) << 20);
            if (p.out_mapped && ctx->h_map_cap < mo) {
                if (ctx->h_map) cudaFreeHost(ctx->h_map);
                ctx->h_map = nullptr;
                ctx->h_map_cap = 0;
                if (cudaHostAlloc(&ctx->h_map, mo + mo / 4, cudaHostAllocMapped) == cudaSuccess) {
                    ctx->h_map_cap = mo + mo / 4;
                } else {
                    cudaGetLastError();
                    p.out_mapped = 0;
                }
            }
            if (p.out_mapped) {
                p.hmap.hdr = (DeviceHeader *)(ctx->h_map + m_hdr);
                p.hmap.det_off = (uint32_t *)(ctx->h_map + m_det_off);
                p.hmap.obs_off = (uint32_t *)(ctx->h_map + m_obs_off);
                p.hmap.probs = (double *)(ctx->h_map + m_prob);
                p.hmap.det_ids = (uint32_t *)(ctx->h_map + m_det);
                p.hmap.obs_ids = (uint32_t *)(ctx->h_map + m_obs);
                p.hmap.edge_off = (uint64_t *)(ctx->h_map + m_edge);
            }
        }
        p.tiny = 0;
        if (tiny_cap && p.out_mapped) {
            p.tiny = 1;
            p.tiny_cap = tiny_cap;
            p.tiny_smem = tiny_smem;
            p.tiny_meta = M[0];
            p.img = ctx->h_stage;  // pinned host memory, read in place (unified addressing)
        } else if (!uploaded) {  // (no mapped output after all: the general pipeline, after the upload)
            e = cudaMemcpyAsync(ctx->d_img, ctx->h_stage, pp.image_bytes(), cudaMemcpyHostToDevice, ctx->stream);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "upload");
            uploaded = true;
        }
        if (ctx->trav_debug & 4) {  // experiments: per-step walk timestamps of every CTA
            if (!ctx->d_dbg) cudaMalloc(&ctx->d_dbg, (size_t)8192 * 512 * 4 * 8);
            cudaMemsetAsync(ctx->d_dbg, 0, (size_t)8192 * 512 * 4 * 8, ctx->stream);
            p.dbg = t.groups <= 8192 || p.tiny ? ctx->d_dbg : nullptr;
        }
        static const bool lat = std::getenv("GP_LAT_TRACE") != nullptr;  // experiments: host phase times
        const uint64_t t_pre = lat ? ns_since(t0) : 0;
        launches += launch_pipeline(ctx, p, &e);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
        if (!p.out_mapped)
            e = cudaMemcpyAsync(ctx->h_hdr, p.hdr, sizeof(DeviceHeader), cudaMemcpyDeviceToHost, ctx->stream);
        cudaEventRecord(ctx->ev_end, ctx->stream);
        const uint64_t t_launch = lat ? ns_since(t0) : 0;
        if (ctx->overlap) {  // the caller's host work, instead of idling in the synchronize
            const std::function<void()> f = std::move(ctx->overlap);
            ctx->overlap = nullptr;
            f();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (lat)
            std::fprintf(stderr, "lat: pack %.1f  carve+plan %.1f  launch %.1f  sync %.1f us\n", pack_ns / 1e3,
                         (t_pre - pack_ns) / 1e3, (t_launch - t_pre) / 1e3, (ns_since(t0) - t_launch) / 1e3);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "device pipeline");
        hdr = p.out_mapped ? *p.hmap.hdr : *ctx->h_hdr;
        const bool retry = hdr.items_overflow || hdr.pool_overflow || hdr.record_overflow ||
                           hdr.num_det_ids == 0xFFFFFFFFu;
        if (retry && attempt >= 5) return fail(ctx, GP_ERR_CUDA, "capacity retry loop did not converge");
        if (hdr.items_overflow) {  // more nonempty signatures than items: use every source
            items_cap = t.sources + 16;
            ctx->items_hint = items_cap;
            continue;
        }
        if (hdr.pool_overflow) {  // the record pool was too small
            pool = 2 * std::max<uint64_t>(pool, hdr.pool_chunks);
            ctx->pool_hint = pool;
            continue;
        }
        if (hdr.record_overflow) {  // a signature spans more words than inline slots
            K = std::min<uint32_t>(64, std::max<uint32_t>(hdr.record_overflow, 2 * K));  // (red::kMaxRecords)
            if (hdr.record_overflow > 64)
                return fail(ctx, GP_ERR_UNSUPPORTED, "signature spans more than 64 detector words");
            ctx->record_slots = K;
            continue;
        }
        if (hdr.num_det_ids == 0xFFFFFFFFu) {  // id (or, fused items: edge) capacity overflow
            ids_cap *= 4;
            if (p.fused) items_cap = std::max<uint64_t>(items_cap, t.sources + 16);
            ctx->ids_hint = ids_cap;
            continue;
        }
        break;
    }
    ctx->last_plan = p;
    ctx->has_plan = true;
    if (p.dbg && p.tiny) {  // experiments: the one-CTA kernel's phase timestamps
        uint64_t h[32];
        cudaMemcpy(h, p.dbg, sizeof h, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "tiny phases (us):");
        for (int i = 1; i < 32 && h[i] >= h[i - 1] && h[i] - h[0] < 1000000; i++)
            std::fprintf(stderr, " %.2f", (h[i] - h[i - 1]) / 1e3);
        std::fprintf(stderr, "\n");
    } else if (p.dbg) {
        const char *path = std::getenv("GP_DEBUG_DUMP");
        std::vector<uint64_t> h((size_t)t.groups * 512 * 4);
        cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
        if (path)
            if (FILE *f = std::fopen(path, "wb")) {
                std::fwrite(h.data(), 8, h.size(), f);
                std::fclose(f);
            }
    }
    if (mode == gp::kModeShard) {  // the partial table: sources hdr.num_edges, records hdr.num_det_ids
        const uint64_t n = hdr.num_edges, r = hdr.num_det_ids;
        part->n = n;
        part->r = r;
        if (stats) {
            *stats = gp_stats{};
            stats->num_sources = t.sources;
            stats->h2d_bytes = gen ? L.lay_gate + (uint64_t)t.prob_table_n * 8 : pp.image_bytes();
            stats->kernel_ns = (uint64_t)(elapsed_ms(ctx->ev_h2d, ctx->ev_end) * 1e6);
            stats->kernel_launches = (uint64_t)launches;
        }
        if (part->on_device) {
            part->prob = p.p_prob;
            part->roff = p.p_roff;
            part->word = p.p_word;
            part->bits = p.p_bits;
            if (stats) stats->total_ns = ns_since(t0);
            return GP_OK;
        }
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t at = o;
            o = (size_t)align16(o + bytes);
            return at;
        };
        const size_t a_prob = take(n * 8), a_roff = take((n + 1) * 4), a_word = take(r * 4), a_bits = take(r * 8);
        if ((st = ensure_host(ctx, &ctx->h_out, &ctx->h_out_cap, o)) != GP_OK) return st;
        if (n) e = cudaMemcpyAsync(ctx->h_out + a_prob, p.p_prob, n * 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + a_roff, p.p_roff, (n + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (r && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + a_word, p.p_word, r * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (r && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + a_bits, p.p_bits, r * 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "shard download");
        part->prob = (double *)(ctx->h_out + a_prob);
        part->roff = (uint32_t *)(ctx->h_out + a_roff);
        part->word = (uint32_t *)(ctx->h_out + a_word);
        part->bits = (uint64_t *)(ctx->h_out + a_bits);
        if (stats) {
            stats->d2h_bytes = o;
            stats->total_ns = ns_since(t0);
        }
        return GP_OK;
    }
    const uint64_t E = hdr.num_edges, nd = hdr.num_det_ids, no = hdr.num_obs_ids;
    if (p.out_mapped) {  // already in mapped host memory
        ho.det_off = p.hmap.det_off;
        ho.obs_off = p.hmap.obs_off;
        ho.probs = p.hmap.probs;
        ho.det_ids = p.hmap.det_ids;
        ho.obs_ids = p.hmap.obs_ids;
        ho.edge_off = p.hmap.edge_off;
        if (stats) {
            const double h2d = elapsed_ms(ctx->ev_start, ctx->ev_h2d);
            const bool g = ctx->graph.used || p.tiny;  // (one launch: no stage split)
            const double low = g ? 0 : elapsed_ms(ctx->ev_h2d, ctx->stage_ev.lowered);
            const double trav = g ? 0 : elapsed_ms(ctx->stage_ev.lowered, ctx->stage_ev.traversed);
            const double red = g ? elapsed_ms(ctx->ev_h2d, ctx->stage_ev.reduced)
                                 : elapsed_ms(ctx->stage_ev.traversed, ctx->stage_ev.reduced);
            const double out_ms = elapsed_ms(ctx->stage_ev.reduced, ctx->ev_end);
            *stats = gp_stats{};
            stats->h2d_ns = (uint64_t)(h2d * 1e6);
            stats->lower_ns = pack_ns + (uint64_t)((h2d + low) * 1e6);
            stats->traverse_ns = (uint64_t)(trav * 1e6);
            stats->traverse_kernel_ns = (uint64_t)(trav * 1e6);
            stats->reduce_ns = (uint64_t)((red + out_ms) * 1e6);
            stats->kernel_ns = (uint64_t)((low + trav + red) * 1e6);  // includes the mapped-output copy
            stats->d2h_ns = (uint64_t)(out_ms * 1e6);
            stats->num_sources = t.sources;
            stats->h2d_bytes = gen ? L.lay_gate + (uint64_t)t.prob_table_n * 8 : pp.image_bytes();
            stats->d2h_bytes = sizeof(DeviceHeader) + (E + 1) * 8 + E * 8 + (nd + no) * 4 + (count + 1) * 8;
            stats->kernel_launches = (uint64_t)launches;
            stats->total_ns = ns_since(t0);
        }
        return GP_OK;
    }
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes);
        return at;
    };
    const size_t o_det_off = take((E + 1) * 4), o_obs_off = take((E + 1) * 4), o_prob = take(E * 8),
                 o_det = take(nd * 4), o_obs = take(no * 4), o_edge = take((count + 1) * 8);
    if ((st = ensure_host(ctx, &ctx->h_out, &ctx->h_out_cap, o)) != GP_OK) return st;
    auto d2h = [&](size_t off, const void *src, size_t bytes) {
        if (bytes && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + off, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    };
    d2h(o_det_off, p.o_det_off, (E + 1) * 4);
    d2h(o_obs_off, p.o_obs_off, (E + 1) * 4);
    d2h(o_prob, p.o_prob, E * 8);
    d2h(o_det, p.o_det, nd * 4);
    d2h(o_obs, p.o_obs, no * 4);
    d2h(o_edge, p.o_edge_off, (count + 1) * 8);
    cudaEventRecord(ctx->ev_end, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "download");
    ho.det_off = (uint32_t *)(ctx->h_out + o_det_off);
    ho.obs_off = (uint32_t *)(ctx->h_out + o_obs_off);
    ho.probs = (double *)(ctx->h_out + o_prob);
    ho.det_ids = (uint32_t *)(ctx->h_out + o_det);
    ho.obs_ids = (uint32_t *)(ctx->h_out + o_obs);
    ho.edge_off = (uint64_t *)(ctx->h_out + o_edge);
    if (stats) {
        const double h2d = elapsed_ms(ctx->ev_start, ctx->ev_h2d);
        const bool g = ctx->graph.used || p.tiny;  // one graph launch / one kernel: no stage split
        const double low = g ? 0 : elapsed_ms(ctx->ev_h2d, ctx->stage_ev.lowered);
        const double trav = g ? 0 : elapsed_ms(ctx->stage_ev.lowered, ctx->stage_ev.traversed);
        const double red = g ? elapsed_ms(ctx->ev_h2d, ctx->stage_ev.reduced)
                             : elapsed_ms(ctx->stage_ev.traversed, ctx->stage_ev.reduced);
        const double d2h_ms = elapsed_ms(ctx->stage_ev.reduced, ctx->ev_end);
        *stats = gp_stats{};
        stats->h2d_ns = (uint64_t)(h2d * 1e6);
        stats->lower_ns = pack_ns + (uint64_t)((h2d + low) * 1e6);
        stats->traverse_ns = (uint64_t)(trav * 1e6);
        stats->traverse_kernel_ns = (uint64_t)(trav * 1e6);
        stats->reduce_ns = (uint64_t)((red + d2h_ms) * 1e6);
        stats->kernel_ns = (uint64_t)((low + trav + red) * 1e6);
        stats->d2h_ns = (uint64_t)(d2h_ms * 1e6);
        stats->num_sources = t.sources;
        stats->h2d_bytes = gen ? L.lay_gate + (uint64_t)t.prob_table_n * 8 : pp.image_bytes();
        stats->d2h_bytes = sizeof(DeviceHeader) + o;
        stats->kernel_launches = (uint64_t)launches;
        stats->total_ns = ns_since(t0);
    }
    return GP_OK;
}

}  // namespace

// ---------------------------------------------------------------- device-generated branches
// gp_compile_bb_branches: the check subsets are drawn on the device, the host
// plans the image from the drawn counts (gp_gen.h bb_layer_count: the same
// offsets pack_plan / pack_finish would give the host-generated circuits),
// uploads only the image head, and the fill kernel writes the rest.

namespace {

gp_status bbgen_params(gp_ctx *ctx, const BBGenReq &req, size_t count, uint8_t level, gp::BBGenParams &g) {
    auto &bb = ctx->bb;
    const gp::BBTemplate &T = bb.t;
    g = gp::BBGenParams{};
    const uint32_t lm = T.lm;
    g.xdata = bb.d_tmpl;
    g.zdata = g.xdata + 7 * lm;
    g.zfinal = g.zdata + 7 * lm;
    g.obs_off = g.zfinal + 6 * lm;
    g.obs_q = g.obs_off + T.O + 1;
    g.lm = lm;
    g.nd = T.nd;
    g.n = T.n;
    g.rounds = T.rounds;
    g.refresh = T.refresh;
    g.O = T.O;
    g.MW = (lm + 63) / 64;
    g.level = level;
    g.C = (uint32_t)count;
    g.check_prob = T.check_prob;
    g.pm = T.pm;
    g.seed = T.seed;
    g.first = req.first;
    const size_t masks = count * T.rounds * 2 * g.MW * 8, counts = count * T.rounds * 4;
    gp_status st;
    if ((st = ensure_device(ctx, reinterpret_cast<uint8_t **>(&bb.d_masks), &bb.d_masks_cap, masks)) != GP_OK) return st;
    if (bb.counts_cap < counts) {
        if (bb.d_counts) cudaFree(bb.d_counts);
        if (bb.h_counts) cudaFreeHost(bb.h_counts);
        bb.d_counts = bb.h_counts = nullptr;
        bb.counts_cap = 0;
        if (cudaMalloc(&bb.d_counts, counts + counts / 4) != cudaSuccess ||
            cudaMallocHost(&bb.h_counts, counts + counts / 4) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, GP_ERR_OUT_OF_MEMORY, "branch count buffers");
        }
        bb.counts_cap = counts + counts / 4;
    }
    if (!bb.d_err) {
        if (cudaMalloc(&bb.d_err, 16) != cudaSuccess || cudaMallocHost(&bb.h_err, 16) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, GP_ERR_OUT_OF_MEMORY, "generator status");
        }
    }
    g.masks = bb.d_masks;
    g.counts = bb.d_counts;
    g.err = bb.d_err;
    return GP_OK;
}

// Draws every branch's check subsets (masks and counts stay on the device;
// the counts also come back to the host for planning).
gp_status bbgen_draw(gp_ctx *ctx, const BBGenReq &req, size_t count, uint8_t level) {
    auto &bb = ctx->bb;
    gp::BBGenParams g;
    gp_status st = bbgen_params(ctx, req, count, level, g);
    if (st != GP_OK) return st;
    cudaMemsetAsync(bb.d_err, 0, 4, ctx->stream);
    gp::launch_bbgen_draw(g, ctx->stream);
    cudaError_t e = cudaMemcpyAsync(bb.h_counts, bb.d_counts, count * bb.t.rounds * 4, cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? GP_OK : cuda_fail(ctx, e, "branch draws");
}

// Image plan of branches [c0, c0 + count) of the drawn batch (host only).
gp_status bbgen_plan(gp_ctx *ctx, size_t c0, size_t count, uint8_t level, gp::PackPlan &pp, uint32_t *pi_out) {
    auto &bb = ctx->bb;
    const gp::BBTemplate &T = bb.t;
    // probability table (channel -> index; identical values share one entry)
    pp.prob_table.clear();
    auto index = [&](double v) {
        for (size_t i = 0; i < pp.prob_table.size(); i++)
            if (std::memcmp(&pp.prob_table[i], &v, 8) == 0) return (uint32_t)i;
        pp.prob_table.push_back(v);
        return (uint32_t)pp.prob_table.size() - 1;
    };
    const double ch[5] = {T.p1, T.p2, T.pr, T.pidle, T.pidle_mr};
    gp::BBCountParams q{T.n, T.nd, T.lm, T.rounds, 0, level ? 3u : 2u, level == 0 ? 6u : level == 1 ? 10u : 15u};
    for (int x = 0; x < 5; x++)
        if (ch[x] > 0) q.on |= 1u << x;
    BatchTotals &t = pp.t;
    t = BatchTotals{};
    t.C = (uint32_t)count;
    t.level = level;
    pp.metas.assign(count, CircuitMeta{});
    const uint32_t l = 2 + 9 * T.rounds, O = T.O, obs_entries = T.obs_off[O];
    for (size_t c = 0; c < count; c++) {  // pack_plan + pack_finish, from the counts
        CircuitMeta &m = pp.metas[c];
        const uint32_t *cnt = bb.h_counts + (c0 + c) * T.rounds;
        uint64_t gates = 0, noise = 0, meas = 0, src = 0;
        uint32_t max_noise = 0, max_meas = 0, D = T.lm, de = 7 * T.lm;
        for (uint32_t li = 0; li < l; li++) {
            const uint32_t r = li == 0 ? 0 : std::min((li - 1) / 9, T.rounds - 1);
            const uint32_t ne = cnt[r] & 0xFFFF, nz = cnt[r] >> 16;
            const gp::BBLayerCount lc = gp::bb_layer_count(q, li, ne, nz);
            gates += lc.gates;
            noise += lc.noise;
            meas += lc.meas;
            src += lc.src;
            max_noise = std::max(max_noise, lc.noise);
            max_meas = std::max(max_meas, lc.meas);
        }
        for (uint32_t r = 0; r < T.rounds; r++) {  // DetectorTracker: Z from the first round, X from the second
            const uint32_t ne = cnt[r] & 0xFFFF, nz = cnt[r] >> 16;
            D += nz + (r ? ne : 0);
            de += (r ? 2 : 1) * nz + (r ? 2 * ne : 0);
        }
        if ((uint64_t)l * (level == 0 ? 2 : level == 1 ? 4 : 7) * T.n + meas >= 0xFFFFFFFFull)
            return fail(ctx, GP_ERR_INVALID_ARGUMENT, "circuit exceeds 32-bit node index space");
        m.n = T.n;
        m.l = l;
        m.M = (uint32_t)meas;
        m.D = D;
        m.O = O;
        m.W = (uint32_t)(((uint64_t)D + O + 63) / 64);
        m.layer_base = (uint32_t)t.layer_slots;
        m.meas_base = (uint32_t)t.meas;
        m.det_base = (uint32_t)t.det_slots;
        m.obs_base = (uint32_t)t.obs_slots;
        m.tile_base = (uint32_t)t.tiles;
        m.bucket_base = (uint32_t)t.buckets;
        m.ell_base = t.ell;
        m.leaf_base = t.leaf;
        m.gate_base = t.gates;
        m.noise_base = t.noise;
        m.det_entry_base = t.det_entries;
        m.obs_entry_base = t.obs_entries;
        m.circ_layer_base = t.layers;
        m.src_noise = (uint32_t)src;
        m.max_layer_noise = max_noise;
        m.src_base = t.sources;
        t.sources += src + m.M;
        t.max_n = std::max(t.max_n, m.n);
        t.max_W = std::max(t.max_W, m.W);
        t.max_l = std::max(t.max_l, m.l);
        t.max_layer_noise = std::max(t.max_layer_noise, max_noise);
        t.max_layer_meas = std::max(t.max_layer_meas, max_meas);
        t.layers += l;
        t.layer_slots += l + 1;
        t.gates += gates;
        t.noise += noise;
        t.meas += m.M;
        t.det_slots += D + 1;
        t.det_entries += de;
        t.obs_slots += O + 1;
        t.obs_entries += obs_entries;
        t.dets += D;
        t.obss += O;
        t.tiles += m.W;
        t.ell += (uint64_t)(l - 1) * gp::ell_stride(m.n);
        t.leaf += (uint64_t)m.W * gp::leaf_stride(m.M);
        t.buckets += (uint64_t)D + 1;
    }
    uint32_t pi[5];
    for (int x = 0; x < 5; x++) pi[x] = ch[x] > 0 ? index(ch[x]) : 0xFFFFFFFFu;
    std::memcpy(pi_out, pi, sizeof pi);
    uint32_t max_m = 0;
    for (const CircuitMeta &m : pp.metas) max_m = std::max(max_m, m.M);
    if (T.n > gp::kNarrowMaxQubits || max_m > gp::kNarrowMaxMeas || pp.prob_table.size() > gp::kNarrowMaxProbs)
        return fail(ctx, GP_ERR_UNSUPPORTED, "device-generated branches need narrow words (<= 4096 qubits, 32768 measurements)");
    t.wide_prob = 0;
    t.narrow = 1;
    t.prob_table_n = (uint32_t)pp.prob_table.size();
    pp.L = gp::stage_layout(t);
    pp.err = gp::kPackOk;
    return GP_OK;
}

// Writes branches [c0, c0 + pp.t.C) into the device image img on stream st
// (its head -- metas, cumulative tables, probability table -- uploaded first).
gp_status bbgen_fill(gp_ctx *ctx, const BBGenReq &req, size_t c0, uint8_t level, const gp::PackPlan &pp,
                     const uint32_t *pi, uint8_t *img, cudaStream_t st) {
    const gp::BBTemplate &T = ctx->bb.t;
    gp::BBGenParams g;
    const gp_status s = bbgen_params(ctx, req, 0, level, g);  // (buffers exist: bbgen_draw sized them)
    if (s != GP_OK) return s;
    const uint64_t MW = (T.lm + 63) / 64;
    g.C = pp.t.C;
    g.first = req.first + c0;
    g.masks = ctx->bb.d_masks + c0 * T.rounds * 2 * MW;
    g.counts = ctx->bb.d_counts + c0 * T.rounds;
    std::memcpy(g.pi, pi, sizeof g.pi);
    g.img = img;
    g.L = pp.L;
    g.gates = pp.t.gates;
    g.noise = pp.t.noise;
    gp::launch_bbgen_fill(g, st);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? GP_OK : cuda_fail(ctx, e, "branch fill");
}

}  // namespace

// ---------------------------------------------------------------- pipelined batches
// A large batch is compiled as P sub-batches in a software pipeline: while
// the GPU runs sub-batch k, the host packs k+1 (into the other pinned
// staging lane) and a copy stream uploads it; each sub-batch's DEM is copied
// by copy_out_kernel on a third stream straight into the mapped pinned batch
// view at its global offsets (the device keeps the running offsets), so the
// download overlaps later sub-batches too. Device capacities come from the
// context's learned hints; any overflow re-runs the batch unpipelined (which
// learns larger hints).

namespace {
struct PipeLane {
    gp::PackPlan pp;
    uint8_t *h_stage = nullptr, *d_img = nullptr, *d_out = nullptr, *d_ws = nullptr;
    size_t h_stage_cap = 0, d_img_cap = 0, d_out_cap = 0, d_ws_cap = 0;
    cudaStream_t s_comp = nullptr;  // the lane's device pipeline (lanes overlap each other's tails)
    cudaEvent_t ev_in = nullptr, ev_done = nullptr, ev_out = nullptr, ev_written = nullptr;
    bool used = false;
};
}  // namespace

namespace gp {
constexpr size_t kLanes = 4;         // lanes allocated: sub-batches in flight (staging, image, output buffers)
// lanes used (GP_PIPE_LANES): with per-sub-batch output regions a lane is
// reused without waiting for a download; two lanes measured best for 4,096
// branches (host circuits 13.6 ms against 14.8 with three and 15.0 with four)
constexpr size_t kLanesDefault = 2;
struct PipeState {
    PipeLane lane[kLanes];
    cudaStream_t s_in = nullptr, s_out = nullptr;
    uint8_t *h_map = nullptr;  // mapped pinned DEM arrays
    size_t h_map_cap = 0;
    uint8_t *h_misc = nullptr;  // mapped: bases [(kMaxSub + 1) * 4], status, headers [kMaxSub]
    uint64_t e_hint = 0, ids_hint = 0;
    // per sub-batch: device output region and completion event (a lane is
    // reused before its previous sub-batch's download has run)
    std::vector<uint8_t *> outs;
    std::vector<size_t> out_caps;
    std::vector<cudaEvent_t> done;
};
void pipe_destroy(PipeState *ps) {
    if (!ps) return;
    for (PipeLane &l : ps->lane) {
        if (l.h_stage) cudaFreeHost(l.h_stage);
        if (l.d_img) cudaFree(l.d_img);
        if (l.d_out) cudaFree(l.d_out);
        if (l.d_ws) cudaFree(l.d_ws);
        if (l.s_comp) cudaStreamDestroy(l.s_comp);
        for (cudaEvent_t e : {l.ev_in, l.ev_done, l.ev_out, l.ev_written})
            if (e) cudaEventDestroy(e);
    }
    if (ps->s_in) cudaStreamDestroy(ps->s_in);
    if (ps->s_out) cudaStreamDestroy(ps->s_out);
    if (ps->h_map) cudaFreeHost(ps->h_map);
    if (ps->h_misc) cudaFreeHost(ps->h_misc);
    for (uint8_t *o : ps->outs)
        if (o) cudaFree(o);
    for (cudaEvent_t e : ps->done)
        if (e) cudaEventDestroy(e);
    delete ps;
}
}  // namespace gp

namespace {

constexpr size_t kMaxSub = 64, kSubCircuits = 512;
constexpr bool kRampDefault = false;  // half-size first / last sub-batches (GP_PIPE_RAMP)

gp_status ensure_host_plain(uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t want = need + need / 4 + 4096;
    if (cudaHostAlloc(buf, want, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return GP_ERR_OUT_OF_MEMORY;
    }
    *cap = want;
    return GP_OK;
}

gp_status ensure_dev_plain(uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t want = need + need / 4;
    if (cudaMalloc(buf, want) != cudaSuccess) {
        cudaGetLastError();
        return GP_ERR_OUT_OF_MEMORY;
    }
    *cap = want;
    return GP_OK;
}

bool pipeline_wanted(gp_ctx *ctx, size_t count) {
    if (ctx->pipeline == 0 || count < 2 * kSubCircuits) return false;
    return ctx->pipe && ctx->pipe->e_hint;  // needs learned output sizes (one unpipelined run)
}

gp_status run_batch_pipelined(gp_ctx *ctx, const gp_circuit_view *cs, size_t count, uint8_t level, HostOut &ho,
                              DeviceHeader &hdr, gp_stats *stats, const BBGenReq *gen = nullptr) {
    const auto t0 = clk::now();
    gp::PipeState &ps = *ctx->pipe;
    gp_status st = GP_OK;
    // device generation: every branch's check subsets drawn up front; each
    // sub-batch is then planned on the host and written on the device
    if (gen && (st = bbgen_draw(ctx, *gen, count, level)) != GP_OK) return st;
    uint32_t gen_pi[gp::kLanes][5] = {};
    const char *ps_env = std::getenv("GP_PIPE_SUB");  // tuning knobs (read per call)
    const size_t sub = ps_env ? std::max<size_t>(64, (size_t)std::atoi(ps_env)) : kSubCircuits;
    const char *pl_env = std::getenv("GP_PIPE_LANES");
    const size_t NL = pl_env ? std::min<size_t>(gp::kLanes, std::max(1, std::atoi(pl_env))) : gp::kLanesDefault;
    const char *pr_env = std::getenv("GP_PIPE_RAMP");
    const bool ramp = pr_env ? std::atoi(pr_env) != 0 : kRampDefault;
    // (device generation: GP_GEN_SUB tunes its sub-batch size separately;
    // measured 13.2 ms per 4,096 branches at 512, 15.8 at 1,024 -- a lane's
    // next sub-batch waits for its download)
    const char *gs = std::getenv("GP_GEN_SUB");
    const size_t gen_sub = gs ? std::max<size_t>(64, (size_t)std::atoi(gs)) : kSubCircuits;
    const size_t P = std::min(kMaxSub, std::max<size_t>(2, count / (gen ? gen_sub : sub)));
    // Mapped host arrays of the whole batch view, sized by the learned hints.
    const uint64_t e_cap = ps.e_hint, ids_cap = ps.ids_hint, c_cap = count + 1;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes);
        return at;
    };
    const size_t o_det_off = take(e_cap * 4), o_obs_off = take(e_cap * 4), o_prob = take(e_cap * 8),
                 o_det = take(ids_cap * 4), o_obs = take(ids_cap * 4), o_edge = take(c_cap * 8);
    if (ps.h_map_cap < o) {
        if (ps.h_map) cudaFreeHost(ps.h_map);
        ps.h_map = nullptr;
        ps.h_map_cap = 0;
        if (cudaHostAlloc(&ps.h_map, o + o / 4, cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, GP_ERR_OUT_OF_MEMORY, "mapped host allocation failed");
        }
        ps.h_map_cap = o + o / 4;
    }
    uint64_t *bases = reinterpret_cast<uint64_t *>(ps.h_misc);
    uint32_t *status = reinterpret_cast<uint32_t *>(bases + (kMaxSub + 1) * 4);
    DeviceHeader *hdrs = reinterpret_cast<DeviceHeader *>(ps.h_misc + ((kMaxSub + 1) * 4 * 8 + 64));
    std::fill(bases, bases + 4, 0);
    *status = 0;
    struct {
        uint32_t *det_off, *obs_off;
        uint64_t *edge_off;
        double *probs;
        uint32_t *det_ids, *obs_ids;
        uint64_t e_cap, ids_cap, c_cap;
    } hm{};
    hm.det_off = (uint32_t *)(ps.h_map + o_det_off);
    hm.obs_off = (uint32_t *)(ps.h_map + o_obs_off);
    hm.probs = (double *)(ps.h_map + o_prob);
    hm.det_ids = (uint32_t *)(ps.h_map + o_det);
    hm.obs_ids = (uint32_t *)(ps.h_map + o_obs);
    hm.edge_off = (uint64_t *)(ps.h_map + o_edge);
    hm.e_cap = e_cap;
    hm.ids_cap = ids_cap;
    hm.c_cap = c_cap;

    const PoolLease lease(true);
    gp::HostPool *hpool = lease.pool;
    uint64_t h2d_bytes = 0, sources = 0;
    int launches = 0;
    auto drain = [&] {
        cudaStreamSynchronize(ps.s_in);
        for (PipeLane &l : ps.lane) cudaStreamSynchronize(l.s_comp);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ps.s_out);
    };
    // Download of sub-batch j by the copy engine: sizes and global offsets
    // are in mapped memory (written by its write_kernel) once it is done.
    std::vector<DevPlan> plans(P);
    std::vector<uint8_t> downloaded(P, 0);
    if (ps.outs.size() < P) {
        ps.outs.resize(P, nullptr);
        ps.out_caps.resize(P, 0);
    }
    while (ps.done.size() < P) {
        ps.done.push_back(nullptr);
        cudaEventCreateWithFlags(&ps.done.back(), cudaEventDisableTiming);
    }
    // GP_PIPE_TRACE=1: per sub-batch host pack time and device event times (stderr)
    const bool trace = std::getenv("GP_PIPE_TRACE") != nullptr;
    // six events per sub-batch: upload start / end, kernels start / end,
    // download start / end; host: pack start / enqueue end
    std::vector<cudaEvent_t> tev(trace ? 6 * P : 0, nullptr);
    for (cudaEvent_t &ev : tev) cudaEventCreate(&ev);
    std::vector<double> tpack0(P, 0.0), tpack1(P, 0.0);
    auto download = [&](size_t j) {
        const DevPlan &pj = plans[j];
        cudaEventSynchronize(ps.done[j]);
        const DeviceHeader &h = hdrs[j];
        downloaded[j] = 1;
        if (trace) cudaEventRecord(tev[6 * j + 4], ps.s_out);
        if (h.num_det_ids == 0xFFFFFFFFu || h.items_overflow || h.record_overflow || h.pool_overflow) {
            *status |= 2;
        } else {
            const uint64_t bE = bases[4 * j], bD = bases[4 * j + 1], bO = bases[4 * j + 2], bC = bases[4 * j + 3];
            const uint64_t E = h.num_edges, nd = h.num_det_ids, no = h.num_obs_ids, C = pj.tot.C;
            if (bD + nd >= 0xFFFFFFFFull || bO + no >= 0xFFFFFFFFull) {
                *status |= 4;  // 32-bit id offsets of the batch view exceeded
            } else if (bE + E + 1 > hm.e_cap || bD + nd > hm.ids_cap || bO + no > hm.ids_cap ||
                       bC + C + 1 > hm.c_cap) {
                *status |= 1;
            } else {
                cudaMemcpyAsync(hm.det_off + bE, pj.o_det_off, (E + 1) * 4, cudaMemcpyDeviceToHost, ps.s_out);
                cudaMemcpyAsync(hm.obs_off + bE, pj.o_obs_off, (E + 1) * 4, cudaMemcpyDeviceToHost, ps.s_out);
                if (E) cudaMemcpyAsync(hm.probs + bE, pj.o_prob, E * 8, cudaMemcpyDeviceToHost, ps.s_out);
                if (nd) cudaMemcpyAsync(hm.det_ids + bD, pj.o_det, nd * 4, cudaMemcpyDeviceToHost, ps.s_out);
                if (no) cudaMemcpyAsync(hm.obs_ids + bO, pj.o_obs, no * 4, cudaMemcpyDeviceToHost, ps.s_out);
                cudaMemcpyAsync(hm.edge_off + bC, pj.o_edge_off, (C + 1) * 8, cudaMemcpyDeviceToHost, ps.s_out);
            }
        }
        if (trace) cudaEventRecord(tev[6 * j + 5], ps.s_out);
    };
    cudaEventRecord(ctx->ev_start, ctx->stream);
    for (size_t k = 0; k < P; k++) {
        PipeLane &ln = ps.lane[k % NL];
        for (size_t j = 0; j < k; j++)  // finished ones: download now (in order)
            if (!downloaded[j]) {
                if (cudaEventQuery(ps.done[j]) != cudaSuccess) break;
                download(j);
            }
        if (trace) tpack0[k] = ns_since(t0) / 1e3;
        // sub-batch k: [bound(k), bound(k + 1)); with the ramp the first and
        // the last are half size (the pipeline fills and drains sooner)
        auto bound = [&](size_t x) -> size_t {
            if (!ramp || P < 3) return count * x / P;
            if (x == 0) return 0;
            if (x >= P) return count;
            const double u = 0.5 + (double)(x - 1);  // units: halves at both ends, P - 1 in all
            return (size_t)((double)count * u / (double)(P - 1));
        };
        const size_t c0 = bound(k), c1 = bound(k + 1), n = c1 - c0;
        if (ln.used) cudaEventSynchronize(ln.ev_in);  // the lane's previous staging was uploaded
        gp::PackPlan &pp = ln.pp;
        pp.force_wide = false;
        pp.no_narrow = false;
        if (gen) {
            if ((st = bbgen_plan(ctx, c0, n, level, pp, gen_pi[k % NL])) != GP_OK) return drain(), st;
            if ((st = ensure_host_plain(&ln.h_stage, &ln.h_stage_cap, pp.L.total)) != GP_OK)
                return drain(), fail(ctx, st, "pinned host allocation of " + std::to_string(pp.L.total) + " bytes failed");
        } else {
    repack:
        gp::pack_plan(hpool, cs + c0, n, level, pp);
        if (pp.err == gp::kPackIndexSpace || pp.err == gp::kPackTooWide) {
            drain();
            const int leaf_err = gp::validate_leaves(cs + c0, 0, pp.err_circuit);
            return fail_pack(ctx, leaf_err ? leaf_err : pp.err);
        }
        if ((st = ensure_host_plain(&ln.h_stage, &ln.h_stage_cap, pp.L.total)) != GP_OK)
            return drain(), fail(ctx, st, "pinned host allocation of " + std::to_string(pp.L.total) + " bytes failed");
        gp::pack_range(hpool, cs + c0, pp, ln.h_stage, 0, n);
        if (pp.err) return drain(), fail_pack(ctx, pp.err);
        if ((pp.need_wide.load() && !pp.force_wide) || (pp.need_wide_words.load() && !pp.no_narrow)) {
            if (pp.need_wide.load()) pp.force_wide = true;
            pp.no_narrow = true;
            goto repack;
        }
        gp::pack_finish(pp, ln.h_stage);
        }  // (host packing)
        BatchTotals t = pp.t;
        if (t.sources >= 0xFFFFFFFFull || t.tiles >= 0xFFFFFFFFull || t.gates >= 0xFFFFFFFFull ||
            t.noise >= 0xFFFFFFFFull || t.meas >= 0xFFFFFFFFull || t.layer_slots >= 0xFFFFFFFFull)
            return drain(), fail(ctx, GP_ERR_UNSUPPORTED, "batch exceeds 32-bit device indexing; split it");
        gp::TravCfg tcfg;
        size_t tsmem;
        if (!gp::plan_traversal(t, ctx->device, &tcfg, &tsmem))
            return drain(), fail(ctx, GP_ERR_UNSUPPORTED, "circuit too wide for on-chip traversal state (2n words)");
        t.groups = 0;
        for (const CircuitMeta &m : pp.metas) t.groups += (m.W + tcfg.T - 1) / tcfg.T;
        gp::pack_head(pp, tcfg.T, ln.h_stage);
        // Device capacities from the learned hints (scaled to the sub-batch).
        const uint32_t K = tcfg.direct ? std::max<uint32_t>(ctx->record_slots, tcfg.T) : ctx->record_slots;
        uint64_t pool = 0;
        if (!tcfg.direct && !tcfg.split)
            pool = (2 * t.sources) / gp::kPoolChunk + t.groups * tcfg.emit_warps + 16;
        const uint64_t slabs = tcfg.split ? t.groups * t.max_l : 0;
        const uint64_t sub_ids = std::max<uint64_t>(3 * t.sources + 1024, ids_cap / P * 2);
        const uint64_t sub_items = t.sources + 16;
        DevPlan &p = plans[k];
        p = DevPlan{};
        p.lay = pp.L;
        p.tot = t;
        p.trav = tcfg;
        p.trav_smem = tsmem;
        const size_t need_ws = carve(ctx, p, t, nullptr, K, sub_ids, pool, slabs, sub_items, false);
        const size_t need_out = carve_out(p, nullptr, sub_items, sub_ids, t.C);
        if (need_ws > ln.d_ws_cap) {  // the lane's workspace serves its sub-batches in stream order
            cudaStreamSynchronize(ln.s_comp);
            if ((st = ensure_device(ctx, &ln.d_ws, &ln.d_ws_cap, need_ws)) != GP_OK) return drain(), st;
        }
        if (ln.used && pp.L.total > ln.d_img_cap) cudaEventSynchronize(ln.ev_done);
        if (ensure_dev_plain(&ps.outs[k], &ps.out_caps[k], need_out) != GP_OK ||
            ensure_dev_plain(&ln.d_img, &ln.d_img_cap, pp.L.total) != GP_OK)
            return drain(), fail(ctx, GP_ERR_OUT_OF_MEMORY, "device allocation failed");
        carve(ctx, p, t, ln.d_ws, K, sub_ids, pool, slabs, sub_items, false);
        carve_out(p, ps.outs[k], sub_items, sub_ids, t.C);
        p.img = ln.d_img;
        p.base_in = bases + 4 * k;
        p.base_out = bases + 4 * (k + 1);
        p.hdr_out = hdrs + k;  // mapped: the host reads it for the download
        // upload (copy stream) -> pipeline (compute stream) -> download (third
        // stream); the upload overwrites the lane's image only once the lane's
        // previous kernels are done reading it
        if (ln.used) cudaStreamWaitEvent(ps.s_in, ln.ev_done, 0);
        if (trace) cudaEventRecord(tev[6 * k], ps.s_in);
        const uint64_t up = gen ? pp.L.lay_gate : pp.image_bytes();  // device generation: the head only
        cudaError_t e = cudaMemcpyAsync(ln.d_img, ln.h_stage, up, cudaMemcpyHostToDevice, ps.s_in);
        if (gen && e == cudaSuccess)
            e = cudaMemcpyAsync(ln.d_img + pp.L.prob_table, ln.h_stage + pp.L.prob_table, t.prob_table_n * 8,
                                cudaMemcpyHostToDevice, ps.s_in);
        cudaEventRecord(ln.ev_in, ps.s_in);
        cudaStreamWaitEvent(ln.s_comp, ln.ev_in, 0);
        if (gen && e == cudaSuccess &&
            (st = bbgen_fill(ctx, *gen, c0, level, pp, gen_pi[k % NL], ln.d_img, ln.s_comp)) != GP_OK)
            return drain(), st;
        if (trace) {
            cudaEventRecord(tev[6 * k + 1], ps.s_in);
            cudaEventRecord(tev[6 * k + 2], ln.s_comp);
        }
        cudaEvent_t prev_written = k ? ps.lane[(k - 1) % NL].ev_written : nullptr;
        launches += gp::enqueue_pipeline(p, ln.s_comp, nullptr, nullptr, &e, prev_written, ln.ev_written);
        if (trace) {
            cudaEventRecord(tev[6 * k + 3], ln.s_comp);
            tpack1[k] = ns_since(t0) / 1e3;
        }
        cudaEventRecord(ln.ev_done, ln.s_comp);
        cudaEventRecord(ps.done[k], ln.s_comp);
        ln.used = true;
        if (e != cudaSuccess) return drain(), cuda_fail(ctx, e, "pipelined launch");
        h2d_bytes += gen ? up + t.prob_table_n * 8 : pp.image_bytes();
        sources += t.sources;
    }
    for (size_t j = 0; j < P; j++)
        if (!downloaded[j]) download(j);
    const uint64_t pack_ns = ns_since(t0);
    cudaEventRecord(ctx->ev_h2d, ctx->stream);
    drain();
    if (gen) cudaMemcpy(ctx->bb.h_err, ctx->bb.d_err, 4, cudaMemcpyDeviceToHost);
    cudaEventRecord(ctx->ev_end, ps.s_out);
    cudaEventSynchronize(ctx->ev_end);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "pipelined batch");
    if (trace) {
        auto at = [&](size_t x) { return elapsed_ms(ctx->ev_start, tev[x]) * 1e3; };
        for (size_t k = 0; k < P; k++)
            std::fprintf(stderr, "sub %zu host %.0f-%.0f  up %.0f-%.0f  kern %.0f-%.0f  down %.0f-%.0f (us)\n", k,
                         tpack0[k], tpack1[k], at(6 * k), at(6 * k + 1), at(6 * k + 2), at(6 * k + 3), at(6 * k + 4),
                         at(6 * k + 5));
        for (cudaEvent_t ev : tev) cudaEventDestroy(ev);
    }
    if (*status & 4) return fail(ctx, GP_ERR_UNSUPPORTED, "batch exceeds 2^32 detector or observable ids; split it");
    if (*status) {  // capacity: let the unpipelined path learn larger hints
        ps.e_hint = 0;
        return GP_ERR_UNSUPPORTED;  // caller falls back
    }
    const uint64_t E = bases[4 * P], nd = bases[4 * P + 1], no = bases[4 * P + 2];
    hdr = DeviceHeader{};
    hdr.num_edges = (uint32_t)E;
    hdr.num_det_ids = (uint32_t)nd;
    hdr.num_obs_ids = (uint32_t)no;
    ps.e_hint = std::max(ps.e_hint, E + E / 8 + 1024);
    ps.ids_hint = std::max(ps.ids_hint, std::max(nd, no) + std::max(nd, no) / 8 + 1024);
    ho.det_off = hm.det_off;
    ho.obs_off = hm.obs_off;
    ho.probs = hm.probs;
    ho.det_ids = hm.det_ids;
    ho.obs_ids = hm.obs_ids;
    ho.edge_off = hm.edge_off;
    if (stats) {
        *stats = gp_stats{};
        const double all = elapsed_ms(ctx->ev_start, ctx->ev_end);
        stats->lower_ns = pack_ns;
        stats->kernel_ns = (uint64_t)(all * 1e6);
        stats->num_sources = sources;
        stats->h2d_bytes = h2d_bytes;
        stats->d2h_bytes = (E + 1) * 8 + E * 8 + (nd + no) * 4 + (count + 1) * 8;
        stats->kernel_launches = (uint64_t)launches;
        stats->total_ns = ns_since(t0);
    }
    return GP_OK;
}

gp_status run_batch_any(gp_ctx *ctx, const gp_circuit_view *cs, size_t count, uint8_t level, HostOut &ho,
                        DeviceHeader &hdr, gp_stats *stats, const BBGenReq *gen = nullptr) {
    if (level > 2) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "correlation level must be 0, 1 or 2");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GP_ERR_CUDA, "cudaSetDevice failed");
    if (pipeline_wanted(ctx, count)) {
        const gp_status st = run_batch_pipelined(ctx, cs, count, level, ho, hdr, stats, gen);
        if (st != GP_ERR_UNSUPPORTED || !ctx->err.empty()) return st;
        ctx->err.clear();  // capacity miss: learn with the unpipelined path
    }
    const gp_status st = run_batch(ctx, cs, count, level, ho, hdr, stats, gp::kModeFull, 0, 0xFFFFFFFFu, nullptr, gen);
    if (st == GP_OK && ctx->pipeline != 0 && count >= 2 * kSubCircuits) {  // learn the pipeline's output sizes
        if (!ctx->pipe) {
            ctx->pipe = new gp::PipeState();
            gp::PipeState &ps = *ctx->pipe;
            cudaStreamCreateWithFlags(&ps.s_in, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&ps.s_out, cudaStreamNonBlocking);
            for (PipeLane &l : ps.lane) {
                cudaStreamCreateWithFlags(&l.s_comp, cudaStreamNonBlocking);
                cudaEventCreateWithFlags(&l.ev_in, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&l.ev_done, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&l.ev_out, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&l.ev_written, cudaEventDisableTiming);
            }
            if (cudaHostAlloc(&ps.h_misc, (kMaxSub + 1) * 4 * 8 + 64 + kMaxSub * sizeof(DeviceHeader),
                              cudaHostAllocMapped) != cudaSuccess) {
                cudaGetLastError();
                ps.h_misc = nullptr;
            }
        }
        if (ctx->pipe->h_misc) {
            const uint64_t E = hdr.num_edges, m = std::max(hdr.num_det_ids, hdr.num_obs_ids);
            ctx->pipe->e_hint = std::max(ctx->pipe->e_hint, E + E / 8 + 1024);
            ctx->pipe->ids_hint = std::max(ctx->pipe->ids_hint, m + m / 8 + 1024);
        }
    }
    return st;
}

}  // namespace

extern "C" {

gp_status gp_ctx_create(int device, gp_ctx **out) {
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return GP_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= n) return GP_ERR_NO_DEVICE;
    gp_ctx *ctx = new gp_ctx();
    ctx->device = device;
    cudaSetDevice(device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMallocHost(&ctx->h_hdr, sizeof(DeviceHeader)) != cudaSuccess) {
        delete ctx;
        return GP_ERR_CUDA;
    }
    cudaEventCreate(&ctx->ev_start);
    cudaEventCreate(&ctx->ev_h2d);
    cudaEventCreate(&ctx->ev_end);
    cudaEventCreate(&ctx->stage_ev.lowered);
    cudaEventCreate(&ctx->stage_ev.traversed);
    cudaEventCreate(&ctx->stage_ev.reduced);
    if (cudaMalloc(&ctx->d_bases, 8 * sizeof(uint64_t)) != cudaSuccess ||
        cudaMemset(ctx->d_bases, 0, 8 * sizeof(uint64_t)) != cudaSuccess) {
        delete ctx;
        return GP_ERR_CUDA;
    }
    *out = ctx;
    return GP_OK;
}

void gp_ctx_destroy(gp_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    if (ctx->h_map) cudaFreeHost(ctx->h_map);
    if (ctx->h_hdr) cudaFreeHost(ctx->h_hdr);
    if (ctx->d_img) cudaFree(ctx->d_img);
    if (ctx->d_ws) cudaFree(ctx->d_ws);
    if (ctx->d_flush) cudaFree(ctx->d_flush);
    if (ctx->d_merge) cudaFree(ctx->d_merge);
    if (ctx->d_bases) cudaFree(ctx->d_bases);
    for (void *d : {(void *)ctx->bb.d_tmpl, (void *)ctx->bb.d_masks, (void *)ctx->bb.d_counts, (void *)ctx->bb.d_err})
        if (d) cudaFree(d);
    for (void *hp : {(void *)ctx->bb.h_counts, (void *)ctx->bb.h_err})
        if (hp) cudaFreeHost(hp);
    if (ctx->graph.exec) cudaGraphExecDestroy(ctx->graph.exec);
    gp::pipe_destroy(ctx->pipe);
    for (cudaEvent_t ev : ctx->prof)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : {ctx->ev_start, ctx->ev_h2d, ctx->ev_end, ctx->stage_ev.lowered, ctx->stage_ev.traversed,
                           ctx->stage_ev.reduced})
        if (ev) cudaEventDestroy(ev);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *gp_last_error(gp_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

gp_status gp_ctx_set_option(gp_ctx *ctx, int option, int64_t value) {
    switch (option) {
        case GP_OPT_FORCE_HASH_COLLISIONS:
            ctx->force_collisions = value != 0;
            return GP_OK;
        case GP_OPT_RECORD_SLOTS:
            if (value < 1 || value > 64) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "record slots must be 1..64");
            ctx->record_slots = (uint32_t)value;
            return GP_OK;
        case GP_OPT_SYNC_TIMING:
            return GP_OK;  // stage events are always recorded
        case GP_OPT_PIPELINE:
            if (value < -1 || value > 1) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "pipeline must be -1, 0 or 1");
            ctx->pipeline = (int)value;
            return GP_OK;
        case 99:  // traversal experiments (not part of the ABI contract)
            ctx->trav_debug = (uint32_t)value;
            return GP_OK;
    }
    return fail(ctx, GP_ERR_INVALID_ARGUMENT, "unknown option");
}

gp_status gp_compile(gp_ctx *ctx, const gp_circuit_view *circuit, uint8_t level, gp_dem_view *out,
                     gp_stats *stats) {
    ctx->err.clear();
    HostOut ho{};
    DeviceHeader hdr{};
    gp_status st = run_batch(ctx, circuit, 1, level, ho, hdr, stats);
    if (st != GP_OK) return st;
    out->num_detectors = circuit->num_detectors;
    out->num_observables = circuit->num_observables;
    out->num_edges = hdr.num_edges;
    out->det_offsets = ho.det_off;
    out->det_ids = ho.det_ids;
    out->obs_offsets = ho.obs_off;
    out->obs_ids = ho.obs_ids;
    out->probs = ho.probs;
    return GP_OK;
}

gp_status gp_compile_batch(gp_ctx *ctx, const gp_circuit_view *circuits, size_t count, uint8_t level,
                           gp_dem_batch_view *out, gp_stats *stats) {
    ctx->err.clear();
    HostOut ho{};
    DeviceHeader hdr{};
    gp_status st = run_batch_any(ctx, circuits, count, level, ho, hdr, stats);
    if (st != GP_OK) return st;
    ctx->out_ndet.resize(count);
    ctx->out_nobs.resize(count);
    for (size_t c = 0; c < count; c++) {
        ctx->out_ndet[c] = circuits[c].num_detectors;
        ctx->out_nobs[c] = circuits[c].num_observables;
    }
    out->num_circuits = count;
    out->edge_offsets = ho.edge_off;
    out->num_detectors = ctx->out_ndet.data();
    out->num_observables = ctx->out_nobs.data();
    out->num_edges = hdr.num_edges;
    out->det_offsets = ho.det_off;
    out->det_ids = ho.det_ids;
    out->obs_offsets = ho.obs_off;
    out->obs_ids = ho.obs_ids;
    out->probs = ho.probs;
    return GP_OK;
}

gp_status gp_compile_bb_branches(gp_ctx *ctx, const gp_bb_spec *spec, uint64_t first_branch, size_t count,
                                 uint8_t level, gp_dem_batch_view *out, gp_stats *stats) {
    ctx->err.clear();
    if (!spec || !out) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "null argument");
    if (level > 2) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "correlation level must be 0, 1 or 2");
    if (count == 0 || count >= (1u << 31)) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "branch count must be 1 .. 2^31 - 1");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GP_ERR_CUDA, "cudaSetDevice failed");
    auto &bb = ctx->bb;
    if (!bb.valid || std::memcmp(&bb.spec, spec, sizeof *spec) != 0) {  // (re)build the template
        bb.valid = false;
        if (const char *why = gp::bb_template(*spec, &bb.t)) return fail(ctx, GP_ERR_INVALID_ARGUMENT, why);
        if (bb.t.lm > 0xFFFF) return fail(ctx, GP_ERR_UNSUPPORTED, "more than 65535 checks per type");
        std::vector<uint32_t> h;
        for (const auto *v : {&bb.t.xdata, &bb.t.zdata, &bb.t.zfinal, &bb.t.obs_off, &bb.t.obs_q})
            h.insert(h.end(), v->begin(), v->end());
        gp_status st = ensure_device(ctx, reinterpret_cast<uint8_t **>(&bb.d_tmpl), &bb.d_tmpl_cap, h.size() * 4);
        if (st != GP_OK) return st;
        if (cudaMemcpy(bb.d_tmpl, h.data(), h.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            return fail(ctx, GP_ERR_CUDA, "template upload");
        bb.spec = *spec;
        bb.valid = true;
    }
    HostOut ho{};
    DeviceHeader hdr{};
    const BBGenReq req{first_branch};
    gp_status st = run_batch_any(ctx, nullptr, count, level, ho, hdr, stats, &req);
    if (st != GP_OK) return st;
    if (*bb.h_err) return fail(ctx, GP_ERR_CUDA, "device branch generator disagreed with its plan");
    ctx->out_ndet.resize(count);
    ctx->out_nobs.resize(count);
    for (size_t c = 0; c < count; c++) {  // (DetectorTracker: Z checks from the first round, X from the second)
        const uint32_t *cnt = bb.h_counts + c * bb.t.rounds;
        uint32_t D = bb.t.lm;
        for (uint32_t r = 0; r < bb.t.rounds; r++) D += (cnt[r] >> 16) + (r ? cnt[r] & 0xFFFF : 0);
        ctx->out_ndet[c] = D;
        ctx->out_nobs[c] = bb.t.O;
    }
    out->num_circuits = count;
    out->edge_offsets = ho.edge_off;
    out->num_detectors = ctx->out_ndet.data();
    out->num_observables = ctx->out_nobs.data();
    out->num_edges = hdr.num_edges;
    out->det_offsets = ho.det_off;
    out->det_ids = ho.det_ids;
    out->obs_offsets = ho.obs_off;
    out->obs_ids = ho.obs_ids;
    out->probs = ho.probs;
    return GP_OK;
}

gp_status gp_compile_shard(gp_ctx *ctx, const gp_circuit_view *circuit, uint8_t level, uint32_t shard,
                           uint32_t nshards, uint32_t memory, gp_partial_view *out, gp_stats *stats) {
    ctx->err.clear();
    if (!circuit || !out) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "null argument");
    if (memory != GP_MEM_HOST && memory != GP_MEM_DEVICE) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "bad memory kind");
    if (nshards == 0 || shard >= nshards) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "shard index out of range");
    const uint64_t l = circuit->num_layers;
    const uint32_t lo = (uint32_t)(l * shard / nshards), hi = (uint32_t)(l * (shard + 1) / nshards);
    HostOut ho{};
    DeviceHeader hdr{};
    PartialOut part;
    part.on_device = memory == GP_MEM_DEVICE;
    const gp_status st = run_batch(ctx, circuit, 1, level, ho, hdr, stats, gp::kModeShard, lo,
                                   shard + 1 == nshards ? 0xFFFFFFFFu : hi, &part);
    if (st != GP_OK) return st;
    out->num_detectors = circuit->num_detectors;
    out->num_observables = circuit->num_observables;
    out->num_sources = part.n;
    out->num_records = part.r;
    out->memory = memory;
    out->reserved = 0;
    out->probs = part.prob;
    out->rec_offsets = part.roff;
    out->rec_words = part.word;
    out->rec_bits = part.bits;
    return GP_OK;
}

// The union of the shards' partial tables as ONE synthetic circuit whose
// sources are the table entries: the parts are copied (host or device) into
// one device buffer, unpack_kernel lays them out as the emit stage would
// (counts, probabilities, slot-major records), and the device reduce runs
// unchanged (mode Merge).
gp_status gp_merge_partials(gp_ctx *ctx, const gp_partial_view *parts, size_t nparts, gp_dem_view *out,
                            gp_stats *stats) {
    const auto t0 = clk::now();
    ctx->err.clear();
    if (!parts || !out || nparts == 0) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "no partial tables");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GP_ERR_CUDA, "cudaSetDevice failed");
    const uint32_t D = parts[0].num_detectors, O = parts[0].num_observables;
    const uint32_t W = (uint32_t)(((uint64_t)D + O + 63) / 64);
    uint64_t S = 0, R = 0;
    std::vector<uint4> desc(nparts);
    for (size_t k = 0; k < nparts; k++) {
        const gp_partial_view &v = parts[k];
        if (v.num_detectors != D || v.num_observables != O)
            return fail(ctx, GP_ERR_INVALID_ARGUMENT, "partial tables of different circuits");
        if (v.memory != GP_MEM_HOST && v.memory != GP_MEM_DEVICE)
            return fail(ctx, GP_ERR_INVALID_ARGUMENT, "bad memory kind");
        if (!v.rec_offsets || (v.num_sources && !v.probs) || (v.num_records && (!v.rec_words || !v.rec_bits)))
            return fail(ctx, GP_ERR_INVALID_ARGUMENT, "null partial table array");
        desc[k] = make_uint4((uint32_t)S, (uint32_t)(S + k), (uint32_t)R, (uint32_t)v.num_records);
        S += v.num_sources;
        R += v.num_records;
    }
    if (S + nparts >= 0xFFFFFFFFull || R >= 0xFFFFFFFFull || (uint64_t)D + 1 >= 0xFFFFFFFFull)
        return fail(ctx, GP_ERR_UNSUPPORTED, "merge exceeds 32-bit device indexing");

    BatchTotals t{};
    t.C = 1;
    t.sources = S;
    t.buckets = (uint64_t)D + 1;
    t.dets = D;
    t.obss = O;
    t.tiles = W;
    t.max_W = W;
    const StageLayout L = gp::stage_layout(t);
    // Concatenated input: probs [S] | offsets [S + parts] | words [R] | bits [R] | descriptors.
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes + 16);
        return at;
    };
    const size_t a_prob = take(S * 8), a_roff = take((S + nparts) * 4), a_word = take(R * 4), a_bits = take(R * 8),
                 a_desc = take(nparts * 16);
    gp_status st = GP_OK;
    cudaError_t e = cudaSuccess;
    // (the parts may be views into this ctx's workspace: copy them out first)
    if ((st = ensure_device(ctx, &ctx->d_merge, &ctx->d_merge_cap, o)) != GP_OK) return st;
    if ((st = ensure_host(ctx, &ctx->h_stage, &ctx->h_stage_cap, L.total + nparts * 16)) != GP_OK) return st;
    cudaEventRecord(ctx->ev_start, ctx->stream);
    uint8_t *m = ctx->d_merge;
    auto cp = [&](size_t dst, const void *src, size_t bytes, uint32_t mem) {
        if (bytes && e == cudaSuccess)
            e = cudaMemcpyAsync(m + dst, src, bytes, mem == GP_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                         : cudaMemcpyHostToDevice, ctx->stream);
    };
    uint64_t h2d = 0;
    for (size_t k = 0; k < nparts; k++) {
        const gp_partial_view &v = parts[k];
        const uint4 d = desc[k];
        cp(a_prob + (size_t)d.x * 8, v.probs, v.num_sources * 8, v.memory);
        cp(a_roff + (size_t)d.y * 4, v.rec_offsets, (v.num_sources + 1) * 4, v.memory);
        cp(a_word + (size_t)d.z * 4, v.rec_words, v.num_records * 4, v.memory);
        cp(a_bits + (size_t)d.z * 8, v.rec_bits, v.num_records * 8, v.memory);
        if (v.memory == GP_MEM_HOST) h2d += v.num_sources * 12 + 4 + v.num_records * 12;
    }
    uint8_t *h = ctx->h_stage;  // synthetic circuit image + part descriptors
    std::memset(h, 0, L.total);
    CircuitMeta cm{};
    cm.D = D;
    cm.O = O;
    cm.W = W;
    cm.src_noise = (uint32_t)S;
    std::memcpy(h + L.meta, &cm, sizeof cm);
    const uint64_t circ_src[2] = {0, S};
    const uint32_t circ_bkt[2] = {0, D + 1};
    std::memcpy(h + L.circ_src, circ_src, sizeof circ_src);
    std::memcpy(h + L.circ_bkt, circ_bkt, sizeof circ_bkt);
    std::memcpy(h + L.total, desc.data(), nparts * 16);
    cp(a_desc, h + L.total, nparts * 16, GP_MEM_HOST);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "merge input copy");
    if ((st = ensure_device(ctx, &ctx->d_img, &ctx->d_img_cap, L.total)) != GP_OK) return st;
    e = cudaMemcpyAsync(ctx->d_img, h, L.total, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "merge upload");
    ctx->has_plan = false;  // the staged circuit image is replaced

    const uint32_t K = 16;  // record slots: the widest signature the reduce accepts
    uint64_t ids_cap = std::max<uint64_t>(ctx->ids_hint, 3 * S + 1024);
    const uint64_t items_cap = S + 16;
    DevPlan p{};
    int launches = 0;
    DeviceHeader hdr{};
    cudaEventRecord(ctx->ev_h2d, ctx->stream);
    for (int attempt = 0;; attempt++) {
        p = DevPlan{};
        p.img = ctx->d_img;
        p.lay = L;
        p.tot = t;
        p.mode = gp::kModeMerge;
        const size_t need = carve(ctx, p, t, nullptr, K, ids_cap, 0, 0, items_cap, true);
        if ((st = ensure_device(ctx, &ctx->d_ws, &ctx->d_ws_cap, need)) != GP_OK) return st;
        carve(ctx, p, t, ctx->d_ws, K, ids_cap, 0, 0, items_cap, true);
        p.base_in = ctx->d_bases;
        p.base_out = ctx->d_bases + 4;
        p.p_prob = (double *)(m + a_prob);
        p.p_roff = (uint32_t *)(m + a_roff);
        p.p_word = (uint32_t *)(m + a_word);
        p.p_bits = (uint64_t *)(m + a_bits);
        p.m_desc = (const uint4 *)(m + a_desc);
        p.m_parts = (uint32_t)nparts;
        launches += gp::enqueue_pipeline(p, ctx->stream, &ctx->stage_ev, nullptr, &e);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
        e = cudaMemcpyAsync(ctx->h_hdr, p.hdr, sizeof(DeviceHeader), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "merge pipeline");
        hdr = *ctx->h_hdr;
        if (hdr.bad_input)
            return fail(ctx, GP_ERR_INVALID_ARGUMENT,
                        "malformed partial table: " + std::to_string(hdr.bad_input) +
                            " entries without records, wider than 16 words or outside the circuit");
        if (hdr.num_det_ids == 0xFFFFFFFFu) {  // id capacity overflow
            if (attempt >= 5) return fail(ctx, GP_ERR_CUDA, "capacity retry loop did not converge");
            ids_cap *= 4;
            ctx->ids_hint = ids_cap;
            continue;
        }
        break;
    }
    const uint64_t E = hdr.num_edges, nd = hdr.num_det_ids, no = hdr.num_obs_ids;
    size_t q = 0;
    auto otake = [&](size_t bytes) {
        const size_t at = q;
        q = (size_t)align16(q + bytes);
        return at;
    };
    const size_t o_det_off = otake((E + 1) * 4), o_obs_off = otake((E + 1) * 4), o_prob = otake(E * 8),
                 o_det = otake(nd * 4), o_obs = otake(no * 4);
    if ((st = ensure_host(ctx, &ctx->h_out, &ctx->h_out_cap, q)) != GP_OK) return st;
    auto d2h = [&](size_t off, const void *src, size_t bytes) {
        if (bytes && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + off, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    };
    d2h(o_det_off, p.o_det_off, (E + 1) * 4);
    d2h(o_obs_off, p.o_obs_off, (E + 1) * 4);
    d2h(o_prob, p.o_prob, E * 8);
    d2h(o_det, p.o_det, nd * 4);
    d2h(o_obs, p.o_obs, no * 4);
    cudaEventRecord(ctx->ev_end, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "merge download");
    out->num_detectors = D;
    out->num_observables = O;
    out->num_edges = E;
    out->det_offsets = (uint32_t *)(ctx->h_out + o_det_off);
    out->obs_offsets = (uint32_t *)(ctx->h_out + o_obs_off);
    out->probs = (double *)(ctx->h_out + o_prob);
    out->det_ids = (uint32_t *)(ctx->h_out + o_det);
    out->obs_ids = (uint32_t *)(ctx->h_out + o_obs);
    if (stats) {
        *stats = gp_stats{};
        stats->h2d_ns = (uint64_t)(elapsed_ms(ctx->ev_start, ctx->ev_h2d) * 1e6);
        stats->reduce_ns = (uint64_t)(elapsed_ms(ctx->ev_h2d, ctx->stage_ev.reduced) * 1e6);
        stats->kernel_ns = stats->reduce_ns;
        stats->d2h_ns = (uint64_t)(elapsed_ms(ctx->stage_ev.reduced, ctx->ev_end) * 1e6);
        stats->num_sources = S;
        stats->h2d_bytes = h2d + L.total + nparts * 16;
        stats->d2h_bytes = q;
        stats->kernel_launches = (uint64_t)launches;
        stats->total_ns = ns_since(t0);
    }
    return GP_OK;
}

gp_status gp_replay(gp_ctx *ctx, uint32_t iterations, int flush_l2, gp_stats *stats) {
    if (!ctx->has_plan) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "gp_replay needs a previous successful compile");
    cudaSetDevice(ctx->device);
    constexpr size_t kFlush = 256ull << 20;  // > 126 MB L2
    if (flush_l2 && !ctx->d_flush && cudaMalloc(&ctx->d_flush, kFlush) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "flush buffer");
    }
    for (cudaEvent_t &ev : ctx->prof)
        if (!ev) cudaEventCreate(&ev);
    std::fill(std::begin(ctx->prof_ns), std::end(ctx->prof_ns), 0);
    uint64_t total = 0, trav = 0;
    int launches = 0;
    for (uint32_t it = 0; it < iterations; it++) {
        if (flush_l2) cudaMemsetAsync(ctx->d_flush, it & 0xFF, kFlush, ctx->stream);
        cudaError_t e;
        launches = gp::enqueue_pipeline(ctx->last_plan, ctx->stream, nullptr, ctx->prof, &e);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "replay");
        for (int k = 1; k < gp::kProfCount; k++)
            ctx->prof_ns[k] += (uint64_t)(elapsed_ms(ctx->prof[k - 1], ctx->prof[k]) * 1e6);
        total += (uint64_t)(elapsed_ms(ctx->prof[0], ctx->prof[gp::kProfCount - 1]) * 1e6);
        trav += (uint64_t)(elapsed_ms(ctx->prof[gp::kProfLower], ctx->prof[gp::kProfEmit]) * 1e6);
    }
    if (stats) {
        *stats = gp_stats{};
        stats->kernel_ns = total;
        stats->traverse_kernel_ns = trav;
        stats->traverse_ns = trav;
        stats->kernel_launches = (uint64_t)launches;
        stats->num_sources = ctx->last_plan.tot.sources;
    }
    return GP_OK;
}

int gp_profile_stages(gp_ctx *ctx, uint64_t *ns, const char **names, int cap) {
    int n = 0;
    for (int k = 1; k < gp::kProfCount && n < cap; k++, n++) {
        if (ns) ns[n] = ctx->prof_ns[k];
        if (names) names[n] = gp::kProfNames[k];
    }
    return n;
}

gp_status gp_circuit_metrics(const gp_circuit_view *v, uint8_t level, gp_metrics *out) {
    *out = gp_metrics{};
    const uint32_t n = v->num_qubits, l = v->num_layers;
    out->base_nodes = (uint64_t)l * 2 * n;
    out->words = ((uint64_t)v->num_detectors + v->num_observables + 63) / 64;
    out->measurements = v->num_measurements;
    std::vector<uint8_t> refs(n);
    for (uint32_t i = 1; i < l; i++) {  // layer i shapes boundary i - 1
        std::fill(refs.begin(), refs.end(), 2);  // idle: X -> X, Z -> Z
        for (uint32_t g = v->gate_offsets[i]; g < v->gate_offsets[i + 1]; g++) {
            const uint32_t q = v->gate_q0[g];
            switch (v->gate_kind[g]) {
                case GP_GATE_CX:
                    refs[q] = 3;
                    refs[v->gate_q1[g]] = 3;
                    break;
                case GP_GATE_R:
                    refs[q] = 0;
                    break;
                case GP_GATE_MR:
                    refs[q] = 1;
                    break;
                default:  // H: 2, M: leaf + X
                    refs[q] = 2;
            }
        }
        for (uint32_t q = 0; q < n; q++) out->succ_refs += refs[q];
    }
    static const uint8_t kDep2[15] = {4, 8, 1, 5, 2, 10, 12, 9, 3, 6, 13, 7, 15, 11, 14};
    for (uint32_t o = 0; o < v->noise_offsets[l]; o++) {
        const uint8_t k = v->noise_kind[o];
        const uint32_t nc = components(k, level);
        out->sources += nc;
        if (k <= GP_NOISE_Z_ERROR) out->source_rows += 1;
        else if (k == GP_NOISE_DEPOLARIZE1) out->source_rows += nc == 2 ? 2 : 4;
        else
            for (uint32_t c = 0; c < nc; c++) out->source_rows += (uint64_t)__builtin_popcount(kDep2[c]);
    }
    for (uint32_t g = 0; g < v->gate_offsets[l]; g++)
        if ((v->gate_kind[g] == GP_GATE_M || v->gate_kind[g] == GP_GATE_MR) && v->gate_flip[g] > 0) {
            out->sources++;
            out->source_rows++;
        }
    return GP_OK;
}

char *gp_serialize_dem(const gp_dem_view *d, size_t *len) {
    // serialize_dem (dem.cpp:144-157) with format_double = std::to_chars
    // shortest round-trip (util.hpp:24-28). Large DEMs are formatted once, in
    // edge pieces on the shared host pool, each into its worker's scratch
    // (kept across calls), then copied into place. A DEM holds few distinct
    // folded probabilities (37 over the 87k hyperedges of surface d25), so
    // each piece keeps the text of the doubles it formatted (direct-mapped by
    // their bits) and copies it for repeats: the same std::to_chars bytes.
    const uint64_t E = d->num_edges;
    const size_t k = E < 4096 ? 1 : std::min<uint64_t>(256, E / 1024);
    // bound of a piece: error(<= 24 chars)\n per edge, " D" / " L" + <= 10 digits per id
    auto bound = [&](uint64_t e0, uint64_t e1) {
        return (size_t)((e1 - e0) * 40 +
                        ((uint64_t)(d->det_offsets[e1] - d->det_offsets[e0]) + (d->obs_offsets[e1] - d->obs_offsets[e0])) * 12);
    };
    struct ProbText {
        uint64_t bits[64];
        uint8_t n[64];
        char s[64][32];
    };
    auto format = [&](uint64_t e0, uint64_t e1, char *p, char *const end) {
        ProbText pt;
        std::memset(pt.n, 0, sizeof pt.n);
        char *const start = p;
        for (uint64_t e = e0; e < e1; e++) {
            std::memcpy(p, "error(", 6);
            p += 6;
            const double v = d->probs[e];
            uint64_t b;
            std::memcpy(&b, &v, 8);
            const uint32_t h = (uint32_t)((b * 0x9E3779B97F4A7C15ull) >> 58);
            if (pt.n[h] && pt.bits[h] == b) {
                std::memcpy(p, pt.s[h], 32);  // (fixed-size copy; the bound leaves room)
                p += pt.n[h];
            } else {
                char *const q = std::to_chars(p, end, v).ptr;
                const size_t m = (size_t)(q - p);
                if (m < 32) {
                    std::memcpy(pt.s[h], p, m);
                    pt.n[h] = (uint8_t)m;
                    pt.bits[h] = b;
                }
                p = q;
            }
            *p++ = ')';
            for (uint64_t x = d->det_offsets[e]; x < d->det_offsets[e + 1]; x++) {
                p[0] = ' ';
                p[1] = 'D';
                p = std::to_chars(p + 2, end, d->det_ids[x]).ptr;
            }
            for (uint64_t x = d->obs_offsets[e]; x < d->obs_offsets[e + 1]; x++) {
                p[0] = ' ';
                p[1] = 'L';
                p = std::to_chars(p + 2, end, d->obs_ids[x]).ptr;
            }
            *p++ = '\n';
        }
        return (size_t)(p - start);
    };
    if (k == 1) {
        char *out = (char *)std::malloc(bound(0, E) + 1 + 64);
        const size_t n = format(0, E, out, out + bound(0, E) + 32);
        out[n] = 0;
        if (len) *len = n;
        return out;
    }
    // pass 1: piece i formatted at scratch `buf[i]` + `off[i]` (the worker's
    // scratch, reset by the first piece it takes in this call)
    static std::atomic<uint64_t> calls{0};
    const uint64_t call = ++calls;
    std::vector<std::vector<char> *> buf(k);
    std::vector<size_t> off(k), at(k + 1, 0);
    gp::host_parallel_for(k, [&](size_t i) {
        thread_local std::vector<char> scratch;
        thread_local uint64_t used = 0, gen = 0;
        if (gen != call) {
            gen = call;
            used = 0;
        }
        const uint64_t e0 = E * i / k, e1 = E * (i + 1) / k;
        const size_t b = bound(e0, e1) + 32;
        if (scratch.size() < used + b) scratch.resize(std::max(used + b, 2 * scratch.size()));
        const size_t n = format(e0, e1, scratch.data() + used, scratch.data() + used + b);
        buf[i] = &scratch;
        off[i] = used;
        at[i + 1] = n;
        used += n;
    });
    for (size_t i = 0; i < k; i++) at[i + 1] += at[i];
    char *out = (char *)std::malloc(at[k] + 1 + 64);
    gp::host_parallel_for(k, [&](size_t i) { std::memcpy(out + at[i], buf[i]->data() + off[i], at[i + 1] - at[i]); });
    out[at[k]] = 0;
    if (len) *len = at[k];
    return out;
}

}  // extern "C"

namespace {

uint64_t dg_mix(uint64_t h, uint64_t w) {
    uint64_t x = h + w + 0x9e3779b97f4a7c15ull;
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// Digest of edges [e0, e1) of flat DEM arrays (gp_dem_digest's definition).
uint64_t digest_range(uint32_t D, uint32_t O, uint64_t e0, uint64_t e1, const uint32_t *doff, const uint32_t *dids,
                      const uint32_t *ooff, const uint32_t *oids, const double *probs) {
    uint64_t h = 0x6a09e667f3bcc909ull;
    h = dg_mix(h, (uint64_t)D << 32 | O);
    h = dg_mix(h, e1 - e0);
    for (uint64_t e = e0; e < e1; e++) {
        h = dg_mix(h, (uint64_t)(doff[e + 1] - doff[e]) << 32 | (ooff[e + 1] - ooff[e]));
        for (uint64_t k = doff[e]; k < doff[e + 1]; k++) h = dg_mix(h, dids[k]);
        for (uint64_t k = ooff[e]; k < ooff[e + 1]; k++) h = dg_mix(h, oids[k]);
        uint64_t bits;
        std::memcpy(&bits, &probs[e], 8);
        h = dg_mix(h, bits);
    }
    return h;
}

}  // namespace

extern "C" {

uint64_t gp_dem_digest(const gp_dem_view *d) {
    return digest_range(d->num_detectors, d->num_observables, 0, d->num_edges, d->det_offsets, d->det_ids,
                        d->obs_offsets, d->obs_ids, d->probs);
}

void gp_dem_batch_digest(const gp_dem_batch_view *b, uint64_t *out) {
    const size_t n = b->num_circuits;
    const unsigned nt = (unsigned)std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), (n + 63) / 64);
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t c; (c = next.fetch_add(16)) < n;)
            for (size_t i = c; i < std::min(n, c + 16); i++)
                out[i] = digest_range(b->num_detectors[i], b->num_observables[i], b->edge_offsets[i],
                                      b->edge_offsets[i + 1], b->det_offsets, b->det_ids, b->obs_offsets,
                                      b->obs_ids, b->probs);
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; t++) pool.emplace_back(work);
    work();
    for (auto &t : pool) t.join();
}

void *gp_host_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void gp_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

void gp_free(void *p) { std::free(p); }

}  // extern "C"
