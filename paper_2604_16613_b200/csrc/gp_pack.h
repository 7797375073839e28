// gp_pack.h -- host side of the upload: a persistent worker pool and the
// task-parallel packer that turns flat circuit views (include/greenpeas.h)
// into the device staging image (gp_layout.h).
//
// Replaces the host half of lower() (stepg.cpp:165-315): only what the device
// cannot do is done here -- the reference's validation (stepg.cpp:171-174,
// eec.cpp:44-54), compact 8-byte op words, per-layer offset tables. The work
// is split into (circuit, layer range) and (circuit, detector range) tasks so
// a single large circuit packs on every host core, and a batch of small ones
// on every core too.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/greenpeas.h"
#include "gp_layout.h"

namespace gp {

// Persistent workers: a job is a counted range of task indices; the caller
// runs tasks too. Workers spin briefly after a job (back-to-back compiles
// wake them without a syscall), then sleep on a condition variable.
class HostPool {
public:
    explicit HostPool(unsigned workers);
    ~HostPool();
    size_t threads() const { return th_.size() + 1; }
    void run(size_t n, const std::function<void(size_t)> &f);

private:
    struct Job {
        const std::function<void(size_t)> *fn = nullptr;
        size_t n = 0;
        std::atomic<size_t> next{0}, left{0};
    };
    void loop();
    static void work(Job &j);
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::shared_ptr<Job> job_;
    std::atomic<uint64_t> gen_{0};
    bool stop_ = false;
};

// Per-circuit results of the packer (validation codes in reference order).
enum PackErr : int { kPackOk = 0, kPackIndexSpace = 1, kPackDetLeaf = 2, kPackObsLeaf = 3, kPackTooWide = 4 };

struct PackPlan {
    BatchTotals t{};
    std::vector<CircuitMeta> metas;
    StageLayout L{};
    std::vector<double> prob_table;  // sorted distinct noise probabilities (bit patterns)
    int err = kPackOk;               // first failing circuit's error
    size_t err_circuit = 0;
};

// Byte offsets of every array of a staging image with these totals.
StageLayout stage_layout(const BatchTotals &t);

// Phase 0 (sizes, bases, index-space checks) + probability table. Cheap:
// O(C) plus one parallel pass over noise probabilities.
void pack_plan(HostPool *pool, const gp_circuit_view *cs, size_t C, uint8_t level, PackPlan &pp);

// Leaf checks of circuits [c0, c1) only (init_leaves, eec.cpp:40-58): the
// first circuit's error code in reference order, kPackOk if none.
int validate_leaves(const gp_circuit_view *cs, size_t c0, size_t c1);

// Phase 1: writes circuits [c0, c1) into img (every section) and validates
// their detector / observable lists. Parallel over tasks. Returns the first
// error code found in [c0, c1) (kPackOk if none) in *err / *err_circuit.
void pack_range(HostPool *pool, const gp_circuit_view *cs, PackPlan &pp, uint8_t *img, size_t c0, size_t c1);

// Phase 2: per-circuit prefix tables (layer measurement / source offsets),
// source bases, maxima. Must run after every pack_range.
void pack_finish(PackPlan &pp, uint8_t *img);

// Phase 3: meta and cumulative per-circuit tables at the head of the image
// (needs the traversal group width T).
void pack_head(const PackPlan &pp, uint32_t T, uint8_t *img);

}  // namespace gp
