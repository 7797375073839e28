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

// Distinct noise probabilities (bit patterns) -> table index, filled
// concurrently while the noise ops are packed (first come, first indexed):
// the probabilities are read once, by the packer itself.
class ProbDict {
public:
    static constexpr uint32_t kSlots = 1u << 16;  // >= 4 x table capacity
    static constexpr uint32_t kFull = 0xFFFFFFFFu;
    ProbDict();
    void clear();                  // O(entries)
    uint32_t index(uint64_t bits);  // inserts; kFull beyond kNoisePidxMax + 1 entries
    uint32_t size() const;
    void values(std::vector<double> &out) const;  // by index

private:
    static constexpr uint32_t kEmpty = 0xFFFFFFFFu, kBusy = 0xFFFFFFFEu;
    static constexpr uint32_t kSlotLog = kNoisePidxMax + 1 + 4096;  // claims logged for clear() (+ racing threads)
    std::unique_ptr<std::atomic<uint64_t>[]> key_;
    std::unique_ptr<std::atomic<uint32_t>[]> val_;
    std::unique_ptr<uint32_t[]> slot_of_;  // [kSlotLog] index -> slot
    std::atomic<uint32_t> n_{0};
};

struct PackPlan {
    BatchTotals t{};
    std::vector<CircuitMeta> metas;
    StageLayout L{};
    std::vector<double> prob_table;  // distinct noise probabilities by table index (pack_head)
    ProbDict dict;
    bool force_wide = false;            // in: per-op fp64 probabilities
    std::atomic<bool> need_wide{false};  // out: more distinct probabilities than the table holds
    bool no_narrow = false;                    // in: 8-byte op words even where narrow ones fit
    std::atomic<bool> need_wide_words{false};  // out: a narrow batch met a 65th probability
    int err = kPackOk;               // first failing circuit's error
    size_t err_circuit = 0;
    // Bytes of the packed image to upload (the probability table is last and
    // reserved at its maximum size).
    uint64_t image_bytes() const { return L.prob_table + (uint64_t)t.prob_table_n * 8; }
};

// Byte offsets of every array of a staging image with these totals.
StageLayout stage_layout(const BatchTotals &t);

// Phase 0 (sizes, bases, index-space checks, layout). O(C). With
// force_wide unset the noise probabilities go through the table; if
// pack_range then sets need_wide, plan and pack again with force_wide.
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
// (needs the traversal group width T), the probability table at its end.
void pack_head(const PackPlan &pp, uint32_t T, uint8_t *img);

}  // namespace gp
