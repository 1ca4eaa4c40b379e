// me_space.hpp -- host-side configuration-space tables for the sweep kernels.
//
// The flat index space is the canonical enumeration of DESIGN.md §4
// (model -> N -> t, c, p ascending with t*c*p | N -> b -> s -> rc -> do).
// Invalid (t, c, p) tuples and (b, s) pairs consume no index, so the space is
// ragged.  It is made addressable without per-index division chains by:
//   * validity classes: models with the same (t | k, t | v, t | h_ffn) pattern
//     over every candidate t and the same (p <= L, p | L) pattern over every
//     candidate p share one tuple list per world size;
//   * per (class, N) lists of valid tuples with the segment-local prefix of
//     their sizes;
//   * per model x N segment prefix offsets;
//   * per tuple a slice of a pooled list of the valid (b, s) pairs, stored as
//     (u = b*s/c, m = gbs/(d*b)) -- the two numbers the estimator needs.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/me.h"

namespace me {

struct DevTuple {          // 32 B
    uint32_t t, c, p, d;
    uint32_t w;            // configs in this tuple's row: n_pairs * n_rcdo
    uint32_t pair_off;     // first pair in the pool
    uint32_t n_pairs;
    uint32_t fence_off;    // the pool's fences in pair_fence (20 u32)
};

struct DevPair {           // 8 B
    uint32_t u;            // tokens per microbatch per CP rank: (s/c) * b
    uint32_t m;            // microbatches per step gbs/(d b); 0xFFFFFFFF in paper mode
};

struct Limits {            // domain of exact u64 evaluation (me.h, me_sweep)
    static constexpr uint32_t h = 1u << 15, f = 1u << 17, L = 1u << 8, v = 1u << 19;
    static constexpr uint32_t s = 1u << 20, b = 1u << 6, N = 1u << 20;
    static constexpr uint64_t index = 1ull << 56;
};

class HostSpace {
  public:
    // (b, s) pair of tuple (c, d, p) kept: c | s, and with a global batch
    // (d b) | gbs (R17) and, interleaved, p | gbs/(d b) (R29)
    bool pair_ok(uint32_t c, uint32_t d, uint32_t p, uint32_t b, uint32_t s) const {
        if (s % c) return false;
        if (!gbs) return true;
        if (gbs % ((uint64_t)d * b)) return false;
        return vpp < 2 || (gbs / ((uint64_t)d * b)) % p == 0;
    }
    // returns ME_* status; `detail` receives a message on failure
    int build(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
              bool for_sweep, std::string* detail);
    int decode(uint64_t index, uint32_t* model_id, uint32_t* world, me_parallel* out) const;
    // global row (model, N, tuple run) holding flat index `index` (< total)
    uint64_t row_of(uint64_t index) const;
    // flat index of the first config of global row g (total for g >= total_rows)
    uint64_t row_start(uint64_t g) const;

    // inputs (copied)
    std::vector<me_model> models;
    std::vector<uint32_t> world, mbs, seq;
    std::vector<uint64_t> caps;
    uint32_t gpus_per_node = 0, gbs = 0, max_t = 0, max_c = 0, max_p = 0;
    uint8_t rc_mask = 0, do_mask = 0, uneven = 0, stage_max = 0, zero_stage = 0;
    uint8_t sp_off = 0, vpp = 0, wb = 0, gb = 0, ob = 0;  // NEXT-4 variants of every configuration
    // (rc, do) digits of the innermost axes
    uint32_t n_rcdo = 0, lg_rcdo = 0, rcdo_rc = 0, rcdo_do = 0;

    // tables
    std::vector<DevTuple> tuples;       // grouped by world size: tup_begin[n] .. tup_begin[n+1]
    std::vector<uint32_t> tup_begin;
    std::vector<DevPair> pairs;
    std::vector<uint32_t> pair_b;       // micro-batch size of each pooled pair (planner)
    std::vector<uint32_t> pair_su;      // per pooled pair list: its u values sorted ascending
    std::vector<uint32_t> pair_fence;   // per pool: 4 + 16 fences over its sorted u values (K0's search index)
    bool fenced = true;                 // every pool has <= 128 pairs (the fences cover it)
    std::vector<uint32_t> model_class;  // per model
    uint32_t n_class = 0;
    std::vector<uint32_t> list_off;     // n_class * n_world + 1
    std::vector<uint32_t> list_tuple;   // tuple ids
    std::vector<uint64_t> list_prefix;  // segment-local exclusive prefix of w
    std::vector<uint64_t> class_seg;    // size of the segment of (class, n)
    std::vector<uint64_t> seg_prefix;   // n_models * n_world + 1
    std::vector<uint64_t> seg_row;      // n_models * n_world + 1: rows before each segment
    uint64_t total = 0, total_rows = 0;
};

}  // namespace me
