// me_abi.cu -- the extern "C" boundary of libme.so (see include/me.h).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/me.h"
#include "me_kernels.cuh"
#include "me_space.hpp"

using namespace me;

extern "C" int me_partition(uint64_t, uint64_t, int, int, uint64_t*, uint64_t*);
extern "C" int me_join_counts(const uint64_t*, int, uint32_t, uint32_t, int, uint64_t*, uint64_t*, uint64_t*);

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_detail;

static int err(int st, const std::string& msg) {
    g_detail = msg;
    return st;
}
static int cuda_err(cudaError_t e, const char* where) {
    return err(ME_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CU(call)                                            \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return cuda_err(e_, #call);  \
    } while (0)

// restores the caller's current device on scope exit
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---------------------------------------------------------------------------
// allocation
// ---------------------------------------------------------------------------
struct Alloc {
    me_alloc_fn alloc = nullptr;
    me_free_fn free = nullptr;
    void* ctx = nullptr;
    cudaStream_t stream = nullptr;

    void* get(size_t bytes) {
        if (!bytes) bytes = 8;
        if (alloc) return alloc(bytes, (void*)stream, ctx);
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) return nullptr;
        return p;
    }
    void put(void* p) {
        if (!p) return;
        if (free) free(p, (void*)stream, ctx);
        else cudaFreeAsync(p, stream);
    }
};

template <typename T>
static int upload(Alloc& A, const std::vector<T>& v, T** out) {
    *out = (T*)A.get(v.size() * sizeof(T));
    if (!*out) return err(ME_ENOMEM, "device allocation of a table failed");
    if (!v.empty()) CU(cudaMemcpyAsync(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, A.stream));
    return ME_OK;
}

// ---------------------------------------------------------------------------
// comm
// ---------------------------------------------------------------------------
struct me_comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, nranks = 1, device = 0;
};

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
constexpr uint32_t kMaxSets = 4;

struct me_plan {
    HostSpace hs;
    DevSpace ds{};
    Alloc A;
    int device = 0;
    std::vector<void*> owned;  // device allocations owned by the plan
    int sms = 148;
    // K0 (rows) + scan on the plan's own stream, overlapping the output kernel
    // of the previous sub-range on the caller's stream (0), or everything on
    // the caller's stream (1; ME_SERIAL)
    int serial = 0;
    // Scratch sets, alternated by successive sub-ranges, so that K0 of
    // sub-range i+1 (plan stream) overlaps the output kernel of sub-range i
    // (caller's stream).
    struct Scratch {
        RowEnt* rows = nullptr;         // the sub-range's rows
        StEnt* st = nullptr;            // their last-stage terms per digit (stage_max)
        uint32_t* rcnt = nullptr;       // survivors per row
        uint32_t* ucnt = nullptr;       // survivors per 32-row unit
        uint64_t* uoff = nullptr;       // output row of each unit's first survivor
        uint32_t* rnext = nullptr;      // output kernel: next unit to take
        cudaEvent_t free_ev = nullptr;  // recorded after the kernel that last used the set
    } scratch[kMaxSets];
    uint32_t n_sets = 2;                // scratch sets in rotation (ME_SETS, 2..kMaxSets)
    uint32_t max_rows = 0;              // rows per sub-range
    int fused_bps[4] = {0, 0, 0, 0};    // resident K3 blocks per SM per output mode
    int k3_caps[4] = {1, 1, 1, 1};      // per output mode: per-capacity counts in K3 (1) or K0 (0) (ME_K3_CAPS)
    int fused_minb[4] = {2, 3, 2, 3};   // K3 register budget per output mode: 2 or 3 blocks per SM
    int k0_bps = 0;                     // count-only K0: grid-stride blocks per SM (ME_K0_BPS; 0 = resident)
    int k0_wbps = 0;                    // K0 with row entries: the same (ME_K0_WBPS; 0 = one block per 128 rows)
                                        // (measured on C5: records 3 -> 351 ms/step, 2 -> 358; INDEX
                                        // 3 -> 193, 2 -> 220 despite a few spilled registers; FULL
                                        // spills more at 3; ME_FUSED_MINB)
    uint32_t turn = 0;
    cudaStream_t cstream = nullptr;     // K0 + scan
    cudaEvent_t ready_ev = nullptr;     // tables uploaded
    // K3 of successive sub-ranges of one call alternate between two streams so
    // that the next K3 fills the tail of the previous one; the caller's stream
    // is ordered before the first and after the last of a call's K3s
    // (ME_K3_STREAMS=1: K3 on the caller's stream)
    cudaStream_t k3s[2] = {nullptr, nullptr};
    cudaEvent_t k3_ev[2] = {nullptr, nullptr};  // the last K3 queued on each
    int k3_streams = 2;
    // Survivor counts of a sweep are accumulated on the plan stream in a
    // plan-owned slot (the result's own stats block comes from the caller's
    // allocator on the caller's stream, so the plan stream may not touch it
    // without waiting for everything queued there before); the caller's stream
    // copies the slot into the result.  stat_ev[j]: that copy is done.
    static constexpr uint32_t kStatSlots = 8;
    uint64_t* pstats = nullptr;         // kStatSlots x 16 u64
    cudaEvent_t stat_ev[kStatSlots] = {};
    uint32_t stat_turn = 0;
};

// a8: the deferred join of a cyclic partition (me_result_join), shared by the
// results it joined.  out (device): [0] global survivors, [1..8] per capacity,
// [9..16] unused, [17 + k] global position of the first row of this rank's
// k-th result.
struct JoinState {
    Alloc A;
    uint64_t* buf = nullptr;   // gather buffer + out
    uint64_t* out = nullptr;
    uint32_t n = 0;            // this rank's results
    cudaEvent_t done = nullptr;
    int refs = 0;
    bool resolved = false;
    std::vector<uint64_t> host;
};

struct me_result {
    me_plan* plan = nullptr;
    bool own_plan = false;
    Alloc A;
    cudaStream_t stream = nullptr;
    me_out_mode mode = ME_OUT_COUNT;
    uint32_t n_cap = 0;
    uint64_t begin = 0, end = 0;
    uint64_t* stats = nullptr;       // device: [0] count, [1..8] per-cap
    uint64_t* gathered = nullptr;    // device: nranks * 9 (comm)
    uint64_t* cols[ME_N_COLS] = {};  // this rank's columns
    bool own_cols = false;
    uint64_t capacity = 0;
    uint64_t* gcols[ME_N_COLS] = {};  // gathered columns (comm + gather)
    uint64_t g_rows = 0;
    me_comm* comm = nullptr;
    bool gather = false;
    // ev[0] sweep start (plan stream), ev[1] unused, ev[2] K0/scan work done
    // (plan stream), ev[3] output kernels done, ev[4] result complete (caller's
    // stream), ev[5] entry (caller's stream)
    cudaEvent_t ev[6] = {};
    std::vector<cudaEvent_t> tev;  // per sub-range: rows start/end, scan end, output start/end
    std::vector<cudaEvent_t> xev;  // other events of the call (destroyed with the result)
    bool ran_count = false, ran_write = false;
    JoinState* join = nullptr;     // set by me_result_join
    uint32_t join_k = 0;           // this result's position in the join
    me_sweep_partition partition = ME_PART_EVEN;
    // host-side results (valid after `resolved`)
    bool resolved = false;
    uint64_t local = 0, global = 0, offset = 0;
    uint64_t caps[8] = {};
};

// floor(cap * num / den), clamped to 2^63 (every total is < 2^63, so the
// clamp never changes a verdict; the exact quotient may not fit 64 bits)
static uint64_t threshold_of(uint64_t cap, me_threshold thr) {
    const unsigned __int128 q = (unsigned __int128)cap * thr.num / thr.den;
    return q >= ((unsigned __int128)1 << 63) ? (1ull << 63) : (uint64_t)q;
}

static int plan_create(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
                       me_threshold thr, int device, void* stream, me_alloc_fn al, me_free_fn fr, void* ctx,
                       me_plan** out) {
    if (!out) return err(ME_EINVAL, "null out");
    if (thr.num < 1 || thr.den < 1 || thr.num > 1024 || thr.den > 1024)
        return err(ME_EINVAL, "threshold num/den must be in [1, 1024]");
    me_plan* P = new (std::nothrow) me_plan();
    if (!P) return err(ME_ENOMEM, "host allocation");
    std::string detail;
    int st = P->hs.build(models, cluster, cfg, true, &detail);
    if (st) {
        delete P;
        return err(st, detail);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        delete P;
        return err(ME_ECUDA, "no CUDA device");
    }
    if (device < 0 || device >= ndev) {
        delete P;
        return err(ME_EINVAL, "bad device ordinal");
    }
    DeviceGuard g(device);
    P->device = device;
    P->A.alloc = al;
    P->A.free = fr;
    P->A.ctx = ctx;
    P->A.stream = (cudaStream_t)stream;
    const HostSpace& H = P->hs;
    DevSpace& D = P->ds;
    DevModel* dm;
    std::vector<DevModel> dmodels;
    for (const me_model& m : H.models) dmodels.push_back(dev_model(m));
    uint32_t *dcls, *dlo, *dlt, *dpb, *dsu, *dfe;
    uint64_t *dsp, *dlp, *dsr;
    DevTuple* dtu;
    DevPair* dpr;
    if ((st = upload(P->A, dmodels, &dm)) || (P->owned.push_back(dm), false) ||
        (st = upload(P->A, H.model_class, &dcls)) || (P->owned.push_back(dcls), false) ||
        (st = upload(P->A, H.seg_prefix, &dsp)) || (P->owned.push_back(dsp), false) ||
        (st = upload(P->A, H.seg_row, &dsr)) || (P->owned.push_back(dsr), false) ||
        (st = upload(P->A, H.list_off, &dlo)) || (P->owned.push_back(dlo), false) ||
        (st = upload(P->A, H.list_tuple, &dlt)) || (P->owned.push_back(dlt), false) ||
        (st = upload(P->A, H.list_prefix, &dlp)) || (P->owned.push_back(dlp), false) ||
        (st = upload(P->A, H.tuples, &dtu)) || (P->owned.push_back(dtu), false) ||
        (st = upload(P->A, H.pairs, &dpr)) || (P->owned.push_back(dpr), false) ||
        (st = upload(P->A, H.pair_b, &dpb)) || (P->owned.push_back(dpb), false) ||
        (st = upload(P->A, H.pair_su, &dsu)) || (P->owned.push_back(dsu), false) ||
        (st = upload(P->A, H.pair_fence, &dfe)) || (P->owned.push_back(dfe), false)) {
        me_plan_free(P);
        return st;
    }
    D.models = dm;
    D.model_class = dcls;
    D.seg_prefix = dsp;
    D.seg_row = dsr;
    D.list_off = dlo;
    D.list_tuple = dlt;
    D.list_prefix = dlp;
    D.tuples = dtu;
    D.pairs = dpr;
    D.pair_b = dpb;
    D.pair_su = dsu;
    D.pair_fence = dfe;
    D.n_fence = (uint32_t)H.pair_fence.size();
    D.fenced = H.fenced ? 1u : 0u;
    if (const char* e = getenv("ME_K0_FENCE")) D.fenced = D.fenced && atoi(e) ? 1u : 0u;
    D.n_seg = (uint32_t)(H.seg_prefix.size() - 1);
    D.n_world = (uint32_t)H.world.size();
    D.n_pairs = (uint32_t)H.pairs.size();
    D.lg_rcdo = H.lg_rcdo;
    D.rcdo_rc = H.rcdo_rc;
    D.rcdo_do = H.rcdo_do;
    D.n_cap = (uint32_t)H.caps.size();
    D.gbs_mode = H.gbs ? 1u : 0u;
    D.stage_max = H.stage_max ? 1u : 0u;
    D.zero_stage = H.zero_stage;
    {
        const Policy Q = make_policy(H.zero_stage, H.sp_off, H.vpp, H.wb, H.gb, H.ob);
        D.sp_off = Q.sp_off;
        D.vpp = Q.vpp;
        D.wb = Q.wb;
        D.gb = Q.gb;
        D.ob = Q.ob;
    }
    for (int q = 0; q < 8; q++) D.thr[q] = 0, D.thr1[q] = 1;
    D.thr_max = 0;
    for (size_t q = 0; q < H.caps.size(); q++) {
        D.thr[q] = threshold_of(H.caps[q], thr);
        D.thr1[q] = (D.thr[q] < (1ull << 62) ? D.thr[q] : (1ull << 62)) + 1;
        if (q == 0 || D.thr[q] > D.thr_max) D.thr_max = D.thr[q];
    }
    cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, device);
    if (const char* e = getenv("ME_SERIAL")) P->serial = atoi(e);
    D.sparse = 2;  // measured on C5 (records, list-based two-phase path): 2 -> 346 ms/step, 4 -> 348, 8 -> 352
    if (const char* e = getenv("ME_SPARSE")) D.sparse = (uint32_t)atoi(e);
    if (const char* e = getenv("ME_K3_CAPS"))
        for (int& x : P->k3_caps) x = atoi(e) ? 1 : 0;
    P->max_rows = (uint32_t)(H.total_rows < kMaxRows ? H.total_rows : kMaxRows);
    // (tests: a small cap exercises the cutting of sub-ranges by rows)
    if (const char* e = getenv("ME_MAX_ROWS")) P->max_rows = std::min(P->max_rows, (uint32_t)std::max(1, atoi(e)));
    if (P->max_rows < 1) P->max_rows = 1;
    if (const char* e = getenv("ME_FUSED_MINB"))
        for (int& x : P->fused_minb) x = atoi(e) >= 3 ? 3 : 2;
    int fbps = 0;  // 0 = as many as fit
    if (const char* e = getenv("ME_FUSED_BPS")) fbps = std::max(1, atoi(e));
    for (int m = 1; m < 4; m++) {
        const int fb = fused_blocks_per_sm((me_out_mode)m, D.n_cap, P->fused_minb[m]);
        P->fused_bps[m] = fbps ? std::min(fb, fbps) : fb;
    }
    D.k0_smem = 1;
    if (const char* e = getenv("ME_K0_SMEM")) D.k0_smem = (uint32_t)atoi(e);
    P->k0_bps = rowcount_blocks_per_sm(D);
    if (const char* e = getenv("ME_K0_BPS")) P->k0_bps = atoi(e) > 0 ? atoi(e) : 0;  // 0: one block per 128 rows
    if (const char* e = getenv("ME_K0_WBPS")) P->k0_wbps = std::max(0, atoi(e));
    if (const char* e = getenv("ME_SETS")) P->n_sets = (uint32_t)std::min(std::max(atoi(e), 2), (int)kMaxSets);
    const uint32_t max_units = fused_units_of(P->max_rows) + 1;
    for (uint32_t si = 0; si < P->n_sets; si++) {
        me_plan::Scratch& sc = P->scratch[si];
        sc.rows = (RowEnt*)P->A.get((size_t)P->max_rows * sizeof(RowEnt));
        sc.rcnt = (uint32_t*)P->A.get((size_t)P->max_rows * 4);
        sc.ucnt = (uint32_t*)P->A.get((size_t)max_units * 4);
        sc.uoff = (uint64_t*)P->A.get((size_t)max_units * 8);
        sc.rnext = (uint32_t*)P->A.get(256);
        for (void* x : {(void*)sc.rows, (void*)sc.rcnt, (void*)sc.ucnt, (void*)sc.uoff, (void*)sc.rnext})
            P->owned.push_back(x);
        bool ok = sc.rows && sc.rcnt && sc.ucnt && sc.uoff && sc.rnext;
        if (H.stage_max) {
            sc.st = (StEnt*)P->A.get((size_t)P->max_rows * H.n_rcdo * sizeof(StEnt));
            P->owned.push_back(sc.st);
            ok = ok && sc.st;
        }
        if (!ok) {
            me_plan_free(P);
            return err(ME_ENOMEM, "scratch allocation");
        }
        if (cudaEventCreateWithFlags(&sc.free_ev, cudaEventDisableTiming) != cudaSuccess) {
            me_plan_free(P);
            return cuda_err(cudaGetLastError(), "cudaEventCreate");
        }
        cudaEventRecord(sc.free_ev, (cudaStream_t)stream);
    }
    P->pstats = (uint64_t*)P->A.get((size_t)me_plan::kStatSlots * 16 * 8);
    if (!P->pstats) {
        me_plan_free(P);
        return err(ME_ENOMEM, "stats slots");
    }
    P->owned.push_back(P->pstats);
    for (auto& x : P->stat_ev) {
        if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) {
            me_plan_free(P);
            return cuda_err(cudaGetLastError(), "cudaEventCreate");
        }
        cudaEventRecord(x, (cudaStream_t)stream);
    }
    if (cudaStreamCreateWithFlags(&P->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ready_ev, cudaEventDisableTiming) != cudaSuccess) {
        me_plan_free(P);
        return cuda_err(cudaGetLastError(), "plan stream");
    }
    if (const char* e = getenv("ME_K3_STREAMS")) P->k3_streams = atoi(e) >= 2 ? 2 : 1;
    for (int i = 0; i < 2 && P->k3_streams == 2; i++)
        if (cudaStreamCreateWithFlags(&P->k3s[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&P->k3_ev[i], cudaEventDisableTiming) != cudaSuccess) {
            me_plan_free(P);
            return cuda_err(cudaGetLastError(), "K3 stream");
        }
    cudaEventRecord(P->ready_ev, (cudaStream_t)stream);
    if (cudaError_t ce = cudaGetLastError()) {
        me_plan_free(P);
        return cuda_err(ce, "plan_create");
    }
    *out = P;
    return ME_OK;
}

extern "C" int me_plan_create(const me_model_range* models, const me_cluster* cluster,
                              const me_cfg_range* cfg, me_threshold thr, int device, void* stream,
                              me_alloc_fn alloc, me_free_fn free, void* alloc_ctx, me_plan** out) {
    return plan_create(models, cluster, cfg, thr, device, stream, alloc, free, alloc_ctx, out);
}

extern "C" int me_plan_size(const me_plan* plan, uint64_t* n) {
    if (!plan || !n) return err(ME_EINVAL, "null argument");
    *n = plan->hs.total;
    return ME_OK;
}

extern "C" int me_plan_table_bytes(const me_plan* plan, uint64_t* bytes) {
    if (!plan || !bytes) return err(ME_EINVAL, "null argument");
    const HostSpace& H = plan->hs;
    *bytes = H.models.size() * sizeof(DevModel) + H.model_class.size() * 4 + H.seg_prefix.size() * 8 +
             H.seg_row.size() * 8 + H.list_off.size() * 4 + H.list_tuple.size() * 4 + H.list_prefix.size() * 8 +
             H.tuples.size() * sizeof(DevTuple) + H.pairs.size() * sizeof(DevPair) + H.pair_b.size() * 4 +
             H.pair_su.size() * 4 + H.pair_fence.size() * 4;
    return ME_OK;
}

extern "C" void me_plan_free(me_plan* P) {
    if (!P) return;
    {
        DeviceGuard g(P->device);
        // the scratch sets may still be read by an output kernel on a sweep's
        // stream (free_ev) or written by K0 on the plan stream
        if (P->cstream) cudaStreamSynchronize(P->cstream);
        for (auto& sc : P->scratch)
            if (sc.free_ev) cudaEventSynchronize(sc.free_ev);
        for (auto& x : P->stat_ev)
            if (x) cudaEventSynchronize(x);
        for (void* p : P->owned) P->A.put(p);
        for (auto& sc : P->scratch)
            if (sc.free_ev) cudaEventDestroy(sc.free_ev);
        for (auto& x : P->stat_ev)
            if (x) cudaEventDestroy(x);
        if (P->ready_ev) cudaEventDestroy(P->ready_ev);
        if (P->cstream) cudaStreamDestroy(P->cstream);
        for (int i = 0; i < 2; i++) {
            if (P->k3s[i]) cudaStreamSynchronize(P->k3s[i]), cudaStreamDestroy(P->k3s[i]);
            if (P->k3_ev[i]) cudaEventDestroy(P->k3_ev[i]);
        }
    }
    delete P;
}

static void result_release(me_result* R) {
    if (!R) return;
    DeviceGuard g(R->plan ? R->plan->device : -1);
    // the plan stream and the caller's stream may still use the buffers
    if (R->ev[2]) cudaEventSynchronize(R->ev[2]);
    if (R->ev[4]) cudaEventSynchronize(R->ev[4]);
    for (int i = 0; i < 6; i++)
        if (R->ev[i]) cudaEventDestroy(R->ev[i]);
    for (cudaEvent_t x : R->tev) cudaEventDestroy(x);
    if (R->join && --R->join->refs == 0) {
        JoinState* J = R->join;
        if (J->done) {
            cudaEventSynchronize(J->done);
            cudaEventDestroy(J->done);
        }
        J->A.put(J->buf);
        delete J;
    }
    R->A.put(R->stats);
    R->A.put(R->gathered);
    if (R->own_cols)
        for (int j = 0; j < ME_N_COLS; j++) R->A.put(R->cols[j]);
    for (int j = 0; j < ME_N_COLS; j++) R->A.put(R->gcols[j]);
    if (R->own_plan) me_plan_free(R->plan);
    delete R;
}

static int n_cols_of(me_out_mode m) {
    return m == ME_OUT_FULL ? ME_N_COLS : (m == ME_OUT_INDEX || m == ME_OUT_RECORDS ? 1 : 0);
}
// u64 words per row of each output column (RECORDS: one column of 8-word rows)
static uint64_t words_of(me_out_mode m) { return m == ME_OUT_RECORDS ? ME_N_COLS : 1; }

static int resolve(me_result* R);

// One pass of the hot path over [b, e): sub-ranges of at most
// kMaxSub indices and max_rows rows; per sub-range K0 and the scan on the plan
// stream `cs`, the output kernel K3 on the caller's stream
// `st`.  write = false: counts only.  Accumulates stats[0] (survivors) and
// stats[1 + j] (per capacity); the caller orders `st` after `cs` afterwards.
static int run_pipeline(me_plan* P, me_result* R, uint64_t* stats, uint64_t b, uint64_t e, cudaStream_t cs,
                        cudaStream_t st, me_out_mode mode, bool write, Cols cols, uint64_t capacity) {
    const HostSpace& H = P->hs;
    if (cudaMemsetAsync(stats, 0, 9 * 8, cs) != cudaSuccess) return cuda_err(cudaGetLastError(), "memset");
    const auto seg_of = [&](uint64_t g) {
        return (uint32_t)(std::upper_bound(H.seg_row.begin(), H.seg_row.end(), g) - H.seg_row.begin() - 1);
    };
    // K3 streams: ordered after the caller's stream at the call's entry
    const bool alt = write && P->k3_streams == 2 && !P->serial;
    bool used[2] = {false, false};
    uint32_t n_sub = 0;
    if (alt) {
        cudaEvent_t entry = nullptr;
        if (cudaEventCreateWithFlags(&entry, cudaEventDisableTiming) != cudaSuccess)
            return cuda_err(cudaGetLastError(), "cudaEventCreate");
        R->xev.push_back(entry);
        cudaEventRecord(entry, st);
        cudaStreamWaitEvent(P->k3s[0], entry, 0);
        cudaStreamWaitEvent(P->k3s[1], entry, 0);
    }
    for (uint64_t lo = b, hi = b; lo < e; lo = hi) {
        hi = e - lo < kMaxSub ? e : lo + kMaxSub;
        // sub-ranges end at row boundaries: only the call's own first and last
        // rows can be cut
        const uint64_t g0 = H.row_of(lo);
        if (hi < e) {
            const uint64_t cut = H.row_start(H.row_of(hi));
            if (cut > lo) hi = cut;
        }
        if (H.row_of(hi - 1) + 1 - g0 > P->max_rows) {
            const uint64_t cut = H.row_start(g0 + P->max_rows);
            if (cut > lo) hi = cut;
        }
        const uint32_t n_rows = (uint32_t)(H.row_of(hi - 1) + 1 - g0);
        // segments of rows g0 and g0 + n_rows - 1 (K0 searches only between them)
        const uint32_t seg_lo = seg_of(g0);
        const uint32_t n_seg_sub = seg_of(g0 + n_rows - 1) - seg_lo + 2;
        me_plan::Scratch& sc = P->scratch[P->turn++ % P->n_sets];
        cudaEvent_t tev[5];
        for (auto& x : tev) {
            if (cudaEventCreate(&x) != cudaSuccess) return cuda_err(cudaGetLastError(), "cudaEventCreate");
            R->tev.push_back(x);
        }
        cudaStreamWaitEvent(cs, sc.free_ev, 0);
        cudaEventRecord(tev[0], cs);
        cudaError_t ce;
        ce = launch_rowcount(P->ds, g0, n_rows, seg_lo, n_seg_sub, lo, hi, sc.rows, sc.st, sc.rcnt, sc.ucnt,
                             stats, !write || !P->k3_caps[mode], write,
                             (uint32_t)(P->sms * (write ? P->k0_wbps : P->k0_bps)), cs);
        if (ce != cudaSuccess) return cuda_err(ce, "row kernel");
        cudaEventRecord(tev[1], cs);
        if (write) {
            // counts only: K0 summed them
            ce = launch_scan(sc.ucnt, fused_units_of(n_rows), sc.uoff, stats, cs);
            if (ce != cudaSuccess) return cuda_err(ce, "scan kernel");
        }
        cudaEventRecord(tev[2], cs);
        if (write) {
            cudaStream_t ks = alt ? P->k3s[n_sub & 1] : st;
            if (alt) used[n_sub & 1] = true;
            n_sub++;
            cudaStreamWaitEvent(ks, tev[2], 0);
            cudaEventRecord(tev[3], ks);
            DevSpace dsk = P->ds;
            dsk.k3_caps = (uint32_t)P->k3_caps[mode];
            ce = launch_fused(dsk, sc.rows, sc.st, sc.rcnt, sc.ucnt, sc.uoff, n_rows, lo, hi, mode, cols, capacity,
                              (uint32_t)(P->sms * P->fused_bps[mode]), P->fused_minb[mode], sc.rnext, stats, ks);
            if (ce != cudaSuccess) return cuda_err(ce, "fused kernel");
            cudaEventRecord(tev[4], ks);
            cudaEventRecord(sc.free_ev, ks);
        } else {
            cudaEventRecord(tev[3], cs);
            cudaEventRecord(tev[4], cs);
            cudaEventRecord(sc.free_ev, cs);
        }
    }
    // the caller's stream waits for the call's K3s (output rows, capacity counts)
    for (int i = 0; i < 2; i++)
        if (used[i]) {
            cudaEventRecord(P->k3_ev[i], P->k3s[i]);
            cudaStreamWaitEvent(st, P->k3_ev[i], 0);
        }
    return ME_OK;
}

static int plan_sweep(me_plan* P, const me_sweep_opts* o, bool own_plan, me_result** out) {
    if (!P || !o || !out) return err(ME_EINVAL, "null argument");
    if (o->mode != ME_OUT_COUNT && o->mode != ME_OUT_INDEX && o->mode != ME_OUT_FULL && o->mode != ME_OUT_RECORDS)
        return err(ME_EINVAL, "bad output mode");
    DeviceGuard g(P->device);
    cudaStream_t st = (cudaStream_t)o->stream;
    uint64_t total = P->hs.total;
    uint64_t b = o->begin, e = o->end ? o->end : total;
    if (e > total) e = total;
    if (b > e) b = e;
    if (o->partition != ME_PART_EVEN && o->partition != ME_PART_CYCLIC) return err(ME_EINVAL, "bad partition");
    if (o->comm && o->partition == ME_PART_EVEN) {
        uint64_t lo = 0, hi = 0;
        me_partition(b, e, o->comm->rank, o->comm->nranks, &lo, &hi);
        b = lo;
        e = hi;
    }
    me_result* R = new (std::nothrow) me_result();
    if (!R) return err(ME_ENOMEM, "host allocation");
    R->plan = P;
    R->A = P->A;
    R->A.stream = st;
    R->stream = st;
    R->mode = o->mode;
    R->n_cap = P->ds.n_cap;
    R->begin = b;
    R->end = e;
    R->partition = o->partition;
    // a CYCLIC call is one block of a cyclic deal: swept by this rank alone,
    // joined with the others later by me_result_join
    R->comm = o->partition == ME_PART_EVEN ? o->comm : nullptr;
    R->gather = R->comm && o->gather;
    int rc = ME_OK;
    auto fail = [&](int s) {
        R->own_plan = false;
        result_release(R);
        return s;
    };
    for (int i = 0; i < 6; i++)
        if (cudaEventCreate(&R->ev[i]) != cudaSuccess) return fail(cuda_err(cudaErrorUnknown, "cudaEventCreate"));
    R->stats = (uint64_t*)R->A.get(9 * 8);
    if (!R->stats) return fail(err(ME_ENOMEM, "stats allocation"));

    // K0 + scan run on the plan stream, which waits for the tables and, per
    // sub-range, for the output kernel that last used the scratch set: K0 of
    // sub-range i+1 (or of the next call) runs while the caller's stream still
    // writes the rows of sub-range i.  Counts go to a plan-owned slot (see
    // me_plan::pstats) that the caller's stream copies into the result.
    // COUNT: K0 alone, nothing to overlap -- it runs on the caller's stream
    // and counts straight into the result (no stream hand-offs per call).
    const int nc = n_cols_of(o->mode);
    const bool direct = nc == 0;
    cudaStream_t cs = P->serial || direct ? st : P->cstream;
    const uint32_t slot = direct ? 0u : P->stat_turn++ % me_plan::kStatSlots;
    uint64_t* pst = direct ? R->stats : P->pstats + (size_t)slot * 16;
    if (!direct) cudaStreamWaitEvent(cs, P->stat_ev[slot], 0);
    cudaStreamWaitEvent(cs, P->ready_ev, 0);
    const uint64_t len = e - b;
    cudaEventRecord(R->ev[0], cs);
    Cols cols{};
    if (nc && len) {
        if (o->out_cols) {
            for (int j = 0; j < nc; j++) {
                R->cols[j] = o->out_cols[j];
                if (!R->cols[j]) return fail(err(ME_EINVAL, "null caller column"));
            }
            R->capacity = o->out_capacity;
        } else {
            // exact allocation: a counting pass first (K0 + scan; synchronises the host once)
            if ((rc = run_pipeline(P, R, pst, b, e, cs, st, o->mode, false, cols, 0))) return fail(rc);
            uint64_t cnt = 0;
            cudaEventRecord(R->ev[2], cs);
            cudaStreamWaitEvent(st, R->ev[2], 0);
            if (cudaMemcpyAsync(&cnt, pst, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                return fail(cuda_err(cudaGetLastError(), "count readback"));
            R->own_cols = true;
            for (int j = 0; j < nc; j++) {
                R->cols[j] = (uint64_t*)R->A.get(cnt * 8 * words_of(o->mode));
                if (!R->cols[j]) return fail(err(ME_ENOMEM, "result column allocation"));
            }
            R->capacity = cnt;
            for (cudaEvent_t x : R->tev) cudaEventDestroy(x);
            R->tev.clear();
        }
        for (int j = 0; j < ME_N_COLS; j++) cols.c[j] = R->cols[j];
    }
    if ((rc = run_pipeline(P, R, pst, b, e, cs, st, o->mode, nc != 0, cols, R->capacity))) return fail(rc);
    R->ran_count = len != 0;
    R->ran_write = nc && len;
    cudaEventRecord(R->ev[2], cs);
    cudaStreamWaitEvent(st, R->ev[2], 0);  // counts complete before the caller's stream reads them
    if (!direct) {
        if (cudaMemcpyAsync(R->stats, pst, 9 * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return fail(cuda_err(cudaGetLastError(), "stats copy"));
        cudaEventRecord(P->stat_ev[slot], st);
    }
    cudaEventRecord(R->ev[3], st);
    if (o->comm && o->partition == ME_PART_EVEN) {
        R->gathered = (uint64_t*)R->A.get((size_t)o->comm->nranks * 9 * 8);
        if (!R->gathered) return fail(err(ME_ENOMEM, "gather buffer"));
        ncclResult_t nr = ncclAllGather(R->stats, R->gathered, 9, ncclUint64, o->comm->nccl, st);
        if (nr != ncclSuccess) return fail(err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr)));
        if (R->gather && nc) {
            if ((rc = resolve(R))) return fail(rc);
            // variable-size allgather of the columns: one broadcast per rank
            const int nr_ = o->comm->nranks;
            std::vector<uint64_t> cnt(nr_), off(nr_ + 1, 0);
            std::vector<uint64_t> h((size_t)nr_ * 9);
            if (cudaMemcpy(h.data(), R->gathered, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
                return fail(cuda_err(cudaGetLastError(), "gathered readback"));
            for (int r = 0; r < nr_; r++) {
                cnt[r] = h[(size_t)r * 9];
                off[r + 1] = off[r] + cnt[r];
            }
            R->g_rows = off[nr_];
            // every rank must enter the broadcasts or none: agree on failures
            // (caller columns overflowed, allocation failed) first
            uint64_t bad = R->capacity < R->local ? 1u : 0u;
            for (int j = 0; j < nc && !bad; j++) {
                R->gcols[j] = (uint64_t*)R->A.get(R->g_rows * 8 * words_of(o->mode));
                if (!R->gcols[j]) bad = 2;
            }
            uint64_t* dflag = (uint64_t*)R->A.get((size_t)(nr_ + 1) * 8);
            if (!dflag) return fail(err(ME_ENOMEM, "flag buffer"));  // (allocation of a few bytes)
            std::vector<uint64_t> flags(nr_, 0);
            if (cudaMemcpyAsync(dflag, &bad, 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
                R->A.put(dflag);
                return fail(cuda_err(cudaGetLastError(), "flag upload"));
            }
            nr = ncclAllGather(dflag, dflag + 1, 1, ncclUint64, o->comm->nccl, st);
            cudaError_t fe = nr == ncclSuccess ? cudaMemcpyAsync(flags.data(), dflag + 1, (size_t)nr_ * 8,
                                                                 cudaMemcpyDeviceToHost, st)
                                               : cudaSuccess;
            if (fe == cudaSuccess) fe = cudaStreamSynchronize(st);
            R->A.put(dflag);
            if (nr != ncclSuccess) return fail(err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr)));
            if (fe != cudaSuccess) return fail(cuda_err(fe, "flag readback"));
            uint64_t any = 0;
            for (uint64_t f : flags) any |= f;
            if (any & 1) return fail(err(ME_ERANGE, "a rank's caller columns overflowed; cannot gather"));
            if (any) return fail(err(ME_ENOMEM, "a rank could not allocate the gathered columns"));
            ncclGroupStart();
            for (int j = 0; j < nc; j++)
                for (int r = 0; r < nr_; r++) {
                    if (!cnt[r]) continue;
                    const uint64_t wd = words_of(o->mode);
                    nr = ncclBroadcast(r == o->comm->rank ? (const void*)R->cols[j] : nullptr,
                                       R->gcols[j] + off[r] * wd, cnt[r] * wd, ncclUint64, r, o->comm->nccl, st);
                    if (nr != ncclSuccess) break;
                }
            ncclResult_t ng = ncclGroupEnd();
            if (nr != ncclSuccess || ng != ncclSuccess)
                return fail(err(ME_ENCCL, std::string("ncclBroadcast: ") + ncclGetErrorString(nr != ncclSuccess ? nr : ng)));
        }
    }
    cudaEventRecord(R->ev[4], st);
    if (cudaError_t ce = cudaGetLastError()) return fail(cuda_err(ce, "me_plan_sweep"));
    R->own_plan = own_plan;
    *out = R;
    return ME_OK;
}

extern "C" int me_plan_sweep(me_plan* plan, const me_sweep_opts* opts, me_result** out) {
    return plan_sweep(plan, opts, false, out);
}

extern "C" int me_sweep(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
                        me_threshold thr, const me_sweep_opts* opts, me_result** out) {
    if (!opts || !out) return err(ME_EINVAL, "null argument");
    me_plan* P = nullptr;
    int st = plan_create(models, cluster, cfg, thr, opts->device, opts->stream, opts->alloc, opts->free,
                         opts->alloc_ctx, &P);
    if (st) return st;
    st = plan_sweep(P, opts, true, out);
    if (st) me_plan_free(P);
    return st;
}

// read device stats (waits)
static int resolve(me_result* R) {
    if (R->resolved) return ME_OK;
    DeviceGuard g(R->plan->device);
    CU(cudaStreamSynchronize(R->stream));
    uint64_t h[9];
    CU(cudaMemcpy(h, R->stats, sizeof h, cudaMemcpyDeviceToHost));
    R->local = h[0];
    for (int q = 0; q < 8; q++) R->caps[q] = h[1 + q];
    R->global = R->local;
    R->offset = 0;
    if (R->join) {
        JoinState* J = R->join;
        if (!J->resolved) {
            CU(cudaEventSynchronize(J->done));
            J->host.resize(17 + (size_t)J->n);
            CU(cudaMemcpy(J->host.data(), J->out, J->host.size() * 8, cudaMemcpyDeviceToHost));
            J->resolved = true;
        }
        R->global = J->host[0];
        for (int q = 0; q < 8; q++) R->caps[q] = J->host[1 + q];
        R->offset = J->host[17 + R->join_k];
    }
    if (R->comm) {
        std::vector<uint64_t> all((size_t)R->comm->nranks * 9);
        CU(cudaMemcpy(all.data(), R->gathered, all.size() * 8, cudaMemcpyDeviceToHost));
        me_join_counts(all.data(), R->comm->nranks, 9, 8, R->comm->rank, &R->offset, &R->global, R->caps);
    }
    R->resolved = true;
    return ME_OK;
}

extern "C" int me_result_wait(me_result* R) {
    if (!R) return err(ME_EINVAL, "null result");
    DeviceGuard g(R->plan->device);
    CU(cudaEventSynchronize(R->ev[4]));
    return ME_OK;
}

extern "C" int me_result_counts(me_result* R, uint64_t* local, uint64_t* global, uint64_t* rank_offset) {
    if (!R) return err(ME_EINVAL, "null result");
    int st = resolve(R);
    if (st) return st;
    if (local) *local = R->local;
    if (global) *global = R->global;
    if (rank_offset) *rank_offset = R->offset;
    return ME_OK;
}

extern "C" int me_result_cap_counts(me_result* R, uint64_t* per_cap) {
    if (!R || !per_cap) return err(ME_EINVAL, "null argument");
    int st = resolve(R);
    if (st) return st;
    for (uint32_t q = 0; q < R->n_cap; q++) per_cap[q] = R->caps[q];
    return ME_OK;
}

extern "C" int me_result_status(me_result* R) {
    if (!R) return err(ME_EINVAL, "null result");
    int st = resolve(R);
    if (st) return st;
    if (n_cols_of(R->mode) && R->local > R->capacity)
        return err(ME_ERANGE, "caller columns too small: need " + std::to_string(R->local) + " rows");
    return ME_OK;
}

extern "C" int me_result_columns(me_result* R, uint64_t** cols, uint64_t* n_rows) {
    if (!R || !cols) return err(ME_EINVAL, "null argument");
    int st = resolve(R);
    if (st) return st;
    const bool g = R->gather && n_cols_of(R->mode);
    for (int j = 0; j < ME_N_COLS; j++) cols[j] = g ? R->gcols[j] : R->cols[j];
    if (n_rows) {
        uint64_t n = g ? R->g_rows : R->local;
        if (!g && n > R->capacity) n = R->capacity;
        *n_rows = n_cols_of(R->mode) ? n : 0;
    }
    return ME_OK;
}

extern "C" int me_result_copy_to_host(me_result* R, uint64_t first, uint64_t n, uint64_t* const* cols_host) {
    if (!R || !cols_host) return err(ME_EINVAL, "null argument");
    uint64_t* cols[ME_N_COLS];
    uint64_t rows = 0;
    int st = me_result_columns(R, cols, &rows);
    if (st) return st;
    if (first > rows || n > rows - first) return err(ME_ERANGE, "rows out of bounds");
    if (!n) return ME_OK;
    DeviceGuard g(R->plan->device);
    for (int j = 0; j < ME_N_COLS; j++) {
        if (!cols_host[j]) continue;
        if (!cols[j]) return err(ME_EINVAL, "column not produced in this mode");
        const uint64_t wd = words_of(R->mode);
        CU(cudaMemcpyAsync(cols_host[j], cols[j] + first * wd, n * 8 * wd, cudaMemcpyDeviceToHost, R->stream));
    }
    CU(cudaStreamSynchronize(R->stream));
    return ME_OK;
}

extern "C" int me_result_timing(me_result* R, float* ms) {
    if (!R || !ms) return err(ME_EINVAL, "null argument");
    DeviceGuard g(R->plan->device);
    CU(cudaEventSynchronize(R->ev[4]));
    CU(cudaEventElapsedTime(&ms[0], R->ev[0], R->ev[4]));
    ms[1] = ms[2] = ms[3] = 0.f;
    for (size_t k = 0; k + 5 <= R->tev.size(); k += 5) {
        float a = 0, b = 0, c = 0;
        CU(cudaEventElapsedTime(&a, R->tev[k], R->tev[k + 1]));
        CU(cudaEventElapsedTime(&b, R->tev[k + 1], R->tev[k + 2]));
        CU(cudaEventElapsedTime(&c, R->tev[k + 3], R->tev[k + 4]));
        ms[1] += a;
        ms[2] += b;
        ms[3] += c;
    }
    if (!R->ran_write) ms[3] = 0.f;
    return ME_OK;
}

extern "C" void me_result_free(me_result* R) { result_release(R); }

extern "C" int me_result_rank(me_result* R, const me_rank_opts* o, me_rank_row* out) {
    if (!R || !o || !out) return err(ME_EINVAL, "null argument");
    if (o->k < 1) return err(ME_EINVAL, "k must be >= 1");
    if (o->green_cap >= R->n_cap || (o->yellow_cap != ME_RANK_NONE && o->yellow_cap >= R->n_cap))
        return err(ME_EINVAL, "capacity slot out of range");
    if (R->mode == ME_OUT_COUNT) return err(ME_EINVAL, "ranking needs an INDEX, FULL or RECORDS result");
    uint64_t* cols[ME_N_COLS];
    uint64_t rows = 0;
    int st = me_result_columns(R, cols, &rows);
    if (st) return st;
    if (!R->gather && R->local > R->capacity) return err(ME_ERANGE, "caller columns overflowed");
    me_plan* P = R->plan;
    const HostSpace& H = P->hs;
    DeviceGuard g(P->device);
    const size_t n_seg = H.seg_prefix.size() - 1, m = n_seg * o->k;
    // a sharded comm result: every rank ranks its own rows, the candidates of
    // all ranks are allgathered and merged per segment (collective)
    const int nr = R->comm && !R->gather ? R->comm->nranks : 1;
    // scratch from the result's allocator, ordered on its stream
    uint64_t* keys = (uint64_t*)R->A.get((rows ? rows : 1) * 8);
    uint64_t* sel = (uint64_t*)R->A.get(m * 8);
    uint64_t* dout = (uint64_t*)R->A.get(m * 16 * (size_t)(nr > 1 ? nr + 1 : 1));
    std::vector<uint64_t> h(2 * m * (size_t)nr);
    cudaError_t ce = keys && sel && dout ? cudaSuccess : cudaErrorMemoryAllocation;
    if (ce == cudaSuccess)
        ce = launch_rank(P->ds, cols[0], (uint32_t)words_of(R->mode), rows, o->green_cap,
                         o->yellow_cap == ME_RANK_NONE ? 8u : o->yellow_cap, o->gpus_per_node, o->k, keys, sel, dout,
                         R->stream);
    ncclResult_t ncr = ncclSuccess;
    if (ce == cudaSuccess && nr > 1)
        ncr = ncclAllGather(dout, dout + 2 * m, 2 * m, ncclUint64, R->comm->nccl, R->stream);
    if (ce == cudaSuccess && ncr == ncclSuccess)
        ce = cudaMemcpyAsync(h.data(), nr > 1 ? dout + 2 * m : dout, h.size() * 8, cudaMemcpyDeviceToHost, R->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(R->stream);
    R->A.put(keys);
    R->A.put(sel);
    R->A.put(dout);
    if (ncr != ncclSuccess) return err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(ncr));
    if (ce == cudaErrorMemoryAllocation) return err(ME_ENOMEM, "rank scratch");
    if (ce != cudaSuccess) return cuda_err(ce, "me_result_rank");
    if (nr > 1) {
        // per segment the k smallest (key, flat index) of the nr * k candidates
        std::vector<uint64_t> merged(2 * m);
        std::vector<std::pair<uint64_t, uint64_t>> cand;
        for (size_t sgi = 0; sgi < n_seg; sgi++) {
            cand.clear();
            for (int r = 0; r < nr; r++)
                for (uint32_t q = 0; q < o->k; q++) {
                    const uint64_t* x = &h[2 * ((size_t)r * m + sgi * o->k + q)];
                    if (x[0] != ~0ull) cand.emplace_back(x[1], x[0]);
                }
            std::sort(cand.begin(), cand.end(), [](const std::pair<uint64_t, uint64_t>& a,
                                                  const std::pair<uint64_t, uint64_t>& b) {
                return a.first != b.first ? a.first < b.first
                                          : (a.second & ((1ull << 56) - 1)) < (b.second & ((1ull << 56) - 1));
            });
            for (uint32_t q = 0; q < o->k; q++) {
                merged[2 * (sgi * o->k + q)] = q < cand.size() ? cand[q].second : ~0ull;
                merged[2 * (sgi * o->k + q) + 1] = q < cand.size() ? cand[q].first : ~0ull;
            }
        }
        h.swap(merged);
    }
    // decode the selected rows on the host (n_seg * k of them)
    for (size_t i = 0; i < m; i++) {
        me_rank_row x{};
        x.index = h[2 * i] == ~0ull ? ~0ull : (h[2 * i] & ((1ull << 56) - 1));
        x.key = h[2 * i + 1];
        if (x.index != ~0ull) {
            if (H.decode(x.index, &x.model_id, &x.world_size, &x.cfg)) return err(ME_ECUDA, "rank decode");
            x.cls = (uint32_t)(x.key >> 62);
            if (H.gbs) {
                x.microbatches = (uint32_t)(H.gbs / ((uint64_t)x.cfg.dp * x.cfg.mbs));
                x.bubble_num = x.cfg.pp - 1;
                x.bubble_den = x.microbatches;
            }
        }
        out[i] = x;
    }
    return ME_OK;
}

extern "C" int me_result_digest(me_result* R, uint64_t* digest) {
    if (!R || !digest) return err(ME_EINVAL, "null argument");
    if (R->mode == ME_OUT_COUNT) return err(ME_EINVAL, "a COUNT result has no rows to digest");
    uint64_t* cols[ME_N_COLS];
    uint64_t rows = 0;
    int st = me_result_columns(R, cols, &rows);
    if (st) return st;
    if (!(R->gather) && R->local > R->capacity) return err(ME_ERANGE, "caller columns overflowed");
    DeviceGuard g(R->plan->device);
    const bool sharded = R->comm && !R->gather;
    const int nr = sharded ? R->comm->nranks : 1;
    uint64_t* d = (uint64_t*)R->A.get((size_t)(2 + 2 * nr) * 8);
    if (!d) return err(ME_ENOMEM, "digest scratch");
    const uint32_t n_cols = R->mode == ME_OUT_FULL ? ME_N_COLS : 1;
    cudaError_t ce = launch_digest(cols, n_cols, (uint32_t)words_of(R->mode), rows, d, R->stream);
    std::vector<uint64_t> h((size_t)2 * nr);
    if (ce == cudaSuccess && sharded) {
        // collective: every rank's digest, merged in rank order with the
        // global offsets: D = sum_r M^offset_r D_r
        ncclResult_t r = ncclAllGather(d, d + 2, 2, ncclUint64, R->comm->nccl, R->stream);
        if (r != ncclSuccess) {
            R->A.put(d);
            return err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
        }
        ce = cudaMemcpyAsync(h.data(), d + 2, h.size() * 8, cudaMemcpyDeviceToHost, R->stream);
    } else if (ce == cudaSuccess) {
        ce = cudaMemcpyAsync(h.data(), d, 16, cudaMemcpyDeviceToHost, R->stream);
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(R->stream);
    R->A.put(d);
    if (ce != cudaSuccess) return cuda_err(ce, "me_result_digest");
    if (!sharded) {
        digest[0] = h[0];
        digest[1] = R->mode == ME_OUT_INDEX ? 0 : h[1];
        return ME_OK;
    }
    std::vector<uint64_t> all((size_t)nr * 9);
    CU(cudaMemcpy(all.data(), R->gathered, all.size() * 8, cudaMemcpyDeviceToHost));
    uint64_t off = 0, di = 0, dr = 0;
    for (int r = 0; r < nr; r++) {
        const uint64_t sh = digest_pow_host(off);
        di += sh * h[2 * r];
        dr += sh * h[2 * r + 1];
        off += all[(size_t)r * 9];
    }
    digest[0] = di;
    digest[1] = R->mode == ME_OUT_INDEX ? 0 : dr;
    return ME_OK;
}

extern "C" int me_digest_merge(uint64_t n, const uint64_t* counts, const uint64_t* digests, uint64_t out[2]) {
    if (!out || (n && (!counts || !digests))) return err(ME_EINVAL, "null argument");
    uint64_t off = 0, di = 0, dr = 0;
    for (uint64_t i = 0; i < n; i++) {
        const uint64_t sh = digest_pow_host(off);
        di += sh * digests[2 * i];
        dr += sh * digests[2 * i + 1];
        off += counts[i];
    }
    out[0] = di;
    out[1] = dr;
    return ME_OK;
}

extern "C" int me_comm_check(me_comm* c) {
    if (!c) return err(ME_EINVAL, "null comm");
    ncclResult_t a = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->nccl, &a);
    if (r != ncclSuccess) return err(ME_ENCCL, std::string("ncclCommGetAsyncError: ") + ncclGetErrorString(r));
    if (a != ncclSuccess && a != ncclInProgress)
        return err(ME_ENCCL, std::string("asynchronous NCCL error: ") + ncclGetErrorString(a));
    return ME_OK;
}

// ---------------------------------------------------------------------------
// single estimates
// ---------------------------------------------------------------------------
static bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

extern "C" int me_estimate_batch(const me_model* models, uint32_t n_models, const uint32_t* ids,
                                 const me_parallel* cfgs, uint64_t n, const uint64_t* caps, uint32_t n_cap,
                                 me_threshold thr, me_breakdown* out, uint8_t* mask, uint8_t* status,
                                 void* stream) {
    if (!models || !n_models || !cfgs) return err(ME_EINVAL, "null argument");
    if (n_cap > 8 || (n_cap && !caps)) return err(ME_EINVAL, "n_cap must be <= 8");
    if (thr.num < 1 || thr.den < 1 || thr.num > 1024 || thr.den > 1024)
        return err(ME_EINVAL, "threshold num/den must be in [1, 1024]");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return err(ME_ECUDA, "no CUDA device");
    }
    if (!n) return ME_OK;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<void*> tmp;
    // scratch: stream-ordered allocations on the caller's stream (the call has
    // no allocator argument; me.h: cudaMallocAsync when none is given)
    auto stage_in = [&](const void* p, size_t bytes, const void** dp) -> int {
        if (!p) { *dp = nullptr; return ME_OK; }
        if (is_device_ptr(p)) { *dp = p; return ME_OK; }
        void* d = nullptr;
        CU(cudaMallocAsync(&d, bytes, st));
        tmp.push_back(d);
        CU(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, st));
        *dp = d;
        return ME_OK;
    };
    auto stage_out = [&](void* p, size_t bytes, void** dp) -> int {
        if (!p) { *dp = nullptr; return ME_OK; }
        if (is_device_ptr(p)) { *dp = p; return ME_OK; }
        void* d = nullptr;
        CU(cudaMallocAsync(&d, bytes, st));
        tmp.push_back(d);
        *dp = d;
        return ME_OK;
    };
    uint64_t thr_h[8] = {0};
    for (uint32_t q = 0; q < n_cap; q++) {
        uint64_t c;
        if (is_device_ptr(caps)) {
            CU(cudaMemcpy(&c, caps + q, 8, cudaMemcpyDeviceToHost));
        } else {
            c = caps[q];
        }
        thr_h[q] = threshold_of(c, thr);
    }
    const void *dm, *di, *dc, *dt;
    void *dout, *dmask, *dstat;
    int rc;
    auto cleanup = [&]() {
        for (void* p : tmp) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
    };
    if ((rc = stage_in(models, (size_t)n_models * sizeof(me_model), &dm)) ||
        (rc = stage_in(ids, n * 4, &di)) || (rc = stage_in(cfgs, n * sizeof(me_parallel), &dc)) ||
        (rc = stage_in(thr_h, sizeof thr_h, &dt)) || (rc = stage_out(out, n * sizeof(me_breakdown), &dout)) ||
        (rc = stage_out(mask, n, &dmask))) {
        cleanup();
        return rc;
    }
    // per-config status is always produced on the device
    if (status && is_device_ptr(status)) {
        dstat = status;
    } else {
        if (cudaMallocAsync(&dstat, n, st) != cudaSuccess) { cleanup(); return cuda_err(cudaGetLastError(), "cudaMallocAsync"); }
        tmp.push_back(dstat);
    }
    cudaError_t ce = launch_estimate((const me_model*)dm, n_models, (const uint32_t*)di, (const me_parallel*)dc,
                                     n, (const uint64_t*)dt, n_cap, (me_breakdown*)dout, (uint8_t*)dmask,
                                     (uint8_t*)dstat, st);
    if (ce != cudaSuccess) { cleanup(); return cuda_err(ce, "estimate kernel"); }
    std::vector<uint8_t> hstat(n);
    int first_bad = ME_OK;
    ce = cudaMemcpyAsync(hstat.data(), dstat, n, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && out && dout != out)
        ce = cudaMemcpyAsync(out, dout, n * sizeof(me_breakdown), cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && mask && dmask != mask) ce = cudaMemcpyAsync(mask, dmask, n, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess && status && dstat != status) ce = cudaMemcpyAsync(status, dstat, n, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    cleanup();
    if (ce != cudaSuccess) return cuda_err(ce, "estimate readback");
    for (uint64_t i = 0; i < n; i++)
        if (hstat[i]) { first_bad = hstat[i]; break; }
    if (!status && first_bad) return err(first_bad, "a configuration failed its preconditions");
    return ME_OK;
}

extern "C" int me_estimate_stage(const me_model* model, const me_parallel* cfg, uint32_t stage, me_breakdown* out,
                                 uint32_t* which) {
    if (!model || !cfg || !out) return err(ME_EINVAL, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return err(ME_ECUDA, "no CUDA device");
    }
    struct Buf {
        me_model m;
        me_parallel c;
        me_breakdown b;
        uint32_t which;
        int status;
    };
    Buf h{};
    h.m = *model;
    h.c = *cfg;
    Buf* d = nullptr;
    cudaStream_t s0 = nullptr;  // the legacy default stream, like me_estimate
    CU(cudaMallocAsync(&d, sizeof(Buf), s0));
    cudaError_t ce = cudaMemcpyAsync(d, &h, sizeof(Buf), cudaMemcpyHostToDevice, s0);
    if (ce == cudaSuccess) ce = launch_estimate_stage(&d->m, &d->c, stage, &d->b, &d->which, &d->status, s0);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&h, d, sizeof(Buf), cudaMemcpyDeviceToHost, s0);
    cudaFreeAsync(d, s0);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s0);
    if (ce != cudaSuccess) return cuda_err(ce, "me_estimate_stage");
    if (h.status) return err(h.status, "estimator precondition failed");
    *out = h.b;
    if (which) *which = h.which;
    return ME_OK;
}

extern "C" int me_estimate(const me_model* model, const me_parallel* cfg, me_breakdown* out) {
    if (!model || !cfg || !out) return err(ME_EINVAL, "null argument");
    me_breakdown b;
    uint8_t s = 0;
    me_threshold thr{4, 5};
    int st = me_estimate_batch(model, 1, nullptr, cfg, 1, nullptr, 0, thr, &b, nullptr, &s, nullptr);
    if (st) return st;
    if (s) return err(s, "estimator precondition failed");
    *out = b;
    return ME_OK;
}

// ---------------------------------------------------------------------------
// host-only space queries
// ---------------------------------------------------------------------------
extern "C" int me_space_size(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
                             uint64_t* n) {
    if (!n) return err(ME_EINVAL, "null out");
    HostSpace H;
    std::string d;
    int st = H.build(models, cluster, cfg, false, &d);
    if (st) return err(st, d);
    *n = H.total;
    return ME_OK;
}

extern "C" int me_decode(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
                         uint64_t index, uint32_t* model_id, uint32_t* world_size, me_parallel* out) {
    HostSpace H;
    std::string d;
    int st = H.build(models, cluster, cfg, false, &d);
    if (st) return err(st, d);
    st = H.decode(index, model_id, world_size, out);
    if (st) return err(st, "index past the end of the space");
    return ME_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU host logic (used by plan_sweep / resolve; exported for tests)
// ---------------------------------------------------------------------------
extern "C" int me_partition(uint64_t begin, uint64_t end, int rank, int nranks, uint64_t* lo, uint64_t* hi) {
    if (!lo || !hi || nranks < 1 || rank < 0 || rank >= nranks || end < begin)
        return err(ME_EINVAL, "bad partition arguments");
    const uint64_t len = end - begin, n = (uint64_t)nranks, r = (uint64_t)rank;
    const uint64_t q = len / n, rem = len % n;
    *lo = begin + q * r + (rem * r) / n;
    *hi = begin + q * (r + 1) + (rem * (r + 1)) / n;
    return ME_OK;
}

extern "C" int me_join_counts(const uint64_t* stats, int nranks, uint32_t stride, uint32_t n_cap, int rank,
                              uint64_t* offset, uint64_t* global, uint64_t* cap_global) {
    if (!stats || nranks < 1 || rank < 0 || rank >= nranks || stride < 1 + n_cap)
        return err(ME_EINVAL, "bad join arguments");
    uint64_t off = 0, tot = 0;
    for (uint32_t q = 0; q < n_cap && cap_global; q++) cap_global[q] = 0;
    for (int r = 0; r < nranks; r++) {
        const uint64_t* row = stats + (size_t)r * stride;
        if (r < rank) off += row[0];
        tot += row[0];
        for (uint32_t q = 0; q < n_cap && cap_global; q++) cap_global[q] += row[1 + q];
    }
    if (offset) *offset = off;
    if (global) *global = tot;
    return ME_OK;
}


// ---------------------------------------------------------------------------
// a8: cyclic partition + deferred join
// ---------------------------------------------------------------------------
extern "C" int me_cyclic_block(uint64_t begin, uint64_t end, uint64_t block, int rank, int nranks, uint64_t k,
                               uint64_t* lo, uint64_t* hi, uint64_t* n_blocks) {
    if (!block || nranks < 1 || rank < 0 || rank >= nranks || end < begin)
        return err(ME_EINVAL, "bad cyclic partition arguments");
    const uint64_t nb = (end - begin + block - 1) / block;
    if (n_blocks) *n_blocks = nb;
    const uint64_t q = k * (uint64_t)nranks + (uint64_t)rank;
    if (k >= nb || q >= nb) return err(ME_ERANGE, "this rank has no such block");
    if (lo) *lo = begin + q * block;
    if (hi) *hi = std::min(end, begin + (q + 1) * block);
    return ME_OK;
}

extern "C" int me_result_join(me_result* const* rs, uint32_t n, uint64_t n_blocks, me_comm* comm) {
    if (!rs || !comm) return err(ME_EINVAL, "null argument");
    const uint64_t N = (uint64_t)comm->nranks, r = (uint64_t)comm->rank;
    const uint64_t mine = n_blocks > r ? (n_blocks - r + N - 1) / N : 0;
    if (n != mine) return err(ME_EINVAL, "me_result_join needs exactly this rank's blocks of the cyclic deal");
    const uint64_t kmax = (n_blocks + N - 1) / N;
    me_result* R0 = n ? rs[0] : nullptr;
    for (uint32_t k = 0; k < n; k++) {
        if (!rs[k] || rs[k]->partition != ME_PART_CYCLIC) return err(ME_EINVAL, "results must come from CYCLIC sweeps");
        if (rs[k]->join) return err(ME_EINVAL, "a result is already joined");
        if (rs[k]->plan != R0->plan || rs[k]->stream != R0->stream)
            return err(ME_EINVAL, "joined results must share a plan and stream");
    }
    if (!R0) {
        // a rank without blocks (more ranks than blocks) still takes part in
        // the collective, with zero counts, so that the others do not wait
        DeviceGuard g(comm->device);
        const size_t words = (size_t)kmax * 9;
        uint64_t* d = nullptr;
        cudaStream_t s0 = nullptr;
        if (cudaMallocAsync(&d, words * 8 * (1 + N), s0) != cudaSuccess) return cuda_err(cudaGetLastError(), "join");
        cudaMemsetAsync(d, 0, words * 8, s0);
        ncclResult_t nr = ncclAllGather(d, d + words, words, ncclUint64, comm->nccl, s0);
        cudaFreeAsync(d, s0);
        cudaStreamSynchronize(s0);
        if (nr != ncclSuccess) return err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr));
        return ME_OK;
    }
    DeviceGuard g(R0->plan->device);
    cudaStream_t st = R0->stream;
    JoinState* J = new (std::nothrow) JoinState();
    if (!J) return err(ME_ENOMEM, "host allocation");
    J->A = R0->A;
    J->n = n;
    const size_t local = (size_t)kmax * 9, all = (size_t)N * kmax * 9;
    J->buf = (uint64_t*)J->A.get((local + all + 17 + kmax) * 8);
    if (!J->buf) {
        delete J;
        return err(ME_ENOMEM, "join buffer");
    }
    J->out = J->buf + local + all;
    auto bail = [&](int s) {
        cudaStreamSynchronize(st);
        J->A.put(J->buf);
        if (J->done) cudaEventDestroy(J->done);
        delete J;
        return s;
    };
    if (cudaEventCreateWithFlags(&J->done, cudaEventDisableTiming) != cudaSuccess)
        return bail(cuda_err(cudaGetLastError(), "cudaEventCreate"));
    // this rank's per-block counts, in block order (the results' stats were
    // written on this stream)
    cudaError_t ce = cudaMemsetAsync(J->buf, 0, local * 8, st);
    for (uint32_t k = 0; k < n && ce == cudaSuccess; k++)
        ce = cudaMemcpyAsync(J->buf + (size_t)k * 9, rs[k]->stats, 72, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return bail(cuda_err(ce, "join staging"));
    ncclResult_t nr = ncclAllGather(J->buf, J->buf + local, local, ncclUint64, comm->nccl, st);
    if (nr != ncclSuccess) return bail(err(ME_ENCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr)));
    ce = launch_join(J->buf + local, comm->nranks, comm->rank, (uint32_t)kmax, n_blocks, J->out, st);
    if (ce != cudaSuccess) return bail(cuda_err(ce, "join kernel"));
    cudaEventRecord(J->done, st);
    for (uint32_t k = 0; k < n; k++) {
        rs[k]->join = J;
        rs[k]->join_k = k;
        rs[k]->resolved = false;
        J->refs++;
    }
    return ME_OK;
}

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
extern "C" int me_comm_unique_id(uint8_t id[128]) {
    if (!id) return err(ME_EINVAL, "null id");
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return err(ME_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(id, &u, 128);
    return ME_OK;
}

extern "C" int me_comm_init(const uint8_t id[128], int rank, int nranks, int device, me_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return err(ME_EINVAL, "bad comm arguments");
    DeviceGuard g(device);
    me_comm* c = new (std::nothrow) me_comm();
    if (!c) return err(ME_ENOMEM, "host allocation");
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return err(ME_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    *out = c;
    return ME_OK;
}

extern "C" int me_comm_rank(const me_comm* c, int* rank, int* nranks) {
    if (!c) return err(ME_EINVAL, "null comm");
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->nranks;
    return ME_OK;
}

extern "C" void me_comm_destroy(me_comm* c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
}

// ---------------------------------------------------------------------------
extern "C" const char* me_strerror(int s) {
    switch (s) {
        case ME_OK: return "ok";
        case ME_EINVAL: return "invalid argument";
        case ME_EDIV: return "estimator precondition (divisibility) failed";
        case ME_EOVERFLOW: return "value outside the exact 64-bit range";
        case ME_ENOMEM: return "out of memory";
        case ME_ECUDA: return "CUDA error";
        case ME_ENCCL: return "NCCL error";
        case ME_ERANGE: return "out of range / buffer too small";
        default: return "unknown status";
    }
}

extern "C" const char* me_last_error_detail(void) { return g_detail.c_str(); }

extern "C" const char* me_version(void) { return "me-b200 0.2.0 sm_100a"; }
