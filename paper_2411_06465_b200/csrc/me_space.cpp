// me_space.cpp -- builds the HostSpace tables (see me_space.hpp).
#include "me_space.hpp"

#include <algorithm>
#include <map>
#include <tuple>
#include <unordered_map>

namespace me {

static int fail(std::string* detail, int st, const std::string& msg) {
    if (detail) *detail = msg;
    return st;
}

static int popc2(uint32_t m) { return (m & 1) + ((m >> 1) & 1); }

int HostSpace::build(const me_model_range* mr, const me_cluster* cl, const me_cfg_range* cr,
                     bool for_sweep, std::string* detail) {
    if (!mr || !cl || !cr || !mr->models || !mr->n_models || !cl->world_sizes || !cl->n_world ||
        !cr->mbs || !cr->n_mbs || !cr->seq || !cr->n_seq)
        return fail(detail, ME_EINVAL, "null or empty axis");
    if (cl->n_cap > 8 || (cl->n_cap && !cl->capacity_bytes))
        return fail(detail, ME_EINVAL, "n_cap must be <= 8");
    if (!(cr->recompute_mask & 3) || (cr->recompute_mask & ~3u) || !(cr->dist_opt_mask & 3) ||
        (cr->dist_opt_mask & ~3u))
        return fail(detail, ME_EINVAL, "recompute_mask / dist_opt_mask must be 1, 2 or 3");
    models.assign(mr->models, mr->models + mr->n_models);
    world.assign(cl->world_sizes, cl->world_sizes + cl->n_world);
    caps.assign(cl->capacity_bytes, cl->capacity_bytes + cl->n_cap);
    mbs.assign(cr->mbs, cr->mbs + cr->n_mbs);
    seq.assign(cr->seq, cr->seq + cr->n_seq);
    gpus_per_node = cl->gpus_per_node;
    gbs = cr->gbs;
    max_t = cr->max_tp;
    max_c = cr->max_cp;
    max_p = cr->max_pp;
    rc_mask = cr->recompute_mask;
    do_mask = cr->dist_opt_mask;
    uneven = cr->allow_uneven_pp ? 1 : 0;
    if (cr->stage_policy > 1) return fail(detail, ME_EINVAL, "stage_policy must be 0 or 1");
    stage_max = cr->stage_policy;
    if (cr->zero_stage > 3) return fail(detail, ME_EINVAL, "zero_stage must be 0..3");
    zero_stage = (uint8_t)cr->zero_stage;
    if (cr->sp_off > 1 || cr->w_bytes > 8 || cr->g_bytes > 8 || cr->o_bytes > 16)
        return fail(detail, ME_EINVAL, "sp_off must be 0/1, w_bytes/g_bytes <= 8, o_bytes <= 16");
    sp_off = cr->sp_off;
    vpp = cr->vpp < 2 ? 0 : cr->vpp;
    wb = cr->w_bytes;
    gb = cr->g_bytes;
    ob = cr->o_bytes;
    if (vpp && (uneven || stage_max))
        return fail(detail, ME_EINVAL, "interleaved 1F1B (vpp >= 2) excludes allow_uneven_pp and ME_STAGE_MAX");

    for (size_t i = 0; i < models.size(); i++) {
        const me_model& m = models[i];
        if (!m.hidden || !m.ffn_hidden || !m.layers || !m.heads || !m.kv_heads || !m.vocab)
            return fail(detail, ME_EINVAL, "model " + std::to_string(i) + ": zero field");
        if (m.heads % m.kv_heads || m.hidden % m.heads)
            return fail(detail, ME_EINVAL, "model " + std::to_string(i) + ": needs k | a and a | h");
        if (for_sweep && (m.hidden > Limits::h || m.ffn_hidden > Limits::f ||
                          m.layers > Limits::L || m.vocab > Limits::v))
            return fail(detail, ME_EINVAL,
                        "model " + std::to_string(i) + " outside the exact-u64 sweep domain");
    }
    for (uint32_t N : world) {
        if (!N) return fail(detail, ME_EINVAL, "zero world size");
        if (for_sweep && N > Limits::N) return fail(detail, ME_EINVAL, "world size > 2^20");
    }
    for (uint32_t b : mbs) {
        if (!b) return fail(detail, ME_EINVAL, "zero mbs");
        if (for_sweep && b > Limits::b) return fail(detail, ME_EINVAL, "mbs > 2^6");
    }
    for (uint32_t s : seq) {
        if (!s) return fail(detail, ME_EINVAL, "zero seq");
        if (for_sweep && s > Limits::s) return fail(detail, ME_EINVAL, "seq > 2^20");
    }

    // innermost (rc, do) digits, rc outer, do inner
    n_rcdo = 0;
    rcdo_rc = rcdo_do = 0;
    for (uint32_t rc = 0; rc < 2; rc++) {
        if (!((rc_mask >> rc) & 1)) continue;
        for (uint32_t dd = 0; dd < 2; dd++) {
            if (!((do_mask >> dd) & 1)) continue;
            rcdo_rc |= rc << n_rcdo;
            rcdo_do |= dd << n_rcdo;
            n_rcdo++;
        }
    }
    lg_rcdo = n_rcdo == 4 ? 2 : (n_rcdo == 2 ? 1 : 0);

    // per world size: every (t, c, p) with t c p | N that passes the global
    // limits, ascending; the pooled (b, s) pairs of each
    tuples.clear();
    pairs.clear();
    pair_b.clear();
    pair_su.clear();
    pair_fence.clear();
    fenced = true;
    tup_begin.assign(1, 0);
    // (c, d|0, p|0) -> (off, n, fence offset)
    std::map<std::tuple<uint32_t, uint32_t, uint32_t>, std::tuple<uint32_t, uint32_t, uint32_t>> pool;
    std::vector<uint32_t> tvals, pvals;
    for (uint32_t N : world) {
        for (uint32_t t = 1; t <= N; t++) {
            if (N % t) continue;
            if (max_t && t > max_t) continue;
            if (gpus_per_node && t > gpus_per_node) continue;
            for (uint32_t c = 1; c <= N / t; c++) {
                if ((N / t) % c) continue;
                if (max_c && c > max_c) continue;
                for (uint32_t p = 1; p <= N / t / c; p++) {
                    if ((N / t / c) % p) continue;
                    if (max_p && p > max_p) continue;
                    uint32_t d = N / t / c / p;
                    auto key = std::make_tuple(c, gbs ? d : 0u, gbs && vpp ? p : 0u);
                    auto it = pool.find(key);
                    if (it == pool.end()) {
                        uint32_t off = (uint32_t)pairs.size();
                        for (uint32_t b : mbs)
                            for (uint32_t s : seq) {
                                if (!pair_ok(c, d, p, b, s)) continue;
                                DevPair pr;
                                pr.u = (s / c) * b;
                                pr.m = gbs ? (uint32_t)(gbs / ((uint64_t)d * b)) : 0xFFFFFFFFu;
                                pairs.push_back(pr);
                                pair_b.push_back(b);
                            }
                        const uint32_t n = (uint32_t)pairs.size() - off;
                        it = pool.emplace(key, std::make_tuple(off, n, (uint32_t)pair_fence.size())).first;
                        for (size_t q = off; q < pairs.size(); q++) pair_su.push_back(pairs[q].u);
                        std::sort(pair_su.begin() + off, pair_su.end());
                        // the pool's search index (K0): the largest u of each
                        // 32-entry group (4), then of each 8-entry block (16);
                        // past the pool's end 0xFFFFFFFF
                        if (n > 128) fenced = false;
                        for (uint32_t span : {32u, 8u})
                            for (uint32_t i = 0; i < 128 / span; i++)
                                pair_fence.push_back(n && i * span < n ? pair_su[off + std::min(n, (i + 1) * span) - 1]
                                                                       : 0xFFFFFFFFu);
                    }
                    DevTuple tu;
                    tu.t = t; tu.c = c; tu.p = p; tu.d = d;
                    tu.pair_off = std::get<0>(it->second);
                    tu.n_pairs = std::get<1>(it->second);
                    tu.fence_off = std::get<2>(it->second);
                    tu.w = tu.n_pairs * n_rcdo;
                    if (tu.w == 0) continue;  // no (b, s) pair survives: consumes no index
                    tuples.push_back(tu);
                    tvals.push_back(t);
                    pvals.push_back(p);
                }
            }
        }
        tup_begin.push_back((uint32_t)tuples.size());
    }
    std::sort(tvals.begin(), tvals.end());
    tvals.erase(std::unique(tvals.begin(), tvals.end()), tvals.end());
    std::sort(pvals.begin(), pvals.end());
    pvals.erase(std::unique(pvals.begin(), pvals.end()), pvals.end());

    // validity classes: signature = (t | k, v, f) over tvals, (p <= L, p | L) over pvals
    std::unordered_map<std::string, uint32_t> cls_of;
    std::vector<std::string> cls_sig;
    model_class.resize(models.size());
    std::string sig(tvals.size() + pvals.size(), '0');
    for (size_t i = 0; i < models.size(); i++) {
        const me_model& m = models[i];
        for (size_t q = 0; q < tvals.size(); q++) {
            uint32_t t = tvals[q];
            sig[q] = (m.kv_heads % t == 0 && m.vocab % t == 0 && m.ffn_hidden % t == 0) ? '1' : '0';
        }
        for (size_t q = 0; q < pvals.size(); q++) {
            uint32_t p = pvals[q];
            sig[tvals.size() + q] = (p <= m.layers && (uneven || m.layers % p == 0) &&
                                     (!vpp || (p >= 2 && m.layers % (p * vpp) == 0)))
                                        ? '1'
                                        : '0';
        }
        auto it = cls_of.find(sig);
        if (it == cls_of.end()) {
            it = cls_of.emplace(sig, (uint32_t)cls_sig.size()).first;
            cls_sig.push_back(sig);
        }
        model_class[i] = it->second;
    }
    n_class = (uint32_t)cls_sig.size();

    // per (class, N) tuple lists
    const uint32_t nW = (uint32_t)world.size();
    list_off.assign(1, 0);
    list_tuple.clear();
    list_prefix.clear();
    class_seg.assign((size_t)n_class * nW, 0);
    for (uint32_t k = 0; k < n_class; k++) {
        const std::string& s = cls_sig[k];
        for (uint32_t n = 0; n < nW; n++) {
            uint64_t acc = 0;
            for (uint32_t j = tup_begin[n]; j < tup_begin[n + 1]; j++) {
                const DevTuple& tu = tuples[j];
                size_t qt = std::lower_bound(tvals.begin(), tvals.end(), tu.t) - tvals.begin();
                size_t qp = std::lower_bound(pvals.begin(), pvals.end(), tu.p) - pvals.begin();
                if (s[qt] != '1' || s[tvals.size() + qp] != '1') continue;
                list_tuple.push_back(j);
                list_prefix.push_back(acc);
                acc += tu.w;
            }
            list_off.push_back((uint32_t)list_tuple.size());
            class_seg[(size_t)k * nW + n] = acc;
        }
    }

    // segment prefix
    seg_prefix.resize(models.size() * nW + 1);
    uint64_t acc = 0;
    for (size_t i = 0; i < models.size(); i++)
        for (uint32_t n = 0; n < nW; n++) {
            seg_prefix[i * nW + n] = acc;
            acc += class_seg[(size_t)model_class[i] * nW + n];
        }
    seg_prefix[models.size() * nW] = acc;
    total = acc;
    // rows (= (model, N, tuple) runs of configs) before each segment
    seg_row.resize(models.size() * nW + 1);
    uint64_t rows = 0;
    for (size_t i = 0; i < models.size(); i++)
        for (uint32_t n = 0; n < nW; n++) {
            seg_row[i * nW + n] = rows;
            const size_t ln = (size_t)model_class[i] * nW + n;
            rows += list_off[ln + 1] - list_off[ln];
        }
    seg_row[models.size() * nW] = rows;
    total_rows = rows;
    if (for_sweep && total >= Limits::index)
        return fail(detail, ME_EOVERFLOW, "space has >= 2^56 configurations");
    return ME_OK;
}

uint64_t HostSpace::row_of(uint64_t index) const {
    const uint32_t nW = (uint32_t)world.size();
    const size_t seg = std::upper_bound(seg_prefix.begin(), seg_prefix.end(), index) - seg_prefix.begin() - 1;
    const uint64_t within = index - seg_prefix[seg];
    const size_t ln = (size_t)model_class[seg / nW] * nW + seg % nW;
    const size_t j = std::upper_bound(list_prefix.begin() + list_off[ln], list_prefix.begin() + list_off[ln + 1],
                                      within) - list_prefix.begin() - 1;
    return seg_row[seg] + (j - list_off[ln]);
}

uint64_t HostSpace::row_start(uint64_t g) const {
    if (g >= total_rows) return total;
    const uint32_t nW = (uint32_t)world.size();
    const size_t seg = std::upper_bound(seg_row.begin(), seg_row.end(), g) - seg_row.begin() - 1;
    const size_t ln = (size_t)model_class[seg / nW] * nW + seg % nW;
    return seg_prefix[seg] + list_prefix[list_off[ln] + (g - seg_row[seg])];
}

int HostSpace::decode(uint64_t index, uint32_t* model_id, uint32_t* world_size,
                      me_parallel* out) const {
    if (index >= total) return ME_ERANGE;
    const uint32_t nW = (uint32_t)world.size();
    // last segment starting at or before index (it is non-empty)
    size_t seg = std::upper_bound(seg_prefix.begin(), seg_prefix.end(), index) - seg_prefix.begin() - 1;
    uint32_t mdl = (uint32_t)(seg / nW), n = (uint32_t)(seg % nW);
    uint64_t within = index - seg_prefix[seg];
    uint32_t cls = model_class[mdl];
    uint32_t lb = list_off[(size_t)cls * nW + n], le = list_off[(size_t)cls * nW + n + 1];
    size_t j = std::upper_bound(list_prefix.begin() + lb, list_prefix.begin() + le, within) -
               list_prefix.begin() - 1;
    uint64_t r = within - list_prefix[j];
    const DevTuple& tu = tuples[list_tuple[j]];
    uint32_t q = (uint32_t)(r >> lg_rcdo), sel = (uint32_t)(r & (n_rcdo - 1));
    // recover (b, s) of the q-th valid pair in (b, s) order
    uint32_t k = 0, b = 0, s = 0;
    for (uint32_t bb : mbs) {
        for (uint32_t ss : seq) {
            if (!pair_ok(tu.c, tu.d, tu.p, bb, ss)) continue;
            if (k == q) { b = bb; s = ss; }
            k++;
        }
    }
    me_parallel c{};
    c.dp = tu.d; c.tp = tu.t; c.pp = tu.p; c.cp = tu.c; c.mbs = b; c.seq = s;
    c.gbs = gbs; c.first_stage_layers = 0;
    c.recompute = (uint8_t)((rcdo_rc >> sel) & 1);
    c.dist_opt = (uint8_t)((rcdo_do >> sel) & 1);
    c.allow_uneven_pp = uneven;
    c.zero_stage = zero_stage;
    c.sp_off = sp_off;
    c.vpp = vpp;
    c.w_bytes = wb;
    c.g_bytes = gb;
    c.o_bytes = ob;
    if (model_id) *model_id = mdl;
    if (world_size) *world_size = world[n];
    if (out) *out = c;
    return ME_OK;
}

}  // namespace me
