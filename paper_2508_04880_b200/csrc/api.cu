// C ABI (include/tusq.h) and the TEM executor: depth-first traversal of a DFS leaf range with
// rollback by uncomputation, hybrid re-anchoring, fused
// tile sweeps (K5) or per-gate kernels (K1-K4), leaf sampling (K6) into shot slots.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "fused.h"
#include "kernels.h"

namespace tq {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

tusq_status fail(tusq_status st, const std::string &msg)
{
    g_err = msg;
    return st;
}

#define TQ_CUDA(call)                                                                             \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(TUSQ_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(e_)); \
    } while (0)

static tusq_status validate_ops(uint32_t n, const tusq_op *ops, uint64_t L)
{
    if (n == 0 || n > 62) return fail(TUSQ_ERR_INVALID_ARG, "n_qubits must be in [1, 62]");
    if (L && !ops) return fail(TUSQ_ERR_INVALID_ARG, "ops is NULL");
    for (uint64_t i = 0; i < L; ++i) {
        const tusq_op &o = ops[i];
        if (o.kind >= NKINDS) return fail(TUSQ_ERR_INVALID_ARG, "unknown gate kind at op " + std::to_string(i));
        if (o.q0 >= n) return fail(TUSQ_ERR_INVALID_ARG, "qubit out of range at op " + std::to_string(i));
        if (two_qubit(o.kind) && (o.q1 >= n || o.q1 == o.q0))
            return fail(TUSQ_ERR_INVALID_ARG, "bad target qubit at op " + std::to_string(i));
    }
    return TUSQ_OK;
}

static bool prec_ok(uint32_t p) { return p == 128 || p == 64; }
static uint32_t block_bits_for(uint32_t n) { return n < 12 ? n : 12; }
// the 2^n state's byte count must fit 63 bits (n <= 58 c128, 59 c64: far above any device)
static bool state_fits(uint32_t n, int prec) { return n + (prec == 128 ? 4u : 3u) <= 62u; }

// Stream-ordered device scratch from the device's default memory pool.  The pool keeps freed
// memory (release threshold raised once per device), so per-call scratch costs no cudaMalloc /
// cudaFree round trip and no device-wide synchronization.
static cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st)
{
    static std::once_flag once[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::call_once(once[dev & 63], [dev]() {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = 1ull << 30;   // keep up to 1 GiB of freed scratch
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    return cudaMallocAsync(p, bytes, st);
}

}  // namespace tq

using namespace tq;

extern "C" {

const char *tusq_last_error(void) { return g_err.c_str(); }
const char *tusq_version(void) { return "tusq-b200 0.2 (sm_100a)"; }

tusq_status tusq_build_error_tree(uint32_t n, const tusq_op *ops, uint64_t L, const tusq_noise *noise,
                                  uint64_t shots, uint64_t seed, const tusq_prune *prune, tusq_tree **out)
{
    if (!out) return fail(TUSQ_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    tusq_status s = validate_ops(n, ops, L);
    if (s) return s;
    if (!noise) return fail(TUSQ_ERR_INVALID_ARG, "noise is NULL");
    auto okp = [](double p) { return p >= 0.0 && p <= 1.0; };
    if (noise->flags & ~TUSQ_NOISE_PAULI) return fail(TUSQ_ERR_INVALID_ARG, "unknown noise flags");
    if (noise->flags & TUSQ_NOISE_PAULI) {
        for (const double *c : {noise->pauli1, noise->pauli2, noise->pauli_meas})
            if (!okp(c[0]) || !okp(c[1]) || !okp(c[2]) || !(c[0] + c[1] + c[2] <= 1.0))
                return fail(TUSQ_ERR_INVALID_ARG, "Pauli channel probabilities outside [0, 1] or summing above 1");
    } else if (!okp(noise->p1) || !okp(noise->p2) || !okp(noise->p_meas)) {
        return fail(TUSQ_ERR_INVALID_ARG, "p outside [0, 1]");
    }
    if (shots == 0) return fail(TUSQ_ERR_INVALID_ARG, "shots must be > 0");
    tusq_prune pr = prune ? *prune : tusq_prune{1, 100, 100, 1};
    if (pr.enabled && (pr.alpha_den == 0 || pr.alpha_num > pr.alpha_den))
        return fail(TUSQ_ERR_INVALID_ARG, "alpha must be in (0, 1]");
    if (pr.enabled && pr.beta == 0) return fail(TUSQ_ERR_INVALID_ARG, "beta must be >= 1 (shot conservation)");
    try {
        return build_tree(n, ops, L, *noise, shots, seed, pr, out);
    } catch (const std::bad_alloc &) {
        return fail(TUSQ_ERR_OOM, "host allocation failed in tusq_build_error_tree");
    } catch (...) {
        return fail(TUSQ_ERR_INTERNAL, "exception in tusq_build_error_tree");
    }
}

tusq_status tusq_twirl_decoherence(double t, double T1, double T2, double out[3])
{
    if (!out) return fail(TUSQ_ERR_INVALID_ARG, "out is NULL");
    if (!(t >= 0.0) || !(T1 > 0.0) || !(T2 > 0.0)) return fail(TUSQ_ERR_INVALID_ARG, "need t >= 0, T1 > 0, T2 > 0");
    // Eq. 2: Pauli-twirled amplitude and phase damping
    const double a = (1.0 - std::exp(-t / T1)) / 4.0;
    const double z = (1.0 - std::exp(-t / T2)) / 2.0 - a;
    if (z < 0.0) return fail(TUSQ_ERR_INVALID_ARG, "unphysical decoherence: p_Z < 0 (T2 > 2 T1)");
    out[0] = a;
    out[1] = a;
    out[2] = z;
    return TUSQ_OK;
}

tusq_status tusq_tree_get_info(const tusq_tree *t, tusq_tree_info *out)
{
    if (!t || !out) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    tree_info(*t, out);
    return TUSQ_OK;
}

tusq_status tusq_tree_serialize(const tusq_tree *t, uint8_t *buf, uint64_t *inout_len)
{
    if (!t || !inout_len) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    uint64_t need = 8 + 4 + 4 + 10 * 8;
    for (auto &l : t->leaves) need += 8 + 8 + 4 + 12ull * l.tr.size();
    if (!buf) { *inout_len = need; return TUSQ_OK; }
    if (*inout_len < need) { *inout_len = need; return fail(TUSQ_ERR_CAPACITY, "serialize buffer too small"); }
    uint8_t *p = buf;
    auto put = [&](const void *src, size_t len) { memcpy(p, src, len); p += len; };
    uint32_t zero = 0;
    put("TUSQTRE1", 8);
    put(&t->n, 4);
    put(&zero, 4);
    uint64_t L = t->gates.size(), nl = t->leaves.size();
    uint64_t hdr[10] = {L, t->shots, t->seed, t->S2, t->S3, t->p0, t->n_sig, t->n_insig, t->n_selected, nl};
    put(hdr, sizeof(hdr));
    for (auto &l : t->leaves) {
        uint32_t m = (uint32_t)l.tr.size();
        put(&l.count, 8);
        put(&l.offset, 8);
        put(&m, 4);
        for (auto &x : l.tr) { put(&x.pos, 4); put(&x.q, 4); put(&x.p, 4); }
    }
    *inout_len = need;
    return TUSQ_OK;
}

tusq_status tusq_tree_leaf(const tusq_tree *t, uint64_t leaf, uint64_t *count, uint64_t *offset, uint32_t *triples,
                           uint32_t *inout_n)
{
    if (!t || !count || !offset || !inout_n) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    if (leaf >= t->leaves.size()) return fail(TUSQ_ERR_INVALID_ARG, "leaf out of range");
    const Leaf &l = t->leaves[leaf];
    if (*inout_n < l.tr.size() || (!triples && l.tr.size())) {
        *inout_n = (uint32_t)l.tr.size();
        return fail(TUSQ_ERR_CAPACITY, "triples buffer too small");
    }
    *count = l.count;
    *offset = l.offset;
    for (size_t i = 0; i < l.tr.size(); ++i) {
        triples[3 * i] = l.tr[i].pos; triples[3 * i + 1] = l.tr[i].q; triples[3 * i + 2] = l.tr[i].p;
    }
    *inout_n = (uint32_t)l.tr.size();
    return TUSQ_OK;
}

void tusq_tree_free(tusq_tree *t) { delete t; }

tusq_status tusq_tree_partition(const tusq_tree *t, uint32_t nranks, uint32_t precision, uint64_t *bounds)
{
    if (!t || !bounds || nranks == 0) return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    if (!prec_ok(precision)) return fail(TUSQ_ERR_INVALID_ARG, "precision must be 128 or 64");
    const uint64_t nl = t->leaves.size();
    const uint32_t L = (uint32_t)t->gates.size();
    const uint64_t budget = precision == 128 ? 1000000ull : 20000ull;
    // replay the scheduler of tusq_run_tree on the executed (core) leaves: hybrid reset vs
    // uncompute, and a forced re-anchor whenever the precision's budget would be exceeded
    std::vector<double> cum(nl + 1, 0.0);
    uint64_t since = 0;
    Leaf prev;
    for (uint64_t i = 0; i < nl; ++i) {
        const Leaf cur = core_of(t->leaves[i], L, nullptr);
        uint64_t idx;
        double re, im;
        const uint64_t reset = suffix_len(*t, cur, fold_prefix(*t, cur, &idx, &re, &im));
        uint64_t cost = reset;
        if (i) {
            const Cursor c = common_prefix(*t, prev, cur);
            const uint64_t unc = suffix_len(*t, prev, c) + suffix_len(*t, cur, c);
            // the default (live-tile) scheduler's rule: uncompute only when the reset's replay is at
            // least 16x longer (tusq_run_tree's reset_bias)
            if (reset >= 16 * unc && since + unc <= budget) { cost = unc; since += unc; }
            else since = reset;
        } else {
            since = reset;
        }
        cum[i + 1] = cum[i] + (double)cost;
        prev = cur;
    }
    bounds[0] = 0;
    uint64_t i = 0;
    for (uint32_t r = 1; r < nranks; ++r) {
        double target = cum[nl] * r / nranks;
        while (i < nl && cum[i] < target) ++i;
        bounds[r] = std::max<uint64_t>(i, bounds[r - 1]);
    }
    bounds[nranks] = nl;
    return TUSQ_OK;
}

tusq_status tusq_init_basis(void *d_state, uint32_t n, uint32_t precision, uint64_t index, double re, double im,
                            void *stream)
{
    if (!d_state || n == 0 || !prec_ok(precision) || !state_fits(n, (int)precision) || index >= (1ull << n))
        return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    launch_init_basis(d_state, n, (int)precision, index, re, im, (cudaStream_t)stream);
    TQ_CUDA(cudaGetLastError());
    return TUSQ_OK;
}

tusq_status tusq_apply_ops(void *d_state, uint32_t n, uint32_t precision, const tusq_op *ops, uint64_t L,
                           uint32_t flags, void *stream)
{
    if (!d_state || !prec_ok(precision)) return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    tusq_status s = validate_ops(n, ops, L);
    if (s) return s;
    if (!state_fits(n, (int)precision)) return fail(TUSQ_ERR_CAPACITY, "2^n state too large");
    std::vector<Op> v(L);
    for (uint64_t i = 0; i < L; ++i) v[i] = Op{ops[i].kind, ops[i].q0, ops[i].q1, ops[i].theta};
    if (flags & TUSQ_APPLY_INVERSE) {
        std::vector<Op> r;
        r.reserve(L);
        for (uint64_t i = L; i-- > 0;) r.push_back(inverse_op(v[i]));
        v.swap(r);
    }
    tusq_run_stats stats{};
    Ctx ctx;
    ctx.psi = d_state; ctx.n = n; ctx.prec = (int)precision; ctx.st = (cudaStream_t)stream; ctx.stats = &stats;
    ctx.dry = (flags & TUSQ_APPLY_PLAN_ONLY) != 0;
    FusedPlanner planner(n, (int)precision);
    const bool fused = !(flags & TUSQ_APPLY_UNFUSED) && planner.enabled();
    // second buffer for the layout-changing sweeps: allocated only if the ops form >= 2 groups
    if (fused) planner.set_alt_lazy((precision == 128 ? 16ull : 8ull) << n);
    try {
        if (fused) {
            planner.execute(v, ctx);
            planner.materialize(ctx);
        } else {
            execute_unfused(v, ctx);
        }
    } catch (const std::exception &e) {
        planner.release(ctx.st);
        return fail(TUSQ_ERR_INTERNAL, e.what());
    }
    planner.release(ctx.st);
    if (!ctx.dry) TQ_CUDA(cudaGetLastError());
    return TUSQ_OK;
}

tusq_status tusq_sample(const void *d_state, uint32_t n, uint32_t precision, uint64_t n_draws, uint64_t seed,
                        uint64_t leaf, uint64_t *d_out, void *stream)
{
    if (!d_state || !d_out || n == 0 || !prec_ok(precision) || !state_fits(n, (int)precision))
        return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    if (!n_draws) return TUSQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t bb = block_bits_for(n);
    uint64_t nb = 1ull << (n - bb);
    void *scr = nullptr;
    const size_t nblk = 2 * nb + 16;
    TQ_CUDA(scratch_alloc(&scr, nblk * sizeof(double) + 16, st));
    double *d_blocks = (double *)scr;
    uint32_t *d_edges = (uint32_t *)(d_blocks + nblk);
    TQ_CUDA(cudaMemsetAsync(d_edges, 0, sizeof(uint32_t), st));
    launch_block_sums(d_state, n, (int)precision, bb, d_blocks, st);
    launch_scan_blocks(d_blocks, d_blocks + nb, nb, 0, st);
    launch_draws(d_state, n, (int)precision, bb, d_blocks, d_blocks + nb, n_draws, seed, leaf, nullptr, 0, 0, 1e-9, 0,
                 d_out, d_edges, st);
    TQ_CUDA(cudaGetLastError());
    TQ_CUDA(cudaFreeAsync(scr, st));
    return TUSQ_OK;
}

tusq_status tusq_run_tree(const tusq_tree *t, const tusq_exec *ex, uint64_t *out_slots, tusq_run_stats *stats_out)
{
    auto t0 = std::chrono::steady_clock::now();
    if (!t || !ex) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    if (!prec_ok(ex->precision)) return fail(TUSQ_ERR_INVALID_ARG, "precision must be 128 or 64");
    if (ex->fuse_qubits != 0 && ex->fuse_qubits != 12)
        return fail(TUSQ_ERR_UNSUPPORTED, "fuse_qubits: this build compiles 12-qubit tiles only (0 or 12)");
    if (!state_fits(t->n, (int)ex->precision)) return fail(TUSQ_ERR_CAPACITY, "2^n state too large");
    if (ex->mode == TUSQ_MODE_SHARDED) {
        try {
            return run_tree_sharded(t, ex, out_slots, stats_out);
        } catch (const std::bad_alloc &) {
            return fail(TUSQ_ERR_OOM, "host allocation failed in tusq_run_tree");
        }
    }
    if (ex->mode != TUSQ_MODE_REPLICA) return fail(TUSQ_ERR_INVALID_ARG, "mode must be TUSQ_MODE_REPLICA or TUSQ_MODE_SHARDED");
    const bool dry = ex->flags & TUSQ_EXEC_PLAN_ONLY;
    const bool sample = !(ex->flags & TUSQ_EXEC_NO_SAMPLE);
    if (sample && !dry && !out_slots) return fail(TUSQ_ERR_INVALID_ARG, "out_slots is NULL");
    const uint32_t n = t->n;
    const uint32_t L = (uint32_t)t->gates.size();
    const int prec = (int)ex->precision;
    const uint64_t amp_bytes = prec == 128 ? 16 : 8;
    const uint64_t need = amp_bytes << n;
    const uint64_t nl = t->leaves.size();
    tusq_comm *comm = ex->comm;
    int crank = 0, cranks = 1;
    if (comm) {
        if (comm_is_local(comm)) return fail(TUSQ_ERR_INVALID_ARG, "replica mode: a local communicator has no ranks to reduce over");
        crank = comm_rank(comm);
        cranks = comm_nranks(comm);
    }
    uint64_t lb = ex->leaf_begin, le = ex->leaf_end ? ex->leaf_end : nl;
    if (comm && ex->leaf_begin == 0 && ex->leaf_end == 0) {   // this rank's cost-balanced range
        std::vector<uint64_t> bounds(cranks + 1);
        tusq_status ps = tusq_tree_partition(t, (uint32_t)cranks, ex->precision, bounds.data());
        if (ps) return ps;
        lb = bounds[crank];
        le = bounds[crank + 1];
    }
    if (lb > le || le > nl) return fail(TUSQ_ERR_INVALID_ARG, "leaf range out of bounds");
    if (!dry && ex->device >= 0) TQ_CUDA(cudaSetDevice(ex->device));
    cudaStream_t st = (cudaStream_t)ex->stream;
    void *psi = ex->d_state;
    bool own_state = false;
    if (psi) {
        if (ex->state_bytes < need) return fail(TUSQ_ERR_CAPACITY, "state buffer smaller than 2^n amplitudes");
    } else if (!dry) {
        if (cudaMalloc(&psi, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(TUSQ_ERR_CAPACITY, "cannot allocate the 2^n state vector on this device");
        }
        own_state = true;
    }
    tusq_run_stats stats{};
    // slot window written by this call: the range's shots, or all S1 slots when reduced over ranks
    const uint64_t off0 = comm ? 0 : (lb < le ? t->leaves[lb].offset : 0);
    const uint64_t off1 = comm ? t->shots : (lb < le ? t->leaves[le - 1].offset + t->leaves[le - 1].count : 0);
    const uint32_t bb = block_bits_for(n);
    const uint64_t nb = 1ull << (n - bb);

    // ---- executed (core) leaves and sampling groups: consecutive leaves with the same core share
    // one state vector; their draws run in one launch with per-leaf readout masks (reading #7)
    std::vector<Leaf> core(le - lb);
    std::vector<uint64_t> tmask(le - lb, 0);
    for (uint64_t li = lb; li < le; ++li) core[li - lb] = core_of(t->leaves[li], L, &tmask[li - lb]);
    Leaf prev_core;
    const bool cont = (ex->flags & TUSQ_EXEC_CONTINUE) && lb > 0;
    if (cont) prev_core = core_of(t->leaves[lb - 1], L, nullptr);
    struct SGroup { uint64_t l0, l1, tab; };   // leaves [l0, l1), table offset (u64 words), 0 = none
    std::vector<SGroup> groups;
    std::vector<uint64_t> htab;
    for (uint64_t i = 0; i < core.size();) {
        uint64_t j = i + 1;
        while (j < core.size() && same_core(core[j], core[i])) ++j;
        SGroup g{lb + i, lb + j, 0};
        if (j - i > 1) {
            g.tab = htab.size() + 1;   // +1: 0 means "no table"
            for (uint64_t k = i; k <= j; ++k)
                htab.push_back(k < j ? t->leaves[lb + k].offset - t->leaves[lb + i].offset
                                     : t->leaves[lb + j - 1].offset + t->leaves[lb + j - 1].count - t->leaves[lb + i].offset);
            for (uint64_t k = i; k < j; ++k) htab.push_back(tmask[k]);
        }
        groups.push_back(g);
        i = j;
    }

    // ---- device scratch: slots, block sums + prefix, edge counter, group tables
    void *scr = nullptr;
    const size_t nslots = std::max<uint64_t>(1, off1 - off0);
    const size_t nblk = 2 * nb + 16;
    uint64_t maxdraws = 1;   // the most draws one state vector takes (sums-only block lists)
    for (const SGroup &g : groups) {
        uint64_t d = 0;
        for (uint64_t li = g.l0; li < g.l1; ++li) d += t->leaves[li].count;
        maxdraws = std::max(maxdraws, d);
    }
    const size_t scr_bytes = (nslots + nblk + htab.size() + maxdraws + 2) * 8;
    uint64_t *d_slots = nullptr, *d_tab = nullptr, *d_blist = nullptr;
    double *d_blocks = nullptr;
    uint32_t *d_edges = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    GateTimer timer(!dry && (ex->flags & TUSQ_EXEC_PROFILE));
    void *alt_buf = nullptr;   // set below, freed here
    auto cleanup = [&]() {
        if (scr) cudaFreeAsync(scr, st);
        if (own_state || alt_buf) cudaStreamSynchronize(st);
        if (own_state) cudaFree(psi);
        if (alt_buf) cudaFree(alt_buf);
        for (auto &e : ev) if (e) cudaEventDestroy(e);
    };
#define TQ_RUN_CUDA(call)                                                                            \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) { cleanup(); return fail(TUSQ_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); } \
    } while (0)
    if (!dry) {
        for (auto &e : ev) TQ_RUN_CUDA(cudaEventCreate(&e));
        TQ_RUN_CUDA(cudaEventRecord(ev[0], st));
        TQ_RUN_CUDA(scratch_alloc(&scr, scr_bytes, st));
        d_slots = (uint64_t *)scr;
        d_blocks = (double *)(d_slots + nslots);
        d_tab = (uint64_t *)(d_blocks + nblk);
        d_blist = d_tab + htab.size();
        d_edges = (uint32_t *)(d_blist + maxdraws);
        if (comm) TQ_RUN_CUDA(cudaMemsetAsync(d_slots, 0, nslots * sizeof(uint64_t), st));
        TQ_RUN_CUDA(cudaMemsetAsync(d_edges, 0, sizeof(uint32_t), st));
        if (!htab.empty())
            TQ_RUN_CUDA(cudaMemcpyAsync(d_tab, htab.data(), htab.size() * 8, cudaMemcpyHostToDevice, st));
    }
    stats.h2d_bytes += (double)htab.size() * 8;
    const bool hybrid = !(ex->flags & TUSQ_EXEC_NO_RESET);
    const bool fold = !(ex->flags & TUSQ_EXEC_NO_FOLD);
    const uint64_t budget = ex->reanchor_budget ? ex->reanchor_budget : (prec == 128 ? 1000000ull : 20000ull);
    const double eps = ex->edge_eps > 0 ? ex->edge_eps : (prec == 128 ? 1e-9 : 1e-5);
    FusedPlanner planner(n, prec);
    planner.set_live(!(ex->flags & TUSQ_EXEC_NO_LIVE));
    const bool fuse = !(ex->flags & TUSQ_EXEC_NO_FUSE) && planner.enabled();
    // small n: the whole range in ONE launch, one sub-range per CTA, state on chip (smallsim.cu)
    const bool small = !(ex->flags & (TUSQ_EXEC_NO_FUSE | TUSQ_EXEC_NO_BATCH)) && n <= small_max_qubits(prec);
    // the fused path's second buffer (layout-changing sweeps run out of place); without the memory
    // for it every sweep keeps the identity layout and runs in place
    void *alt = nullptr;
    if (fuse && !small && !dry && le > lb) {
        if (cudaMalloc(&alt, need) != cudaSuccess) { cudaGetLastError(); alt = nullptr; }
        planner.set_alt(alt);
        alt_buf = alt;
    }
    Ctx ctx;
    ctx.psi = psi; ctx.n = n; ctx.prec = prec; ctx.st = st; ctx.dry = dry; ctx.stats = &stats;
    ctx.timer = timer.on() ? &timer : nullptr;
    std::vector<Op> ops;
    ops.reserve(4 * t->gates.size() + 64);
    uint64_t since_anchor = 0;
    bool phys_sums_valid = false;
    bool virt = false;                 // the device state is the basis state vstate, not yet written
    InitState vstate{0, 1.0, 0.0};
    std::vector<uint64_t> fills;       // (slot - off0, count, value) of the virtual leaves' draws
    try {
        if (small) {
            tusq_status ss = run_tree_small(t, ex, lb, le, psi, d_slots, off0, d_edges, eps, stats);
            if (ss != TUSQ_OK) { cleanup(); return ss; }
            groups.clear();
        }
        // transition decisions (reset vs uncompute), made one group AHEAD: a state that the next
        // transition discards (it resets) need not be stored after sampling (sums-only sweeps)
        struct Dec { bool reset; Cursor cf, c; InitState init; uint64_t sa_after; };
        // Reset when its replay is shorter than bias x the uncompute.  With live tiles a reset's replay
        // starts from one basis state and mostly visits a few tiles, while an uncompute sweeps a
        // dense state and its state must be stored for it (no sums-only sampling): measured on C4,
        // bias 1 / 2 / 1e6 = 21.4 / 15.1 / 13.2 s (debug build), plan bytes flat above 16; keeping
        // the gate-count rule for replays longer than 40-80 % of the circuit measured 17.7-19.7 s.  The
        // plain dense path (TUSQ_EXEC_NO_LIVE) keeps the gate-count rule (bias 1).
        uint64_t reset_bias = (ex->flags & TUSQ_EXEC_NO_LIVE) ? 1 : 16;
#ifdef TUSQ_DEBUG_KNOBS
        if (getenv("TUSQ_DBG_RESET_BIAS")) reset_bias = (uint64_t)atoll(getenv("TUSQ_DBG_RESET_BIAS"));
#endif
        auto decide = [&](size_t gi, uint64_t sa) {
            const SGroup &g = groups[gi];
            const Leaf &l = core[g.l0 - lb];
            const Leaf *prev = g.l0 > lb ? &core[g.l0 - lb - 1] : (cont ? &prev_core : nullptr);
            Dec d;
            d.init = InitState{0, 1.0, 0.0};
            d.cf = fold ? fold_prefix(*t, l, &d.init.index, &d.init.re, &d.init.im) : Cursor{0, 0};
            d.c = Cursor{0, 0};
            const uint64_t reset_cost = suffix_len(*t, l, d.cf);
            d.reset = prev == nullptr;
            if (!d.reset) {
                d.c = common_prefix(*t, *prev, l);
                const uint64_t up = suffix_len(*t, *prev, d.c), down = suffix_len(*t, l, d.c);
                if ((hybrid && reset_cost < reset_bias * (up + down)) || sa + up + down > budget) d.reset = true;
                else d.sa_after = sa + up + down;
            }
            if (d.reset) d.sa_after = reset_cost;
            return d;
        };
        Dec next{};
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            const SGroup &g = groups[gi];
            // ---- transition to the group's core (uncompute to the divergence slot, then forward)
            const Leaf &l = core[g.l0 - lb];
            const Leaf *prev = g.l0 > lb ? &core[g.l0 - lb - 1] : (cont ? &prev_core : nullptr);
            const Dec cur = gi == 0 ? decide(0, since_anchor) : next;
            if (gi + 1 < groups.size()) next = decide(gi + 1, cur.sa_after);
            const bool next_resets = gi + 1 < groups.size() && next.reset;
            ops.clear();
            InitState init = cur.init;
            const Cursor cf = cur.cf;
            bool reset = cur.reset;
            if (!reset) {
                append_inverse(*t, *prev, cur.c, ops);
                append_forward(*t, l, cur.c, ops);
            } else {
                stats.resets++;
                append_forward(*t, l, cf, ops);
            }
            since_anchor = cur.sa_after;
            stats.gate_apps += ops.size();
            // A leaf whose whole executed stream folds (reset with nothing left to apply) is the basis
            // state amp|x>: it stays VIRTUAL -- no device pass -- and its draws are x ^ readout mask
            // (a single-outcome CDF: every draw picks x exactly).  A later uncompute from it starts
            // by resetting to that basis state, fused into its first sweep.
            if (reset && ops.empty()) {
                virt = true;
                vstate = init;
                phys_sums_valid = false;
                if (sample)
                    for (uint64_t li = g.l0; li < g.l1; ++li)
                        if (t->leaves[li].count) {
                            fills.push_back(t->leaves[li].offset - off0);
                            fills.push_back(t->leaves[li].count);
                            fills.push_back(init.index ^ tmask[li - lb]);
                            stats.draws += t->leaves[li].count;
                        }
                stats.leaves += g.l1 - g.l0;
                stats.sampled_vectors++;
                continue;
            }
            const bool from_virtual = virt && !reset;   // uncompute from a basis state never written
            if (from_virtual) { reset = true; init = vstate; }
            virt = false;
            const uint64_t sweeps_before = stats.sweeps;
            uint64_t draws = 0;
            for (uint64_t li = g.l0; li < g.l1; ++li) draws += t->leaves[li].count;
            bool sums = false;
            const bool want_sums = sample && draws && n >= 12;
            if (fuse) {
                // (plan-only runs pass a placeholder pointer: nothing is launched)
                double *sums_dst = want_sums ? (dry ? reinterpret_cast<double *>(16) : d_blocks) : nullptr;
                planner.execute_ex(ops, ctx, reset ? &init : nullptr, sums_dst, &sums, want_sums && next_resets);
            } else {
                if (reset) {
                    if (ctx.timer) ctx.timer->begin(st);
                    double b = dry ? (double)need : launch_init_basis(psi, n, prec, init.index, init.re, init.im, st);
                    if (ctx.timer) ctx.timer->end(st, b);
                    stats.launches++;
                    stats.hbm_bytes += b;
                }
                execute_unfused(ops, ctx);
            }
            // per-block |amp|^2 sums are PHYSICAL-block sums: still valid after a transition that only
            // relabelled (pending X mask), recomputed when the state changed without an epilogue
            if (sums) phys_sums_valid = true;
            else if (reset || stats.sweeps != sweeps_before) phys_sums_valid = false;
            // ---- sampling: one CDF, the draws of every leaf of the group in one launch
            if (sample && draws) {
                const uint64_t xm = fuse ? planner.xmask() : 0;
                if (ctx.timer) ctx.timer->begin(st);
                if (!phys_sums_valid) {
                    uint64_t vf = ~0ull, vx = 0;   // K5 live tiles may leave the buffer valid on a subset
                    if (fuse) {
                        planner.close_blocks(ctx, bb);
                        planner.valid_set(&vf, &vx);
                    }
                    stats.sample_bytes += dry ? (double)need : launch_block_sums(psi, n, prec, bb, d_blocks, st, vf, vx);
                    stats.launches++;
                    phys_sums_valid = true;
                }
                const Leaf &l0 = t->leaves[g.l0];
                if (!dry) {
                    launch_scan_blocks(d_blocks, d_blocks + nb, nb, xm >> bb, st);
                    if (fuse && planner.pending_tiles()) {
                        // sums-only sweep: find the blocks the draws land in, compute and store
                        // just those tiles, then draw as usual
                        launch_draws(psi, n, prec, bb, d_blocks, d_blocks + nb, draws, t->seed, g.l0,
                                     g.tab ? d_tab + (g.tab - 1) : nullptr, (uint32_t)(g.l1 - g.l0), tmask[g.l0 - lb],
                                     eps, xm, d_slots + (l0.offset - off0), d_edges, st, d_blist);
                        planner.replay_tiles(ctx, d_blist, draws, xm >> bb);
                    }
                    stats.sample_bytes += launch_draws(psi, n, prec, bb, d_blocks, d_blocks + nb, draws, t->seed, g.l0,
                                                       g.tab ? d_tab + (g.tab - 1) : nullptr, (uint32_t)(g.l1 - g.l0),
                                                       tmask[g.l0 - lb], eps, xm, d_slots + (l0.offset - off0), d_edges,
                                                       st);
                } else {
                    stats.sample_bytes += (double)draws * (double)(amp_bytes << bb);
                }
                if (ctx.timer) ctx.timer->end(st, 0.0, 1);
                stats.launches += 3;
                stats.draws += draws;
                stats.sampled_vectors++;
            }
            stats.leaves += g.l1 - g.l0;
            if (!dry) {
                cudaError_t e = cudaPeekAtLastError();
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    cleanup();
                    return fail(TUSQ_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
                }
            }
        }
        if (virt) {   // the call ends on a virtual leaf: write its basis state (K7)
            if (!dry) launch_init_basis(psi, n, prec, vstate.index, vstate.re, vstate.im, st);
            stats.launches++;
            stats.hbm_bytes += (double)need;
            if (fuse) planner.note_basis(vstate.index);
        }
        if (fuse) {   // leave the caller's buffer in logical order, whole
            planner.materialize(ctx);
            planner.finish(ctx);
        }
        if (!dry && !fills.empty()) {   // the virtual leaves' draws, one launch
            void *fb = nullptr;
            TQ_RUN_CUDA(scratch_alloc(&fb, fills.size() * 8, st));
            TQ_RUN_CUDA(cudaMemcpyAsync(fb, fills.data(), fills.size() * 8, cudaMemcpyHostToDevice, st));
            launch_fill_slots((const uint64_t *)fb, fills.size() / 3, d_slots, st);
            TQ_RUN_CUDA(cudaFreeAsync(fb, st));
            stats.launches++;
            stats.h2d_bytes += (double)fills.size() * 8;
        }
        if (!dry) {
            TQ_RUN_CUDA(cudaEventRecord(ev[1], st));
            if (comm && sample) {   // the disjoint slot arrays of all ranks, summed on the device
                std::string err;
                TQ_RUN_CUDA(cudaEventRecord(ev[2], st));
                if (comm_allreduce_u64(comm, d_slots, nslots, st, err) != TUSQ_OK) {
                    cleanup();
                    return fail(TUSQ_ERR_NCCL, err);
                }
                TQ_RUN_CUDA(cudaEventRecord(ev[3], st));
            }
            if (sample && off1 > off0) {
                TQ_RUN_CUDA(cudaMemcpyAsync(out_slots + off0, d_slots, (off1 - off0) * sizeof(uint64_t),
                                            cudaMemcpyDeviceToHost, st));
                stats.d2h_bytes += (double)(off1 - off0) * 8;
            }
            uint32_t h_edges = 0;
            TQ_RUN_CUDA(cudaMemcpyAsync(&h_edges, d_edges, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            stats.d2h_bytes += 4;
            TQ_RUN_CUDA(cudaStreamSynchronize(st));
            float ms = 0;
            if (cudaEventElapsedTime(&ms, ev[0], ev[1]) == cudaSuccess) stats.device_seconds = ms * 1e-3;
            if (comm && sample && cudaEventElapsedTime(&ms, ev[2], ev[3]) == cudaSuccess) stats.reduce_seconds = ms * 1e-3;
            stats.edge_draws = h_edges;
            timer.flush();
            stats.gate_kernel_launches = timer.launches;
            stats.gate_kernel_seconds = timer.seconds;
            stats.gate_kernel_bytes = timer.bytes;
            stats.sample_kernel_seconds = timer.sample_seconds;
            stats.dense_sweep_launches = timer.dense_launches;
            stats.dense_sweep_seconds = timer.dense_seconds;
            stats.dense_sweep_bytes = timer.dense_bytes;
        }
    } catch (const std::exception &e) {
        cleanup();
        return fail(TUSQ_ERR_INTERNAL, e.what());
    }
    cleanup();
    stats.host_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats_out) *stats_out = stats;
    return TUSQ_OK;
#undef TQ_RUN_CUDA
}

}  // extern "C"
