// C ABI (include/tusq.h) and the TEM executor: depth-first traversal of a DFS leaf range with
// rollback by uncomputation, hybrid re-anchoring, fused
// tile sweeps (K5) or per-gate kernels (K1-K4), leaf sampling (K6) into shot slots.
#include <algorithm>
#include <chrono>
#include <cstring>
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

// Host cost model of one transition (gate applications): hybrid min(uncompute, reset).
static uint64_t transition_cost(const tusq_tree &t, const Leaf *prev, const Leaf &l, bool hybrid, bool fold)
{
    uint64_t idx;
    double re, im;
    Cursor cf = fold ? fold_prefix(t, l, &idx, &re, &im) : Cursor{0, 0};
    uint64_t reset = suffix_len(t, l, cf);
    if (!prev) return reset;
    Cursor c = common_prefix(t, *prev, l);
    uint64_t unc = suffix_len(t, *prev, c) + suffix_len(t, l, c);
    return hybrid ? std::min(unc, reset) : unc;
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
    if (!okp(noise->p1) || !okp(noise->p2) || !okp(noise->p_meas)) return fail(TUSQ_ERR_INVALID_ARG, "p outside [0, 1]");
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
    (void)precision;
    if (!t || !bounds || nranks == 0) return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    const uint64_t nl = t->leaves.size();
    std::vector<double> cum(nl + 1, 0.0);
    for (uint64_t i = 0; i < nl; ++i)
        cum[i + 1] = cum[i] + (double)transition_cost(*t, i ? &t->leaves[i - 1] : nullptr, t->leaves[i], true, true);
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
    if (!d_state || n == 0 || n > 62 || !prec_ok(precision) || index >= (1ull << n))
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
    FusedPlanner planner(n, (int)precision, 0);
    try {
        if (!(flags & TUSQ_APPLY_UNFUSED) && planner.enabled()) {
            planner.execute(v, ctx);
            planner.materialize(ctx);
        } else {
            execute_unfused(v, ctx);
        }
    } catch (const std::exception &e) {
        return fail(TUSQ_ERR_INTERNAL, e.what());
    }
    if (!ctx.dry) TQ_CUDA(cudaGetLastError());
    return TUSQ_OK;
}

tusq_status tusq_sample(const void *d_state, uint32_t n, uint32_t precision, uint64_t n_draws, uint64_t seed,
                        uint64_t leaf, uint64_t *d_out, void *stream)
{
    if (!d_state || !d_out || n == 0 || n > 62 || !prec_ok(precision)) return fail(TUSQ_ERR_INVALID_ARG, "bad argument");
    if (!n_draws) return TUSQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t bb = block_bits_for(n);
    uint64_t nb = 1ull << (n - bb);
    double *d_blocks = nullptr;
    uint32_t *d_edges = nullptr;
    TQ_CUDA(cudaMallocAsync((void **)&d_blocks, (2 * nb + 16) * sizeof(double), st));
    TQ_CUDA(cudaMallocAsync((void **)&d_edges, sizeof(uint32_t), st));
    TQ_CUDA(cudaMemsetAsync(d_edges, 0, sizeof(uint32_t), st));
    launch_block_sums(d_state, n, (int)precision, bb, d_blocks, st);
    launch_scan_blocks(d_blocks, d_blocks + nb, nb, 0, st);
    launch_draws(d_state, n, (int)precision, bb, d_blocks, d_blocks + nb, n_draws, seed, leaf, 1e-9, 0, d_out,
                 d_edges, st);
    TQ_CUDA(cudaGetLastError());
    TQ_CUDA(cudaFreeAsync(d_blocks, st));
    TQ_CUDA(cudaFreeAsync(d_edges, st));
    return TUSQ_OK;
}

tusq_status tusq_run_tree(const tusq_tree *t, const tusq_exec *ex, uint64_t *out_slots, tusq_run_stats *stats_out)
{
    auto t0 = std::chrono::steady_clock::now();
    if (!t || !ex) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    if (!prec_ok(ex->precision)) return fail(TUSQ_ERR_INVALID_ARG, "precision must be 128 or 64");
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
    const int prec = (int)ex->precision;
    const uint64_t amp_bytes = prec == 128 ? 16 : 8;
    const uint64_t need = amp_bytes << n;
    const uint64_t nl = t->leaves.size();
    const uint64_t lb = ex->leaf_begin, le = ex->leaf_end ? ex->leaf_end : nl;
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
    const uint64_t off0 = lb < le ? t->leaves[lb].offset : 0;
    const uint64_t off1 = lb < le ? t->leaves[le - 1].offset + t->leaves[le - 1].count : 0;
    uint64_t *d_slots = nullptr;
    double *d_blocks = nullptr;
    uint32_t *d_edges = nullptr;
    const uint32_t bb = block_bits_for(n);
    const uint64_t nb = 1ull << (n - bb);
    GateTimer timer(!dry && (ex->flags & TUSQ_EXEC_PROFILE));
    auto cleanup = [&]() {
        if (d_slots) cudaFree(d_slots);
        if (d_blocks) cudaFree(d_blocks);
        if (d_edges) cudaFree(d_edges);
        if (own_state) cudaFree(psi);
    };
#define TQ_RUN_CUDA(call)                                                                            \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) { cleanup(); return fail(TUSQ_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); } \
    } while (0)
    if (!dry) {
        TQ_RUN_CUDA(cudaMalloc((void **)&d_slots, std::max<uint64_t>(1, off1 - off0) * sizeof(uint64_t)));
        TQ_RUN_CUDA(cudaMalloc((void **)&d_blocks, (2 * nb + 16) * sizeof(double)));
        TQ_RUN_CUDA(cudaMalloc((void **)&d_edges, sizeof(uint32_t)));
        TQ_RUN_CUDA(cudaMemsetAsync(d_edges, 0, sizeof(uint32_t), st));
    }
    const bool hybrid = !(ex->flags & TUSQ_EXEC_NO_RESET);
    const bool fold = !(ex->flags & TUSQ_EXEC_NO_FOLD);
    const uint64_t budget = ex->reanchor_budget ? ex->reanchor_budget : (prec == 128 ? 1000000ull : 20000ull);
    const double eps = ex->edge_eps > 0 ? ex->edge_eps : (prec == 128 ? 1e-9 : 1e-5);
    FusedPlanner planner(n, prec, ex->fuse_qubits);
    const bool fuse = !(ex->flags & TUSQ_EXEC_NO_FUSE) && planner.enabled();
    Ctx ctx;
    ctx.psi = psi; ctx.n = n; ctx.prec = prec; ctx.st = st; ctx.dry = dry; ctx.stats = &stats;
    ctx.timer = timer.on() ? &timer : nullptr;
    std::vector<Op> ops;
    ops.reserve(4 * t->gates.size() + 64);
    uint64_t since_anchor = 0;
    bool phys_sums_valid = false;
    try {
        for (uint64_t li = lb; li < le; ++li) {
            const Leaf &l = t->leaves[li];
            const Leaf *prev = li > lb ? &t->leaves[li - 1]
                               : ((ex->flags & TUSQ_EXEC_CONTINUE) && lb > 0) ? &t->leaves[lb - 1] : nullptr;
            ops.clear();
            InitState init{0, 1.0, 0.0};
            Cursor cf = fold ? fold_prefix(*t, l, &init.index, &init.re, &init.im) : Cursor{0, 0};
            uint64_t reset_cost = suffix_len(*t, l, cf);
            bool reset = prev == nullptr;
            if (!reset) {
                Cursor c = common_prefix(*t, *prev, l);
                uint64_t up = suffix_len(*t, *prev, c), down = suffix_len(*t, l, c);
                if ((hybrid && reset_cost < up + down) || since_anchor + up + down > budget) {
                    reset = true;
                } else {
                    append_inverse(*t, *prev, c, ops);
                    append_forward(*t, l, c, ops);
                    since_anchor += up + down;
                }
            }
            if (reset) {
                stats.resets++;
                append_forward(*t, l, cf, ops);
                since_anchor = ops.size();
            }
            stats.gate_apps += ops.size();
            const uint64_t sweeps_before = stats.sweeps;
            bool sums = false;
            const bool want_sums = sample && l.count && n >= 12;
            if (fuse) {
                // (plan-only runs pass a placeholder pointer: nothing is launched)
                double *sums_dst = want_sums ? (dry ? reinterpret_cast<double *>(16) : d_blocks) : nullptr;
                planner.execute_ex(ops, ctx, reset ? &init : nullptr, sums_dst, &sums);
            } else {
                if (reset) {
                    double b = dry ? (double)need : launch_init_basis(psi, n, prec, init.index, init.re, init.im, st);
                    stats.launches++;
                    stats.hbm_bytes += b;
                }
                execute_unfused(ops, ctx);
            }
            // per-block |amp|^2 sums are PHYSICAL-block sums: still valid after a transition that only
            // relabelled (pending X mask), recomputed when the state changed without an epilogue
            if (sums) phys_sums_valid = true;
            else if (reset || stats.sweeps != sweeps_before) phys_sums_valid = false;
            if (sample && l.count) {
                const uint64_t xm = fuse ? planner.xmask() : 0;
                if (!phys_sums_valid) {
                    stats.sample_bytes += dry ? (double)need : launch_block_sums(psi, n, prec, bb, d_blocks, st);
                    stats.launches++;
                    phys_sums_valid = true;
                }
                if (!dry) {
                    launch_scan_blocks(d_blocks, d_blocks + nb, nb, xm >> bb, st);
                    stats.sample_bytes += launch_draws(psi, n, prec, bb, d_blocks, d_blocks + nb, l.count, t->seed,
                                                       li, eps, xm, d_slots + (l.offset - off0), d_edges, st);
                } else {
                    stats.sample_bytes += (double)l.count * (double)(amp_bytes << bb);
                }
                stats.launches += 2;
                stats.draws += l.count;
            }
            stats.leaves++;
            if (!dry) {
                cudaError_t e = cudaPeekAtLastError();
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    cleanup();
                    return fail(TUSQ_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
                }
            }
        }
        if (fuse) planner.materialize(ctx);   // leave the caller's buffer in logical order
        if (!dry) {
            if (sample && off1 > off0)
                TQ_RUN_CUDA(cudaMemcpyAsync(out_slots + off0, d_slots, (off1 - off0) * sizeof(uint64_t),
                                            cudaMemcpyDeviceToHost, st));
            uint32_t h_edges = 0;
            TQ_RUN_CUDA(cudaMemcpyAsync(&h_edges, d_edges, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            TQ_RUN_CUDA(cudaStreamSynchronize(st));
            stats.edge_draws = h_edges;
            timer.flush();
            stats.gate_kernel_launches = timer.launches;
            stats.gate_kernel_seconds = timer.seconds;
            stats.gate_kernel_bytes = timer.bytes;
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
