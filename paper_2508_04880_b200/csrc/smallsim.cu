// Batched sub-trees with on-chip state for small n ("traverse
// multiple sub-trees in parallel", Fig. P:325 (B)).
//
// For n <= 13 (complex128) / n <= 14 (complex64) a whole state vector fits one CTA's shared memory
// (<= 128 KiB).  The DFS leaf range is cut into contiguous, cost-balanced sub-ranges, one per CTA;
// the host compiles each sub-range's transitions (uncompute to the divergence slot + forward, or
// reset + replay -- the same scheduler as the per-transition path) and its leaf samplings into a
// linear program of 32-byte instructions, and ONE launch runs every program: each CTA keeps its
// state in shared memory for its whole sub-range, applies gates as shared-memory passes, builds
// the |amp|^2 CDF on chip (fp64) and writes its leaves' draws straight into the shot slots.
// Instead of ~3 launches per transition and 3 per sampled vector (2071 launches for C1), a
// circuit of this size is one kernel launch.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fused.h"
#include "kernels.h"

namespace tq {
namespace sm {

enum : uint8_t { S_END = 0, S_INIT, S_U2, S_DIAG, S_X, S_Y, S_Z, S_CX, S_CPH, S_SAMPLE, S_STORE };

struct SInst {
    uint8_t op, q0, q1, _pad;
    uint32_t pi;          // parameter (double) index, or table (u64) index for S_SAMPLE
    uint64_t x, y, z;     // S_INIT: index; S_SAMPLE: leaf0, slot0, draws
};
static_assert(sizeof(SInst) == 32, "SInst is 32 bytes");

constexpr int TPB = 512;
constexpr int CH = 16;    // CDF chunk (amplitudes per prefix entry)

template <typename R> struct CVs;
template <> struct CVs<double> { using T = double2; };
template <> struct CVs<float> { using T = float2; };

__device__ __forceinline__ uint32_t ins0(uint32_t j, uint32_t q) { return ((j >> q) << (q + 1)) | (j & ((1u << q) - 1)); }

template <typename R>
__global__ void __launch_bounds__(TPB) k_small(uint32_t n, const SInst *__restrict__ prog,
                                               const uint64_t *__restrict__ prog_off, const double *__restrict__ prm,
                                               const uint64_t *__restrict__ tabs, uint32_t k0, uint32_t k1,
                                               double eps, uint64_t *__restrict__ slots, uint32_t *__restrict__ edges,
                                               typename CVs<R>::T *__restrict__ out_state)
{
    using V = typename CVs<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    const uint32_t N = 1u << n;
    V *a = reinterpret_cast<V *>(smraw);
    double *pre = reinterpret_cast<double *>(smraw + (size_t)N * sizeof(V));   // chunk prefix, N/CH + 1
    __shared__ double wsum[TPB / 32];
    const uint32_t tid = threadIdx.x;
    const SInst *ip = prog + prog_off[blockIdx.x];
    for (;; ++ip) {
        const SInst in = *ip;   // uniform across the CTA
        if (in.op == S_END) break;
        switch (in.op) {
        case S_INIT:
            for (uint32_t i = tid; i < N; i += TPB) {
                V v;
                v.x = i == in.x ? (R)prm[in.pi] : R(0);
                v.y = i == in.x ? (R)prm[in.pi + 1] : R(0);
                a[i] = v;
            }
            break;
        case S_U2: {
            const double *m = prm + in.pi;
            const R u0r = (R)m[0], u0i = (R)m[1], u1r = (R)m[2], u1i = (R)m[3];
            const R u2r = (R)m[4], u2i = (R)m[5], u3r = (R)m[6], u3i = (R)m[7];
            for (uint32_t j = tid; j < N / 2; j += TPB) {
                const uint32_t i0 = ins0(j, in.q0), i1 = i0 | (1u << in.q0);
                const V x = a[i0], y = a[i1];
                V nx, ny;
                nx.x = u0r * x.x - u0i * x.y + u1r * y.x - u1i * y.y;
                nx.y = u0r * x.y + u0i * x.x + u1r * y.y + u1i * y.x;
                ny.x = u2r * x.x - u2i * x.y + u3r * y.x - u3i * y.y;
                ny.y = u2r * x.y + u2i * x.x + u3r * y.y + u3i * y.x;
                a[i0] = nx;
                a[i1] = ny;
            }
            break;
        }
        case S_DIAG: {
            const double *d = prm + in.pi;
            const R d0r = (R)d[0], d0i = (R)d[1], d1r = (R)d[2], d1i = (R)d[3];
            for (uint32_t i = tid; i < N; i += TPB) {
                const bool b = (i >> in.q0) & 1u;
                const R pr = b ? d1r : d0r, pi = b ? d1i : d0i;
                const V x = a[i];
                V y;
                y.x = x.x * pr - x.y * pi;
                y.y = x.x * pi + x.y * pr;
                a[i] = y;
            }
            break;
        }
        case S_X: case S_Y:
            for (uint32_t j = tid; j < N / 2; j += TPB) {
                const uint32_t i0 = ins0(j, in.q0), i1 = i0 | (1u << in.q0);
                V x = a[i0], y = a[i1];
                if (in.op == S_Y) {   // (Y psi)_0 = -i psi_1, (Y psi)_1 = i psi_0
                    const V t0 = {y.y, -y.x}, t1 = {-x.y, x.x};
                    a[i0] = t0;
                    a[i1] = t1;
                } else {
                    a[i0] = y;
                    a[i1] = x;
                }
            }
            break;
        case S_Z:
            for (uint32_t j = tid; j < N / 2; j += TPB) {
                const uint32_t i1 = ins0(j, in.q0) | (1u << in.q0);
                V x = a[i1];
                x.x = -x.x;
                x.y = -x.y;
                a[i1] = x;
            }
            break;
        case S_CX: {
            const uint32_t lo = min(in.q0, in.q1), hi = max(in.q0, in.q1);
            for (uint32_t j = tid; j < N / 4; j += TPB) {
                const uint32_t i0 = ins0(ins0(j, lo), hi) | (1u << in.q0), i1 = i0 | (1u << in.q1);
                const V x = a[i0], y = a[i1];
                a[i0] = y;
                a[i1] = x;
            }
            break;
        }
        case S_CPH: {
            const R pr = (R)prm[in.pi], pi = (R)prm[in.pi + 1];
            const uint32_t lo = min(in.q0, in.q1), hi = max(in.q0, in.q1);
            for (uint32_t j = tid; j < N / 4; j += TPB) {
                const uint32_t i = ins0(ins0(j, lo), hi) | (1u << in.q0) | (1u << in.q1);
                const V x = a[i];
                V y;
                y.x = x.x * pr - x.y * pi;
                y.y = x.x * pi + x.y * pr;
                a[i] = y;
            }
            break;
        }
        case S_STORE:   // the final state of the call's last leaf, for the caller's buffer
            for (uint32_t i = tid; i < N; i += TPB) out_state[i] = a[i];
            break;
        case S_SAMPLE: {
            // CDF on chip: chunk sums of |amp|^2 (fp64), an exclusive prefix over the chunks, then
            // per draw a binary search over chunks and a sequential walk inside one chunk
            const uint32_t nch = (N + CH - 1) / CH;
            double s = 0.0;
            const uint32_t c0 = tid;   // one chunk per thread per pass
            for (uint32_t c = c0; c < nch; c += TPB) {
                double cs = 0.0;
                for (uint32_t i = c * CH; i < min(N, c * CH + CH); ++i) {
                    const double re = a[i].x, im = a[i].y;
                    cs += re * re + im * im;
                }
                pre[c + 1] = cs;
            }
            __syncthreads();
            // exclusive prefix over nch chunk sums (nch <= 1024): each thread owns a contiguous run
            const uint32_t per = (nch + TPB - 1) / TPB, b0 = tid * per, b1 = min(nch, b0 + per);
            for (uint32_t c = b0; c < b1; ++c) s += pre[c + 1];
            double incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, o);
                if ((tid & 31) >= (uint32_t)o) incl += y;
            }
            if ((tid & 31) == 31) wsum[tid >> 5] = incl;
            __syncthreads();
            double woff = 0.0;
            for (uint32_t w = 0; w < (tid >> 5); ++w) woff += wsum[w];
            double run = woff + incl - s;
            __syncthreads();
            for (uint32_t c = b0; c < b1; ++c) {
                const double v = pre[c + 1];
                pre[c] = run;
                run += v;
            }
            if (tid == TPB - 1 || (b1 == nch && b0 < b1)) pre[nch] = run;
            __syncthreads();
            const double T = pre[nch];
            // draws: one thread each; the group's leaves via its table (nlt+1 offsets, nlt masks)
            const uint64_t *tb = tabs + in.pi;
            const uint32_t nlt = (uint32_t)(in.z >> 40);
            const uint64_t nd = in.z & ((1ull << 40) - 1);
            for (uint64_t w = tid; w < nd; w += TPB) {
                uint32_t lo = 0, hi = nlt - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (tb[mid] <= w) lo = mid; else hi = mid - 1;
                }
                const uint64_t leaf = in.x + lo, j = w - tb[lo];
                const U4 rnd = philox10(U4{(uint32_t)j, (uint32_t)leaf, (uint32_t)(leaf >> 32), TAG_SHOT}, k0, k1);
                const uint64_t xr = (uint64_t)rnd.x | ((uint64_t)rnd.y << 32);
                const double t = (double)(xr >> 11) * 0x1.0p-53 * T;
                // last chunk whose start prefix <= t (chunks are exclusive prefixes)
                uint32_t cl = 0, ch = nch - 1;
                while (cl < ch) {
                    const uint32_t mid = (cl + ch + 1) >> 1;
                    if (pre[mid] <= t) cl = mid; else ch = mid - 1;
                }
                double runc = pre[cl], prev = runc;
                uint32_t k = N;
                for (uint32_t c = cl; c < nch && k == N; ++c) {
                    runc = pre[c];
                    for (uint32_t i = c * CH; i < min(N, c * CH + CH); ++i) {
                        const double re = a[i].x, im = a[i].y;
                        const double nr = runc + (re * re + im * im);
                        if (nr > t) { k = i; prev = runc; runc = nr; break; }
                        runc = nr;
                    }
                }
                bool edge;
                if (k == N) {   // rounding: no C(k) > t -- the last nonzero amplitude
                    k = N - 1;
                    while (k > 0 && a[k].x == R(0) && a[k].y == R(0)) --k;
                    edge = true;
                } else {
                    edge = fmin(t - prev, runc - t) < eps;
                }
                slots[in.y + w] = (uint64_t)k ^ tb[nlt + 1 + lo];
                if (edge) atomicAdd(edges, 1u);
            }
            break;
        }
        default: break;
        }
        __syncthreads();
    }
}

}  // namespace sm

static bool diag_vals(const Op &o, double d[4])
{
    const double s2 = M_SQRT1_2;
    d[0] = 1; d[1] = 0;
    switch (o.kind) {
    case I: d[2] = 1; d[3] = 0; return true;
    case S: d[2] = 0; d[3] = 1; return true;
    case SDG: d[2] = 0; d[3] = -1; return true;
    case T: d[2] = s2; d[3] = s2; return true;
    case TDG: d[2] = s2; d[3] = -s2; return true;
    case P: d[2] = cos(o.theta); d[3] = sin(o.theta); return true;
    case RZ: d[0] = cos(o.theta / 2); d[1] = -sin(o.theta / 2); d[2] = cos(o.theta / 2); d[3] = sin(o.theta / 2);
        return true;
    default: return false;
    }
}

uint32_t small_max_qubits(int prec) { return prec == 128 ? 13u : 14u; }

// Compile one gate / Pauli into the program.
static void emit_op(const Op &o, std::vector<sm::SInst> &pg, std::vector<double> &prm)
{
    using namespace sm;
    SInst s{};
    s.q0 = (uint8_t)o.q0;
    s.q1 = (uint8_t)o.q1;
    double d[4];
    switch (o.kind) {
    case X: s.op = S_X; break;
    case Y: s.op = S_Y; break;
    case Z: s.op = S_Z; break;
    case CX: s.op = S_CX; break;
    case CZ: case CP:
        s.op = S_CPH;
        s.pi = (uint32_t)prm.size();
        prm.push_back(o.kind == CZ ? -1.0 : cos(o.theta));
        prm.push_back(o.kind == CZ ? 0.0 : sin(o.theta));
        break;
    case H: case RX: case RY: {
        s.op = S_U2;
        s.pi = (uint32_t)prm.size();
        const double c = cos(o.theta / 2), sn = sin(o.theta / 2), r = M_SQRT1_2;
        if (o.kind == H) prm.insert(prm.end(), {r, 0, r, 0, r, 0, -r, 0});
        else if (o.kind == RX) prm.insert(prm.end(), {c, 0, 0, -sn, 0, -sn, c, 0});
        else prm.insert(prm.end(), {c, 0, -sn, 0, sn, 0, c, 0});
        break;
    }
    default:
        if (!diag_vals(o, d)) throw std::runtime_error("small-n path: unsupported op");
        if (o.kind == I) return;
        s.op = S_DIAG;
        s.pi = (uint32_t)prm.size();
        prm.insert(prm.end(), {d[0], d[1], d[2], d[3]});
        break;
    }
    pg.push_back(s);
}

tusq_status run_tree_small(const tusq_tree *t, const tusq_exec *ex, uint64_t lb, uint64_t le, void *psi,
                           uint64_t *d_slots, uint64_t off0, uint32_t *d_edges, double eps, tusq_run_stats &stats)
{
    using namespace sm;
    const uint32_t n = t->n;
    const uint32_t L = (uint32_t)t->gates.size();
    const int prec = (int)ex->precision;
    const bool dry = ex->flags & TUSQ_EXEC_PLAN_ONLY;
    const bool sample = !(ex->flags & TUSQ_EXEC_NO_SAMPLE);
    const bool hybrid = !(ex->flags & TUSQ_EXEC_NO_RESET);
    const bool fold = !(ex->flags & TUSQ_EXEC_NO_FOLD);
    const uint64_t budget = ex->reanchor_budget ? ex->reanchor_budget : (prec == 128 ? 1000000ull : 20000ull);
    cudaStream_t st = (cudaStream_t)ex->stream;
    const uint64_t nl = le - lb;
    if (!nl) return TUSQ_OK;
    // executed (core) leaves
    std::vector<Leaf> core(nl);
    std::vector<uint64_t> tmask(nl);
    for (uint64_t i = 0; i < nl; ++i) core[i] = core_of(t->leaves[lb + i], L, &tmask[i]);
    // sub-ranges: contiguous, balanced by the replay cost of a fresh descent per leaf (a
    // conservative proxy); about 16 leaves per CTA, at most 4 CTAs per SM
    const uint64_t maxc = (uint64_t)(dry ? 148 : device_sm_count()) * 4;
    const uint64_t C = std::max<uint64_t>(1, std::min<uint64_t>(maxc, (nl + 15) / 16));
    std::vector<double> cum(nl + 1, 0.0);
    for (uint64_t i = 0; i < nl; ++i) {
        uint64_t idx;
        double re, im;
        cum[i + 1] = cum[i] + 1.0 + (double)suffix_len(*t, core[i], fold_prefix(*t, core[i], &idx, &re, &im));
    }
    std::vector<uint64_t> bnd(C + 1, 0);
    for (uint64_t c = 1, i = 0; c < C; ++c) {
        const double target = cum[nl] * (double)c / (double)C;
        while (i < nl && cum[i] < target) ++i;
        bnd[c] = std::max(i, bnd[c - 1]);
    }
    bnd[C] = nl;
    std::vector<SInst> pg;
    std::vector<uint64_t> poff;
    std::vector<double> prm;
    std::vector<uint64_t> tabs;
    std::vector<Op> ops;
    for (uint64_t c = 0; c < C; ++c) {
        if (bnd[c] == bnd[c + 1]) continue;
        poff.push_back(pg.size());
        uint64_t since = 0;
        for (uint64_t g0 = bnd[c]; g0 < bnd[c + 1];) {
            uint64_t g1 = g0 + 1;
            while (g1 < bnd[c + 1] && same_core(core[g1], core[g0])) ++g1;
            const Leaf &l = core[g0];
            const Leaf *prev = g0 > bnd[c] ? &core[g0 - 1] : nullptr;
            ops.clear();
            InitState init{0, 1.0, 0.0};
            const Cursor cf = fold ? fold_prefix(*t, l, &init.index, &init.re, &init.im) : Cursor{0, 0};
            const uint64_t reset_cost = suffix_len(*t, l, cf);
            bool reset = prev == nullptr;
            if (!reset) {
                const Cursor cc = common_prefix(*t, *prev, l);
                const uint64_t up = suffix_len(*t, *prev, cc), down = suffix_len(*t, l, cc);
                if ((hybrid && reset_cost < up + down) || since + up + down > budget) {
                    reset = true;
                } else {
                    append_inverse(*t, *prev, cc, ops);
                    append_forward(*t, l, cc, ops);
                    since += up + down;
                }
            }
            if (reset) {
                SInst s{};
                s.op = S_INIT;
                s.x = init.index;
                s.pi = (uint32_t)prm.size();
                prm.push_back(init.re);
                prm.push_back(init.im);
                pg.push_back(s);
                append_forward(*t, l, cf, ops);
                since = ops.size();
                stats.resets++;
            }
            for (const Op &o : ops) emit_op(o, pg, prm);
            stats.gate_apps += ops.size();
            uint64_t draws = 0;
            for (uint64_t k = g0; k < g1; ++k) draws += t->leaves[lb + k].count;
            if (sample && draws) {
                SInst s{};
                s.op = S_SAMPLE;
                s.x = lb + g0;
                s.y = t->leaves[lb + g0].offset - off0;
                s.z = draws | ((uint64_t)(g1 - g0) << 40);
                s.pi = (uint32_t)tabs.size();
                for (uint64_t k = g0; k <= g1; ++k)
                    tabs.push_back(k < g1 ? t->leaves[lb + k].offset - t->leaves[lb + g0].offset : draws);
                for (uint64_t k = g0; k < g1; ++k) tabs.push_back(tmask[k]);
                pg.push_back(s);
                stats.draws += draws;
                stats.sampled_vectors++;
            }
            stats.leaves += g1 - g0;
            g0 = g1;
        }
        if (bnd[c + 1] == nl) {   // the sub-range holding the call's last leaf leaves its state behind
            SInst s{};
            s.op = S_STORE;
            pg.push_back(s);
        }
        pg.push_back(SInst{});   // S_END
    }
    const double bytes_state = (double)(1ull << n) * (prec == 128 ? 16 : 8);
    stats.launches += 1;
    stats.sweeps += 0;
    stats.hbm_bytes += bytes_state;   // the final state written back; everything else is on chip
    const size_t pbytes = pg.size() * sizeof(SInst), obytes = poff.size() * 8, mbytes = prm.size() * 8,
                 tbytes = tabs.size() * 8;
    stats.h2d_bytes += (double)(pbytes + obytes + mbytes + tbytes);
    if (dry) return TUSQ_OK;
    char *buf = nullptr;
    const size_t total = pbytes + obytes + mbytes + tbytes + 64;
    if (cudaMallocAsync((void **)&buf, total, st) != cudaSuccess) return fail(TUSQ_ERR_OOM, "small-n program buffer");
    size_t at = 0;
    auto put = [&](const void *src, size_t len) {
        void *dst = buf + at;
        if (len) cudaMemcpyAsync(dst, src, len, cudaMemcpyHostToDevice, st);
        at += (len + 15) & ~(size_t)15;
        return dst;
    };
    const SInst *d_pg = (const SInst *)put(pg.data(), pbytes);
    const uint64_t *d_off = (const uint64_t *)put(poff.data(), obytes);
    const double *d_prm = (const double *)put(prm.data(), mbytes);
    const uint64_t *d_tab = (const uint64_t *)put(tabs.data(), tbytes);
    const size_t smem = ((size_t)1 << n) * (prec == 128 ? 16 : 8) + (((1u << n) + CH - 1) / CH + 1) * 8;
    const uint32_t k0 = (uint32_t)t->seed, k1 = (uint32_t)(t->seed >> 32);
    GateTimer *timer = nullptr;
    (void)timer;
    if (prec == 128) {
        cudaFuncSetAttribute(k_small<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_small<double><<<(unsigned)poff.size(), TPB, smem, st>>>(n, d_pg, d_off, d_prm, d_tab, k0, k1, eps, d_slots,
                                                                   d_edges, (double2 *)psi);
    } else {
        cudaFuncSetAttribute(k_small<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_small<float><<<(unsigned)poff.size(), TPB, smem, st>>>(n, d_pg, d_off, d_prm, d_tab, k0, k1, eps, d_slots,
                                                                  d_edges, (float2 *)psi);
    }
    cudaFreeAsync(buf, st);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TUSQ_ERR_CUDA, std::string("k_small launch: ") + cudaGetErrorString(e));
    return TUSQ_OK;
}

}  // namespace tq
