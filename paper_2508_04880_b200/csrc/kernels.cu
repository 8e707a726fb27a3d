// sm_100a gate, Pauli, init and sampler kernels (K1-K4, K6, K7) -- the unfused path.
//
// Every kernel is HBM-bound streaming work (no dense contraction, so no tensor cores):
// coalesced 128-bit (c128) / 64-bit (c64) amplitude loads, grid-stride loops sized to the
// SM count, two independent pairs per thread in flight.  Bytes per launch are the
// algorithmic bytes of SURVEY.md 8(d): 2*2^n*s for dense/X-type, 2^n*s for the
// half-touching CX / diagonal / Z-only kernels (s = 16 B c128, 8 B c64).
#include <atomic>
#include <cstdio>

#include "kernels.h"

namespace tq {

template <typename R> struct CV;
template <> struct CV<double> { using T = double2; };
template <> struct CV<float> { using T = float2; };

template <typename R> struct Cx { R re, im; };

template <typename R, typename V>
__device__ __forceinline__ V cmul(Cx<R> u, V a)
{
    V r;
    r.x = u.re * a.x - u.im * a.y;
    r.y = u.re * a.y + u.im * a.x;
    return r;
}

template <typename R, typename V>
__device__ __forceinline__ V cmac2(Cx<R> u0, V a, Cx<R> u1, V b)
{
    V r;
    r.x = u0.re * a.x - u0.im * a.y + u1.re * b.x - u1.im * b.y;
    r.y = u0.re * a.y + u0.im * a.x + u1.re * b.y + u1.im * b.x;
    return r;
}

__device__ __forceinline__ uint64_t insert0(uint64_t j, uint32_t q)
{
    uint64_t lo = j & ((1ull << q) - 1);
    return ((j >> q) << (q + 1)) | lo;
}

int device_sm_count()
{
    // per-device cache (benign concurrent first fills: every writer stores the same value)
    static std::atomic<int> sms[64];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int> &slot = sms[dev & 63];
    int v = slot.load(std::memory_order_relaxed);
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        slot.store(v, std::memory_order_relaxed);
    }
    return v;
}

static unsigned grid_for(uint64_t work, unsigned threads, unsigned per_thread)
{
    uint64_t need = (work + (uint64_t)threads * per_thread - 1) / ((uint64_t)threads * per_thread);
    uint64_t cap = (uint64_t)device_sm_count() * 16;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

constexpr unsigned TPB = 256;

// ------------------------------------------------------------------ K1: dense 1q
template <typename R>
__global__ void __launch_bounds__(TPB) k_dense1(typename CV<R>::T *__restrict__ psi, uint64_t npairs, uint32_t q,
                                                Cx<R> u00, Cx<R> u01, Cx<R> u10, Cx<R> u11)
{
    using V = typename CV<R>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t bit = 1ull << q;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npairs; j += 2 * stride) {
        uint64_t i0 = insert0(j, q);
        uint64_t j2 = j + stride;
        bool two = j2 < npairs;
        uint64_t k0 = two ? insert0(j2, q) : i0;
        V a = psi[i0], b = psi[i0 | bit];
        V c = psi[k0], d = psi[k0 | bit];
        psi[i0] = cmac2(u00, a, u01, b);
        psi[i0 | bit] = cmac2(u10, a, u11, b);
        if (two) {
            psi[k0] = cmac2(u00, c, u01, d);
            psi[k0 | bit] = cmac2(u10, c, u11, d);
        }
    }
}

// ------------------------------------------------------------------ K2: diagonal 1q
// d0 == 1: touch only the bit-1 half.  Otherwise multiply both halves.
template <typename R>
__global__ void __launch_bounds__(TPB) k_diag1_half(typename CV<R>::T *__restrict__ psi, uint64_t nhalf, uint32_t q,
                                                    Cx<R> d1)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t bit = 1ull << q;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nhalf; j += stride) {
        uint64_t i = insert0(j, q) | bit;
        psi[i] = cmul(d1, psi[i]);
    }
}

template <typename R>
__global__ void __launch_bounds__(TPB) k_diag1_full(typename CV<R>::T *__restrict__ psi, uint64_t N, uint32_t q,
                                                    Cx<R> d0, Cx<R> d1)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride)
        psi[i] = cmul(((i >> q) & 1) ? d1 : d0, psi[i]);
}

// ------------------------------------------------------------------ K3: CX / CZ / CP
template <typename R>
__global__ void __launch_bounds__(TPB) k_cx(typename CV<R>::T *__restrict__ psi, uint64_t nq, uint32_t c, uint32_t t)
{
    // two independent quartets per thread per iteration (4 loads in flight before the stores)
    using V = typename CV<R>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t lo = c < t ? c : t, hi = c < t ? t : c;
    const uint64_t tb = 1ull << t;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += 2 * stride) {
        const uint64_t k0 = insert0(insert0(j, lo), hi) | (1ull << c);
        const bool two = j + stride < nq;
        const uint64_t k1 = two ? insert0(insert0(j + stride, lo), hi) | (1ull << c) : k0;
        const V a0 = __ldcs(psi + k0), b0 = __ldcs(psi + (k0 | tb));
        const V a1 = __ldcs(psi + k1), b1 = __ldcs(psi + (k1 | tb));
        __stcs(psi + k0, b0);
        __stcs(psi + (k0 | tb), a0);
        if (two) {
            __stcs(psi + k1, b1);
            __stcs(psi + (k1 | tb), a1);
        }
    }
}

template <typename R>
__global__ void __launch_bounds__(TPB) k_cphase(typename CV<R>::T *__restrict__ psi, uint64_t nq, uint32_t c,
                                                uint32_t t, Cx<R> ph)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t lo = c < t ? c : t, hi = c < t ? t : c;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nq; j += stride) {
        uint64_t k = insert0(insert0(j, lo), hi) | (1ull << c) | (1ull << t);
        psi[k] = cmul(ph, psi[k]);
    }
}

// ------------------------------------------------------------------ K4: Pauli string
// (P psi)(k) = i^ny (-1)^popc((k ^ xm) & zm) psi(k ^ xm)   (Y = i X Z)
template <typename R>
__global__ void __launch_bounds__(TPB) k_pauli_x(typename CV<R>::T *__restrict__ psi, uint64_t nhalf, uint32_t lowbit,
                                                 uint64_t xm, uint64_t zm, Cx<R> gph)
{
    // two independent pairs per thread per iteration (4 loads in flight before the stores)
    using V = typename CV<R>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nhalf; j += 2 * stride) {
        const bool two = j + stride < nhalf;
        const uint64_t k0 = insert0(j, lowbit), k1 = k0 ^ xm;
        const uint64_t m0 = two ? insert0(j + stride, lowbit) : k0, m1 = m0 ^ xm;
        const V a = __ldcs(psi + k0), b = __ldcs(psi + k1);
        const V c = __ldcs(psi + m0), d = __ldcs(psi + m1);
        // new[k0] = ph(k0) psi[k1], ph(k0) uses (k0 ^ xm) = k1
        auto put = [&](uint64_t p0, uint64_t p1, const V &x, const V &y) {
            const R s0 = (__popcll(p1 & zm) & 1) ? R(-1) : R(1);
            const R s1 = (__popcll(p0 & zm) & 1) ? R(-1) : R(1);
            V na = cmul(gph, y), nb = cmul(gph, x);
            na.x *= s0; na.y *= s0;
            nb.x *= s1; nb.y *= s1;
            __stcs(psi + p0, na);
            __stcs(psi + p1, nb);
        };
        put(k0, k1, a, b);
        if (two) put(m0, m1, c, d);
    }
}

template <typename R>
__global__ void __launch_bounds__(TPB) k_pauli_z(typename CV<R>::T *__restrict__ psi, uint64_t nhalf, uint32_t lowz,
                                                 uint64_t zm)
{
    using V = typename CV<R>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nhalf; j += stride) {
        uint64_t k0 = insert0(j, lowz);
        uint64_t k = (__popcll(k0 & zm) & 1) ? k0 : (k0 | (1ull << lowz));   // the odd-parity partner
        V a = psi[k];
        a.x = -a.x;
        a.y = -a.y;
        psi[k] = a;
    }
}

// ------------------------------------------------------------------ K7: init basis
template <typename R>
__global__ void __launch_bounds__(TPB) k_init(typename CV<R>::T *__restrict__ psi, uint64_t N, uint64_t index, R re,
                                              R im)
{
    using V = typename CV<R>::T;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
        V v;
        v.x = (i == index) ? re : R(0);
        v.y = (i == index) ? im : R(0);
        psi[i] = v;
    }
}

// ------------------------------------------------------------------ launch helpers
template <typename R>
static Cx<R> cx_of(double re, double im) { return Cx<R>{(R)re, (R)im}; }

struct M2 { double r[4], i[4]; };

static bool matrix_1q(const Op &o, M2 &m)
{
    const double s2 = M_SQRT1_2;
    double c = cos(o.theta / 2), s = sin(o.theta / 2);
    auto set = [&](double a, double ai, double b, double bi, double cc, double ci, double d, double di) {
        m.r[0] = a; m.i[0] = ai; m.r[1] = b; m.i[1] = bi; m.r[2] = cc; m.i[2] = ci; m.r[3] = d; m.i[3] = di;
    };
    switch (o.kind) {
    case H: set(s2, 0, s2, 0, s2, 0, -s2, 0); return true;
    case RX: set(c, 0, 0, -s, 0, -s, c, 0); return true;
    case RY: set(c, 0, -s, 0, s, 0, c, 0); return true;
    default: return false;
    }
}

static bool diag_1q(const Op &o, double d[4])
{
    // d = {d0re, d0im, d1re, d1im}
    const double s2 = M_SQRT1_2;
    d[0] = 1; d[1] = 0;
    switch (o.kind) {
    case I: d[2] = 1; d[3] = 0; return true;
    case Z: d[2] = -1; d[3] = 0; return true;
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

template <typename R>
static double gate_impl(void *psi_, uint32_t n, const Op &o, cudaStream_t st)
{
    using V = typename CV<R>::T;
    V *psi = (V *)psi_;
    const uint64_t N = 1ull << n;
    const double s = sizeof(V);
    M2 m;
    double d[4];
    if (o.kind == X || o.kind == Y || (o.kind == Z)) {
        uint64_t xm = (o.kind == Z) ? 0 : (1ull << o.q0), zm = (o.kind == X) ? 0 : (1ull << o.q0);
        return launch_pauli_string(psi_, n, sizeof(R) == 8 ? 128 : 64, xm, zm, st);
    }
    if (matrix_1q(o, m)) {
        uint64_t np = N / 2;
        k_dense1<R><<<grid_for(np, TPB, 2), TPB, 0, st>>>(psi, np, o.q0, cx_of<R>(m.r[0], m.i[0]), cx_of<R>(m.r[1], m.i[1]),
                                                          cx_of<R>(m.r[2], m.i[2]), cx_of<R>(m.r[3], m.i[3]));
        return 2.0 * N * s;
    }
    if (diag_1q(o, d)) {
        if (o.kind == I) return 0.0;
        if (d[0] == 1.0 && d[1] == 0.0) {
            uint64_t nh = N / 2;
            k_diag1_half<R><<<grid_for(nh, TPB, 1), TPB, 0, st>>>(psi, nh, o.q0, cx_of<R>(d[2], d[3]));
            return 1.0 * N * s;
        }
        k_diag1_full<R><<<grid_for(N, TPB, 1), TPB, 0, st>>>(psi, N, o.q0, cx_of<R>(d[0], d[1]), cx_of<R>(d[2], d[3]));
        return 2.0 * N * s;
    }
    if (o.kind == CX) {
        uint64_t nq = N / 4;
        k_cx<R><<<grid_for(nq, TPB, 2), TPB, 0, st>>>(psi, nq, o.q0, o.q1);
        return 1.0 * N * s;
    }
    if (o.kind == CZ || o.kind == CP) {
        uint64_t nq = N / 4;
        double th = (o.kind == CZ) ? M_PI : o.theta;
        double cr = (o.kind == CZ) ? -1.0 : cos(th), ci = (o.kind == CZ) ? 0.0 : sin(th);
        k_cphase<R><<<grid_for(nq, TPB, 1), TPB, 0, st>>>(psi, nq, o.q0, o.q1, cx_of<R>(cr, ci));
        return 0.5 * N * s;
    }
    return 0.0;
}

double launch_gate(void *psi, uint32_t n, int prec, const Op &op, cudaStream_t st)
{
    return prec == 64 ? gate_impl<float>(psi, n, op, st) : gate_impl<double>(psi, n, op, st);
}

template <typename R>
static double pauli_impl(void *psi_, uint32_t n, uint64_t xm, uint64_t zm, cudaStream_t st)
{
    using V = typename CV<R>::T;
    V *psi = (V *)psi_;
    const uint64_t N = 1ull << n;
    const double s = sizeof(V);
    if (xm == 0 && zm == 0) return 0.0;
    if (xm) {
        int ny = __builtin_popcountll(xm & zm);
        static const double gr[4] = {1, 0, -1, 0}, gi[4] = {0, 1, 0, -1};
        uint32_t low = (uint32_t)__builtin_ctzll(xm);
        uint64_t nh = N / 2;
        k_pauli_x<R><<<grid_for(nh, TPB, 2), TPB, 0, st>>>(psi, nh, low, xm, zm, cx_of<R>(gr[ny & 3], gi[ny & 3]));
        return 2.0 * N * s;
    }
    uint32_t lowz = (uint32_t)__builtin_ctzll(zm);
    uint64_t nh = N / 2;
    k_pauli_z<R><<<grid_for(nh, TPB, 1), TPB, 0, st>>>(psi, nh, lowz, zm);
    return 1.0 * N * s;
}

double launch_pauli_string(void *psi, uint32_t n, int prec, uint64_t xm, uint64_t zm, cudaStream_t st)
{
    return prec == 64 ? pauli_impl<float>(psi, n, xm, zm, st) : pauli_impl<double>(psi, n, xm, zm, st);
}

// zeros at the elements x of the affine set {x : (x & ~scan_free) == scan_fix} that lie OUTSIDE the
// valid set {x : (x & ~vfree) == vfix}: K5's live-tile sweeps leave stale data outside the valid
// set; this writes the zeros there (a whole-state pass at the end of a call, or the blocks the
// valid set touches before the sampler reads them)
template <typename V>
__global__ void __launch_bounds__(TPB) k_zero_outside(V *__restrict__ psi, uint64_t cnt, uint64_t sfree, uint64_t sfix,
                                                      uint64_t vfree, uint64_t vfix, bool dense)
{
    for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * TPB) {
        uint64_t x = i;
        if (!dense) {
            x = sfix;
            uint64_t y = i;
            for (uint64_t m = sfree; m && y; m &= m - 1, y >>= 1)
                if (y & 1) x |= m & (~m + 1);
        }
        if ((x ^ vfix) & ~vfree) {
            V z;
            z.x = 0;
            z.y = 0;
            __stcs(psi + x, z);
        }
    }
}

double launch_zero_outside(void *psi, uint32_t n, int prec, uint64_t sfree, uint64_t sfix, uint64_t vfree, uint64_t vfix,
                           cudaStream_t st)
{
    const uint64_t all = n >= 64 ? ~0ull : (1ull << n) - 1;
    sfree &= all;
    const uint64_t cnt = 1ull << __builtin_popcountll(sfree);
    const bool dense = sfree == all;
    if (prec == 64) {
        k_zero_outside<float2><<<grid_for(cnt, TPB, 1), TPB, 0, st>>>((float2 *)psi, cnt, sfree, sfix, vfree, vfix, dense);
        return cnt * 8.0;
    }
    k_zero_outside<double2><<<grid_for(cnt, TPB, 1), TPB, 0, st>>>((double2 *)psi, cnt, sfree, sfix, vfree, vfix, dense);
    return cnt * 16.0;
}

double launch_init_basis(void *psi, uint32_t n, int prec, uint64_t index, double re, double im, cudaStream_t st)
{
    const uint64_t N = 1ull << n;
    if (prec == 64) {
        k_init<float><<<grid_for(N, TPB, 1), TPB, 0, st>>>((float2 *)psi, N, index, (float)re, (float)im);
        return N * 8.0;
    }
    k_init<double><<<grid_for(N, TPB, 1), TPB, 0, st>>>((double2 *)psi, N, index, re, im);
    return N * 16.0;
}

// ------------------------------------------------------------------ K6: sampler
// Inverse-CDF draws from |amp|^2: block sums over contiguous blocks of
// 2^block_bits amplitudes -> exclusive prefix over blocks -> per draw a binary search over
// blocks and a warp-shuffle scan inside the chosen block.  Sums in fp64 for both precisions.
template <typename R, int PER>
__global__ void __launch_bounds__(TPB) k_block_sums(const typename CV<R>::T *__restrict__ psi, uint32_t block_bits,
                                                    double *__restrict__ out, uint64_t vfree, uint64_t vfix)
{
    // PER > 0: the block is PER * TPB amplitudes and every load is issued before the first use
    // (PER independent 16-byte loads in flight per thread); PER = 0: generic strided loop
    using V = typename CV<R>::T;
    const uint64_t bs = 1ull << block_bits;
    const uint64_t base = (uint64_t)blockIdx.x * bs;
    // a block outside the valid set holds no amplitude (K5 live tiles: the buffer is stale there);
    // inside a block, positions the valid set fixes mask the elements (read as zero, not loaded)
    if ((base ^ vfix) & ~vfree & ~(bs - 1)) {
        if (threadIdx.x == 0) out[blockIdx.x] = 0.0;
        return;
    }
    double acc = 0.0;
    const uint64_t lowfix = ~vfree & (bs - 1);   // in-block positions the valid set fixes
    if constexpr (PER > 0) {
        V a[PER];
        if (lowfix) {   // elements outside the valid set read as zero (and are not loaded)
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const uint64_t x = base + threadIdx.x + k * TPB;
                if (((x ^ vfix) & lowfix) == 0) a[k] = __ldcs(psi + x);
                else { a[k].x = 0; a[k].y = 0; }
            }
        } else {
#pragma unroll
            for (int k = 0; k < PER; ++k) a[k] = __ldcs(psi + base + threadIdx.x + k * TPB);
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const double re = a[k].x, im = a[k].y;
            acc += re * re + im * im;
        }
    } else {
        for (uint64_t i = threadIdx.x; i < bs; i += blockDim.x) {
            if (((base + i) ^ vfix) & lowfix) continue;
            V a = psi[base + i];
            double re = a.x, im = a.y;
            acc += re * re + im * im;
        }
    }
    __shared__ double red[TPB / 32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < TPB / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) out[blockIdx.x] = v;
    }
}

double launch_block_sums(const void *psi, uint32_t n, int prec, uint32_t block_bits, double *d_blocks,
                         cudaStream_t st, uint64_t vfree, uint64_t vfix)
{
    uint64_t nb = 1ull << (n - block_bits);
    const bool fast = block_bits == 12;
    if (prec == 64) {
        if (fast) k_block_sums<float, 16><<<(unsigned)nb, TPB, 0, st>>>((const float2 *)psi, block_bits, d_blocks, vfree, vfix);
        else k_block_sums<float, 0><<<(unsigned)nb, TPB, 0, st>>>((const float2 *)psi, block_bits, d_blocks, vfree, vfix);
    } else {
        if (fast) k_block_sums<double, 16><<<(unsigned)nb, TPB, 0, st>>>((const double2 *)psi, block_bits, d_blocks, vfree, vfix);
        else k_block_sums<double, 0><<<(unsigned)nb, TPB, 0, st>>>((const double2 *)psi, block_bits, d_blocks, vfree, vfix);
    }
    const uint64_t all = n >= 64 ? ~0ull : (1ull << n) - 1;
    return (double)(1ull << __builtin_popcountll((vfree & all) | ((1ull << block_bits) - 1))) * (prec == 64 ? 8.0 : 16.0);
}

// Two-level CDF over blocks: superblocks of SB logical blocks.  k_super sums each superblock
// (fixed order, deterministic) reading the PHYSICAL block sums (physical block = logical ^ mh);
// k_scan turns the nsb superblock sums into an exclusive prefix (v[nsb] = total).  A draw then
// binary-searches superblocks and scans one superblock's block sums with a warp.
constexpr uint64_t SB = 1024;

__global__ void __launch_bounds__(256) k_super(const double *__restrict__ phys, double *__restrict__ sup, uint64_t nb,
                                               uint64_t mh)
{
    const uint64_t b0 = blockIdx.x * SB;
    double s = 0.0;
    for (int j = 0; j < 4; ++j) {
        const uint64_t i = threadIdx.x * 4 + j;
        if (b0 + i < nb) s += phys[(b0 + i) ^ mh];
    }
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        sup[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_scan(const double *__restrict__ phys, double *__restrict__ v, uint64_t nb,
                                               uint64_t mh)
{
    __shared__ double part[1024];
    const uint64_t chunk = (nb + blockDim.x - 1) / blockDim.x;
    const uint64_t b0 = threadIdx.x * chunk, b1 = b0 + chunk < nb ? b0 + chunk : nb;
    double s = 0.0;
    for (uint64_t i = b0; i < b1; ++i) s += phys[i ^ mh];
    part[threadIdx.x] = s;
    __syncthreads();
    // Hillis-Steele inclusive scan over the 1024 partials
    for (unsigned off = 1; off < blockDim.x; off <<= 1) {
        double x = threadIdx.x >= off ? part[threadIdx.x - off] : 0.0;
        __syncthreads();
        part[threadIdx.x] += x;
        __syncthreads();
    }
    double run = threadIdx.x ? part[threadIdx.x - 1] : 0.0;
    for (uint64_t i = b0; i < b1; ++i) {
        double x = phys[i ^ mh];
        v[i] = run;
        run += x;
    }
    if (threadIdx.x == blockDim.x - 1) v[nb] = part[blockDim.x - 1];
}

void launch_scan_blocks(const double *d_phys, double *d_prefix, uint64_t nb, uint64_t mh, cudaStream_t st)
{
    // d_prefix: nsb superblock sums, then (in place) their exclusive prefix + total
    const uint64_t nsb = (nb + SB - 1) / SB;
    double *sup = d_prefix + nsb + 1;   // scratch for the raw superblock sums
    k_super<<<(unsigned)nsb, 256, 0, st>>>(d_phys, sup, nb, mh);
    k_scan<<<1, 1024, 0, st>>>(sup, d_prefix, nsb, 0);
}

// one warp per draw
template <typename R>
__global__ void __launch_bounds__(TPB) k_draws(const typename CV<R>::T *__restrict__ psi, uint32_t block_bits,
                                               const double *__restrict__ phys, const double *__restrict__ sprefix,
                                               uint64_t nb, uint64_t n_draws, uint32_t k0, uint32_t k1,
                                               uint64_t leaf, const uint64_t *__restrict__ ltab, uint32_t nlt,
                                               uint64_t omask, double edge_eps, uint64_t xm,
                                               uint64_t *__restrict__ out, uint32_t *__restrict__ edges,
                                               double tg_total, double tg_lo, double tg_hi, uint64_t ohi,
                                               uint64_t *__restrict__ blist)
{
    // Leaves that share one state vector (they differ only in terminal X flips, DESIGN reading #7:
    // measurement noise relabels the drawn bitstring) are drawn in ONE launch: ltab holds
    // the group's nlt + 1 slot offsets (relative, ascending) then its nlt readout masks; warp w is
    // slot w of the group, draw j = w - ltab[k] of leaf leaf + k, outcome XOR masks[k].  Without a
    // table: draw w of `leaf`, outcome XOR omask.
    // sharded mode (tg_total > 0): the draw's point t = u * tg_total on the CDF over all shards in
    // logical order; this shard owns [tg_lo, tg_hi) and searches t - tg_lo locally, writing
    // ohi | local index (ohi = the shard's global bits)
    // logical index i is stored at physical i ^ xm (pending X relabels of the fused path)
    using V = typename CV<R>::T;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (warp >= n_draws) return;
    uint64_t dj = warp, dl = leaf;
    uint64_t om = omask;
    if (ltab) {
        uint32_t lo = 0, hi = nlt - 1;   // last k with ltab[k] <= warp
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (ltab[mid] <= warp) lo = mid; else hi = mid - 1;
        }
        dj = warp - ltab[lo];
        dl = leaf + lo;
        om = ltab[nlt + 1 + lo];
    }
    U4 w = philox10(U4{(uint32_t)dj, (uint32_t)dl, (uint32_t)(dl >> 32), TAG_SHOT}, k0, k1);
    uint64_t x = (uint64_t)w.x | ((uint64_t)w.y << 32);
    const uint64_t nsb = (nb + SB - 1) / SB;
    const uint64_t mh = xm >> block_bits;
    const double T = sprefix[nsb];
    double t;
    if (tg_total > 0.0) {
        const double tg = (double)(x >> 11) * 0x1.0p-53 * tg_total;
        if (!(tg >= tg_lo && tg < tg_hi)) return;   // another shard's draw (warp-uniform)
        t = tg - tg_lo;
    } else {
        t = (double)(x >> 11) * 0x1.0p-53 * T;
    }
    // superblock: first sb whose inclusive prefix sprefix[sb+1] exceeds t
    uint64_t lo = 0, hi = nsb - 1;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (sprefix[mid + 1] > t) hi = mid; else lo = mid + 1;
    }
    const uint64_t sb = lo;
    // block inside the superblock: lane l owns blocks [sb*SB + 32 l, +32)
    const uint64_t bl0 = sb * SB + 32 * lane;
    double ls = 0.0;
    for (uint64_t j = 0; j < 32 && bl0 + j < nb; ++j) ls += phys[(bl0 + j) ^ mh];
    double lincl = ls;
    for (int o = 1; o < 32; o <<= 1) {
        double y = __shfl_up_sync(0xffffffffu, lincl, o);
        if (lane >= (unsigned)o) lincl += y;
    }
    const double sbase = sprefix[sb];
    unsigned bhit = __ballot_sync(0xffffffffu, sbase + lincl > t);
    unsigned bl = bhit ? __ffs(bhit) - 1 : 31;
    while (!bhit && bl > 0 && !__shfl_sync(0xffffffffu, ls > 0.0 ? 1 : 0, bl)) --bl;   // rounding fallback
    uint64_t b = 0;
    double bbase = 0.0;
    if (lane == bl) {
        double run = sbase + lincl - ls;
        uint64_t bb = bl0;
        for (uint64_t j = 0; j < 32 && bl0 + j < nb; ++j) {
            const double v = phys[(bl0 + j) ^ mh];
            bb = bl0 + j;
            if (run + v > t) break;
            run += v;
        }
        b = bb;
        bbase = run;
    }
    b = __shfl_sync(0xffffffffu, b, bl);
    bbase = __shfl_sync(0xffffffffu, bbase, bl);
    if (blist) {   // blocks-only pass: the block this draw lands in (K5 then computes those tiles)
        if (lane == 0) blist[warp] = b;
        return;
    }
    const uint64_t bs = 1ull << block_bits;
    const uint64_t chunk = (bs + 31) / 32;
    const uint64_t c0 = lane * chunk < bs ? lane * chunk : bs, c1 = c0 + chunk < bs ? c0 + chunk : bs;
    const V *blk0 = psi + ((b * bs) ^ (xm & ~(bs - 1)));
    const uint64_t ml = xm & (bs - 1);
    struct Blk {
        const V *p;
        uint64_t m;
        __device__ V operator[](uint64_t i) const { return p[i ^ m]; }
    } blk{blk0, ml};
    double s = 0.0;
    for (uint64_t i = c0; i < c1; ++i) {
        V a = blk[i];
        double re = a.x, im = a.y;
        s += re * re + im * im;
    }
    double incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        double y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    const double base = bbase;
    unsigned hit = __ballot_sync(0xffffffffu, base + incl > t);
    uint64_t k = b * bs + bs - 1;
    bool edge = false;
    if (hit) {
        unsigned L = __ffs(hit) - 1;
        if (lane == L) {
            double run = base + incl - s, prev = run;
            uint64_t kk = c1 - 1;
            bool found = false;
            for (uint64_t i = c0; i < c1; ++i) {
                V a = blk[i];
                double re = a.x, im = a.y;
                double nr = run + (re * re + im * im);
                if (nr > t) { kk = i; prev = run; run = nr; found = true; break; }
                run = nr;
            }
            k = b * bs + kk;
            double gap = fmin(t - prev, run - t);
            edge = !found || gap < edge_eps;
            out[warp] = (k | ohi) ^ om;
            if (edge) atomicAdd(edges, 1u);
        }
    } else {
        // rounding: no C(k) > t in this block -- last nonzero amplitude of the block
        if (lane == 0) {
            uint64_t kk = bs - 1;
            for (uint64_t i = bs; i-- > 0;) {
                V a = blk[i];
                if (a.x != 0 || a.y != 0) { kk = i; break; }
            }
            out[warp] = ((b * bs + kk) | ohi) ^ om;
            atomicAdd(edges, 1u);
        }
    }
}

double launch_draws(const void *psi, uint32_t n, int prec, uint32_t block_bits, const double *d_phys,
                    const double *d_sprefix, uint64_t n_draws, uint64_t seed, uint64_t leaf, const uint64_t *d_ltab,
                    uint32_t nlt, uint64_t omask, double edge_eps, uint64_t xm, uint64_t *d_out, uint32_t *d_edges,
                    cudaStream_t st, uint64_t *d_blist)
{
    if (!n_draws) return 0.0;
    uint64_t nb = 1ull << (n - block_bits);
    unsigned grid = (unsigned)((n_draws * 32 + TPB - 1) / TPB);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    if (prec == 64)
        k_draws<float><<<grid, TPB, 0, st>>>((const float2 *)psi, block_bits, d_phys, d_sprefix, nb, n_draws, k0, k1,
                                             leaf, d_ltab, nlt, omask, edge_eps, xm, d_out, d_edges, 0.0, 0.0, 0.0, 0,
                                             d_blist);
    else
        k_draws<double><<<grid, TPB, 0, st>>>((const double2 *)psi, block_bits, d_phys, d_sprefix, nb, n_draws, k0,
                                              k1, leaf, d_ltab, nlt, omask, edge_eps, xm, d_out, d_edges, 0.0, 0.0, 0.0,
                                              0, d_blist);
    return (double)n_draws * (double)(1ull << block_bits) * (prec == 64 ? 8.0 : 16.0);
}

// sharded mode: the draws of one leaf that fall into this shard's CDF window [t_lo, t_hi)
double launch_draws_window(const void *psi, uint32_t n, int prec, uint32_t block_bits, const double *d_phys,
                           const double *d_sprefix, uint64_t n_draws, uint64_t seed, uint64_t leaf, uint64_t omask,
                           double edge_eps, uint64_t *d_out, uint32_t *d_edges, double t_total, double t_lo,
                           double t_hi, uint64_t ohi, cudaStream_t st)
{
    if (!n_draws) return 0.0;
    uint64_t nb = 1ull << (n - block_bits);
    unsigned grid = (unsigned)((n_draws * 32 + TPB - 1) / TPB);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    if (prec == 64)
        k_draws<float><<<grid, TPB, 0, st>>>((const float2 *)psi, block_bits, d_phys, d_sprefix, nb, n_draws, k0, k1,
                                             leaf, nullptr, 0, omask, edge_eps, 0, d_out, d_edges, t_total, t_lo, t_hi,
                                             ohi, nullptr);
    else
        k_draws<double><<<grid, TPB, 0, st>>>((const double2 *)psi, block_bits, d_phys, d_sprefix, nb, n_draws, k0,
                                              k1, leaf, nullptr, 0, omask, edge_eps, 0, d_out, d_edges, t_total, t_lo,
                                              t_hi, ohi, nullptr);
    return (double)n_draws * (double)(1ull << block_bits) * (prec == 64 ? 8.0 : 16.0);
}

// draws of leaves whose state is a known basis state (every draw = that index ^ readout mask):
// trip = ntrip (slot offset, count, value) triples, one warp per triple
__global__ void __launch_bounds__(TPB) k_fill_slots(const uint64_t *__restrict__ trip, uint64_t ntrip,
                                                    uint64_t *__restrict__ slots)
{
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= ntrip) return;
    const uint64_t off = trip[3 * w], cnt = trip[3 * w + 1], val = trip[3 * w + 2];
    for (uint64_t j = threadIdx.x & 31; j < cnt; j += 32) slots[off + j] = val;
}

void launch_fill_slots(const uint64_t *d_trip, uint64_t ntrip, uint64_t *d_slots, cudaStream_t st)
{
    if (!ntrip) return;
    k_fill_slots<<<(unsigned)((ntrip * 32 + TPB - 1) / TPB), TPB, 0, st>>>(d_trip, ntrip, d_slots);
}

}  // namespace tq
