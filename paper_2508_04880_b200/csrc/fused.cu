// K5: fused-tile gate kernel and its host planner.
//
// One launch applies a run of gates (a "group") to the whole 2^n state in ONE HBM sweep
// (read + write 2 * 2^n * s bytes), instead of one sweep per gate (Eq. 1: a k-qubit
// gate touches only its own amplitude pairs, so gates confined to a 12-qubit tile commute with
// the tiling).  Design:
//   - a tile = the 4096 amplitudes that share the values of the n-12 "outer" qubits; tile qubits
//     are qubits 0,1,2 (128-byte contiguous runs) plus the group's exchange qubits plus fillers;
//   - 128 threads x 32 register-resident amplitudes; 5 "register" tile bits, 5 lane bits, 2 warp
//     bits.  A gate that exchanges amplitudes (H, RX, RY, U, X, Y, CX target) needs its qubit in a
//     register bit: the planner splits the group into phases with different register sets and the
//     kernel switches phases by one shared-memory transpose (XOR-swizzled, conflict-free when
//     lanes 0-2 carry qubits 0-2);
//   - diagonal gates and CX/CZ/CP controls act on ANY qubit: register bits at compile-time
//     positions, thread/outer bits through per-thread predicates on the logical index;
//   - H is applied as an unscaled butterfly; the (1/sqrt2)^h factor (and global phases of
//     relabelled Y) is applied once at the store;
//   - X (and the X part of Y) on a qubit's first or last touch in a group is a free RELABEL:
//     the state is stored as physical = logical XOR mask, loads/stores XOR their addresses,
//     and the tile part of the mask is materialized by the next sweep at no cost;
//   - a reset to a basis state (K7) is fused into the first sweep (no load);
//   - the last sweep before sampling can emit per-4096-block |amp|^2 sums (K6 epilogue).
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "fused.h"
#include "kernels.h"

namespace tq {
namespace fk {

constexpr int TB = 12;     // tile bits
#ifndef TQ_RB
#define TQ_RB 5
#endif
constexpr int RB = TQ_RB;          // register bits (5: 32 amplitudes per thread, 4: 16)
constexpr int NR = 1 << RB;        // amplitudes per thread
constexpr int NTB = TB - RB;       // thread bits (5 lane bits + warp bits)
constexpr int NT = 1 << NTB;       // threads per CTA
constexpr int MAXPH = 24;
#ifndef TQ_NG
#define TQ_NG 2
#endif
#ifndef TQ_NBUF
#define TQ_NBUF 3
#endif
constexpr int NG = TQ_NG;      // tile groups (of NT threads) per CTA
constexpr int NBUF = TQ_NBUF;  // tile buffers per CTA (shared memory)
// One mbarrier per (buffer, group) pair, i.e. per tile index mod NBUF * NG: the tiles of a buffer
// alternate between the groups, and with one barrier per buffer a group could wait on the phase
// two ahead of the one in flight and see its parity as already complete (phase aliasing; it let a
// group read a tile still landing and over-arrive on the barrier -- a launch failure at 24q).
// Per pair, every barrier has ONE consumer that waits its phases in order.
constexpr int NMB = NBUF * NG;
constexpr int MAXG = 400;
constexpr int MAXP = 1600;

enum Code : uint16_t {
    C_H = 0,      // +r      unscaled butterfly
    C_U = 5,      // +r      generic 2x2 (8 params)
    C_X = 10,     // +r
    C_Y = 15,     // +r
    C_D1 = 20,    // +r      bit 1 *= p (2 params)
    C_D2 = 25,    // +r      bit 0 *= p0, bit 1 *= p1 (4 params)
    C_CX = 30,    // +5c+t   (c != t)
    C_CPH = 55,   // +5a+b   (a < b) both bits 1 *= p
    C_TX = 80,    // +t      if pred(q): X on reg t
    C_TD1 = 85,   // +r      if pred(q): bit 1 of reg r *= p
    C_TPH = 90,   //         all *= pred(q0)&pred(q1) ? p1 : p0 (4 params)
    C_DK = 91,    // +mask   a[r] *= tab[pext(r, mask)]  (2 * 2^popc(mask) params)
    C_CX2 = 123,  // +25c+5t1+t2 (t1 < t2): CX(c->t1) CX(c->t2) as ONE swap pass
    C_CU = 248,   // +6p+j   2x2 on bit p per pattern of the control pair j (Toffoli cores), 32 params
    C_CCX = 278,  // +6p+j   Toffoli on register bits: swap bit p where both controls of pair j are 1
    C_TDK = 308,  // +r      bit 1 of reg r *= prod_k (pred(q_k) ? e^{i t_k} : 1), a = k count: 2a params
                  //         (q_k, t_k as a u64 turn fraction), or b = 1: 2 params (c, M), t_k = c << q_k
    C_DKC = 313,  // +16t+m  bit t of r set: a[r] *= tab[pext(r, M)], M = the 4-bit m spread over the
                  //         register bits other than t (2 * 2^popc(m) params): a diagonal table whose
                  //         entries with bit t clear are 1 (a CP ladder onto t), half the multiplies
    C_N = 393,    // number of gate codes
    C_XPOSE = 393 // transpose registers to phase a
};

// the j-th (0..5) pair {u < v} of register bits other than p, as a mask (with p): the diagonal of a
// Toffoli core H(t) DK(a, b, t) H(t)
__host__ __device__ constexpr int hdh_mask(int p, int j)
{
    int k = 0;
    for (int u = 0; u < 5; ++u)
        for (int v = u + 1; v < 5; ++v) {
            if (u == p || v == p) continue;
            if (k == j) return (1 << p) | (1 << u) | (1 << v);
            ++k;
        }
    return 0;
}

// m (4 bits) spread over the 5 register bits other than t
__host__ __device__ constexpr int spread_skip(int m, int t)
{
    int o = 0, k = 0;
    for (int b = 0; b < 5; ++b) {
        if (b == t) continue;
        if ((m >> k) & 1) o |= 1 << b;
        ++k;
    }
    return o;
}

__host__ __device__ constexpr int pext5(int r, int m)
{
    int o = 0, k = 0;
    for (int b = 0; b < 5; ++b)
        if ((m >> b) & 1) { o |= ((r >> b) & 1) << k; ++k; }
    return o;
}

struct Phase {
    uint16_t g0, g1;      // gate range
    uint8_t rl[RB];       // tile-local bit of each register bit
    uint8_t tl[8];        // tile-local bit of each thread bit (lanes 0-4, then warp bits)
    uint16_t so[NR];      // entering this phase: tile-local index read into register r
    uint16_t so_out[NR];  // leaving this phase: tile-local index register r is written to
                          // (they differ when register permutations are absorbed, host-computed)
};

struct GRec {
    uint16_t code;
    uint8_t a, b;         // TX/TD1: a = global control qubit; TPH: a, b = global qubits
    uint16_t pi;          // parameter index into prm
    uint16_t _pad;
};

enum : uint32_t { F_INIT = 1, F_SUMS = 2, F_SCALE = 4, F_LBASE = 8, F_BULK = 16, F_LIVE = 32, F_VMASK = 64, F_TSTORE = 128,
                  F_NOSTORE = 256,   // block sums only: the state is not written (the sampler's chosen
                                     // tiles are recomputed by an F_TLIST launch of the same group)
                  F_TLIST = 512,     // visit only the tiles tlist[i] ^ tl_xor, i < nlist (device list)
                  F_DBG_NOSTORE = 1u << 31 };   // (debug-knob builds only: skip the stores, for timing)
constexpr int NCH = 4;             // 8-bit chunks of the tile index (n <= TB + 8 * NCH = 44 fused)

// Qubit layout: the state may be stored with its qubits permuted (logical qubit q at physical bit
// position pi(q)); logical index l lives at physical address pi(l ^ xm).  A sweep reads with the
// layout pi_in and writes with pi_out, chosen by the planner so that the NEXT group's 12 tile
// qubits sit at physical positions 0..11 -- every tile read after the first group of a transition
// is one contiguous 64 KiB block; transitions begin and end in the
// identity layout.
struct Params {
    uint64_t xm_load, xm_store;   // logical X-relabel mask at load / at store (outer bits only)
    uint64_t xin, xout;           // xm_store in the read / write layout
    uint32_t init_t, init_r;      // F_INIT: the state is init_re + i init_im at ONE element: register
                                  //   init_r of thread init_t of the (single, F_LIVE) tile, 0 elsewhere
    uint64_t lfree, lfix;         // F_LIVE: only the tiles T = pdep(i, lfree) | lfix, i < nlive, can hold
    uint64_t nlive;               //   nonzero amplitudes (support analysis); the rest stay zero
    const uint64_t *tlist;        // F_TLIST: device list of tile indices (XOR tl_xor), nlist of them
    uint64_t nlist, tl_xor;
    uint64_t vfree, vfix;         // F_VMASK (read layout = identity): the buffer holds the state only on
                                  //   {x : (x & ~vfree) == vfix}; elsewhere it is zero but not written:
                                  //   tiles outside are not loaded (zeros), elements outside read as 0
    uint32_t vl_mask, vl_val;     //   the same condition on the tile-local bits
    // F_TSTORE: the tile is written through shared memory by bulk copies (TMA engine): registers go
    // to the tile buffer in WRITE order (tile bits sorted by write position), whose runs of 2^ts_l0
    // elements are contiguous in both places; run i lands at the tile base + pdep(i, ts_hi) where
    // ts_hi holds the write positions of write-order bits ts_l0..11
    uint8_t ts_l0;
    uint8_t ts_hipos[TB];         //   write position of write-order bit ts_l0 + k
    uint8_t wpos[TB];             //   write-order bit of tile-local bit b
    uint16_t wreg[NR];            //   write-order offset (bytes at launch) of register r in the last phase
    double init_re, init_im;
    double scale_re, scale_im;
    uint64_t ntiles;
    uint32_t flags, nphase, ngate, nout;
    uint8_t qs[TB];               // tile-local bit b <-> logical qubit qs[b] (tile-local order = read order)
    uint8_t pin[TB], pout[TB];    // physical read / write position of tile-local bit b
    uint8_t oo[64], ol[64];       // tile-index bit k (outer qubits in read order): write / logical position
    uint32_t rx;                  // register bits where xm_load is set (folded into gl, kept 0)
    uint16_t mloc;                // tile-local bits of xm_load (applied when copying to shared memory)
    uint16_t last_xpose;          // record index of the last transpose (0xFFFF: none)
    uint16_t gtab;                // 0xFFFF, or: prm + gtab holds a u16[NR][NT] gather table (byte offsets):
                                  // the phase-0 read takes register r of thread t from slot gtab[r][t]
    uint16_t st_pair;             // 0, or v: registers r, r ^ v hold adjacent amplitudes in the last
                                  // layout -> one 2x-wide store per pair
    uint32_t st_odd;              // bit r: register r holds the odd one of its pair
    uint64_t regm_load;           // global mask of the phase-0 register qubits
    uint64_t outer;               // read-layout mask of the outer (non-tile) positions
    uint64_t dstep;               // pdep(gridDim.x * NG, outer): next tile of the same group (read layout)
    uint64_t dissue[NG];          // pdep(T(j + NBUF) - T(j), outer) for a tile j of group g
    // gj, gs, sj and the phases' so / so_out are BYTE offsets at launch (element offsets while
    // the host plans): the kernel adds them to byte pointers with no index scaling
    uint64_t gj[NR];              // global offset of tile-local index (j << NTB) (copy slots)
    uint16_t sj[NR];              // swz(j << NTB): swizzled shared-memory part of copy slot j
    uint16_t so0[NR];             // F_BULK: phase-0 read offsets (bytes) into the LINEAR tile buffer
    uint64_t gl[NR];              // phase 0: global element offset of register r (additive)
    uint64_t gs[NR];              // last phase: global offset of register r (additive)
    Phase ph[MAXPH];
    GRec g[MAXG];
    double prm[MAXP];
};
static_assert(sizeof(Params) < 32000, "kernel parameter block too large");

template <typename R> struct CV;
template <> struct CV<double> { using T = double2; };
template <> struct CV<float> { using T = float2; };

__device__ __forceinline__ uint64_t ins0(uint64_t j, uint32_t q)
{
    return ((j >> q) << (q + 1)) | (j & ((1ull << q) - 1));
}

template <typename V, typename R>
__device__ __forceinline__ V mulc(V a, R pr, R pi)
{
    V r;
    r.x = a.x * pr - a.y * pi;
    r.y = a.x * pi + a.y * pr;
    return r;
}

// a *= (pr + i pi) in place.  Written in PTX with read-write operands so the results stay in a's
// registers (C++ lets the compiler allocate fresh registers and copy back at the switch join).
__device__ __forceinline__ void cmul_ip(double2 &a, double pr, double pi)
{
    asm volatile("{\n\t.reg .f64 u, v;\n\t"
                 "mul.f64 u, %1, %3;\n\t"
                 "mul.f64 v, %0, %3;\n\t"
                 "neg.f64 u, u;\n\t"
                 "fma.rn.f64 %0, %0, %2, u;\n\t"
                 "fma.rn.f64 %1, %1, %2, v;\n\t}"
                 : "+d"(a.x), "+d"(a.y) : "d"(pr), "d"(pi));
}
__device__ __forceinline__ void cmul_ip(float2 &a, float pr, float pi)
{
    asm volatile("{\n\t.reg .f32 u, v;\n\t"
                 "mul.f32 u, %1, %3;\n\t"
                 "mul.f32 v, %0, %3;\n\t"
                 "neg.f32 u, u;\n\t"
                 "fma.rn.f32 %0, %0, %2, u;\n\t"
                 "fma.rn.f32 %1, %1, %2, v;\n\t}"
                 : "+f"(a.x), "+f"(a.y) : "f"(pr), "f"(pi));
}
// unscaled butterfly in place: y <- x - y, x <- 2x - y  (= x + y up to one rounding)
__device__ __forceinline__ void bfly_ip(double2 &x, double2 &y)
{
    asm volatile("{\n\t.reg .f64 s, t;\n\t"
                 "sub.rn.f64 %2, %0, %2;\n\tsub.rn.f64 %3, %1, %3;\n\t"
                 "neg.f64 s, %2;\n\tneg.f64 t, %3;\n\t"
                 "fma.rn.f64 %0, 0d4000000000000000, %0, s;\n\tfma.rn.f64 %1, 0d4000000000000000, %1, t;\n\t}"
                 : "+d"(x.x), "+d"(x.y), "+d"(y.x), "+d"(y.y));
}
__device__ __forceinline__ void bfly_ip(float2 &x, float2 &y)
{
    asm volatile("{\n\t.reg .f32 s, t;\n\t"
                 "sub.rn.f32 %2, %0, %2;\n\tsub.rn.f32 %3, %1, %3;\n\t"
                 "neg.f32 s, %2;\n\tneg.f32 t, %3;\n\t"
                 "fma.rn.f32 %0, 0f40000000, %0, s;\n\tfma.rn.f32 %1, 0f40000000, %1, t;\n\t}"
                 : "+f"(x.x), "+f"(x.y), "+f"(y.x), "+f"(y.y));
}

// ---------------------------------------------------------------- register gate ops
// Every op updates its registers IN PLACE (no result lands in a fresh register): the gate loop
// is a switch inside a loop over 128 live registers, and any renaming inside a case costs a
// copy of the whole amplitude set at the join (measured: 66 % of executed instructions were
// moves before this).  Swaps are explicit XOR-swaps in PTX so that ptxas cannot rename them.
__device__ __forceinline__ void xswap(double &x, double &y)
{
    long long a = __double_as_longlong(x), b = __double_as_longlong(y);
    asm volatile("xor.b64 %0, %0, %1;\n\txor.b64 %1, %1, %0;\n\txor.b64 %0, %0, %1;" : "+l"(a), "+l"(b));
    x = __longlong_as_double(a);
    y = __longlong_as_double(b);
}
__device__ __forceinline__ void xswap(float &x, float &y)
{
    int a = __float_as_int(x), b = __float_as_int(y);
    asm volatile("xor.b32 %0, %0, %1;\n\txor.b32 %1, %1, %0;\n\txor.b32 %0, %0, %1;" : "+r"(a), "+r"(b));
    x = __int_as_float(a);
    y = __int_as_float(b);
}
template <typename V>
__device__ __forceinline__ void vswap(V &x, V &y)
{
    xswap(x.x, y.x);
    xswap(x.y, y.y);
}

template <int B, typename V>
__device__ __forceinline__ void g_h(V (&a)[NR])
{
    // unscaled butterfly (x, y) -> (x + y, x - y), in place: y <- x - y, x <- 2x - y
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if (!(i & (1 << B))) bfly_ip(a[i], a[i | (1 << B)]);
}

template <int B, typename V, typename R>
__device__ __forceinline__ void g_u(V (&a)[NR], const double *p)
{
    const R u0r = (R)p[0], u0i = (R)p[1], u1r = (R)p[2], u1i = (R)p[3];
    const R u2r = (R)p[4], u2i = (R)p[5], u3r = (R)p[6], u3i = (R)p[7];
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if (!(i & (1 << B))) {
            V x = a[i], y = a[i | (1 << B)];
            a[i].x = u0r * x.x - u0i * x.y + u1r * y.x - u1i * y.y;
            a[i].y = u0r * x.y + u0i * x.x + u1r * y.y + u1i * y.x;
            a[i | (1 << B)].x = u2r * x.x - u2i * x.y + u3r * y.x - u3i * y.y;
            a[i | (1 << B)].y = u2r * x.y + u2i * x.x + u3r * y.y + u3i * y.x;
        }
}

template <int B, typename V>
__device__ __forceinline__ void g_x(V (&a)[NR])
{
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if (!(i & (1 << B))) vswap(a[i], a[i | (1 << B)]);
}

template <int B, typename V>
__device__ __forceinline__ void g_y(V (&a)[NR])
{
    // (Y psi)_0 = -i psi_1, (Y psi)_1 = i psi_0: swap, then in-place (exact) multiplies by -i / +i
    // (a re/im register exchange here made ptxas copy every amplitude at each gate dispatch)
    using R = decltype(a[0].x);
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if (!(i & (1 << B))) {
            vswap(a[i], a[i | (1 << B)]);
            cmul_ip(a[i], R(0), R(-1));
            cmul_ip(a[i | (1 << B)], R(0), R(1));
        }
}

template <int B, typename V, typename R>
__device__ __forceinline__ void g_d1(V (&a)[NR], R pr, R pi)
{
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if (i & (1 << B)) cmul_ip(a[i], pr, pi);
}

template <int B, typename V, typename R>
__device__ __forceinline__ void g_d2(V (&a)[NR], const double *p)
{
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i & (1 << B)) cmul_ip(a[i], (R)p[2], (R)p[3]);
        else cmul_ip(a[i], (R)p[0], (R)p[1]);
    }
}

// CX(c->t1) then CX(c->t2): control-1 registers r move to r ^ t1 ^ t2 -- 8 swaps, like one CX
template <int C, int T1, int T2, typename V>
__device__ __forceinline__ void g_cx2(V (&a)[NR])
{
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if ((i & (1 << C)) && !(i & (1 << T1))) vswap(a[i], a[i ^ (1 << T1) ^ (1 << T2)]);
}

// CX(c -> t); with MASK, C is a mask of control bits (all must be 1: a Toffoli for two bits)
template <int C, int T, typename V, bool MASK = false>
__device__ __forceinline__ void g_cx(V (&a)[NR])
{
    constexpr int CM = MASK ? C : (1 << C);
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if ((i & CM) == CM && !(i & (1 << T))) vswap(a[i], a[i | (1 << T)]);
}

template <int A, int B, typename V, typename R>
__device__ __forceinline__ void g_cph(V (&a)[NR], R pr, R pi)
{
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if ((i & (1 << A)) && (i & (1 << B))) cmul_ip(a[i], pr, pi);
}

template <int M, typename V, typename R>
__device__ __forceinline__ void g_dk(V (&a)[NR], const double *tab)
{
    // straight-line: the 2^k table entries are loaded up front, then 32 independent complex
    // multiplies (per-entry "skip if 1" branches were measured slower: they serialize the warp)
    constexpr int K = __builtin_popcount(M);
    R tr[1 << K], ti[1 << K];
#pragma unroll
    for (int idx = 0; idx < (1 << K); ++idx) { tr[idx] = (R)tab[2 * idx]; ti[idx] = (R)tab[2 * idx + 1]; }
#pragma unroll
    for (int i = 0; i < NR; ++i) cmul_ip(a[i], tr[pext5(i, M)], ti[pext5(i, M)]);
}

template <int T, int M, typename V, typename R>
__device__ __forceinline__ void g_dkc(V (&a)[NR], const double *tab)
{
    constexpr int K = __builtin_popcount(M);
    R tr[1 << K], ti[1 << K];
#pragma unroll
    for (int idx = 0; idx < (1 << K); ++idx) { tr[idx] = (R)tab[2 * idx]; ti[idx] = (R)tab[2 * idx + 1]; }
#pragma unroll
    for (int i = 0; i < NR; ++i)
        if ((i >> T) & 1) cmul_ip(a[i], tr[pext5(i, M)], ti[pext5(i, M)]);
}

// new (x, y) = (m00 x + m01 y, m10 x + m11 y), in place
__device__ __forceinline__ void mat2_ip(double2 &x, double2 &y, const double *m)
{
    asm volatile("{\n\t.reg .f64 a, b, c, d;\n\t"
                 "mul.f64 a, %4, %0;\n\tneg.f64 b, %5;\n\tfma.rn.f64 a, b, %1, a;\n\t"
                 "neg.f64 d, %7;\n\tfma.rn.f64 a, d, %3, a;\n\tfma.rn.f64 a, %6, %2, a;\n\t"
                 "mul.f64 b, %4, %1;\n\tfma.rn.f64 b, %5, %0, b;\n\tfma.rn.f64 b, %6, %3, b;\n\tfma.rn.f64 b, %7, %2, b;\n\t"
                 "mul.f64 c, %8, %0;\n\tneg.f64 d, %9;\n\tfma.rn.f64 c, d, %1, c;\n\tfma.rn.f64 c, %10, %2, c;\n\t"
                 "neg.f64 d, %11;\n\tfma.rn.f64 c, d, %3, c;\n\t"
                 "mul.f64 d, %8, %1;\n\tfma.rn.f64 d, %9, %0, d;\n\tfma.rn.f64 d, %10, %3, d;\n\tfma.rn.f64 d, %11, %2, d;\n\t"
                 "mov.f64 %0, a;\n\tmov.f64 %1, b;\n\tmov.f64 %2, c;\n\tmov.f64 %3, d;\n\t}"
                 : "+d"(x.x), "+d"(x.y), "+d"(y.x), "+d"(y.y)
                 : "d"(m[0]), "d"(m[1]), "d"(m[2]), "d"(m[3]), "d"(m[4]), "d"(m[5]), "d"(m[6]), "d"(m[7]));
}
__device__ __forceinline__ void mat2_ip(float2 &x, float2 &y, const double *md)
{
    const float m0 = (float)md[0], m1 = (float)md[1], m2 = (float)md[2], m3 = (float)md[3];
    const float m4 = (float)md[4], m5 = (float)md[5], m6 = (float)md[6], m7 = (float)md[7];
    asm volatile("{\n\t.reg .f32 a, b, c, d;\n\t"
                 "mul.f32 a, %4, %0;\n\tneg.f32 b, %5;\n\tfma.rn.f32 a, b, %1, a;\n\t"
                 "neg.f32 d, %7;\n\tfma.rn.f32 a, d, %3, a;\n\tfma.rn.f32 a, %6, %2, a;\n\t"
                 "mul.f32 b, %4, %1;\n\tfma.rn.f32 b, %5, %0, b;\n\tfma.rn.f32 b, %6, %3, b;\n\tfma.rn.f32 b, %7, %2, b;\n\t"
                 "mul.f32 c, %8, %0;\n\tneg.f32 d, %9;\n\tfma.rn.f32 c, d, %1, c;\n\tfma.rn.f32 c, %10, %2, c;\n\t"
                 "neg.f32 d, %11;\n\tfma.rn.f32 c, d, %3, c;\n\t"
                 "mul.f32 d, %8, %1;\n\tfma.rn.f32 d, %9, %0, d;\n\tfma.rn.f32 d, %10, %3, d;\n\tfma.rn.f32 d, %11, %2, d;\n\t"
                 "mov.f32 %0, a;\n\tmov.f32 %1, b;\n\tmov.f32 %2, c;\n\tmov.f32 %3, d;\n\t}"
                 : "+f"(x.x), "+f"(x.y), "+f"(y.x), "+f"(y.y)
                 : "f"(m0), "f"(m1), "f"(m2), "f"(m3), "f"(m4), "f"(m5), "f"(m6), "f"(m7));
}

// Controlled 2x2 on bit P: for each pattern b of the control bits CM, the block of amplitude
// pairs (bit P = 0, 1) gets the matrix m[8b .. 8b+7] (m00, m01, m10, m11 complex).  The host
// classifies each block (2 bits of `kinds` per block): 0 identity (skipped), 1 diagonal,
// 2 anti-diagonal (swap, then the two entries unless bit b of `unit` says they are 1), 3 general.
// This is H(t) DK(a, b, t) H(t) DK(a, b) -- a Toffoli core with its control phases -- which for a
// Toffoli is the identity on three blocks and a plain swap on the fourth.
template <int P, int CM, typename V, typename R>
__device__ __forceinline__ void g_cu(V (&a)[NR], const double *m, uint32_t kinds, uint32_t unit)
{
    constexpr int NB = 1 << __builtin_popcount(CM);
#pragma unroll
    for (int bi = 0; bi < NB; ++bi) {
        const uint32_t kd = (kinds >> (2 * bi)) & 3u;
        const double *q = m + 8 * bi;
        if (kd == 1) {
            const R d0r = (R)q[0], d0i = (R)q[1], d1r = (R)q[6], d1i = (R)q[7];
#pragma unroll
            for (int i = 0; i < NR; ++i)
                if (!(i & (1 << P)) && pext5(i, CM) == bi) {
                    cmul_ip(a[i], d0r, d0i);
                    cmul_ip(a[i | (1 << P)], d1r, d1i);
                }
        } else if (kd == 2) {
#pragma unroll
            for (int i = 0; i < NR; ++i)
                if (!(i & (1 << P)) && pext5(i, CM) == bi) vswap(a[i], a[i | (1 << P)]);
            if (!((unit >> bi) & 1u)) {
                const R xr = (R)q[2], xi = (R)q[3], yr = (R)q[4], yi = (R)q[5];
#pragma unroll
                for (int i = 0; i < NR; ++i)
                    if (!(i & (1 << P)) && pext5(i, CM) == bi) {
                        cmul_ip(a[i], xr, xi);
                        cmul_ip(a[i | (1 << P)], yr, yi);
                    }
            }
        } else if (kd == 3) {
#pragma unroll
            for (int i = 0; i < NR; ++i)
                if (!(i & (1 << P)) && pext5(i, CM) == bi) mat2_ip(a[i], a[i | (1 << P)], q);
        }
    }
}

// One gate record.  C is a compile-time code; the dispatch below is a balanced binary tree of
// compile-time ranges (7 compare-and-branch levels) instead of the linear compare chain ptxas
// emits for a 123-way switch.
// does code C only name register positions < RB (and DK masks < NR)?
__host__ __device__ constexpr bool code_ok(int C)
{
    if (C < C_CX) return (C % 5) < RB;
    if (C < C_CPH) return (C - C_CX) / 5 < RB && (C - C_CX) % 5 < RB;
    if (C < C_TX) return (C - C_CPH) / 5 < RB && (C - C_CPH) % 5 < RB;
    if (C < C_TPH) return (C - C_TX) % 5 < RB;
    if (C == C_TPH) return true;
    if (C < C_CX2) return C - C_DK < NR;
    if (C >= C_DKC) return (C - C_DKC) / 16 < RB;
    if (C >= C_TDK) return (C - C_TDK) < RB;
    if (C >= C_CCX) return hdh_mask((C - C_CCX) / 6, (C - C_CCX) % 6) < NR;
    if (C >= C_CU) return hdh_mask((C - C_CU) / 6, (C - C_CU) % 6) < NR;
    const int c = (C - C_CX2) / 25, t1 = (C - C_CX2) / 5 % 5, t2 = (C - C_CX2) % 5;
    return c < RB && t1 < RB && t2 < RB && t1 < t2 && c != t1 && c != t2;
}

template <int C, typename V, typename R>
__device__ __forceinline__ void gate_case(V (&a)[NR], const double *p, uint64_t lbase, uint32_t ga, uint32_t gb)
{
    if constexpr (!code_ok(C)) {
        return;
    } else if constexpr (C < C_U) {
        g_h<C - C_H>(a);
    } else if constexpr (C < C_X) {
        g_u<C - C_U, V, R>(a, p);
    } else if constexpr (C < C_Y) {
        g_x<C - C_X>(a);
    } else if constexpr (C < C_D1) {
        g_y<C - C_Y>(a);
    } else if constexpr (C < C_D2) {
        g_d1<C - C_D1, V, R>(a, (R)p[0], (R)p[1]);
    } else if constexpr (C < C_CX) {
        g_d2<C - C_D2, V, R>(a, p);
    } else if constexpr (C < C_CPH) {
        constexpr int c = (C - C_CX) / 5, t = (C - C_CX) % 5;
        if constexpr (c != t) g_cx<c, t>(a);
    } else if constexpr (C < C_TX) {
        constexpr int x = (C - C_CPH) / 5, y = (C - C_CPH) % 5;
        if constexpr (x < y) g_cph<x, y, V, R>(a, (R)p[0], (R)p[1]);
    } else if constexpr (C < C_TD1) {
        if ((lbase >> ga) & 1) g_x<C - C_TX>(a);
    } else if constexpr (C < C_TPH) {
        if ((lbase >> ga) & 1) g_d1<C - C_TD1, V, R>(a, (R)p[0], (R)p[1]);
    } else if constexpr (C == C_TPH) {
        const bool pred = ((lbase >> ga) & 1) && ((lbase >> gb) & 1);
        const R fr = (R)(pred ? p[2] : p[0]), fi = (R)(pred ? p[3] : p[1]);
        if (fr != R(1) || fi != R(0)) {
#pragma unroll
            for (int i = 0; i < NR; ++i) cmul_ip(a[i], fr, fi);
        }
    } else if constexpr (C >= C_DKC) {
        constexpr int t = (C - C_DKC) / 16;
        if constexpr (t < RB) g_dkc<t, spread_skip((C - C_DKC) % 16, t), V, R>(a, p);
    } else if constexpr (C >= C_TDK) {
        // a run of controlled phases from outer/thread qubits onto one register bit (QFT ladders):
        // the per-thread factor is e^{2 pi i acc / 2^64}, acc = sum of the set predicates' angles
        // as 64-bit turn fractions (integer adds, no chain of complex products), ONE sincospi.
        // gb = 1 (geometric weights, a QFT ladder: angle_k = c * 2^{q_k} turns / 2^64):
        // acc = (lbase & M) * c, a single multiply.
        uint64_t acc = 0;
        if (gb) {
            acc = (lbase & (uint64_t)__double_as_longlong(p[1])) * (uint64_t)__double_as_longlong(p[0]);
        } else {
            for (uint32_t k = 0; k < ga; ++k)
                if ((lbase >> (uint32_t)__double_as_longlong(p[2 * k])) & 1)
                    acc += (uint64_t)__double_as_longlong(p[2 * k + 1]);
        }
        if (acc) {
            double sn, cs;
            sincospi((double)(long long)acc * 0x1p-63, &sn, &cs);
            g_d1<C - C_TDK, V, R>(a, (R)cs, (R)sn);
        }
    } else if constexpr (C >= C_CCX) {
        constexpr int pb = (C - C_CCX) / 6;
        g_cx<(hdh_mask(pb, (C - C_CCX) % 6) & ~(1 << pb)), pb, V, true>(a);
    } else if constexpr (C >= C_CU) {
        constexpr int pb = (C - C_CU) / 6;
        g_cu<pb, hdh_mask(pb, (C - C_CU) % 6) & ~(1 << pb), V, R>(a, p, gb, ga);
    } else if constexpr (C >= C_CX2) {
        constexpr int c = (C - C_CX2) / 25, t1 = (C - C_CX2) / 5 % 5, t2 = (C - C_CX2) % 5;
        g_cx2<c, t1, t2>(a);
    } else if constexpr (C < C_N) {
        if constexpr (C - C_DK > 0) g_dk<C - C_DK, V, R>(a, p);
    }
}

template <int LO, int HI, typename V, typename R>
__device__ __forceinline__ void dispatch(int code, V (&a)[NR], const double *p, uint64_t lbase, uint32_t ga,
                                         uint32_t gb)
{
    if constexpr (HI - LO == 1) {
        gate_case<LO, V, R>(a, p, lbase, ga, gb);
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (code < MID) dispatch<LO, MID, V, R>(code, a, p, lbase, ga, gb);
        else dispatch<MID, HI, V, R>(code, a, p, lbase, ga, gb);
    }
}

template <typename V, typename R>
__device__ __forceinline__ void apply_gate(V (&a)[NR], const GRec &g, const double *prm, uint64_t lbase)
{
    // fast paths for the two hottest classes (H and diagonal tables: ~2/3 of all records)
    // ordered by frequency in Adder groups: Toffoli swaps, CX, diagonal tables, H, CU, rest
    const int c = g.code;
    if (c >= C_DKC) dispatch<C_DKC, C_N, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c >= C_TDK) dispatch<C_TDK, C_DKC, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c >= C_CCX) dispatch<C_CCX, C_TDK, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c >= C_CX && c < C_CPH) dispatch<C_CX, C_CPH, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c >= C_DK && c < C_DK + NR) dispatch<C_DK, C_DK + NR, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c < C_U) dispatch<0, C_U, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c >= C_CU) dispatch<C_CU, C_CCX, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c < C_CX) dispatch<C_U, C_CX, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else if (c < C_DK) dispatch<C_CPH, C_DK, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
    else dispatch<C_CX2, C_CU, V, R>(c, a, prm + g.pi, lbase, g.a, g.b);
}

// shared-memory swizzle of a 12-bit tile index: the 16-byte slot's low 3 bits (its bank group
// within a 128-byte wavefront) XOR a fold of the 9 high bits, so that the 8 lanes of a
// quarter-warp hit distinct bank groups whichever 3 tile bits the lanes carry in a phase layout
// The swizzle is GF(2)-linear (swz(a ^ b) = swz(a) ^ swz(b)), so per-register parts are
// swizzled on the host (Phase.so / so_out, Params.sj) and the kernel XORs one swizzled thread part.
__host__ __device__ __forceinline__ uint32_t swz(uint32_t t) { return t ^ (((t >> 3) ^ (t >> 6) ^ (t >> 9)) & 7u); }

template <int R_>
__device__ __forceinline__ uint32_t roff32(const uint32_t (&rb)[RB])
{
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < RB; ++k)
        if (R_ & (1 << k)) o |= rb[k];
    return o;
}

// asynchronous global -> shared copies (LDGSTS): the next tile streams into shared memory while the
// current one computes
template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (BYTES == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
// the same copy, or (skip) zeros written without reading global memory (the ignore-src operand)
template <int BYTES>
__device__ __forceinline__ void cp_async_or_zero(void *smem, const void *gmem, bool skip)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const unsigned k = skip;
    if constexpr (BYTES == 16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                     "cp.async.cg.shared.global [%0], [%1], 16, p;\n\t}" ::"r"(s), "l"(gmem), "r"(k));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                     "cp.async.ca.shared.global [%0], [%1], 8, p;\n\t}" ::"r"(s), "l"(gmem), "r"(k));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// tile bases in the read layout: the tile index deposited into the outer positions
__device__ __forceinline__ uint64_t pdep_outer(uint64_t T, uint64_t m)
{
    uint64_t o = 0;
    for (uint64_t b = 1; m; m &= m - 1) {
        if (T & b) o |= m & (~m + 1);
        b <<= 1;
    }
    return o;
}

// Copy a tile into shared memory in LOGICAL tile order: thread tid copies tile-local indices
// p = tid + NT*j from their read-layout addresses (tile-local bits are in read-position order, so
// a warp copies 512 contiguous bytes when the tile's qubits sit at physical 0..11), to slot
// swz(p ^ mloc).
template <typename V>
__device__ __forceinline__ void prefetch_tile(V *sm, const V *psi, uint64_t tbase, const Params &P, uint64_t gt,
                                              uint32_t tid)
{
    // tbase: the tile's base in the read layout (outer positions); all offsets below are in bytes
    const char *src = reinterpret_cast<const char *>(psi + ((tbase ^ P.xin) + gt));
    char *dst = reinterpret_cast<char *>(sm);
    const uint32_t st = swz(tid ^ P.mloc) * (uint32_t)sizeof(V);
    if (P.flags & F_VMASK) {
        // the buffer holds the state only on the valid set: elements outside it are zero, written
        // into shared memory without a global read
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const uint32_t e = tid + (uint32_t)NT * (uint32_t)j;   // physical tile-local index
            cp_async_or_zero<sizeof(V)>(dst + (st ^ P.sj[j]), src + P.gj[j], (e & P.vl_mask) != P.vl_val);
        }
    } else {
#pragma unroll
        for (int j = 0; j < NR; ++j) cp_async<sizeof(V)>(dst + (st ^ P.sj[j]), src + P.gj[j]);
    }
    cp_async_commit();
}

// 32-byte (c128) / 16-byte (c64) streaming store of two adjacent amplitudes
__device__ __forceinline__ void st_pair(double2 *q, const double2 &lo, const double2 &hi)
{
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q), "d"(lo.x), "d"(lo.y), "d"(hi.x), "d"(hi.y)
                 : "memory");
}
__device__ __forceinline__ void st_pair(float2 *q, const float2 &lo, const float2 &hi)
{
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q), "f"(lo.x), "f"(lo.y), "f"(hi.x), "f"(hi.y)
                 : "memory");
}
// store with qubit 0 on register bit K: every lane writes whole 32-byte sectors (a plain 16-byte
// store per register would leave each sector half-written per instruction: 2x L2 sectors)
template <int PV, typename V>
__device__ __forceinline__ void store_pairs(V *q0, const V (&a)[NR], const Params &P)
{
    // PV: the register-index difference of the two registers holding adjacent amplitudes
    constexpr int HB = 31 - __builtin_clz(PV);
    const uint32_t odd = P.st_odd;
    char *qb = reinterpret_cast<char *>(q0);
#pragma unroll
    for (int r = 0; r < NR; ++r)
        if (!(r & (1 << HB))) {
            const int r1 = r ^ PV;
            if ((odd >> r) & 1u) st_pair(reinterpret_cast<V *>(qb + P.gs[r1]), a[r1], a[r]);
            else st_pair(reinterpret_cast<V *>(qb + P.gs[r]), a[r], a[r1]);
        }
}

// ---- tile pipeline: NG independent 128-thread tile groups per CTA share NBUF tile buffers.
// Tile j of a CTA (j = 0, 1, 2, ...) is handled by group j % NG and lives in buffer j % NBUF from
// its load until its last transpose.  At that point its group RELEASES the buffer by issuing the
// load of tile j + NBUF (the other group's) into it; completion is tracked by an mbarrier
// (cp.async.mbarrier.arrive.noinc), so the group that waits need not be the group that issued.
// With NG = 2, NBUF = 3 every tile's load is issued about one tile period before it is needed,
// whatever the position of the group's last transpose (before: one shared buffer per 128-thread
// CTA, so the next load could only start after the last transpose).
__device__ __forceinline__ void named_bar(uint32_t id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NT) : "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t *m, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *m)
{
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     (unsigned)__cvta_generic_to_shared(m))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t *m)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"((unsigned)__cvta_generic_to_shared(m))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(m)),
                 "r"(parity)
                 : "memory");
}

__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t m)
{
    uint64_t o = 0;
    for (; m && x; m &= m - 1, x >>= 1)
        if (x & 1) o |= m & (~m + 1);
    return o;
}

// tile index of this CTA's j-th tile, or ~0 past the end.  F_LIVE (a sweep right after a reset,
// DESIGN.md "Live tiles"): only the nlive tiles the support analysis allows are visited; the
// others hold zeros (K7 wrote them) and the group's gates keep them zero.
__device__ __forceinline__ uint64_t cta_tile(uint64_t j, const Params &P)
{
    const uint64_t t = (uint64_t)blockIdx.x * NG + (j % NG) + (j / NG) * ((uint64_t)gridDim.x * NG);
    if (P.flags & F_LIVE) return t < P.nlive ? pdep64(t, P.lfree) | P.lfix : ~0ull;
    if (P.flags & F_TLIST) return t < P.nlist ? P.tlist[t] ^ P.tl_xor : ~0ull;
    return t < P.ntiles ? t : ~0ull;
}

// F_VMASK: a tile (read-layout base tbase) none of whose elements the buffer holds: it is all zero
__device__ __forceinline__ bool tile_dead(uint64_t tbase, const Params &P)
{
    return (P.flags & F_VMASK) && (((tbase ^ P.xin ^ P.vfix) & ~P.vfree & P.outer) != 0);
}

// Hand buffer j % NBUF over to tile j (issued by the group that held it): load tile j into it, or
// (F_INIT: nothing to load) just arrive.  Called by all NT threads of the issuing group.
template <typename V>
__device__ __forceinline__ void issue_tile(V *smbase, uint64_t *mbar, const V *psi, uint64_t j, uint64_t tbase,
                                           const Params &P, uint64_t gt, uint32_t tid, bool init)
{
    if (cta_tile(j, P) == ~0ull) return;
    const int b = (int)(j % NBUF);
    if (init || tile_dead(tbase, P)) {   // nothing to load: just arrive (one arrival per bulk phase)
        if (!(P.flags & F_BULK) || tid == 0) mbar_arrive(&mbar[j % NMB]);
    } else if (P.flags & F_BULK) {
        // the tile is one contiguous 64 KiB (c128) block: ONE bulk copy (TMA engine, UBLKCP)
        // issued by one thread, completion as transaction bytes on the buffer's mbarrier
        if (tid == 0) {
            constexpr uint32_t bytes = (1u << TB) * (uint32_t)sizeof(V);
            const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar[j % NMB]);
            const unsigned dst = (unsigned)__cvta_generic_to_shared(smbase + (size_t)b * (1u << TB));
            const V *src = psi + (tbase ^ P.xin);
#ifdef TUSQ_DEBUG_CHECKS
            if (((tbase ^ P.xin) & ((1u << TB) - 1)) || (tbase ^ P.xin) >= (P.ntiles << TB)) {
                printf("k_fused bulk: bad tile base %llx (xin %llx, ntiles %llu) block %d j %llu\n",
                       (unsigned long long)tbase, (unsigned long long)P.xin, (unsigned long long)P.ntiles,
                       (int)blockIdx.x, (unsigned long long)j);
                __trap();
            }
#endif
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(src), "r"(bytes), "r"(mb)
                         : "memory");
        }
    } else {
        prefetch_tile(smbase + (size_t)b * (1u << TB), psi, tbase, P, gt, tid);
        mbar_arrive_cp_async(&mbar[j % NMB]);
    }
}

// before a buffer written through the generic proxy (transposes) is refilled by the async proxy
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// tile bases step in the deposited (outer-bit) domain: filling the holes with ones lets the
// carries of an ordinary add run through them (pdep(x + y) = ((pdep x | ~m) + pdep y) & m)
__device__ __forceinline__ uint64_t dep_add(uint64_t x, uint64_t dy, uint64_t m) { return ((x | ~m) + dy) & m; }

template <typename R>
// src: the state in the read layout; dst: where the write layout goes.  A sweep that keeps the
// layout (every tile writes back exactly the block it read) runs in place (src == dst); one that
// changes it is a global permutation and runs out of place into the other buffer.
__global__ void __launch_bounds__(NT * NG, (NG == 1 ? 2 : 1)) k_fused(const typename CV<R>::T *src,
                                                      typename CV<R>::T *dst, const __grid_constant__ Params P,
                                                      double *__restrict__ sums)
{
    using V = typename CV<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    V *smbase = reinterpret_cast<V *>(smraw);
    __shared__ uint64_t mbar[NMB];
    __shared__ double red[NG][NT / 32];
    const uint32_t grp = threadIdx.x / NT;
    const uint32_t tid = threadIdx.x % NT;
    const uint32_t bar = 1 + grp;     // named barrier of this tile group (0 = __syncthreads)
    const bool init = P.flags & F_INIT;
    // gather table (leading transposes folded into the first shared-memory read), after the buffers
    uint16_t *gsm = reinterpret_cast<uint16_t *>(smraw + (size_t)NBUF * (1u << TB) * sizeof(V));
    if (P.gtab != 0xFFFFu) {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(P.prm + P.gtab);
        uint32_t *dst = reinterpret_cast<uint32_t *>(gsm);
        for (uint32_t i = threadIdx.x; i < NR * NT / 2; i += NT * NG) dst[i] = src[i];
    }
    // tile index -> write-layout / logical base: one table per 8-bit chunk of the tile index
    uint64_t(*tabo)[256] = reinterpret_cast<uint64_t(*)[256]>(gsm + NR * NT);
    uint64_t(*tabl)[256] = tabo + NCH;
    uint64_t *rofs = reinterpret_cast<uint64_t *>(tabl + NCH);   // F_TSTORE: run offsets (bytes)
    if (P.flags & F_TSTORE) {
        const uint32_t nrun = 1u << (TB - P.ts_l0);
        for (uint32_t i = threadIdx.x; i < nrun; i += NT * NG) {
            uint64_t o = 0;
            for (uint32_t k = 0; k < (uint32_t)(TB - P.ts_l0); ++k)
                if ((i >> k) & 1u) o |= 1ull << P.ts_hipos[k];
            rofs[i] = o * sizeof(V);
        }
    }
    const bool need_l = P.flags & F_LBASE;
    for (uint32_t i = threadIdx.x; i < NCH * 256; i += NT * NG) {
        const uint32_t c = i >> 8, v = i & 255u;
        uint64_t o = 0, l = 0;
#pragma unroll
        for (uint32_t b = 0; b < 8; ++b) {
            const uint32_t k = c * 8 + b;
            if (((v >> b) & 1u) && k < P.nout) {
                o |= 1ull << P.oo[k];
                l |= 1ull << P.ol[k];
            }
        }
        tabo[c][v] = o;
        tabl[c][v] = l;
    }
    if (threadIdx.x == 0) {
        // arrivals per phase: one expect_tx arrival per bulk copy, or every thread's cp.async
        // arrival / reset arrival
        const uint32_t cnt = (P.flags & F_BULK) ? 1u : (uint32_t)NT;
        for (int b = 0; b < NMB; ++b) mbar_init(&mbar[b], cnt);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto lookup = [&](uint64_t(*tab)[256], uint64_t T) {
        uint64_t o = tab[0][T & 255u];
#pragma unroll
        for (int c = 1; c < NCH; ++c) o |= tab[c][(T >> (8 * c)) & 255u];
        return o;
    };
    // read-layout offset of this thread's copy slot: tile-local bits 0..NTB-1 = tid (tile independent)
    uint64_t gt = 0;
#pragma unroll
    for (int b = 0; b < NTB; ++b) gt |= (uint64_t)((tid >> b) & 1u) << P.pin[b];
    // the first NBUF tiles: tile j is issued by group j % NG
    for (uint64_t j = grp; j < NBUF; j += NG)
        issue_tile(smbase, mbar, src, j, pdep_outer(cta_tile(j, P), P.outer), P, gt, tid, init);
    V a[NR];
    // thread parts of the phase-0 logical index (predicates, init) and of the last phase's write address
    uint64_t gthr0 = 0, gthr_st = 0;
    {
        const Phase &p0 = P.ph[0], &pl = P.ph[P.nphase - 1];
#pragma unroll
        for (int q = 0; q < NTB; ++q) {
            gthr0 |= (uint64_t)((tid >> q) & 1u) << P.qs[p0.tl[q]];
            gthr_st |= (uint64_t)((tid >> q) & 1u) << P.pout[pl.tl[q]];
        }
    }
    // read-layout tile base: the tile index deposited into the outer positions (stepped in place)
    uint64_t base = pdep_outer(cta_tile(grp, P), P.outer);
    const uint64_t dissue = P.dissue[grp];
    for (uint64_t j = grp;; j += NG, base = dep_add(base, P.dstep, P.outer)) {
        const uint64_t T = cta_tile(j, P);
        if (T == ~0ull) break;
        const bool live = P.flags & (F_LIVE | F_TLIST);
        if (live) base = pdep_outer(T, P.outer);   // sparse tile sequence: no incremental bases
        const uint64_t nbase = live ? pdep_outer(cta_tile(j + NBUF, P), P.outer) : dep_add(base, dissue, P.outer);
        V *sm = smbase + (size_t)(j % NBUF) * (1u << TB);
        char *smb = reinterpret_cast<char *>(sm);
        const uint64_t bout = lookup(tabo, T);
        const uint64_t blog = need_l ? lookup(tabl, T) : 0;
        mbar_wait(&mbar[j % NMB], (uint32_t)((j / NMB) & 1));
        const bool dead = tile_dead(base, P);
        if (init || dead) {
            // a reset: every amplitude is 0 but one, whose place in the phase-0 layout (after any
            // leading transposes, folded away on the host) the planner computed
#pragma unroll
            for (int r = 0; r < NR; ++r) { a[r].x = R(0); a[r].y = R(0); }
            if (init && tid == P.init_t) {   // (F_INIT comes with F_LIVE: T is the one live tile)
#pragma unroll
                for (int r = 0; r < NR; ++r)
                    if ((uint32_t)r == P.init_r) { a[r].x = (R)P.init_re; a[r].y = (R)P.init_im; }
            }
        } else {
            // the tile has landed in shared memory in logical order: read it in the phase-0 layout
            if (P.gtab != 0xFFFFu) {
#pragma unroll
                for (int r = 0; r < NR; ++r) a[r] = *reinterpret_cast<const V *>(smb + gsm[r * NT + tid]);
            } else if (P.flags & F_BULK) {   // linear buffer: logical element e at slot e ^ mloc
                uint32_t t0 = 0;
#pragma unroll
                for (int q = 0; q < NTB; ++q) t0 |= ((tid >> q) & 1u) << P.ph[0].tl[q];
                t0 *= (uint32_t)sizeof(V);
#pragma unroll
                for (int r = 0; r < NR; ++r) a[r] = *reinterpret_cast<const V *>(smb + (t0 ^ P.so0[r]));
            } else {
                uint32_t t0 = 0;
#pragma unroll
                for (int q = 0; q < NTB; ++q) t0 |= ((tid >> q) & 1u) << P.ph[0].tl[q];
                t0 = swz(t0) * (uint32_t)sizeof(V);
#pragma unroll
                for (int r = 0; r < NR; ++r) a[r] = *reinterpret_cast<const V *>(smb + (t0 ^ P.ph[0].so[r]));
            }
        }
        // (the buffer then stays ours until the stores read it)
        const bool tstore = (P.flags & F_TSTORE) && !(P.flags & F_NOSTORE);
        if (!tstore && (P.last_xpose == 0xFFFFu || dead)) {   // no transpose: release the buffer right away
            if (P.flags & F_BULK) fence_proxy_async();
            named_bar(bar);
            issue_tile(smbase, mbar, src, j + NBUF, nbase, P, gt, tid, init);
        }

        // ONE flat loop over records; a phase change is just a record (C_XPOSE) so that all paths
        // join at a single loop header with the amplitudes in one canonical register set (nested
        // phase/gate loops made ptxas copy every amplitude at each gate iteration).
        uint32_t ph = 0;
        uint64_t lbase = blog | gthr0;   // logical index bits of this thread (thread + outer) for predicates
        // records are fetched as one 64-bit constant load, one record ahead (the fetch -> decode
        // -> branch chain was the top stall in ncu's source view; a shared-memory copy fetched by
        // a volatile load at the top of the iteration measured ~6 % slower)
        const uint64_t *recw = reinterpret_cast<const uint64_t *>(P.g);
        const uint32_t ngate = dead ? 0u : P.ngate;   // a zero tile stays zero
        uint64_t wnext = ngate ? recw[0] : 0;
        for (uint32_t gi = 0; gi < ngate; ++gi) {
            const uint64_t w = wnext;
            wnext = recw[gi + 1 < P.ngate ? gi + 1 : gi];
            GRec g;
            g.code = (uint16_t)w;
            g.a = (uint8_t)(w >> 16);
            g.b = (uint8_t)(w >> 24);
            g.pi = (uint16_t)(w >> 32);
            g._pad = 0;
            if (g.code != C_XPOSE) {
                apply_gate<V, R>(a, g, P.prm, lbase);
            } else {
                // transpose registers from the current layout to phase g.a through shared memory
                const Phase &prv = P.ph[ph];
                const Phase &cur = P.ph[g.a];
                ph = g.a;
                uint32_t tt = 0;
#pragma unroll
                for (int q = 0; q < NTB; ++q) tt |= ((tid >> q) & 1u) << prv.tl[q];
                // g.b = 1: same thread-bit layout on both sides -- every thread writes and reads
                // back only its own slots (a register permutation), no barrier needed
                if (!g.b) named_bar(bar);
                tt = swz(tt) * (uint32_t)sizeof(V);
#define TQ_ST(r) if constexpr (r < NR) *reinterpret_cast<V *>(smb + (tt ^ prv.so_out[r])) = a[r];
                TQ_ST(0) TQ_ST(1) TQ_ST(2) TQ_ST(3) TQ_ST(4) TQ_ST(5) TQ_ST(6) TQ_ST(7)
                TQ_ST(8) TQ_ST(9) TQ_ST(10) TQ_ST(11) TQ_ST(12) TQ_ST(13) TQ_ST(14) TQ_ST(15)
                TQ_ST(16) TQ_ST(17) TQ_ST(18) TQ_ST(19) TQ_ST(20) TQ_ST(21) TQ_ST(22) TQ_ST(23)
                TQ_ST(24) TQ_ST(25) TQ_ST(26) TQ_ST(27) TQ_ST(28) TQ_ST(29) TQ_ST(30) TQ_ST(31)
#undef TQ_ST
                if (!g.b) named_bar(bar);
                tt = 0;
#pragma unroll
                for (int q = 0; q < NTB; ++q) tt |= ((tid >> q) & 1u) << cur.tl[q];
                tt = swz(tt) * (uint32_t)sizeof(V);
#define TQ_LD(r) if constexpr (r < NR) a[r] = *reinterpret_cast<const V *>(smb + (tt ^ cur.so[r]));
                TQ_LD(0) TQ_LD(1) TQ_LD(2) TQ_LD(3) TQ_LD(4) TQ_LD(5) TQ_LD(6) TQ_LD(7)
                TQ_LD(8) TQ_LD(9) TQ_LD(10) TQ_LD(11) TQ_LD(12) TQ_LD(13) TQ_LD(14) TQ_LD(15)
                TQ_LD(16) TQ_LD(17) TQ_LD(18) TQ_LD(19) TQ_LD(20) TQ_LD(21) TQ_LD(22) TQ_LD(23)
                TQ_LD(24) TQ_LD(25) TQ_LD(26) TQ_LD(27) TQ_LD(28) TQ_LD(29) TQ_LD(30) TQ_LD(31)
#undef TQ_LD
                // logical index bits of this thread (thread + outer bits) for predicates
                if (need_l) {
                    lbase = blog;
#pragma unroll
                    for (int q = 0; q < NTB; ++q) lbase |= (uint64_t)((tid >> q) & 1u) << P.qs[cur.tl[q]];
                }
                if (gi == P.last_xpose && !tstore) {   // the buffer is free until tile j + NBUF: hand it over
                    if (P.flags & F_BULK) fence_proxy_async();
                    named_bar(bar);
                    issue_tile(smbase, mbar, src, j + NBUF, nbase, P, gt, tid, init);
                }
            }
        }

        // ---- store with the last phase's thread layout, into the write layout
        if (P.flags & F_SCALE) {
            const R sr = (R)P.scale_re, si = (R)P.scale_im;
            if (si == R(0)) {
#pragma unroll
                for (int r = 0; r < NR; ++r) { a[r].x *= sr; a[r].y *= sr; }
            } else {
#pragma unroll
                for (int r = 0; r < NR; ++r) cmul_ip(a[r], sr, si);
            }
        }
        if (tstore) {
            // registers -> the tile buffer in write order, then bulk copies of its contiguous runs
            named_bar(bar);   // everyone is done reading the buffer
            uint32_t wt = 0;
#pragma unroll
            for (int q = 0; q < NTB; ++q) wt |= ((tid >> q) & 1u) << P.wpos[P.ph[P.nphase - 1].tl[q]];
            wt *= (uint32_t)sizeof(V);
#pragma unroll
            for (int r = 0; r < NR; ++r) *reinterpret_cast<V *>(smb + (wt ^ P.wreg[r])) = a[r];
            fence_proxy_async();
            named_bar(bar);
            const uint32_t nrun = 1u << (TB - P.ts_l0), rbytes = (1u << P.ts_l0) * (uint32_t)sizeof(V);
            char *tb = reinterpret_cast<char *>(dst + (bout ^ P.xout));
            const unsigned sbase = (unsigned)__cvta_generic_to_shared(smb);
            for (uint32_t i = tid; i < nrun; i += NT)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(tb + rofs[i]),
                             "r"(sbase + i * rbytes), "r"(rbytes)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            named_bar(bar);   // the buffer has been read: hand it to tile j + NBUF
            issue_tile(smbase, mbar, src, j + NBUF, nbase, P, gt, tid, init);
        }
        // xout has no tile bits: register offsets are additive
        V *q0 = dst + ((bout | gthr_st) ^ P.xout);
#ifdef TUSQ_DEBUG_KNOBS
        if (P.flags & F_DBG_NOSTORE) {
            if (a[0].x == R(12345)) q0[0] = a[1];   // keep the registers live
            continue;
        }
#endif
#ifdef TUSQ_DEBUG_CHECKS
        for (int r = 0; r < NR; ++r)
            if (((bout | gthr_st) ^ P.xout) + P.gs[r] / sizeof(V) >= (P.ntiles << TB)) {
                printf("k_fused store: out of range (tile %llu, reg %d)\n", (unsigned long long)T, r);
                __trap();
            }
#endif
        if (tstore || (P.flags & F_NOSTORE)) {
            // (written above / not written: block sums only)
        } else if (P.st_pair) {
            switch (P.st_pair) {
#define TQ_SP(v) case v: if constexpr (v < NR) store_pairs<v>(q0, a, P); break;
                TQ_SP(1) TQ_SP(2) TQ_SP(3) TQ_SP(4) TQ_SP(5) TQ_SP(6) TQ_SP(7) TQ_SP(8) TQ_SP(9) TQ_SP(10)
                TQ_SP(11) TQ_SP(12) TQ_SP(13) TQ_SP(14) TQ_SP(15) TQ_SP(16) TQ_SP(17) TQ_SP(18) TQ_SP(19)
                TQ_SP(20) TQ_SP(21) TQ_SP(22) TQ_SP(23) TQ_SP(24) TQ_SP(25) TQ_SP(26) TQ_SP(27) TQ_SP(28)
                TQ_SP(29) TQ_SP(30) TQ_SP(31)
#undef TQ_SP
            default: break;
            }
        } else {
#pragma unroll
            for (int r = 0; r < NR; ++r) __stcs(reinterpret_cast<V *>(reinterpret_cast<char *>(q0) + P.gs[r]), a[r]);
        }
        if (P.flags & F_SUMS) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                double re = a[r].x, im = a[r].y;
                s += re * re + im * im;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            if ((tid & 31) == 0) red[grp][tid >> 5] = s;
            named_bar(bar);
            if (tid == 0) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < NT / 32; ++w) t += red[grp][w];
                sums[(bout ^ P.xout) >> TB] = t;   // (F_SUMS: identity write layout, tile {0..11})
            }
            named_bar(bar);
        }
    }
    // bulk stores still in flight must land before the CTA retires
    if (P.flags & F_TSTORE) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace fk

// ======================================================================= host planner
namespace {

using namespace fk;

struct KOp {
    Op op;
    bool in_tile_xy = false;   // X/Y applied in registers
    bool zpart = false;        // Z part of a relabelled Y (diag -1 on q)
};

struct Group {
    std::vector<KOp> ops;      // in-kernel ops
    uint64_t xb = 0, xa = 0;   // relabel masks before load / after store
    double fr = 1.0, fi = 0.0; // global phase from relabelled Y
    int nh = 0;                // unscaled H count
    uint64_t tilemask = 0;     // required tile qubits (exchange operands)
};

inline uint64_t bit(uint32_t q) { return 1ull << q; }

bool is_exchange(const Op &o) { return o.kind == H || o.kind == RX || o.kind == RY; }

uint64_t op_qubits(const Op &o) { return bit(o.q0) | (two_qubit(o.kind) ? bit(o.q1) : 0); }

}  // namespace

GateTimer::~GateTimer()
{
    for (auto e : a_) cudaEventDestroy(e);
    for (auto e : b_) cudaEventDestroy(e);
}

void GateTimer::begin(cudaStream_t st)
{
    // the pool grows as needed and is read once, at the end of the call (no host sync mid-run)
    if (!on_) return;
    if (used_ == a_.size()) {
        cudaEvent_t x, y;
        cudaEventCreate(&x);
        cudaEventCreate(&y);
        a_.push_back(x);
        b_.push_back(y);
        by_.push_back(0);
        cat_.push_back(0);
    }
    cudaEventRecord(a_[used_], st);
}

void GateTimer::end(cudaStream_t st, double bytes, int cat)
{
    if (!on_) return;
    cudaEventRecord(b_[used_], st);
    by_[used_] = bytes;
    cat_[used_] = (uint8_t)cat;
    ++used_;
}

void GateTimer::flush()
{
    if (!on_ || !used_) return;
    cudaEventSynchronize(b_[used_ - 1]);
    for (size_t i = 0; i < used_; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, a_[i], b_[i]);
#ifdef TUSQ_DEBUG_KNOBS
        static const bool dbg_trace = getenv("TUSQ_DBG_TRACE") != nullptr;
        if (dbg_trace) fprintf(stderr, "[t] %zu %d %.4f\n", i, (int)cat_[i], ms);
#endif
        if (cat_[i] == 0 || cat_[i] == 2) {   // 2: a dense K5 sweep (also a gate kernel)
            seconds += ms * 1e-3;
            bytes += by_[i];
            ++launches;
            if (cat_[i] == 2) {
                dense_seconds += ms * 1e-3;
                dense_bytes += by_[i];
                ++dense_launches;
            }
        } else {
            sample_seconds += ms * 1e-3;
        }
    }
    used_ = 0;
}

// deposit the low bits of x into the set bits of m (host pdep)
static uint64_t pdep_mask(uint64_t x, uint64_t m)
{
    uint64_t o = 0;
    for (; m && x; m &= m - 1, x >>= 1)
        if (x & 1) o |= m & (~m + 1);
    return o;
}

static void count(Ctx &ctx, double bytes, bool fused)
{
    ctx.stats->launches++;
    // kernel parameters travel with the launch: the K5 block, or a few scalars
    ctx.stats->h2d_bytes += fused ? (double)sizeof(Params) : 64.0;
    ctx.stats->sweeps++;
    ctx.stats->hbm_bytes += bytes;
    if (fused) ctx.stats->fused_launches++;
}

void execute_unfused(const std::vector<Op> &ops, Ctx &ctx)
{
    size_t i = 0;
    while (i < ops.size()) {
        const Op &o = ops[i];
        if (o.kind == X || o.kind == Y || o.kind == Z) {
            uint64_t xm = 0, zm = 0, used = 0;
            size_t j = i;
            while (j < ops.size() && (ops[j].kind == X || ops[j].kind == Y || ops[j].kind == Z) &&
                   !((used >> ops[j].q0) & 1)) {
                used |= bit(ops[j].q0);
                if (ops[j].kind != Z) xm |= bit(ops[j].q0);
                if (ops[j].kind != X) zm |= bit(ops[j].q0);
                ++j;
            }
            double b = 0;
            if (!ctx.dry) {
                if (ctx.timer) ctx.timer->begin(ctx.st);
                b = launch_pauli_string(ctx.psi, ctx.n, ctx.prec, xm, zm, ctx.st);
                if (ctx.timer) ctx.timer->end(ctx.st, b);
            } else {
                b = (double)(1ull << ctx.n) * (ctx.prec == 128 ? 16 : 8) * (xm ? 2.0 : 1.0);
            }
            count(ctx, b, false);
            i = j;
            continue;
        }
        if (o.kind != I) {
            double b;
            if (!ctx.dry) {
                if (ctx.timer) ctx.timer->begin(ctx.st);
                b = launch_gate(ctx.psi, ctx.n, ctx.prec, o, ctx.st);
                if (ctx.timer) ctx.timer->end(ctx.st, b);
            } else {
                double s = (double)(1ull << ctx.n) * (ctx.prec == 128 ? 16 : 8);
                b = (o.kind == CX || o.kind == T || o.kind == TDG || o.kind == S || o.kind == SDG || o.kind == P)
                        ? s
                        : (o.kind == CZ || o.kind == CP) ? 0.5 * s : 2 * s;
            }
            count(ctx, b, false);
        }
        ++i;
    }
}

FusedPlanner::FusedPlanner(uint32_t n, int prec)
    : n_(n), prec_(prec), tile_bits_(TB), enabled_(n >= (uint32_t)TB && n <= (uint32_t)(TB + 8 * NCH))
{
}

static bool diag_of(const Op &o, double d[4]);

// ---- group formation (greedy over the op stream) --------------------------------------
static std::vector<Group> make_groups(const std::vector<Op> &ops, bool strict)
{
    // strict: every qubit an op touches (controls, diagonals) must join the tile, so whole runs
    // stay in registers and fold; otherwise they join only while there is room
    // Tile capacity: qubits 0,1,2 + up to 9 others.  Groups after the first read a layout in which
    // their own tile qubits sit at physical positions 0..11 (FusedPlanner::execute_ex), so any 12
    // qubits would make a contiguous tile -- but the sweep BEFORE such a group writes with runs of
    // 2^m amplitudes, m = the qubits the two tiles share.  Keeping 0,1,2 in every tile keeps
    // m >= 3 (128-byte write runs).  Measured on C4 batches (profiles/r2_k5_anatomy.json): 12 free
    // qubits need 25 % fewer sweeps but each costs 38 % more (short write runs, more transposes);
    // 9 + {0,1,2} with the remap is the fastest (-8 % vs the identity layout).
    uint64_t low = 7;
    int hi_cap = TB - 3;
    // tile qubits a group may claim beyond 0-2 (default all 9; fewer leave fillers 3, 4... in the
    // tile, i.e. longer contiguous runs per tile row, at the price of more sweeps)
    std::vector<Group> groups;
    Group g;
    uint64_t touched = 0;
    std::vector<int> pending(64, -1);   // index (in g.ops) of a pending X/Y on qubit q
    auto popc_hi = [&](uint64_t m) { return __builtin_popcountll(m & ~low); };
    auto close = [&]() {
        // pending X/Y become relabel-after (last touch in the group)
        std::vector<KOp> kept;
        kept.reserve(g.ops.size());
        std::vector<uint8_t> drop(g.ops.size(), 0);
        for (uint32_t q = 0; q < 64; ++q) {
            int idx = pending[q];
            if (idx < 0) continue;
            KOp &k = g.ops[idx];
            g.xa ^= bit(q);
            if (k.op.kind == Y) {     // Y = i X Z: Z here, X after the store, factor i
                k.op.kind = Z;
                k.zpart = true;
                double r = g.fr, im = g.fi;
                g.fr = -im; g.fi = r;
            } else {
                drop[idx] = 1;
            }
            pending[q] = -1;
        }
        for (size_t i = 0; i < g.ops.size(); ++i)
            if (!drop[i]) kept.push_back(g.ops[i]);
        g.ops.swap(kept);
        if (!g.ops.empty() || g.xb || g.xa) groups.push_back(g);
#ifdef TUSQ_DEBUG_KNOBS   // TUSQ_DBG_CAP=12: any 12 tile qubits in the groups after the first
        static const int dbg_cap = getenv("TUSQ_DBG_CAP") ? atoi(getenv("TUSQ_DBG_CAP")) : 0;
        if (dbg_cap == 12 && !groups.empty()) { low = 0; hi_cap = TB; }
#endif
        g = Group();
        touched = 0;
    };
    // a Toffoli core H(t) [classical run] H(t) starting at op i: the qubits it touches (0: none)
    auto core_qubits = [&](size_t i) -> uint64_t {
        const Op &h = ops[i];
        if (h.kind != H) return 0;
        uint64_t m = bit(h.q0);
        double d[4];
        for (size_t j = i + 1; j < ops.size(); ++j) {
            const Op &o = ops[j];
            if (o.kind == H && o.q0 == h.q0) return j > i + 1 ? m : 0;
            if (!(o.kind == CX || o.kind == CZ || o.kind == CP || diag_of(o, d))) return 0;
            m |= op_qubits(o);
        }
        return 0;
    };
    for (size_t oi = 0; oi < ops.size(); ++oi) {
        const Op &o = ops[oi];
        if (o.kind == I) continue;
        const uint64_t qm = op_qubits(o);
        // keep a Toffoli core in one group (it folds into one controlled-2x2 record): close the
        // group before the core's first H when the core's qubits would not fit
        if (!g.ops.empty()) {
            const uint64_t cq = core_qubits(oi);
            if (cq && popc_hi(g.tilemask | cq) > hi_cap) close();
        }
        // requirements of this op on the group's tile set
        const bool xy = (o.kind == X || o.kind == Y);
        uint64_t need = 0;
        if (is_exchange(o)) need |= bit(o.q0);
        if (o.kind == CX) need |= bit(o.q1);
        if (strict && !xy) need |= qm;
        // a pending X/Y on a qubit this op touches must be applied in registers
        for (uint64_t m = qm; m; m &= m - 1) {
            uint32_t q = __builtin_ctzll(m);
            if (pending[q] >= 0) need |= bit(q);
        }
        const bool fits = popc_hi(g.tilemask | need) <= hi_cap && g.ops.size() + 1 < (size_t)MAXG - 8;
        if (!fits) close();
        // re-evaluate after a possible close (pending cleared)
        need = 0;
        if (is_exchange(o)) need |= bit(o.q0);
        if (o.kind == CX) need |= bit(o.q1);
        if (strict && !xy) need |= qm;
        // soft: controls / diagonal qubits join the tile while there is room (never close a group)
        if (!xy && popc_hi(g.tilemask | need | qm) <= hi_cap) need |= qm;
        for (uint64_t m = qm; m; m &= m - 1) {
            uint32_t q = __builtin_ctzll(m);
            if (pending[q] >= 0) {
                need |= bit(q);
                g.ops[pending[q]].in_tile_xy = true;
                pending[q] = -1;
            }
        }
        g.tilemask |= need;
        if (xy) {
            const uint32_t q = o.q0;
            if (!(touched & bit(q))) {
                // first touch: relabel before the load.  Y = (-i) Z X: X first, Z here.
                g.xb ^= bit(q);
                if (o.kind == Y) {
                    KOp k;
                    k.op = Op{Z, q, 0, 0.0};
                    k.zpart = true;
                    g.ops.push_back(k);
                    double r = g.fr, im = g.fi;   // multiply by -i
                    g.fr = im; g.fi = -r;
                }
            } else {
                KOp k;
                k.op = o;
                g.ops.push_back(k);
                pending[q] = (int)g.ops.size() - 1;
            }
            touched |= bit(q);
            continue;
        }
        KOp k;
        k.op = o;
        g.ops.push_back(k);
        touched |= qm;
    }
    close();
    return groups;
}

// ---- phase planning + parameter block ----------------------------------------------------
struct Built {
    Params P;
    uint64_t tile = 0;
    uint8_t pin0[NR];      // absorbed entry permutation of phase 0: register r reads pattern pin0[r]
    uint8_t pout_last[NR]; // absorbed exit permutation of the last phase: register s written as pattern pout[s]
    int h_absorbed = 0;    // H's folded into C_CU records (exactly scaled there)
    size_t prm_used = 0;   // doubles of P.prm the records use
};

}  // namespace tq
struct tq::PlanScratch {
    Built B;
    uint16_t V[tq::fk::NT][tq::fk::NR], M[1 << tq::fk::TB];   // gather-table simulation
    tq::fk::Params replay;       // the last group of a sums-only transition (replay_tiles)
    const void *rsrc = nullptr;
    void *rdst = nullptr;
};
namespace tq {

// parameter doubles a record reads at prm[pi]
static int rec_nparams(const GRec &r)
{
    const uint16_t c = r.code;
    if (c >= C_DKC && c < C_N) return 2 << __builtin_popcount((c - C_DKC) % 16);
    if (c >= C_TDK && c < C_DKC) return r.b ? 2 : 2 * r.a;
    if (c >= C_U && c < C_X) return 8;
    if (c >= C_D1 && c < C_D2) return 2;
    if (c >= C_D2 && c < C_CX) return 4;
    if (c >= C_CPH && c < C_TX) return 2;
    if (c >= C_TD1 && c < C_TPH) return 3;   // cos, sin, theta (theta for C_TDK merges)
    if (c == C_TPH) return 4;
    if (c >= C_DK && c < C_CX2) return 2 << __builtin_popcount(c - C_DK);
    if (c >= C_CU && c < C_CCX) return 32;
    return 0;
}

static bool is_perm_rec(uint16_t c)
{
    if (c >= C_X && c < C_X + 5) return true;
    if (c >= C_CX && c < C_CX + 25) return (c - C_CX) / 5 != (c - C_CX) % 5;
    if (c >= C_CX2 && c < C_CU) return code_ok(c);
    if (c >= C_CCX && c < C_TDK) return code_ok(c);
    return false;
}

static uint32_t perm_apply(uint16_t c, uint32_t r)
{
    if (c < C_X + 5) return r ^ (1u << (c - C_X));
    if (c >= C_CCX && c < C_TDK) {
        const int p = (c - C_CCX) / 6;
        const uint32_t cm = (uint32_t)hdh_mask(p, (c - C_CCX) % 6) & ~(1u << p);
        return (r & cm) == cm ? r ^ (1u << p) : r;
    }
    if (c >= C_CX2) {
        const uint32_t cb = (c - C_CX2) / 25, t1 = (c - C_CX2) / 5 % 5, t2 = (c - C_CX2) % 5;
        return ((r >> cb) & 1) ? r ^ (1u << t1) ^ (1u << t2) : r;
    }
    const uint32_t cb = (c - C_CX) / 5, tb = (c - C_CX) % 5;
    return ((r >> cb) & 1) ? r ^ (1u << tb) : r;
}

static void matrix_u(const Op &o, double m[8])
{
    const double c = cos(o.theta / 2), s = sin(o.theta / 2);
    if (o.kind == RX) { double v[8] = {c, 0, 0, -s, 0, -s, c, 0}; memcpy(m, v, sizeof(v)); }
    else { double v[8] = {c, 0, -s, 0, s, 0, c, 0}; memcpy(m, v, sizeof(v)); }   // RY
}

static bool diag_of(const Op &o, double d[4])
{
    const double s2 = M_SQRT1_2;
    d[0] = 1; d[1] = 0;
    switch (o.kind) {
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

// tile: the group's 12 logical tile qubits; lin / lout: physical position of every logical qubit
// in the read / write layout
static void build_params(const Group &G, uint32_t n, Built &B, uint64_t tile, const uint8_t *lin,
                         const uint8_t *lout)
{
    Params &P = B.P;
    memset(&P, 0, sizeof(P));
    B.tile = tile;
    uint8_t loc[64];
    memset(loc, 0xff, sizeof(loc));
    {
        // tile-local bits in read order: tile-local index = read offset when the tile is contiguous
        std::vector<uint32_t> tq;
        for (uint32_t q = 0; q < n; ++q)
            if (tile & bit(q)) tq.push_back(q);
        std::sort(tq.begin(), tq.end(), [&](uint32_t a, uint32_t b) { return lin[a] < lin[b]; });
        for (int b = 0; b < TB; ++b) {
            P.qs[b] = (uint8_t)tq[b];
            P.pin[b] = lin[tq[b]];
            P.pout[b] = lout[tq[b]];
            loc[tq[b]] = (uint8_t)b;
        }
        // tile index bits: the outer qubits in read order
        std::vector<uint32_t> oq;
        for (uint32_t q = 0; q < n; ++q)
            if (!(tile & bit(q))) oq.push_back(q);
        std::sort(oq.begin(), oq.end(), [&](uint32_t a, uint32_t b) { return lin[a] < lin[b]; });
        P.nout = (uint32_t)oq.size();
        for (size_t k = 0; k < oq.size(); ++k) {
            P.oo[k] = lout[oq[k]];
            P.ol[k] = (uint8_t)oq[k];
            P.outer |= bit(lin[oq[k]]);
        }
    }
    // lane preference: tile bits by write position (the store's lanes 0-2 want write positions
    // 0-2); lanes 0-2 of every layout also need distinct (bit mod 3) classes -- the swizzle maps
    // tile bit b to bank group bit (b mod 3), so that keeps the quarter-warps conflict-free
    uint8_t lp[TB];
    for (int b = 0; b < TB; ++b) lp[b] = (uint8_t)b;
    std::sort(lp, lp + TB, [&](uint8_t a, uint8_t b) { return P.pout[a] < P.pout[b]; });
    // register-need sequence
    // needq: the qubit an op must have in a register (exchange target); ctrlq: a CX control that
    // also triggers a phase switch when it is a tile qubit outside the registers -- a register
    // control turns a whole-register predicated X (TX) into half the swaps and lets Toffoli
    // cores fold into one diagonal table (measured: ~2.5 TX records per Adder group otherwise)
    std::vector<int> needq(G.ops.size(), -1), ctrlq(G.ops.size(), -1);
    for (size_t i = 0; i < G.ops.size(); ++i) {
        const Op &o = G.ops[i].op;
        if (is_exchange(o) || G.ops[i].in_tile_xy) needq[i] = (int)o.q0;
        else if (o.kind == CX) {
            needq[i] = (int)o.q1;
            if (tile & bit(o.q0)) ctrlq[i] = (int)o.q0;
        }
    }
    auto needs_switch = [&](size_t i, uint64_t regs) {
        return (needq[i] >= 0 && !(regs & bit(needq[i]))) || (ctrlq[i] >= 0 && !(regs & bit(ctrlq[i])));
    };
    auto lookahead = [&](size_t from, uint64_t keep) {
        std::vector<uint32_t> rs;
        uint64_t have = 0;
        // upcoming qubits in order of first appearance: exchange targets (hard), and the controls /
        // diagonal qubits next to them (soft: in registers they avoid predicated whole-register work
        // and let monomial folding see the whole run)
        for (size_t i = from; i < G.ops.size() && rs.size() < (size_t)RB; ++i) {
            const Op &o = G.ops[i].op;
            uint32_t cand[2] = {needq[i] >= 0 ? (uint32_t)needq[i] : o.q0, o.q0};
            if (two_qubit(o.kind) && needq[i] < 0) cand[1] = o.q1;
            for (uint32_t q : cand)
                if (rs.size() < (size_t)RB && !(have & bit(q)) && (tile & bit(q))) { have |= bit(q); rs.push_back(q); }
        }
        // fill: keep previous register qubits, then tile qubits touched by diagonals, then any >= 3
        for (uint64_t m = keep; m && rs.size() < (size_t)RB; m &= m - 1) {
            uint32_t q = __builtin_ctzll(m);
            if (!(have & bit(q))) { have |= bit(q); rs.push_back(q); }
        }
        // then the tile bits least wanted as store lanes (largest write positions first)
        for (int i = TB - 1; i >= 0 && rs.size() < (size_t)RB; --i) {
            const uint32_t q = P.qs[lp[i]];
            if (!(have & bit(q))) { have |= bit(q); rs.push_back(q); }
        }
        return rs;
    };
    auto make_phase = [&](const std::vector<uint32_t> &rs, uint16_t g0) {
        Phase ph;
        memset(&ph, 0, sizeof(ph));
        ph.g0 = g0;
        uint32_t rmask = 0;
        for (int k = 0; k < RB; ++k) { ph.rl[k] = loc[rs[k]]; rmask |= 1u << ph.rl[k]; }
        // lanes 0-2: the non-register tile bits of smallest write position with distinct
        // (b mod 3) classes; lanes 3-4: the next by write position; warps: the rest ascending
        uint32_t used = rmask;
        int tj = 0;
        uint32_t cls = 0;
        for (int i = 0; i < TB && tj < 3; ++i) {
            const uint32_t b = lp[i];
            if ((used >> b) & 1u || (cls >> (b % 3)) & 1u) continue;
            used |= 1u << b;
            cls |= 1u << (b % 3);
            ph.tl[tj++] = (uint8_t)b;
        }
        for (int i = 0; i < TB && tj < 5; ++i)
            if (!((used >> lp[i]) & 1u)) { used |= 1u << lp[i]; ph.tl[tj++] = lp[i]; }
        for (uint32_t b = 0; b < (uint32_t)TB && tj < NTB; ++b)
            if (!(used & (1u << b))) { used |= 1u << b; ph.tl[tj++] = (uint8_t)b; }
        for (int r = 0; r < NR; ++r) {
            uint32_t o = 0;
            for (int k = 0; k < RB; ++k)
                if (r & (1 << k)) o |= 1u << ph.rl[k];
            ph.so[r] = (uint16_t)swz(o);        // pre-swizzled (swz is linear)
            ph.so_out[r] = (uint16_t)swz(o);
        }
        return ph;
    };
    std::vector<Phase> phases;
    std::vector<GRec> recs;
    std::vector<double> prm;
    uint64_t regset = 0;
    std::vector<uint32_t> rs;
    auto regpos = [&](uint32_t q) -> int {
        for (int k = 0; k < RB; ++k)
            if (rs[k] == q) return k;
        return -1;
    };
    auto addp = [&](std::initializer_list<double> v) {
        uint16_t i = (uint16_t)prm.size();
        for (double x : v) prm.push_back(x);
        return i;
    };
    // Monomial folding: a run of CX / diagonal / in-register X,Y gates on register qubits whose
    // net permutation is the identity is one diagonal: a[r] *= tab[pext(r, mask)].  (The CX+T
    // core of a Toffoli, P:457's Cuccaro adder, is such a run.)  Tables are built by simulating
    // the run on the 32 register patterns in double.
    auto classical = [&](size_t j) -> bool {
        const KOp &k = G.ops[j];
        const Op &o = k.op;
        auto inreg = [&](uint32_t q) { return (regset & bit(q)) != 0; };
        double d[4];
        if (o.kind == CX || o.kind == CZ || o.kind == CP) return inreg(o.q0) && inreg(o.q1);
        if ((o.kind == X || o.kind == Y) && k.in_tile_xy) return inreg(o.q0);
        if (diag_of(o, d)) return inreg(o.q0);
        return false;
    };
    // net permutation x -> x ^ c (an X translation, c may be 0) folds into the table followed by X's
    auto try_fold = [&](size_t i, size_t &fe, uint32_t &fmask, std::vector<double> &tab, uint32_t &fxor) -> bool {
        uint8_t perm[NR];
        double pr[NR], pi[NR];
        for (int x = 0; x < NR; ++x) { perm[x] = (uint8_t)x; pr[x] = 1.0; pi[x] = 0.0; }
        uint32_t mask = 0;
        size_t best = i;
        uint32_t best_mask = 0, best_xor = 0;
        double br[NR], bi[NR];
        for (size_t j = i; j < G.ops.size() && classical(j); ++j) {
            if (needs_switch(j, regset)) break;
            const Op &o = G.ops[j].op;
            const int a = regpos(o.q0), b = two_qubit(o.kind) ? regpos(o.q1) : -1;
            mask |= 1u << a;
            if (b >= 0) mask |= 1u << b;
            double d[4];
            const bool dg = diag_of(o, d);
            for (int x = 0; x < NR; ++x) {
                uint32_t y = perm[x];
                double fr = 1.0, fi = 0.0;
                if (o.kind == CX) { if ((y >> a) & 1) y ^= 1u << b; }
                else if (o.kind == X) { y ^= 1u << a; }
                else if (o.kind == Y) { fr = 0.0; fi = ((y >> a) & 1) ? -1.0 : 1.0; y ^= 1u << a; }
                else if (o.kind == CZ || o.kind == CP) {
                    if (((y >> a) & 1) && ((y >> b) & 1)) {
                        fr = o.kind == CZ ? -1.0 : cos(o.theta);
                        fi = o.kind == CZ ? 0.0 : sin(o.theta);
                    }
                } else if (dg) {
                    const bool s = (y >> a) & 1;
                    fr = s ? d[2] : d[0];
                    fi = s ? d[3] : d[1];
                }
                const double nr = pr[x] * fr - pi[x] * fi, ni = pr[x] * fi + pi[x] * fr;
                pr[x] = nr; pi[x] = ni;
                perm[x] = (uint8_t)y;
            }
            const uint32_t c = perm[0];
            bool xlat = true;
            for (int x = 0; x < NR && xlat; ++x) xlat = (uint32_t)perm[x] == ((uint32_t)x ^ c);
            // a translation costs one X record per set bit of c; require the fold to pay for them
            if (xlat && (j + 1) - i >= 2 + (size_t)__builtin_popcount(c)) {
                best = j + 1;
                best_mask = mask;
                best_xor = c;
                memcpy(br, pr, sizeof(br));
                memcpy(bi, pi, sizeof(bi));
            }
        }
        if (best < i + 2) return false;
        fe = best;
        fmask = best_mask;
        fxor = best_xor;
        tab.clear();
        const int k = __builtin_popcount(fmask);
        for (int idx = 0; idx < (1 << k); ++idx) {
            uint32_t x = 0;
            int t = 0;
            for (int b = 0; b < RB; ++b)
                if (fmask & (1u << b)) { if ((idx >> t) & 1) x |= 1u << b; ++t; }
            tab.push_back(br[x]);
            tab.push_back(bi[x]);
        }
        return true;
    };
    std::vector<double> ftab;
    // Phase switches are moved back to the start of a Toffoli core: when op i needs a switch and
    // the ops since the last H(t) -- or since the H(t) before it, H(t) run H(t) -- are all
    // classical, the records from that H on are dropped and re-planned in the new phase, so that
    // the core folds into one table (and one C_CU record) instead of being cut in two.
    std::vector<size_t> rec_at(G.ops.size(), SIZE_MAX), prm_at(G.ops.size(), SIZE_MAX);
    size_t phase_op0 = 0;
    auto classical_kind = [&](const Op &o) {
        double d[4];
        return o.kind == CX || o.kind == CZ || o.kind == CP || diag_of(o, d);
    };
    for (size_t i = 0; i < G.ops.size(); ++i) {
        if (phases.empty() || needs_switch(i, regset)) {
            if (!phases.empty()) {
                size_t k = i;
                while (k > phase_op0 && classical_kind(G.ops[k - 1].op)) --k;
                const Op &oi = G.ops[i].op;
                if (k > phase_op0 + 1 && G.ops[k - 1].op.kind == H && classical_kind(oi)) {
                    const uint32_t tq = G.ops[k - 1].op.q0;
                    size_t target = k - 1, m = k - 1;
                    while (m > 0 && classical_kind(G.ops[m - 1].op)) --m;
                    // inside the first run of a core (not the tail after its second H) and op i
                    // still acts on the core's target
                    const bool tail = m > 0 && G.ops[m - 1].op.kind == H && G.ops[m - 1].op.q0 == tq;
                    const bool on_t = oi.q0 == tq || (two_qubit(oi.kind) && oi.q1 == tq);
                    if (!tail && on_t && rec_at[target] != SIZE_MAX) {
                        recs.resize(rec_at[target]);
                        prm.resize(prm_at[target]);
                        i = target;
                    }
                }
            }
            phase_op0 = i;
            if (!phases.empty()) phases.back().g1 = (uint16_t)recs.size();
            rs = lookahead(i, regset);
            regset = 0;
            for (uint32_t q : rs) regset |= bit(q);
            if (!phases.empty()) {
                GRec x;
                memset(&x, 0, sizeof(x));
                x.code = C_XPOSE;
                x.a = (uint8_t)phases.size();
                recs.push_back(x);
            }
            phases.push_back(make_phase(rs, (uint16_t)recs.size()));
        }
        rec_at[i] = recs.size();
        prm_at[i] = prm.size();
        {
            size_t fe = i;
            uint32_t fmask = 0, fxor = 0;
            if (try_fold(i, fe, fmask, ftab, fxor)) {
                // M|x> = ph(x) |x ^ c>: diagonal table on the input pattern, then X on the bits of c
                GRec r;
                memset(&r, 0, sizeof(r));
                r.code = C_DK + fmask;
                r.pi = (uint16_t)prm.size();
                prm.insert(prm.end(), ftab.begin(), ftab.end());
                recs.push_back(r);
                for (int b = 0; b < RB; ++b)
                    if (fxor & (1u << b)) {
                        GRec xr;
                        memset(&xr, 0, sizeof(xr));
                        xr.code = C_X + b;
                        recs.push_back(xr);
                    }
                i = fe - 1;
                continue;
            }
        }
        const KOp &k = G.ops[i];
        const Op &o = k.op;
        GRec r;
        memset(&r, 0, sizeof(r));
        double d[4];
        if (o.kind == H) {
            r.code = C_H + regpos(o.q0);
        } else if (o.kind == RX || o.kind == RY) {
            double m[8];
            matrix_u(o, m);
            r.code = C_U + regpos(o.q0);
            r.pi = addp({m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7]});
        } else if (o.kind == X || o.kind == Y) {   // in-tile
            r.code = (o.kind == X ? C_X : C_Y) + regpos(o.q0);
        } else if (o.kind == CX) {
            int t = regpos(o.q1), c = regpos(o.q0);
            if (c >= 0) r.code = C_CX + 5 * c + t;
            else { r.code = C_TX + t; r.a = (uint8_t)o.q0; }
        } else if (o.kind == CZ || o.kind == CP) {
            double pr = o.kind == CZ ? -1.0 : cos(o.theta), pi = o.kind == CZ ? 0.0 : sin(o.theta);
            int a = regpos(o.q0), b = regpos(o.q1);
            if (a >= 0 && b >= 0) {
                if (a > b) std::swap(a, b);
                r.code = C_CPH + 5 * a + b;
                r.pi = addp({pr, pi});
            } else if (a >= 0 || b >= 0) {
                r.code = C_TD1 + (a >= 0 ? a : b);
                r.a = (uint8_t)(a >= 0 ? o.q1 : o.q0);
                r.pi = addp({pr, pi, o.kind == CZ ? M_PI : o.theta});
            } else {
                r.code = C_TPH;
                r.a = (uint8_t)o.q0;
                r.b = (uint8_t)o.q1;
                r.pi = addp({1.0, 0.0, pr, pi});
            }
        } else if (diag_of(o, d)) {
            int a = regpos(o.q0);
            const bool d0one = d[0] == 1.0 && d[1] == 0.0;
            if (a >= 0) {
                if (d0one) { r.code = C_D1 + a; r.pi = addp({d[2], d[3]}); }
                else { r.code = C_D2 + a; r.pi = addp({d[0], d[1], d[2], d[3]}); }
            } else {
                r.code = C_TPH;
                r.a = r.b = (uint8_t)o.q0;
                r.pi = addp({d[0], d[1], d[2], d[3]});
            }
        } else {
            throw std::runtime_error("fused planner: unsupported op kind");
        }
        recs.push_back(r);
    }
    if (phases.empty()) {
        rs = lookahead(0, 0);
        phases.push_back(make_phase(rs, 0));
    }
    phases.back().g1 = (uint16_t)recs.size();
    // Merge adjacent CX records sharing a control (the two leading CXs of every Cuccaro MAJ and
    // the mirrored pair when uncomputing) into one swap pass.
    {
        std::vector<GRec> m;
        m.reserve(recs.size());
        std::vector<uint16_t> newidx(recs.size() + 1);
        for (size_t j = 0; j < recs.size(); ++j) {
            newidx[j] = (uint16_t)m.size();
            const uint16_t c0 = recs[j].code;
            if (j + 1 < recs.size() && c0 >= C_CX && c0 < C_CX + 25 && recs[j + 1].code >= C_CX &&
                recs[j + 1].code < C_CX + 25) {
                const int c = (c0 - C_CX) / 5, t1 = (c0 - C_CX) % 5;
                const int c2 = (recs[j + 1].code - C_CX) / 5, t2 = (recs[j + 1].code - C_CX) % 5;
                if (c == c2 && t1 != t2 && c != t1 && c != t2) {
                    GRec r = recs[j];
                    r.code = (uint16_t)(C_CX2 + 25 * c + 5 * std::min(t1, t2) + std::max(t1, t2));
                    m.push_back(r);
                    newidx[j + 1] = (uint16_t)m.size();
                    ++j;
                    continue;
                }
            }
            m.push_back(recs[j]);
        }
        newidx[recs.size()] = (uint16_t)m.size();
        for (auto &ph : phases) { ph.g0 = newidx[ph.g0]; ph.g1 = newidx[ph.g1]; }
        recs.swap(m);
    }
    // Runs of controlled phases from non-register qubits onto the same register bit (C_TD1: the CP
    // ladders of a QFT, ~30 per H at 34 qubits) merge into one C_TDK record: the kernel multiplies
    // the per-thread scalar factors first and touches the amplitudes once.
    {
        std::vector<GRec> m;
        m.reserve(recs.size());
        std::vector<uint16_t> newidx(recs.size() + 1);
        for (size_t j = 0; j < recs.size(); ++j) {
            newidx[j] = (uint16_t)m.size();
            const uint16_t c0 = recs[j].code;
            size_t k = j;
            if (c0 >= C_TD1 && c0 < C_TD1 + RB)
                while (k < recs.size() && recs[k].code == c0 && k - j < 255) ++k;
            if (k - j >= 2) {
                GRec r;
                memset(&r, 0, sizeof(r));
                r.code = (uint16_t)(C_TDK + (c0 - C_TD1));
                r.a = (uint8_t)(k - j);
                r.pi = (uint16_t)prm.size();
                // angles as 64-bit fractions of a turn (exact for the dyadic angles of a QFT)
                std::vector<uint64_t> qk, ph;
                for (size_t q = j; q < k; ++q) {
                    double f = prm[recs[q].pi + 2] / (2.0 * M_PI);
                    f -= std::floor(f);
                    const double w = std::ldexp(f, 64);
                    qk.push_back(recs[q].a);
                    ph.push_back(w >= 18446744073709551616.0 ? 0ull : (uint64_t)w);
                    newidx[q] = (uint16_t)m.size();
                }
                // geometric weights (angle_k = c << q_k mod 2^64, a QFT ladder): acc = (lbase & M) * c
                size_t lo = 0;
                for (size_t q = 1; q < qk.size(); ++q) if (qk[q] < qk[lo]) lo = q;
                const uint64_t cgeo = ph[lo] >> qk[lo];
                bool geo = (ph[lo] & ((1ull << qk[lo]) - 1)) == 0;
                uint64_t mq = 0;
                for (size_t q = 0; q < qk.size() && geo; ++q) {
                    geo = (cgeo << qk[q]) == ph[q] && !(mq & bit(qk[q]));
                    mq |= bit(qk[q]);
                }
                auto bits_of = [](uint64_t v) { double d; memcpy(&d, &v, 8); return d; };
                if (geo) {
                    r.b = 1;
                    prm.push_back(bits_of(cgeo));
                    prm.push_back(bits_of(mq));
                } else {
                    for (size_t q = 0; q < qk.size(); ++q) {
                        prm.push_back(bits_of(qk[q]));
                        prm.push_back(bits_of(ph[q]));
                    }
                }
                m.push_back(r);
                j = k - 1;
                continue;
            }
            m.push_back(recs[j]);
        }
        newidx[recs.size()] = (uint16_t)m.size();
        for (auto &ph : phases) { ph.g0 = newidx[ph.g0]; ph.g1 = newidx[ph.g1]; }
        recs.swap(m);
    }
    // Toffoli cores: H(t) DK(a, b, t) H(t) [DK(subset of a, b)] is, per pattern of the controls
    // (a, b), a 2x2 matrix on t -- ONE controlled-2x2 record (C_CU) replaces 3-4 records.  The host
    // multiplies the blocks out exactly as the gates define them (the two H's included, so the
    // group's deferred (1/sqrt2)^h drops 2 per merge) and classifies each block: for an error-free
    // Toffoli three blocks are the identity and the fourth is a plain swap.
    B.h_absorbed = 0;
    {
        std::vector<GRec> m;
        m.reserve(recs.size());
        std::vector<uint16_t> newidx(recs.size() + 1);
        for (size_t j = 0; j < recs.size(); ++j) {
            newidx[j] = (uint16_t)m.size();
            const uint16_t c0 = recs[j].code;
            // X records between the table and the second H (a Pauli error folded into the core):
            // H X_S D H = Z_p^[p in S] X_S' (H D H), S' = S \ {p} -- the Z joins the blocks, the
            // X's follow the record (and conjugate a trailing control diagonal)
            size_t k2 = j + 2;
            uint32_t xs = 0;
            if (j + 1 < recs.size() && recs[j + 1].code >= C_DK && recs[j + 1].code < C_DK + NR)
                while (k2 < recs.size() && recs[k2].code >= C_X && recs[k2].code < C_X + RB &&
                       (((recs[j + 1].code - C_DK) >> (recs[k2].code - C_X)) & 1)) {
                    xs ^= 1u << (recs[k2].code - C_X);
                    ++k2;
                }
            if (k2 < recs.size() && c0 < C_H + RB && recs[k2].code == c0 && recs[j + 1].code >= C_DK &&
                recs[j + 1].code < C_DK + NR) {
                const int p = c0 - C_H, mask = recs[j + 1].code - C_DK;
                int jj = -1;
                for (int q = 0; q < 6; ++q)
                    if (hdh_mask(p, q) == mask) jj = q;
                if (jj >= 0 && code_ok(C_CU + 6 * p + jj)) {
                    const int cm = mask & ~(1 << p);
                    const bool zp = (xs >> p) & 1u;
                    const uint32_t xo = xs & ~(1u << p);
                    const double *t1 = &prm[recs[j + 1].pi];
                    // optional trailing diagonal on the controls
                    const double *t2 = nullptr;
                    int m2 = 0;
                    if (k2 + 1 < recs.size() && recs[k2 + 1].code > C_DK && recs[k2 + 1].code < C_DK + NR &&
                        ((recs[k2 + 1].code - C_DK) & ~cm) == 0) {
                        m2 = recs[k2 + 1].code - C_DK;
                        t2 = &prm[recs[k2 + 1].pi];
                    }
                    auto pextm = [](uint32_t x, uint32_t mk) {
                        uint32_t o = 0, k = 0;
                        for (int b = 0; b < RB; ++b)
                            if (mk & (1u << b)) { o |= ((x >> b) & 1u) << k; ++k; }
                        return o;
                    };
                    std::vector<double> blk(32, 0.0);
                    uint32_t kinds = 0, unit = 0;
                    for (uint32_t bi = 0; bi < 4; ++bi) {
                        uint32_t x = 0, k = 0;   // deposit bi into the control bits
                        for (int b = 0; b < RB; ++b)
                            if (cm & (1 << b)) { if ((bi >> k) & 1u) x |= 1u << b; ++k; }
                        const uint32_t x0 = x, x1 = x | (1u << p);
                        const double d0r = t1[2 * pextm(x0, mask)], d0i = t1[2 * pextm(x0, mask) + 1];
                        const double d1r = t1[2 * pextm(x1, mask)], d1i = t1[2 * pextm(x1, mask) + 1];
                        double fr = 1.0, fi = 0.0;
                        if (t2) { fr = t2[2 * pextm(x0 ^ xo, m2)]; fi = t2[2 * pextm(x0 ^ xo, m2) + 1]; }
                        // (1/2) [[d0 + d1, d0 - d1], [d0 - d1, d0 + d1]] * f   (= H diag(d0, d1) H, then f)
                        const double sr = 0.5 * (d0r + d1r), si = 0.5 * (d0i + d1i);
                        const double ar = 0.5 * (d0r - d1r), ai = 0.5 * (d0i - d1i);
                        double e[8] = {sr * fr - si * fi, sr * fi + si * fr, ar * fr - ai * fi, ar * fi + ai * fr,
                                       ar * fr - ai * fi, ar * fi + ai * fr, sr * fr - si * fi, sr * fi + si * fr};
                        if (zp)
                            for (int q = 4; q < 8; ++q) e[q] = -e[q];   // Z on t after the block
                        // snap to the exact values the algebra gives (errors <= a few ulp)
                        for (double &v : e) {
                            if (fabs(v) < 1e-15) v = 0.0;
                            else if (fabs(v - 1.0) < 1e-15) v = 1.0;    // <= 4 ulp
                            else if (fabs(v + 1.0) < 1e-15) v = -1.0;
                        }
                        const bool offz = e[2] == 0 && e[3] == 0 && e[4] == 0 && e[5] == 0;
                        const bool diagz = e[0] == 0 && e[1] == 0 && e[6] == 0 && e[7] == 0;
                        uint32_t kd = 3;
                        if (offz) kd = (e[0] == 1 && e[1] == 0 && e[6] == 1 && e[7] == 0) ? 0 : 1;
                        else if (diagz) {
                            kd = 2;
                            if (e[2] == 1 && e[3] == 0 && e[4] == 1 && e[5] == 0) unit |= 1u << bi;
                        }
                        kinds |= kd << (2 * bi);
                        for (int q = 0; q < 8; ++q) blk[8 * bi + q] = e[q];
                    }
                    GRec r;
                    memset(&r, 0, sizeof(r));
                    if (kinds == (2u << 6) && unit == 8u && code_ok(C_CCX + 6 * p + jj)) {
                        // an error-free Toffoli: a pure register permutation (compile-time swaps,
                        // no block dispatch; absorbable into phase entry/exit offsets)
                        r.code = (uint16_t)(C_CCX + 6 * p + jj);
                    } else {
                        r.code = (uint16_t)(C_CU + 6 * p + jj);
                        r.a = (uint8_t)unit;
                        r.b = (uint8_t)kinds;
                        r.pi = (uint16_t)prm.size();
                        prm.insert(prm.end(), blk.begin(), blk.end());
                    }
                    m.push_back(r);
                    for (int b = 0; b < RB; ++b)
                        if ((xo >> b) & 1u) {
                            GRec xr;
                            memset(&xr, 0, sizeof(xr));
                            xr.code = (uint16_t)(C_X + b);
                            m.push_back(xr);
                        }
                    B.h_absorbed += 2;
                    const size_t last = t2 ? k2 + 1 : k2;
                    for (size_t q = j + 1; q <= last; ++q) newidx[q] = (uint16_t)m.size();
                    j = last;
                    continue;
                }
            }
            m.push_back(recs[j]);
        }
        newidx[recs.size()] = (uint16_t)m.size();
        for (auto &ph : phases) { ph.g0 = newidx[ph.g0]; ph.g1 = newidx[ph.g1]; }
        recs.swap(m);
    }
    // Absorb register permutations (in-register X, CX between register bits) at the start of a
    // phase into its entry offsets and at its end into its exit offsets: a permutation of the 32
    // registers right after a load/transpose (or before a transpose/store) is free to apply as
    // a permutation of the addresses it reads/writes.
    for (int r = 0; r < NR; ++r) { B.pin0[r] = (uint8_t)r; B.pout_last[r] = (uint8_t)r; }
    {
        std::vector<GRec> kept;
        kept.reserve(recs.size());
        for (size_t p = 0; p < phases.size(); ++p) {
            Phase &ph = phases[p];
            size_t g0 = ph.g0, g1 = ph.g1, a = g0, b = g1;
            while (a < g1 && is_perm_rec(recs[a].code)) ++a;
            while (b > a && is_perm_rec(recs[b - 1].code)) --b;
            uint8_t pin[NR], pout[NR];
            for (uint32_t r = 0; r < (uint32_t)NR; ++r) {
                uint32_t x = r;                      // a_k[r] = a_0[pi_1(...pi_k(r))]
                for (size_t j = a; j-- > g0;) x = perm_apply(recs[j].code, x);
                pin[r] = (uint8_t)x;
                uint32_t y = r;                      // a_fin[r] = a_m[pi_b(...pi_end(r))]
                for (size_t j = g1; j-- > b;) y = perm_apply(recs[j].code, y);
                pout[r] = (uint8_t)y;
            }
            uint16_t base_so[NR];
            memcpy(base_so, ph.so, sizeof(base_so));
            for (int r = 0; r < NR; ++r) {
                ph.so[r] = base_so[pin[r]];          // register r reads the pattern pin[r]
                ph.so_out[pout[r]] = base_so[r];     // register pout[r] holds the value of pattern r
            }
            if (p == 0) memcpy(B.pin0, pin, sizeof(pin));
            if (p + 1 == phases.size())
                for (int r = 0; r < NR; ++r) B.pout_last[pout[r]] = (uint8_t)r;
            if (p > 0) kept.push_back(recs[g0 - 1]);   // the XPOSE record entering this phase
            const uint16_t ng0 = (uint16_t)kept.size();
            for (size_t j = a; j < b; ++j) kept.push_back(recs[j]);
            ph.g0 = ng0;
            ph.g1 = (uint16_t)kept.size();
        }
        recs.swap(kept);
    }
    // Diagonal tables whose entries with some register bit t clear are exactly 1 (a CP ladder onto
    // t: the QFT's in-register phases) become controlled tables: half the multiplies and loads.
    for (auto &r : recs) {
        if (r.code < C_DK || r.code >= C_DK + NR) continue;
        const int M = r.code - C_DK, K = __builtin_popcount((unsigned)M);
        const double *tab = prm.data() + r.pi;
        for (int t = 0; t < RB; ++t) {
            if (!((M >> t) & 1)) continue;
            const int kt = __builtin_popcount((unsigned)(M & ((1 << t) - 1)));   // t's index in the pext
            bool ctl = true;
            for (int e = 0; e < (1 << K) && ctl; ++e)
                if (!((e >> kt) & 1)) ctl = tab[2 * e] == 1.0 && tab[2 * e + 1] == 0.0;
            if (!ctl) continue;
            int m4 = 0, k = 0;   // the other bits of M, numbered over the register bits other than t
            for (int b = 0; b < RB; ++b) {
                if (b == t) continue;
                if ((M >> b) & 1) m4 |= 1 << k;
                ++k;
            }
            std::vector<double> sub;
            for (int e = 0; e < (1 << K); ++e)
                if ((e >> kt) & 1) { sub.push_back(tab[2 * e]); sub.push_back(tab[2 * e + 1]); }
            r.code = (uint16_t)(C_DKC + 16 * t + m4);
            r.pi = (uint16_t)prm.size();
            prm.insert(prm.end(), sub.begin(), sub.end());
            break;
        }
    }
    {   // compact the parameter block (merges leave their inputs' parameters unused)
        std::vector<double> used;
        used.reserve(prm.size());
        for (auto &r : recs) {
            const int np = rec_nparams(r);
            if (!np) continue;
            const uint16_t at = (uint16_t)used.size();
            used.insert(used.end(), prm.begin() + r.pi, prm.begin() + r.pi + np);
            r.pi = at;
        }
        prm.swap(used);
    }
    if (phases.size() > (size_t)MAXPH || recs.size() > (size_t)MAXG || prm.size() > (size_t)MAXP)
        throw std::runtime_error("fused planner: group exceeds the kernel parameter block");
    P.nphase = (uint32_t)phases.size();
    P.ngate = (uint32_t)recs.size();
    // transposes between phases with identical thread-bit layouts are thread-local (no barrier)
    {
        uint32_t cur = 0;
        for (auto &r : recs) {
            if (r.code != C_XPOSE) continue;
            r.b = memcmp(phases[cur].tl, phases[r.a].tl, NTB) == 0 ? 1 : 0;
            cur = r.a;
        }
    }
#ifdef TUSQ_DEBUG_PLAN   // build-time debug aid (TUSQ_NVCC_FLAGS=-DTUSQ_DEBUG_PLAN): print every group plan
    {
        fprintf(stderr, "[plan] ops %zu recs %zu phases %zu prm %zu tile %#llx\n  ops:", G.ops.size(), recs.size(),
                phases.size(), prm.size(), (unsigned long long)tile);
        for (auto &k : G.ops) fprintf(stderr, " %u(%u,%u)", k.op.kind, k.op.q0, k.op.q1);
        fprintf(stderr, "\n  codes:");
        for (auto &r : recs) fprintf(stderr, " %u", r.code);
        fprintf(stderr, "\n  phases:");
        for (auto &ph : phases) {
            fprintf(stderr, " [g%u-%u regs", ph.g0, ph.g1);
            for (int k = 0; k < RB; ++k) fprintf(stderr, " %u", P.qs[ph.rl[k]]);
            fprintf(stderr, "]");
        }
        fprintf(stderr, "\n");
    }
#endif
    std::copy(phases.begin(), phases.end(), P.ph);
    std::copy(recs.begin(), recs.end(), P.g);
    std::copy(prm.begin(), prm.end(), P.prm);
    B.prm_used = (prm.size() + 1) & ~(size_t)1;   // the gather table starts 16-byte aligned
}

// dynamic shared memory of k_fused: NBUF tile buffers, the gather table, the tile-index tables
static size_t smem_bytes(int prec)
{
    return (size_t)NBUF * (1 << TB) * (prec == 128 ? 16 : 8) + NR * NT * 2 + 2 * NCH * 256 * sizeof(uint64_t) +
           (1 << (TB - 3)) * sizeof(uint64_t);   // F_TSTORE run offsets (runs >= 8 elements)
}

static int blocks_per_sm(int prec)
{
    // one-time per device and precision (the attribute is per device); concurrent first calls
    // compute the same value
    static std::atomic<int> occ[64][2];
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int> &slot = occ[dev & 63][prec == 128 ? 1 : 0];
    int o = slot.load(std::memory_order_relaxed);
    if (!o) {
        const size_t smem = smem_bytes(prec);
        if (prec == 128) {
            cudaFuncSetAttribute(k_fused<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused<double>, NT * NG, smem);
        } else {
            cudaFuncSetAttribute(k_fused<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused<float>, NT * NG, smem);
        }
        if (o < 1) o = 1;
        slot.store(o, std::memory_order_relaxed);
    }
    return o;
}

void FusedPlanner::execute(const std::vector<Op> &ops, Ctx &ctx)
{
    execute_ex(ops, ctx, nullptr, nullptr, nullptr, false);
}

bool FusedPlanner::execute_ex(const std::vector<Op> &ops, Ctx &ctx, const InitState *init, double *d_sums,
                              bool *sums_written, bool sums_only)
{
    if (sums_written) *sums_written = false;
    if (pending_tiles_) throw std::runtime_error("fused planner: a sums-only transition was not replayed");
    if (stale_ && !init) throw std::runtime_error("fused planner: uncompute from a state that was not stored");
    stale_ = false;
    // strict grouping when it costs (almost) no extra sweeps -- e.g. ripple-carry ladders --
    // otherwise tile membership for controls/diagonals only while there is room (e.g. QFT)
    bool strict = false;
    std::vector<Group> groups = make_groups(ops, false);
    {
        std::vector<Group> g2 = make_groups(ops, true);
        if (g2.size() * 100 <= groups.size() * 105) { groups.swap(g2); strict = true; }
    }
    // The sampler's per-block sums come free from the last sweep if its tile is the contiguous
    // block {0..11}.  If it is not, try cutting the stream so that the longest suffix touching only
    // qubits < 12 is its own group -- accepted only when it costs no extra sweep.
    if (d_sums && !groups.empty()) {
        size_t s = ops.size();
        while (s > 0) {
            const Op &o = ops[s - 1];
            if (o.q0 >= (uint32_t)TB || (two_qubit(o.kind) && o.q1 >= (uint32_t)TB)) break;
            --s;
        }
        if (s > 0 && s < ops.size()) {
            std::vector<Op> head(ops.begin(), ops.begin() + s), tail(ops.begin() + s, ops.end());
            std::vector<Group> g3 = make_groups(head, strict), g4 = make_groups(tail, strict);
            if (g3.size() + g4.size() <= groups.size()) {
                g3.insert(g3.end(), g4.begin(), g4.end());
                groups.swap(g3);
            }
        }
    }
    const double s = (double)(1ull << n_) * (prec_ == 128 ? 16 : 8);
    bool pending_init = init != nullptr;
    if (groups.empty() && pending_init) {
        if (!ctx.dry) launch_init_basis(ctx.psi, n_, prec_, init->index, init->re, init->im, ctx.st);
        count(ctx, s, false);
        note_basis(init->index);
        return true;
    }
    if (!scratch_) scratch_ = std::make_shared<PlanScratch>();
    Built &B = scratch_->B;
    // ---- tiles and layouts of the launched groups.  The transition
    // starts and ends in the identity layout.  Group k >= 1 reads the layout the group before it
    // wrote: its own 12 tile qubits at physical 0..11 (a contiguous 64 KiB tile), ordered
    // [shared with group k-1][new], then group k-1's other tile qubits right above them (a
    // compact write footprint for group k-1), then the rest ascending.  Fillers of a middle group
    // come from the previous group's tile first (longer write runs for it).
    std::vector<size_t> launched;
    {
        bool pi = pending_init;
        for (size_t gi = 0; gi < groups.size(); ++gi)
            if (!groups[gi].ops.empty() || pi) { launched.push_back(gi); pi = false; }
    }
    const size_t NLG = launched.size();
    std::vector<uint64_t> tiles(NLG);
    for (size_t k = 0; k < NLG; ++k) {
        uint64_t t = groups[launched[k]].tilemask;
        auto fill = [&](uint64_t from) {
            for (uint64_t m = from; m && __builtin_popcountll(t) < TB; m &= m - 1) t |= m & (~m + 1);
        };
        if (k > 0 && k + 1 < NLG) fill(tiles[k - 1]);
        fill(n_ >= 64 ? ~0ull : (1ull << n_) - 1);   // then the lowest unused qubits
        tiles[k] = t;
    }
    // A sweep that changes the layout is a global permutation of the state: it must run out of
    // place (alt_, the caller-provided second buffer).  Buffers alternate from ctx.psi, so the
    // number of layout-changing sweeps must be even for the state to end in ctx.psi: with an odd
    // number of groups, boundary 1 keeps the identity (group 0 runs in place).  Without a second
    // buffer every layout is the identity and every sweep runs in place.
    // ---- live tiles.  After a reset the state is ONE basis state; a gate
    // can only make a qubit vary if it is an exchange gate on it (H, RX, RY, U) or a CX whose
    // control already varies; X / Y / CX with a fixed control just flip a fixed bit; diagonals
    // change nothing.  So before launched group k the nonzero amplitudes lie in {x : x_q = b_q
    // for q outside S_k}, and group k only has to visit the 2^|S_k \ tile_k| tiles with those
    // outer bits -- the others are zero (K7 wrote them) and stay zero (the group's gates act
    // inside tiles).  The leading groups whose live tiles are <= 1/8 of all run IN PLACE in the
    // identity layout over their live tiles only (F_LIVE); the first reset group is one tile.
    // Without a reset the analysis continues from the support known after the previous call
    // (dfree_ / dfix_: physical, identity layout; logical = physical ^ xmask_).
    const uint64_t all = n_ >= 64 ? ~0ull : (1ull << n_) - 1;
    std::vector<uint64_t> supS(NLG, ~0ull), supB(NLG, 0);
    std::vector<char> live(NLG, 0);   // launched group k visits only its live tiles (in place)
    const bool track = live_ && (pending_init || (dfree_ & all) != all);
    uint64_t sup_end = all, bx_end = 0;
    if (track) {
        uint64_t sup = pending_init ? 0 : dfree_ & all;   // qubits that may vary
        uint64_t bx = pending_init ? init->index : (dfix_ ^ xmask_) & ~sup;   // values of the others
        auto step = [&](const Op &o) {
            const uint64_t b0 = bit(o.q0), b1 = two_qubit(o.kind) ? bit(o.q1) : 0;
            switch (o.kind) {
            case Kind::I: case Kind::Z: case Kind::S: case Kind::SDG: case Kind::T: case Kind::TDG:
            case Kind::P: case Kind::RZ: case Kind::CZ: case Kind::CP: break;
            case Kind::X: case Kind::Y: if (!(sup & b0)) bx ^= b0; break;
            case Kind::CX:
                if (sup & b0) sup |= b1;
                else if ((bx & b0) && !(sup & b1)) bx ^= b1;
                break;
            default: sup |= b0 | b1; break;   // H, RX, RY and anything else: the qubits may vary
            }
        };
        bool pi = true;
        size_t k = 0;
        for (const Group &G : groups) {
            const bool launch = !G.ops.empty() || pi;
            pi = false;
            bx ^= G.xb & ~sup;
            if (launch) { supS[k] = sup; supB[k] = bx; ++k; }
            for (const KOp &ko : G.ops) step(ko.op);
            bx ^= G.xa & ~sup;
        }
        sup_end = sup;
        bx_end = bx;
        // live: the group's live tiles are <= 1/8 of all (the reset group is always one tile)
        for (size_t g = 0; g < NLG; ++g)
            live[g] = __builtin_popcountll(supS[g] & ~tiles[g] & all) + 3 <= (int)(n_ - TB) || (g == 0 && pending_init);
    }
    if (!track && pending_init && NLG) live[0] = 1;   // the reset group is always one tile
    std::vector<std::array<uint8_t, 64>> lay(NLG + 1);
#ifdef TUSQ_DEBUG_KNOBS   // debug builds only: TUSQ_DBG_IDENTITY=1 keeps every layout the identity
    static const bool dbg_identity = getenv("TUSQ_DBG_IDENTITY") != nullptr;
#else
    constexpr bool dbg_identity = false;
#endif
    if (!alt_ && alt_lazy_ && NLG >= 2 && !ctx.dry && !dbg_identity) {
        if (cudaMallocAsync(&alt_, alt_lazy_, ctx.st) == cudaSuccess) alt_owned_ = true;
        else { cudaGetLastError(); alt_ = nullptr; alt_lazy_ = 0; }   // no memory: stay in place
    }
    const bool remap = alt_ != nullptr && !dbg_identity && NLG >= 2;
    for (size_t k = 0; k <= NLG; ++k) {
        auto &L = lay[k];
        if (k == 0 || k == NLG || !remap || live[k - 1] || live[k]) {   // (live sweeps: in place, identity)
            for (uint32_t q = 0; q < 64; ++q) L[q] = (uint8_t)q;
            continue;
        }
        const uint64_t a = tiles[k - 1], b = tiles[k], all = n_ >= 64 ? ~0ull : (1ull << n_) - 1;
        uint8_t pos = 0;
#ifdef TUSQ_DEBUG_KNOBS   // TUSQ_DBG_WCONTIG=1: contiguous WRITES instead (group k-1's tile at 0..11)
        static const bool wcontig = getenv("TUSQ_DBG_WCONTIG") != nullptr;
        if (wcontig) {
            for (uint64_t part : {a & b, a & ~b, b & ~a, all & ~(a | b)})
                for (uint64_t m = part; m; m &= m - 1) L[__builtin_ctzll(m)] = pos++;
            continue;
        }
#endif
        for (uint64_t part : {a & b, b & ~a, a & ~b, all & ~(a | b)})
            for (uint64_t m = part; m; m &= m - 1) L[__builtin_ctzll(m)] = pos++;
    }
    // parity: reset remapped boundaries to the identity, first to last, until the number of
    // layout changes is even (all-identity is even, so this terminates)
    for (size_t k = 1; k < NLG; ++k) {
        size_t changes = 0;
        for (size_t j = 0; j < NLG; ++j) changes += lay[j] != lay[j + 1];
        if (!(changes & 1)) break;
        for (uint32_t q = 0; q < 64; ++q) lay[k][q] = (uint8_t)q;
    }
    auto permute = [&](uint64_t x, const std::array<uint8_t, 64> &L) {
        uint64_t o = 0;
        for (; x; x &= x - 1) o |= bit(L[__builtin_ctzll(x)]);
        return o;
    };
    size_t lk = 0;   // launched-group counter
    void *cur = ctx.psi;   // the buffer holding the state in layout lay[lk]
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const Group &G = groups[gi];
        if (G.ops.empty() && !pending_init) {   // pure relabel
            xmask_ ^= G.xb ^ G.xa;
            continue;
        }
        // loads go through shared memory (always coalesced): no load-layout phase needed
        build_params(G, n_, B, tiles[lk], lay[lk].data(), lay[lk + 1].data());
        Params &P = B.P;
        const size_t kq = lk;          // this group's launch index (lk advances below)
        uint64_t init_tile = 0;        // the reset group's one tile (tile-index bits)
        void *src = cur;
        void *dst = lay[lk] == lay[lk + 1] ? cur : (cur == ctx.psi ? alt_ : ctx.psi);
        cur = dst;
        uint64_t m_load = (pending_init ? 0 : xmask_) ^ G.xb;
        P.xm_load = m_load;
        P.xm_store = m_load & ~B.tile;
        P.xin = permute(P.xm_store, lay[lk]);
        P.xout = permute(P.xm_store, lay[lk + 1]);
        ++lk;
        // a contiguous tile (its 12 qubits at read positions 0..11) loads with one bulk copy into a
        // LINEAR buffer; otherwise per-thread cp.async into the swizzled layout
        bool bulk = !pending_init;
        for (int b = 0; b < TB && bulk; ++b) bulk = P.pin[b] == b;
        // ... read conflict-free from the linear buffer only when lanes 0-2 carry tile bits 0-2 (each
        // quarter warp then reads one 128-byte row); a gather (leading transposes folded) reads
        // arbitrary slots and keeps the swizzled staging (ncu: 7x bank conflicts from linear)
        if (((1u << P.ph[0].tl[0]) | (1u << P.ph[0].tl[1]) | (1u << P.ph[0].tl[2])) != 7u) bulk = false;
        if (P.ngate && P.g[0].code == C_XPOSE) bulk = false;
        // a buffer valid on a subset only is read element-wise (invalid elements zero-filled)
        if (!pending_init && (vfree_ & ((n_ >= 64 ? ~0ull : (1ull << n_) - 1))) != (n_ >= 64 ? ~0ull : (1ull << n_) - 1))
            bulk = false;
        {
            const Phase &f = P.ph[0], &l = P.ph[P.nphase - 1];
            P.regm_load = 0;
            P.rx = 0;
            for (int k = 0; k < RB; ++k) {
                P.regm_load |= bit(P.qs[f.rl[k]]);
                if (m_load & bit(P.qs[f.rl[k]])) P.rx |= 1u << k;
            }
            auto goff = [&](const Phase &ph, uint32_t pat, const uint8_t *posn) {
                uint64_t o = 0;
                for (int k = 0; k < RB; ++k)
                    if (pat & (1u << k)) o |= bit(posn[ph.rl[k]]);
                return o;
            };
            // register r loads pattern pin0[r] ^ rx (mask fix-up + absorbed permutation; logical
            // positions: only an init group uses gl, and it reads the identity layout); register s
            // is stored at the pattern pout_last[s], in the write layout
            for (int r = 0; r < NR; ++r) {
                P.gl[r] = goff(f, (uint32_t)B.pin0[r] ^ P.rx, P.qs);
                P.gs[r] = goff(l, B.pout_last[r], P.pout);
            }
            // bulk-copy stores (F_TSTORE): write order = tile bits by write position; the low ts_l0
            // write-order bits must be write positions 0..ts_l0-1 (contiguous, aligned runs)
            {
                uint8_t ord[TB];
                for (int b = 0; b < TB; ++b) ord[b] = (uint8_t)b;
                std::sort(ord, ord + TB, [&](uint8_t x, uint8_t y) { return P.pout[x] < P.pout[y]; });
                for (int k = 0; k < TB; ++k) P.wpos[ord[k]] = (uint8_t)k;
                int l0 = 0;
                while (l0 < TB && P.pout[ord[l0]] == l0) ++l0;
                P.ts_l0 = (uint8_t)l0;
                for (int k = 0; k + l0 < TB; ++k) P.ts_hipos[k] = P.pout[ord[l0 + k]];
                for (int r = 0; r < NR; ++r) {
                    uint32_t w = 0;
                    for (int k = 0; k < RB; ++k)
                        if ((B.pout_last[r] >> k) & 1) w |= 1u << P.wpos[l.rl[k]];
                    P.wreg[r] = (uint16_t)w;
                }
            }
            P.rx = 0;
            // paired stores when qubit 0 is a register bit of the last layout
            P.st_pair = 0;
            P.st_odd = 0;
            for (int v = 1; v < NR && !P.st_pair; ++v) {
                bool ok = true;
                for (int r = 0; r < NR && ok; ++r) ok = P.gs[r ^ v] == (P.gs[r] ^ 1ull);
                if (ok) {
                    P.st_pair = (uint16_t)v;
                    for (int r = 0; r < NR; ++r) P.st_odd |= (uint32_t)(P.gs[r] & 1) << r;
                }
            }
            // shared-memory staging of loads: copy-slot offsets, tile-local XOR mask, last transpose
            P.mloc = 0;
            for (int b = 0; b < TB; ++b)
                if (m_load & bit(P.qs[b])) P.mloc |= (uint16_t)(1u << b);
            for (int j = 0; j < NR; ++j) {
                uint64_t o = 0;
                for (int k = 0; k < RB; ++k)
                    if (j & (1 << k)) o |= bit(P.pin[NTB + k]);
                P.gj[j] = o;
                P.sj[j] = (uint16_t)swz((uint32_t)j << NTB);
            }
            // Leading transposes (phases whose records were all absorbed, e.g. the error-free Toffoli
            // ladders of an Adder group) fold into the first shared-memory read: the data movement of
            // the whole chain is simulated here and the read becomes a gather through a table
            P.gtab = 0xFFFFu;
            init_tile = 0;
            uint32_t kstar = 0;
            while (kstar < P.ngate && P.g[kstar].code == C_XPOSE) ++kstar;
            // A reset group holds ONE nonzero element: its leading transposes fold away entirely
            // -- the host follows that element through them (the same slot simulation as the
            // gather) and the kernel puts it straight into its final register.
            if (pending_init) {
                auto &V = scratch_->V;
                auto &M = scratch_->M;
                auto tt = [&](const Phase &ph, uint32_t t) {
                    uint32_t x = 0;
                    for (int j = 0; j < NTB; ++j) x |= ((t >> j) & 1u) << ph.tl[j];
                    return swz(x);
                };
                for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                    for (int r = 0; r < NR; ++r) V[t][r] = (uint16_t)(tt(P.ph[0], t) ^ P.ph[0].so[r]);
                uint32_t cur = 0;
                for (uint32_t k = 0; k < kstar; ++k) {
                    const Phase &a = P.ph[cur], &b = P.ph[P.g[k].a];
                    for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                        for (int r = 0; r < NR; ++r) M[tt(a, t) ^ a.so_out[r]] = V[t][r];
                    for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                        for (int r = 0; r < NR; ++r) V[t][r] = M[tt(b, t) ^ b.so[r]];
                    cur = P.g[k].a;
                }
                // the nonzero logical element l* (the reset target seen through the load mask), its
                // tile and its tile-local index; find the register that holds it
                const uint64_t lstar = init->index ^ m_load;
                uint32_t estar = 0;
                for (int b = 0; b < TB; ++b) estar |= (uint32_t)((lstar >> P.qs[b]) & 1u) << b;
                init_tile = 0;
                for (uint32_t k = 0; k < P.nout; ++k) init_tile |= ((lstar >> P.ol[k]) & 1ull) << k;
                const uint16_t want = (uint16_t)swz(estar);
                bool found = false;
                for (uint32_t t = 0; t < (uint32_t)NT && !found; ++t)
                    for (int r = 0; r < NR && !found; ++r)
                        if (V[t][r] == want) { P.init_t = t; P.init_r = (uint32_t)r; found = true; }
                if (!found) throw std::runtime_error("fused planner: reset element not found");
                for (uint32_t k = cur; k < P.nphase; ++k) P.ph[k - cur] = P.ph[k];
                P.nphase -= cur;
                for (uint32_t i = kstar; i < P.ngate; ++i) {
                    P.g[i - kstar] = P.g[i];
                    if (P.g[i - kstar].code == C_XPOSE) P.g[i - kstar].a = (uint8_t)(P.g[i - kstar].a - cur);
                }
                P.ngate -= kstar;
                if (P.ngate < (uint32_t)MAXG) P.g[P.ngate] = GRec{};
            } else if (kstar > 0 && B.prm_used + NR * NT / 4 <= (size_t)MAXP) {
                auto &V = scratch_->V;
                auto &M = scratch_->M;
                auto tt = [&](const Phase &ph, uint32_t t) {
                    uint32_t x = 0;
                    for (int j = 0; j < NTB; ++j) x |= ((t >> j) & 1u) << ph.tl[j];
                    return swz(x);
                };
                // initial slot of the element (t, r) reads in phase 0: swizzled (cp.async copy) or
                // linear with the tile part of the load mask (bulk copy; swz is an involution)
                for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                    for (int r = 0; r < NR; ++r) {
                        const uint16_t sw = (uint16_t)(tt(P.ph[0], t) ^ P.ph[0].so[r]);
                        V[t][r] = bulk ? (uint16_t)(swz(sw) ^ P.mloc) : sw;
                    }
                uint32_t cur = 0;
                for (uint32_t k = 0; k < kstar; ++k) {
                    const Phase &a = P.ph[cur], &b = P.ph[P.g[k].a];
                    for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                        for (int r = 0; r < NR; ++r) M[tt(a, t) ^ a.so_out[r]] = V[t][r];
                    for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                        for (int r = 0; r < NR; ++r) V[t][r] = M[tt(b, t) ^ b.so[r]];
                    cur = P.g[k].a;
                }
                const uint32_t esz = prec_ == 128 ? 16 : 8;
                uint16_t *tab = reinterpret_cast<uint16_t *>(P.prm + B.prm_used);
                for (uint32_t t = 0; t < (uint32_t)NT; ++t)
                    for (int r = 0; r < NR; ++r) tab[r * NT + t] = (uint16_t)(V[t][r] * esz);
                P.gtab = (uint16_t)B.prm_used;
                // phase `cur` becomes phase 0; drop the folded records
                for (uint32_t k = cur; k < P.nphase; ++k) P.ph[k - cur] = P.ph[k];
                P.nphase -= cur;
                for (uint32_t i = kstar; i < P.ngate; ++i) {
                    P.g[i - kstar] = P.g[i];
                    if (P.g[i - kstar].code == C_XPOSE) P.g[i - kstar].a = (uint8_t)(P.g[i - kstar].a - cur);
                }
                P.ngate -= kstar;
                if (P.ngate < (uint32_t)MAXG) P.g[P.ngate] = GRec{};
            }
            P.last_xpose = 0xFFFFu;
            for (uint32_t i = 0; i < P.ngate; ++i)
                if (P.g[i].code == C_XPOSE) P.last_xpose = (uint16_t)i;
            // linear phase-0 read offsets of the bulk path (element units; bytes below)
            for (int r = 0; r < NR; ++r) P.so0[r] = (uint16_t)(swz(P.ph[0].so[r]) ^ P.mloc);
        }
        P.ntiles = 1ull << (n_ - TB);
        P.flags = 0;
        for (uint32_t i = 0; i < P.ngate; ++i) {   // records that read the logical index
            const uint16_t c = P.g[i].code;
            if ((c >= C_TX && c <= C_TPH) || (c >= C_TDK && c < C_DKC)) P.flags |= F_LBASE;
        }
        if (bulk) P.flags |= F_BULK;
        {
            int ts_min = 6;   // stores by bulk copies when runs are >= 2^ts_min elements (measured:
                              // 64 KiB runs 6.40 -> 5.81 ms, 128-byte runs 7.74 -> 11.5 ms, 1-2 KiB even)
#ifdef TUSQ_DEBUG_KNOBS       // TUSQ_DBG_TS_L0=k: only runs >= 2^k elements (13: never)
            static const int dbg_ts = getenv("TUSQ_DBG_TS_L0") ? atoi(getenv("TUSQ_DBG_TS_L0")) : 0;
            if (dbg_ts) ts_min = dbg_ts;
#endif
            // (not on a partly valid buffer: its mostly-zero tiles measured slower with it)
            // and only when lanes 0-2 of the last phase carry write-order bits 0-2: the write-order
            // staging is linear (the bulk copies need contiguous runs), so each quarter warp must
            // cover one 128-byte row -- otherwise every STS is 8-way bank conflicted (ncu on a
            // dense C4 sweep: 14 wavefronts per STS, 1.0 G conflicts, ~3 ms of a 15.9 ms sweep)
            const Phase &lp = P.ph[P.nphase - 1];
            const uint32_t lane_w = (1u << P.wpos[lp.tl[0]]) | (1u << P.wpos[lp.tl[1]]) | (1u << P.wpos[lp.tl[2]]);
            if (P.ts_l0 >= ts_min && (vfree_ & all) == all && lane_w == 7u) P.flags |= F_TSTORE;
        }
        if (pending_init) {
            P.flags |= F_INIT;
            P.init_re = init->re;
            P.init_im = init->im;
        }
        if (live[kq]) {   // live-tile sweep (in place, identity layout)
            P.flags |= F_LIVE;
            P.lfree = P.lfix = 0;
            if (pending_init) {
                P.lfix = init_tile;
            } else {
                for (uint32_t j = 0; j < P.nout; ++j) {
                    const uint32_t q = P.ol[j];
                    if (supS[kq] & bit(q)) P.lfree |= 1ull << j;
                    else P.lfix |= ((supB[kq] >> q) & 1ull) << j;
                }
            }
            P.nlive = 1ull << __builtin_popcountll(P.lfree);
        }
        const double tbytes = (double)(1u << TB) * (prec_ == 128 ? 16 : 8);
        double sc = 1.0;
        int nh = 0;
        for (auto &k : G.ops) nh += k.op.kind == H;
        nh -= B.h_absorbed;
        for (int i = 0; i < nh / 2; ++i) sc *= 0.5;
        if (nh & 1) sc *= M_SQRT1_2;
        P.scale_re = sc * G.fr;
        P.scale_im = sc * G.fi;
        if (P.scale_re != 1.0 || P.scale_im != 0.0) P.flags |= F_SCALE;
        const bool last = gi + 1 == groups.size();
        bool want = last && d_sums && B.tile == ((1ull << TB) - 1);
        if (want) P.flags |= F_SUMS;
        // sums only: the caller discards this state right after sampling it (the next transition
        // resets), so the last sweep writes only its block sums; the sampler's chosen tiles are
        // then recomputed and stored by replay_tiles()
        const bool nostore = live_ && want && sums_only && !ctx.dry && !pending_init && !(P.flags & F_LIVE);
        if (nostore) {
            P.flags |= F_NOSTORE;
            P.flags &= ~(uint32_t)F_TSTORE;
            if (P.flags & F_VMASK) {
                // nothing is written, so only the tiles V touches need a visit (the other block sums
                // are zero): a live sweep over V's tiles (T = physical outer bits ^ xin)
                P.lfree = P.lfix = 0;
                uint32_t j = 0;
                for (uint64_t m = P.outer; m; m &= m - 1, ++j) {
                    const uint32_t pos = (uint32_t)__builtin_ctzll(m);
                    if ((P.vfree >> pos) & 1) P.lfree |= 1ull << j;
                    else P.lfix |= (((P.vfix ^ P.xin) >> pos) & 1ull) << j;
                }
                P.nlive = 1ull << __builtin_popcountll(P.lfree);
                P.flags |= F_LIVE;
            }
        }
#ifdef TUSQ_DEBUG_KNOBS   // TUSQ_DBG_NOSTORE=1: the sweeps skip their stores (wrong results; timing only)
        static const bool dbg_nostore = getenv("TUSQ_DBG_NOSTORE") != nullptr;
        if (dbg_nostore) P.flags |= F_DBG_NOSTORE;
#endif
        // F_VMASK: the first sweep reading a buffer that is valid on V only (identity read layout)
        const bool vmask = !pending_init && (vfree_ & all) != all;
        if (vmask) {
            for (int b = 0; b < TB; ++b)
                if (P.pin[b] != P.qs[b])
                    throw std::runtime_error("fused planner: valid-set sweep outside the identity layout");
            P.flags |= F_VMASK;
            P.vfree = vfree_ & all;
            P.vfix = vfix_ & all & ~P.vfree;
            P.vl_mask = P.vl_val = 0;
            for (int b = 0; b < TB; ++b)
                if (!((P.vfree >> P.pin[b]) & 1)) {
                    P.vl_mask |= 1u << b;
                    P.vl_val |= (uint32_t)((P.vfix >> P.pin[b]) & 1) << b;
                }
        }
        // bytes: a reset sweep writes one tile; live sweeps move their tiles; a full sweep on a
        // partly valid buffer reads only the tiles V touches
        double bytes = 2 * s;
        if (pending_init) bytes = live_ ? tbytes : s;
        else if (P.flags & F_LIVE) bytes = 2.0 * (double)P.nlive * tbytes;
        else if (vmask) bytes = s + (double)(1ull << __builtin_popcountll(P.vfree)) * (prec_ == 128 ? 16 : 8);
        if (!ctx.dry) {
            int bps = blocks_per_sm(prec_);
            const uint64_t nt = (P.flags & F_LIVE) ? P.nlive : P.ntiles;
            uint64_t grid = std::min<uint64_t>((nt + NG - 1) / NG, (uint64_t)device_sm_count() * bps);
#ifdef TUSQ_DEBUG_KNOBS   // TUSQ_DBG_GRID=g caps the grid (several tiles per CTA at small n)
            static const uint64_t dbg_grid = getenv("TUSQ_DBG_GRID") ? (uint64_t)atoll(getenv("TUSQ_DBG_GRID")) : 0;
            if (dbg_grid) grid = std::min(grid, dbg_grid);
#endif
            const size_t smem = smem_bytes(prec_);
            // incremental tile bases (deposited steps, read layout) and byte offsets for the kernel
            auto pdep = [&](uint64_t x) {
                uint64_t o = 0;
                for (uint32_t q = 0; q < 64 && x; ++q)
                    if (P.outer & bit(q)) { o |= (x & 1) << q; x >>= 1; }
                return o;
            };
            const uint64_t S = grid * NG;
            P.dstep = pdep(S);
            for (int g = 0; g < NG; ++g) {
                const uint64_t gn = (uint64_t)g + NBUF;
                P.dissue[g] = pdep((gn % NG) + (gn / NG) * S - (uint64_t)g);
            }
            const uint32_t esz = prec_ == 128 ? 16 : 8;
            for (int r = 0; r < NR; ++r) {
                P.gs[r] *= esz;
                P.gj[r] *= esz;
                P.sj[r] = (uint16_t)(P.sj[r] * esz);
                P.so0[r] = (uint16_t)(P.so0[r] * esz);
                P.wreg[r] = (uint16_t)(P.wreg[r] * esz);
            }
            for (uint32_t k = 0; k < P.nphase; ++k)
                for (int r = 0; r < NR; ++r) {
                    P.ph[k].so[r] = (uint16_t)(P.ph[k].so[r] * esz);
                    P.ph[k].so_out[r] = (uint16_t)(P.ph[k].so_out[r] * esz);
                }
            if (ctx.timer) ctx.timer->begin(ctx.st);
            // A reset sweep is ONE CTA computing the tile that holds the basis state (F_LIVE,
            // nlive = 1); the rest of the buffer is not written -- the valid set V shrinks to that
            // tile (the zeros outside V are only written by finish(), once per call).  Without
            // live tiles (TUSQ_EXEC_NO_LIVE) K7 writes the zeros first and V stays everything.
            if (pending_init && !live_) launch_init_basis(dst, n_, prec_, 0, 0.0, 0.0, ctx.st);
            // live-tile sweeps write the sums of their live tiles only: the others are zero
            if ((P.flags & F_LIVE) && want && !(nostore && src == dst) &&
                cudaMemsetAsync(d_sums, 0, (size_t)P.ntiles * sizeof(double), ctx.st) != cudaSuccess)
                throw std::runtime_error("cudaMemsetAsync (block sums) failed");
            if (nostore && src == dst) {
                // The group's gates act inside tiles, and tile {0..11} is the sampler's block: each
                // block's |amp|^2 sum is the same before and after the group (a unitary on the
                // block; outer qubits enter only as controls).  In place and in the identity
                // layout the block keeps its physical index, so the sums are those of the INPUT:
                // one read of the valid set, no K5 sweep (its chosen tiles are replayed later).
                const uint64_t vf = (P.flags & F_VMASK) ? P.vfree : ~0ull, vx = (P.flags & F_VMASK) ? P.vfix : 0;
                launch_block_sums(src, n_, prec_, TB, d_sums, ctx.st, vf, vx);
            } else if (prec_ == 128)
                k_fused<double><<<(unsigned)grid, NT * NG, smem, ctx.st>>>((const double2 *)src, (double2 *)dst, P,
                                                                           d_sums);
            else
                k_fused<float><<<(unsigned)grid, NT * NG, smem, ctx.st>>>((const float2 *)src, (float2 *)dst, P,
                                                                          d_sums);
            if (ctx.timer)
                ctx.timer->end(ctx.st, nostore ? bytes - s : bytes, (P.flags & (F_LIVE | F_VMASK | F_INIT | F_NOSTORE)) ? 0 : 2);
            if (nostore) {
                scratch_->replay = P;
                scratch_->rsrc = src;
                scratch_->rdst = dst;
                pending_tiles_ = true;
            }
#ifdef TUSQ_DEBUG_KNOBS   // TUSQ_DBG_TRACE=1: one line per K5 launch (group shape), for launch-time fits
            static const bool dbg_trace = getenv("TUSQ_DBG_TRACE") != nullptr;
            if (dbg_trace) {
                int cnt[10] = {0};   // H, DK, CX-like, D, XPOSE, XY, T-pred, other, CU, CCX
                for (uint32_t i = 0; i < P.ngate; ++i) {
                    const uint16_t c = P.g[i].code;
                    const int k = c < C_U ? 0 : ((c >= C_DK && c < C_CX2) || (c >= C_DKC && c < C_N)) ? 1
                                : ((c >= C_CX && c < C_CPH) || (c >= C_CX2 && c < C_CU)) ? 2
                                : (c >= C_D1 && c < C_CX) ? 3 : c == C_XPOSE ? 4 : (c >= C_X && c < C_D1) ? 5
                                : ((c >= C_TX && c <= C_TPH) || (c >= C_TDK && c < C_DKC)) ? 6
                                : (c >= C_CU && c < C_CCX) ? 8 : (c >= C_CCX && c < C_TDK) ? 9 : 7;
                    cnt[k]++;
                }
                int contig = 1;
                for (int b = 0; b < TB; ++b) contig &= P.pin[b] == b;
                fprintf(stderr, "[k5] idx %d ops %zu recs %u ph %u init %d contig %d oop %d gtab %d nlive %llu vmask %d ns %d tile %#llx H %d DK %d CX %d D %d XP %d XY %d TP %d O %d CU %d CCX %d\n",
                        ctx.timer ? (int)ctx.timer->pending() - 1 : -1, G.ops.size(), P.ngate, P.nphase, pending_init ? 1 : 0, contig, src != dst ? 1 : 0,
                        P.gtab != 0xFFFFu, (unsigned long long)((P.flags & F_LIVE) ? P.nlive : P.ntiles), (P.flags & F_VMASK) ? 1 : 0, (P.flags & F_NOSTORE) ? 1 : 0, (unsigned long long)B.tile, cnt[0], cnt[1], cnt[2], cnt[3], cnt[4], cnt[5],
                        cnt[6], cnt[7], cnt[8], cnt[9]);
            }
#endif
        }
        count(ctx, nostore ? (bytes - s) : bytes, true);   // (a sums-only sweep reads, writes nothing)
        pending_init = false;
        // the valid set after this sweep: a live sweep (in place, identity layout) wrote its live
        // tiles whole; any other sweep wrote every tile
        if (P.flags & F_NOSTORE) {
            // nothing written: the buffer still holds this group's input (and will be mixed with
            // the replayed tiles); only a reset may follow (stale_)
        } else if ((P.flags & F_LIVE) && live_) {
            uint64_t tpos = 0;
            for (int b = 0; b < TB; ++b) tpos |= bit(P.pin[b]);
            vfree_ = tpos | pdep_mask(P.lfree, P.outer);
            vfix_ = (pdep_mask(P.lfix, P.outer) ^ P.xin) & ~vfree_ & all;
        } else {
            vfree_ = ~0ull;
            vfix_ = 0;
        }
        xmask_ = P.xm_store ^ G.xa;
        if (want && sums_written) *sums_written = true;
    }
    if (cur != ctx.psi) throw std::runtime_error("fused planner: layout parity left the state in the scratch buffer");
    // what the buffer may hold from now on: the final support if every sweep was a live one
    if (track) {   // the support analysis holds whatever the sweeps were
        dfree_ = sup_end;
        dfix_ = (bx_end ^ xmask_) & ~sup_end & all;
    } else {
        dfree_ = ~0ull;
        dfix_ = 0;
    }
    return true;
}

void FusedPlanner::materialize(Ctx &ctx)
{
    if (!xmask_) return;
    dfix_ ^= xmask_ & ~dfree_;   // the XOR moves the known support and the valid set with the state
    vfix_ ^= xmask_ & ~vfree_;
    double b = 0;
    if (!ctx.dry) b = launch_pauli_string(ctx.psi, n_, prec_, xmask_, 0, ctx.st);
    else b = 2.0 * (double)(1ull << n_) * (prec_ == 128 ? 16 : 8);
    count(ctx, b, false);
    xmask_ = 0;
}

void FusedPlanner::close_blocks(Ctx &ctx, uint32_t block_bits)
{
    const uint64_t all = n_ >= 64 ? ~0ull : (1ull << n_) - 1, low = (1ull << block_bits) - 1;
    if ((vfree_ & all) == all || (vfree_ & low) == low) return;
    // zeros in the blocks V touches, at the elements outside V; V becomes those whole blocks
    const uint64_t sf = (vfree_ & all) | low;
    double b = 0;
    if (!ctx.dry) b = launch_zero_outside(ctx.psi, n_, prec_, sf, vfix_ & all & ~sf, vfree_ & all, vfix_ & all & ~vfree_, ctx.st);
    else b = (double)(1ull << __builtin_popcountll(sf)) * (prec_ == 128 ? 16 : 8);
    count(ctx, b, false);
    vfree_ = sf;
    vfix_ &= ~sf;
}

void FusedPlanner::finish(Ctx &ctx)
{
    if (stale_ || pending_tiles_) throw std::runtime_error("fused planner: the call ended on a state that was not stored");
    const uint64_t all = n_ >= 64 ? ~0ull : (1ull << n_) - 1;
    if ((vfree_ & all) == all) return;
    double b = 0;
    if (!ctx.dry) b = launch_zero_outside(ctx.psi, n_, prec_, all, 0, vfree_ & all, vfix_ & all & ~vfree_, ctx.st);
    else b = (double)(1ull << n_) * (prec_ == 128 ? 16 : 8);
    count(ctx, b, false);
    vfree_ = ~0ull;
    vfix_ = 0;
}

void FusedPlanner::replay_tiles(Ctx &ctx, const uint64_t *d_blist, uint64_t n, uint64_t mh)
{
    if (!pending_tiles_) return;
    pending_tiles_ = false;
    stale_ = true;   // the buffer now mixes the group's input and the replayed tiles
    if (!n) return;
    Params &P = scratch_->replay;
    P.flags = (P.flags & ~(uint32_t)(F_NOSTORE | F_SUMS | F_LIVE | F_TSTORE)) | F_TLIST;
    P.tlist = d_blist;
    P.nlist = n;
    P.tl_xor = mh ^ (P.xout >> TB);   // logical block b of the sampler -> tile index (tile {0..11})
    const uint64_t grid = std::min<uint64_t>((n + NG - 1) / NG, (uint64_t)device_sm_count() * blocks_per_sm(prec_));
    const size_t smem = smem_bytes(prec_);
    if (prec_ == 128)
        k_fused<double><<<(unsigned)grid, NT * NG, smem, ctx.st>>>((const double2 *)scratch_->rsrc,
                                                                   (double2 *)scratch_->rdst, P, nullptr);
    else
        k_fused<float><<<(unsigned)grid, NT * NG, smem, ctx.st>>>((const float2 *)scratch_->rsrc,
                                                                  (float2 *)scratch_->rdst, P, nullptr);
    ctx.stats->launches++;
    ctx.stats->fused_launches++;
    ctx.stats->hbm_bytes += 2.0 * (double)n * (double)(1u << TB) * (prec_ == 128 ? 16 : 8);
#ifdef TUSQ_DEBUG_KNOBS   // keep the launch trace aligned with the k_fused launch sequence
    static const bool dbg_trace = getenv("TUSQ_DBG_TRACE") != nullptr;
    if (dbg_trace) fprintf(stderr, "[k5r] replay %llu tiles\n", (unsigned long long)n);
#endif
}

}  // namespace tq
