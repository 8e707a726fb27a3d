// Internal declarations shared by the library's host and device translation units.
// (The oracle in oracle/ is a separate program; nothing here is shared with it.)
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tusq.h"

#if defined(__CUDACC__)
#define TQ_HD __host__ __device__ __forceinline__
#else
#define TQ_HD inline
#endif

namespace tq {

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based generator (Salmon et al. SC'11) with curand's constants; one
// implementation for host (ECM sampling, pruning draws) and device (shot draws).
struct U4 { uint32_t x, y, z, w; };

TQ_HD uint32_t mulhi32(uint32_t a, uint32_t b, uint32_t *lo)
{
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *lo = (uint32_t)p;
    return (uint32_t)(p >> 32);
}

TQ_HD U4 philox10(U4 c, uint32_t k0, uint32_t k1)
{
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0, lo1;
        uint32_t hi0 = mulhi32(0xD2511F53u, c.x, &lo0);
        uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z, &lo1);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Stream tags (third/fourth counter word) -- DESIGN.md reading #9.
constexpr uint32_t TAG_ER = 0x45520000u;      // "ER"  error-realization draws
constexpr uint32_t TAG_PRUNE = 0x50520000u;   // "PR"  pruning selection draws
constexpr uint32_t TAG_SHOT = 0x53000000u;    // "S"   leaf shot draws

// ---------------------------------------------------------------- gates / Paulis
enum Kind : uint32_t { I = 0, X, Y, Z, H, S, SDG, T, TDG, RX, RY, RZ, P, CX, CZ, CP, NKINDS };
TQ_HD bool two_qubit(uint32_t k) { return k == CX || k == CZ || k == CP; }
TQ_HD bool is_diag1(uint32_t k) { return k == Z || k == S || k == SDG || k == T || k == TDG || k == RZ || k == P || k == I; }

// An op of an executed stream: a circuit gate or a frozen Pauli, possibly inverted.
struct Op {
    uint32_t kind;   // Kind (X/Y/Z also used for frozen Paulis)
    uint32_t q0, q1; // q0 = control for 2q gates
    double theta;    // already sign-flipped when inverted
};

// Inverse of a gate (H, Paulis, CX, CZ self-inverse; T<->Tdg, S<->Sdg; R(t) -> R(-t)).
inline Op inverse_op(const Op &o)
{
    Op r = o;
    switch (o.kind) {
    case S: r.kind = SDG; break;
    case SDG: r.kind = S; break;
    case T: r.kind = TDG; break;
    case TDG: r.kind = T; break;
    case RX: case RY: case RZ: case P: case CP: r.theta = -o.theta; break;
    default: break;
    }
    return r;
}

// Canonical triple: Pauli p on qubit q right before gate pos (pos = L: terminal).
struct Triple { uint32_t pos, q, p; };

struct Leaf {
    std::vector<Triple> tr;
    uint64_t count = 0, offset = 0;
};

// The executed part of a leaf: its triples before the readout (pos < L), and the readout flips
// (terminal X triples at pos = L) as a bit mask.  Measurement noise is a classical flip of the
// drawn bitstring (reading #7): leaves that differ only in terminal
// flips share one state vector and one CDF.
inline Leaf core_of(const Leaf &l, uint32_t L, uint64_t *tmask)
{
    Leaf c;
    c.count = l.count;
    c.offset = l.offset;
    uint64_t m = 0;
    for (const Triple &x : l.tr) {
        if (x.pos < L) c.tr.push_back(x);
        else if (x.p == 1 || x.p == 2) m ^= 1ull << x.q;   // terminal X (Y reads as X; Z never emitted)
    }
    if (tmask) *tmask = m;
    return c;
}

inline bool same_core(const Leaf &a, const Leaf &b)
{
    if (a.tr.size() != b.tr.size()) return false;
    for (size_t i = 0; i < a.tr.size(); ++i)
        if (a.tr[i].pos != b.tr[i].pos || a.tr[i].q != b.tr[i].q || a.tr[i].p != b.tr[i].p) return false;
    return true;
}

}  // namespace tq

struct tusq_tree {
    uint32_t n = 0;
    std::vector<tq::Op> gates;        // the circuit, length L
    uint64_t shots = 0, seed = 0;
    uint64_t S2 = 0, S3 = 0, p0 = 0, n_sig = 0, n_insig = 0, n_selected = 0, n_sites = 0;
    std::vector<tq::Leaf> leaves;     // DFS order after pruning
};

namespace tq {
// error reporting (thread-local message)
void set_error(const std::string &msg);
tusq_status fail(tusq_status st, const std::string &msg);

// ECM + tree (ecm.cpp)
tusq_status build_tree(uint32_t n, const tusq_op *ops, uint64_t L, const tusq_noise &noise, uint64_t shots,
                       uint64_t seed, const tusq_prune &prune, tusq_tree **out);

// Event streams (plan.cpp)
// length of the common event prefix of two leaves and the event sequence of a leaf suffix
struct Cursor { uint64_t pos; uint32_t tri; };   // events before: gates [0,pos), triples [0,tri)
Cursor common_prefix(const tusq_tree &t, const Leaf &a, const Leaf &b);
uint64_t suffix_len(const tusq_tree &t, const Leaf &a, const Cursor &c);   // events after the cursor
void append_forward(const tusq_tree &t, const Leaf &a, const Cursor &from, std::vector<Op> &out);
void append_inverse(const tusq_tree &t, const Leaf &a, const Cursor &to, std::vector<Op> &out);
// classical basis-state prefix of a leaf from |0..0>: returns the cursor after it, and the basis
// index and amplitude it produces
Cursor fold_prefix(const tusq_tree &t, const Leaf &a, uint64_t *index, double *re, double *im);
void tree_info(const tusq_tree &t, tusq_tree_info *out);
}  // namespace tq
