// TEM scheduling on the host: leaf event streams, DFS transitions, classical-prefix folding,
// tree statistics and the multi-GPU leaf partition.
//
// A leaf's event stream ("edges represent gates") is, for pos = 0..L:
//   its frozen Paulis at pos (ascending qubit), then gate pos (pos < L).
// Consecutive DFS leaves share the events before their first differing slot; the
// transition uncomputes the previous leaf's remaining events with inverse gates in
// reverse order and applies the next leaf's remaining events forward (Fig. P:204).
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "common.h"

namespace tq {

static inline bool slot_less(const Triple &a, const Triple &b)
{
    return a.pos != b.pos ? a.pos < b.pos : a.q < b.q;
}

Cursor common_prefix(const tusq_tree &t, const Leaf &a, const Leaf &b)
{
    size_t j = 0, m = std::min(a.tr.size(), b.tr.size());
    while (j < m && a.tr[j].pos == b.tr[j].pos && a.tr[j].q == b.tr[j].q && a.tr[j].p == b.tr[j].p) ++j;
    const Triple *d = nullptr;
    if (j < a.tr.size() && j < b.tr.size()) d = slot_less(a.tr[j], b.tr[j]) ? &a.tr[j] : &b.tr[j];
    else if (j < a.tr.size()) d = &a.tr[j];
    else if (j < b.tr.size()) d = &b.tr[j];
    if (!d) return Cursor{(uint64_t)t.gates.size() + 1, (uint32_t)j};   // identical streams
    return Cursor{d->pos, (uint32_t)j};
}

uint64_t suffix_len(const tusq_tree &t, const Leaf &a, const Cursor &c)
{
    uint64_t L = t.gates.size();
    uint64_t g = c.pos < L ? L - c.pos : 0;
    return g + (a.tr.size() - std::min<size_t>(a.tr.size(), c.tri));
}

static inline Op pauli_op(const Triple &tr) { return Op{tr.p, tr.q, 0u, 0.0}; }

void append_forward(const tusq_tree &t, const Leaf &a, const Cursor &from, std::vector<Op> &out)
{
    const uint64_t L = t.gates.size();
    size_t k = from.tri;
    for (uint64_t pos = from.pos; pos <= L; ++pos) {
        while (k < a.tr.size() && a.tr[k].pos == pos) out.push_back(pauli_op(a.tr[k++]));
        if (pos < L) out.push_back(t.gates[pos]);
    }
}

void append_inverse(const tusq_tree &t, const Leaf &a, const Cursor &to, std::vector<Op> &out)
{
    const uint64_t L = t.gates.size();
    if (to.pos > L) return;
    int64_t k = (int64_t)a.tr.size() - 1;
    for (int64_t pos = (int64_t)L; pos >= (int64_t)to.pos; --pos) {
        if (pos < (int64_t)L) out.push_back(inverse_op(t.gates[pos]));
        while (k >= (int64_t)to.tri && a.tr[k].pos == (uint64_t)pos) out.push_back(pauli_op(a.tr[k--]));
    }
}

// Longest prefix of a leaf's event stream whose result from |0..0> is a single basis state times a
// phase, computed exactly on the host (the re-anchor target):
//   - classical events: X, Y, Z, CX, and diagonal gates act on a basis state as a permutation and
//     a phase;
//   - blocks H(t) [classical events] H(t) -- e.g. the 15-gate Toffoli of a Cuccaro adder with its
//     frozen Paulis -- are simulated on their few-entry support: when the block maps the current
//     basis state to a single basis state (every other amplitude below 1e-13, i.e. rounding
//     residue of an exact cancellation), the fold continues past it.  A Pauli error inside a core
//     usually leaves it a superposition: the fold stops before that block's first H.
// The device then starts from amp |index> at the returned cursor instead of replaying the prefix.
Cursor fold_prefix(const tusq_tree &t, const Leaf &a, uint64_t *index, double *re, double *im)
{
    using C = std::complex<double>;
    const uint64_t L = t.gates.size();
    const C iu(0.0, 1.0);
    // apply one classical event (a gate or a Pauli) to a sparse state; false if not classical
    auto classical = [&](const Op &o, std::vector<std::pair<uint64_t, C>> &v) -> bool {
        for (auto &e : v) {
            uint64_t &x = e.first;
            C &amp = e.second;
            const uint64_t b0 = (x >> o.q0) & 1, b1 = (x >> o.q1) & 1;
            switch (o.kind) {
            case I: break;
            case X: x ^= 1ull << o.q0; break;
            case Y: amp *= b0 ? -iu : iu; x ^= 1ull << o.q0; break;
            case Z: if (b0) amp = -amp; break;
            case S: if (b0) amp *= iu; break;
            case SDG: if (b0) amp *= -iu; break;
            case T: if (b0) amp *= C(M_SQRT1_2, M_SQRT1_2); break;
            case TDG: if (b0) amp *= C(M_SQRT1_2, -M_SQRT1_2); break;
            case RZ: amp *= std::exp(iu * (b0 ? 0.5 : -0.5) * o.theta); break;
            case P: if (b0) amp *= std::exp(iu * o.theta); break;
            case CX: if (b0) x ^= 1ull << o.q1; break;
            case CZ: if (b0 && b1) amp = -amp; break;
            case CP: if (b0 && b1) amp *= std::exp(iu * o.theta); break;
            default: return false;
            }
        }
        return true;
    };
    auto hadamard = [&](uint32_t q, std::vector<std::pair<uint64_t, C>> &v) {
        std::vector<std::pair<uint64_t, C>> out;
        for (auto &e : v) {
            const uint64_t x0 = e.first & ~(1ull << q), x1 = x0 | (1ull << q);
            const double sgn = ((e.first >> q) & 1) ? -1.0 : 1.0;
            out.push_back({x0, e.second * M_SQRT1_2});
            out.push_back({x1, e.second * (sgn * M_SQRT1_2)});
        }
        std::sort(out.begin(), out.end(), [](const auto &p, const auto &q2) { return p.first < q2.first; });
        v.clear();
        for (auto &e : out) {
            if (!v.empty() && v.back().first == e.first) v.back().second += e.second;
            else v.push_back(e);
        }
    };
    std::vector<std::pair<uint64_t, C>> st{{0, C(1.0, 0.0)}};
    size_t k = 0;
    uint64_t pos = 0;
    auto pauli = [&](const Triple &tr) { return Op{tr.p, tr.q, 0u, 0.0}; };
    for (; pos <= L; ++pos) {
        while (k < a.tr.size() && a.tr[k].pos == pos) { classical(pauli(a.tr[k]), st); ++k; }
        if (pos == L) break;
        const Op &o = t.gates[pos];
        if (classical(o, st)) continue;
        if (o.kind != H) break;
        // a block H(q) ... H(q): classical events in between, on a copy of the state
        const uint32_t q = o.q0;
        uint64_t e = pos + 1;
        size_t ke = k;
        std::vector<std::pair<uint64_t, C>> w = st;
        hadamard(q, w);
        bool ok = false;
        for (; e < L; ++e) {
            while (ke < a.tr.size() && a.tr[ke].pos == e) { classical(pauli(a.tr[ke]), w); ++ke; }
            const Op &g = t.gates[e];
            if (g.kind == H && g.q0 == q) { hadamard(q, w); ok = true; break; }
            if (!classical(g, w)) break;
        }
        if (!ok) break;
        std::vector<std::pair<uint64_t, C>> keep;
        for (auto &x : w)
            if (std::abs(x.second) > 1e-13) keep.push_back(x);
        if (keep.size() != 1) break;   // the block leaves a superposition: stop before its first H
        st = keep;
        pos = e;                        // gate e (the closing H) is done; triples at e applied
        k = ke;
    }
    *index = st[0].first;
    *re = st[0].second.real();
    *im = st[0].second.imag();
    return Cursor{pos, (uint32_t)k};
}

void tree_info(const tusq_tree &t, tusq_tree_info *o)
{
    *o = tusq_tree_info{};
    o->S1 = t.shots; o->S2 = t.S2; o->S3 = t.S3; o->p0 = t.p0; o->n_sig = t.n_sig; o->n_insig = t.n_insig;
    o->n_selected = t.n_selected; o->n_leaves = t.leaves.size(); o->n_sites = t.n_sites; o->n_ops = t.gates.size();
    uint64_t edges = 0, inv = 0, naive = 0;
    for (size_t i = 0; i < t.leaves.size(); ++i) {
        const Leaf &l = t.leaves[i];
        uint64_t len = t.gates.size() + l.tr.size();
        naive += len;
        if (i == 0) { edges += len; continue; }
        Cursor c = common_prefix(t, t.leaves[i - 1], l);
        edges += suffix_len(t, l, c);
        inv += suffix_len(t, t.leaves[i - 1], c);
    }
    o->edges = edges;
    o->dftt_ops = edges + inv;
    o->naive_ops = naive;
}

}  // namespace tq
