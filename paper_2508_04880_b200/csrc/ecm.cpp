// Error Characterization Module + TEM tree build (host, integer-only, deterministic).
//
//   noise sites + integer thresholds   PAPER.md P:178; readings #1-#4
//   ER sampling (Philox, per shot x site, multi-threaded over shots)   P:178-182; reading #9
//   ER tallying (hash of the sparse ER)                                P:177-182, Fig. P:163
//   ER commutation as a single-pass Pauli FRAME propagation            P:197-224, rules 1-6
//       (symplectic (x, z) bits per qubit; equivalent to the paper's per-qubit stacks)
//   pruning (alpha, beta; Philox selection)                            P:336-340; reading #10
//   DFS leaf order, shot offsets                                       P:312-316; reading #12
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <unordered_map>

#include "common.h"

namespace tq {
namespace {

struct Site {
    uint32_t pos, q;
    uint64_t cI, cX, cY;   // cumulative thresholds: I below cI, X below cX, Y below cY, else Z
};

uint64_t round_u32(double p) { return (uint64_t)std::llround(p * 4294967296.0); }

// The (pX, pY, pZ) channel of each site class: depolarizing p -> (p/3, p/3, p/3), bit flip p ->
// (p, 0, 0) (readings #2, #4), or the caller's general Pauli channels (TUSQ_NOISE_PAULI, Eq. 2).
struct Chan { double x, y, z; };

static void channels(const tusq_noise &nz, Chan &c1, Chan &c2, Chan &cm)
{
    if (nz.flags & TUSQ_NOISE_PAULI) {
        c1 = Chan{nz.pauli1[0], nz.pauli1[1], nz.pauli1[2]};
        c2 = Chan{nz.pauli2[0], nz.pauli2[1], nz.pauli2[2]};
        cm = Chan{nz.pauli_meas[0], nz.pauli_meas[1], nz.pauli_meas[2]};
    } else {
        c1 = Chan{nz.p1 / 3.0, nz.p1 / 3.0, nz.p1 / 3.0};
        c2 = Chan{nz.p2 / 3.0, nz.p2 / 3.0, nz.p2 / 3.0};
        cm = Chan{nz.p_meas, 0.0, 0.0};
    }
}

std::vector<Site> make_sites(uint32_t n, const std::vector<Op> &g, const tusq_noise &nz)
{
    std::vector<Site> s;
    Chan c1, c2, cm;
    channels(nz, c1, c2, cm);
    auto live = [](const Chan &c) { return c.x > 0 || c.y > 0 || c.z > 0; };   // reading #21
    auto add = [&](uint32_t pos, uint32_t q, const Chan &c) {
        const uint64_t one = 4294967296ull;
        uint64_t tX = std::min(round_u32(c.x), one), tY = round_u32(c.y), tZ = round_u32(c.z);
        // rounding may push a channel that sums to 1 past 2^32: the excess comes off Y, then Z
        // (reading #9); tI = 0 then
        if (tX + tY > one) tY = one - tX;
        if (tX + tY + tZ > one) tZ = one - tX - tY;
        const uint64_t tI = one - (tX + tY + tZ);
        s.push_back(Site{pos, q, tI, tI + tX, tI + tX + tY});
    };
    for (uint32_t pos = 0; pos < g.size(); ++pos) {
        if (two_qubit(g[pos].kind)) {
            if (live(c2)) { add(pos, g[pos].q0, c2); add(pos, g[pos].q1, c2); }
        } else if (live(c1)) {
            add(pos, g[pos].q0, c1);
        }
    }
    if (live(cm))
        for (uint32_t q = 0; q < n; ++q) add((uint32_t)g.size(), q, cm);
    return s;
}

// sparse ER entry: site index << 2 | pauli
using ErKey = std::vector<uint32_t>;

struct VecHash {
    size_t operator()(const std::vector<uint32_t> &v) const noexcept
    {
        uint64_t h = 0xcbf29ce484222325ull ^ v.size();
        for (uint32_t x : v) { h ^= x; h *= 0x100000001b3ull; h ^= h >> 29; }
        return (size_t)h;
    }
};

// Pauli <-> symplectic bits: I=(0,0) X=(1,0) Y=(1,1) Z=(0,1)
inline uint8_t xbit(uint32_t p) { return (p == 1 || p == 2) ? 1 : 0; }
inline uint8_t zbit(uint32_t p) { return (p == 2 || p == 3) ? 1 : 0; }
inline uint32_t pauli_of(uint8_t x, uint8_t z) { return x ? (z ? 2u : 1u) : (z ? 3u : 0u); }

// Canonical form by Pauli-frame propagation from the first error position.
// frame x[q], z[q]; a gate either conjugates the frame (Clifford rules) or freezes
// the non-commuting part of one qubit's frame right before itself.
void canonicalize(uint32_t n, const std::vector<Op> &g, const std::vector<Site> &sites, const ErKey &er,
                  std::vector<uint8_t> &fx, std::vector<uint8_t> &fz, std::vector<uint32_t> &out)
{
    out.clear();
    if (er.empty()) return;
    const uint32_t L = (uint32_t)g.size();
    std::fill(fx.begin(), fx.end(), 0);
    std::fill(fz.begin(), fz.end(), 0);
    size_t k = 0;
    uint32_t start = sites[er[0] >> 2].pos;
    auto freeze = [&](uint32_t pos, uint32_t q) {
        out.push_back(pos); out.push_back(q); out.push_back(pauli_of(fx[q], fz[q]));
        fx[q] = 0; fz[q] = 0;
    };
    for (uint32_t pos = start; pos <= L; ++pos) {
        if (pos < L && pos > start) {      // the gate at `start` precedes the first error
            const Op &o = g[pos];
            uint32_t a = o.q0, b = o.q1;
            switch (o.kind) {
            case CX:            // rules 4-6: x_t ^= x_c, z_c ^= z_t
                fx[b] ^= fx[a];
                fz[a] ^= fz[b];
                break;
            case H:             // X <-> Z
                std::swap(fx[a], fz[a]);
                break;
            case I: case X: case Y: case Z:   // rule 2
                break;
            case S: case SDG: case T: case TDG: case RZ: case P:   // rule 3 (Z axis)
                if (fx[a]) freeze(pos, a);
                break;
            case RX:            // X passes; Y, Z frozen
                if (fz[a]) freeze(pos, a);
                break;
            case RY:            // Y passes; X, Z frozen
                if (fx[a] != fz[a]) freeze(pos, a);
                break;
            case CZ: case CP:   // per qubit: Z passes, X/Y frozen
                if (fx[a]) freeze(pos, a);
                if (fx[b]) freeze(pos, b);
                break;
            default: break;
            }
        }
        // rule 1: merge the noise of this position into the frame
        while (k < er.size() && sites[er[k] >> 2].pos == pos) {
            const Site &s = sites[er[k] >> 2];
            uint32_t p = er[k] & 3u;
            fx[s.q] ^= xbit(p);
            fz[s.q] ^= zbit(p);
            ++k;
        }
    }
    // terminal: Z dropped before readout, X/Y read as a flip (reading #7)
    for (uint32_t q = 0; q < n; ++q)
        if (fx[q]) { out.push_back(L); out.push_back(q); out.push_back(1u); }
    // sort triples by (pos, q)
    size_t m = out.size() / 3;
    std::vector<Triple> tmp(m);
    for (size_t i = 0; i < m; ++i) tmp[i] = Triple{out[3 * i], out[3 * i + 1], out[3 * i + 2]};
    std::sort(tmp.begin(), tmp.end(), [](const Triple &x, const Triple &y) {
        return x.pos != y.pos ? x.pos < y.pos : x.q < y.q;
    });
    for (size_t i = 0; i < m; ++i) { out[3 * i] = tmp[i].pos; out[3 * i + 1] = tmp[i].q; out[3 * i + 2] = tmp[i].p; }
}

// DFS order over slots (pos, q), children I < X < Y < Z (reading #12)
bool dfs_less(const std::vector<Triple> &a, const std::vector<Triple> &b)
{
    size_t m = std::min(a.size(), b.size());
    for (size_t j = 0; j < m; ++j) {
        const Triple &x = a[j], &y = b[j];
        if (x.pos != y.pos || x.q != y.q) {
            bool x_earlier = x.pos != y.pos ? x.pos < y.pos : x.q < y.q;
            return !x_earlier;   // the key with a Pauli at the earlier slot has I there in the other
        }
        if (x.p != y.p) return x.p < y.p;
    }
    return a.size() < b.size();
}

}  // namespace

tusq_status build_tree(uint32_t n, const tusq_op *ops, uint64_t L, const tusq_noise &nz, uint64_t shots,
                       uint64_t seed, const tusq_prune &pr, tusq_tree **out)
{
    auto t = new tusq_tree();
    t->n = n;
    t->shots = shots;
    t->seed = seed;
    t->gates.resize(L);
    for (uint64_t i = 0; i < L; ++i) t->gates[i] = Op{ops[i].kind, ops[i].q0, ops[i].q1, ops[i].theta};
    const std::vector<Site> sites = make_sites(n, t->gates, nz);
    const uint64_t M = sites.size();
    t->n_sites = M;
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);

    // ---- ER sampling: each shot independently, threads over shot ranges
    std::vector<ErKey> ers(shots);
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (shots * M < 200000) nth = 1;
    auto sample_range = [&](uint64_t s0, uint64_t s1) {
        for (uint64_t s = s0; s < s1; ++s) {
            ErKey &e = ers[s];
            for (uint64_t i4 = 0; i4 < M; i4 += 4) {
                U4 w = philox10(U4{(uint32_t)(i4 >> 2), (uint32_t)s, (uint32_t)(s >> 32), TAG_ER}, k0, k1);
                uint32_t ws[4] = {w.x, w.y, w.z, w.w};
                for (uint64_t i = i4; i < std::min(M, i4 + 4); ++i) {
                    uint64_t x = ws[i & 3];
                    const Site &st = sites[i];
                    if (x < st.cI) continue;
                    uint32_t p = x < st.cX ? 1u : x < st.cY ? 2u : 3u;
                    e.push_back((uint32_t)(i << 2) | p);
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        uint64_t chunk = (shots + nth - 1) / nth;
        for (unsigned j = 0; j < nth; ++j) {
            uint64_t s0 = j * chunk, s1 = std::min(shots, s0 + chunk);
            if (s0 < s1) th.emplace_back(sample_range, s0, s1);
        }
        for (auto &x : th) x.join();
    }

    // ---- tallying
    std::unordered_map<ErKey, uint64_t, VecHash> tally;
    tally.reserve(shots * 2);
    for (auto &e : ers) tally[e] += 1;
    t->S2 = tally.size();
    ers.clear();
    ers.shrink_to_fit();

    // ---- commutation + merge
    std::unordered_map<std::vector<uint32_t>, uint64_t, VecHash> canon;
    canon.reserve(tally.size() * 2);
    {
        std::vector<uint8_t> fx(n), fz(n);
        std::vector<uint32_t> key;
        for (auto &kv : tally) {
            canonicalize(n, t->gates, sites, kv.first, fx, fz, key);
            canon[key] += kv.second;
        }
    }
    t->S3 = canon.size();

    // ---- DFS order
    std::vector<Leaf> all;
    all.reserve(canon.size());
    for (auto &kv : canon) {
        Leaf l;
        size_t m = kv.first.size() / 3;
        l.tr.resize(m);
        for (size_t i = 0; i < m; ++i) l.tr[i] = Triple{kv.first[3 * i], kv.first[3 * i + 1], kv.first[3 * i + 2]};
        l.count = kv.second;
        all.push_back(std::move(l));
    }
    std::sort(all.begin(), all.end(), [](const Leaf &a, const Leaf &b) { return dfs_less(a.tr, b.tr); });

    // ---- pruning
    uint64_t p0 = 0;
    for (auto &l : all) p0 = std::max(p0, l.count);
    t->p0 = p0;
    std::vector<int> cls(all.size(), 1);  // 0 pruned, 1 significant, 2 kept insignificant
    uint64_t p_insig = 0, n_insig = 0;
    if (pr.enabled) {
        for (size_t i = 0; i < all.size(); ++i) {
            unsigned __int128 lhs = (unsigned __int128)all[i].count * pr.alpha_den;
            unsigned __int128 rhs = (unsigned __int128)pr.alpha_num * p0;
            if (lhs < rhs) { cls[i] = 2; p_insig += all[i].count; ++n_insig; }
        }
    }
    t->n_insig = n_insig;
    t->n_sig = all.size() - n_insig;
    t->n_selected = n_insig;
    if (pr.enabled && n_insig > pr.beta) {
        // insignificant leaves in DFS order with a Fenwick-free linear walk (beta draws)
        std::vector<size_t> idx;
        for (size_t i = 0; i < all.size(); ++i) if (cls[i] == 2) idx.push_back(i);
        std::vector<uint8_t> taken(idx.size(), 0);
        uint64_t w_rem = p_insig;
        for (uint32_t j = 0; j < pr.beta; ++j) {
            U4 w = philox10(U4{j, 0u, 0u, TAG_PRUNE}, k0, k1);
            uint64_t r = ((uint64_t)w.x | ((uint64_t)w.y << 32)) % w_rem;
            uint64_t cum = 0;
            for (size_t u = 0; u < idx.size(); ++u) {
                if (taken[u]) continue;
                cum += all[idx[u]].count;
                if (cum > r) { taken[u] = 1; w_rem -= all[idx[u]].count; break; }
            }
        }
        uint64_t wk = 0;
        for (size_t u = 0; u < idx.size(); ++u) if (taken[u]) wk += all[idx[u]].count;
        uint64_t assigned = 0;
        size_t best = SIZE_MAX;
        std::vector<uint64_t> scaled(all.size(), 0);
        for (size_t u = 0; u < idx.size(); ++u) {
            size_t i = idx[u];
            if (!taken[u]) { cls[i] = 0; continue; }
            scaled[i] = (uint64_t)(((unsigned __int128)p_insig * all[i].count) / wk);
            assigned += scaled[i];
            if (best == SIZE_MAX || all[i].count > all[best].count) best = i;
        }
        scaled[best] += p_insig - assigned;
        for (size_t u = 0; u < idx.size(); ++u) if (taken[u]) all[idx[u]].count = scaled[idx[u]];
        t->n_selected = pr.beta;
    }
    uint64_t off = 0;
    for (size_t i = 0; i < all.size(); ++i) {
        if (cls[i] == 0) continue;
        all[i].offset = off;
        off += all[i].count;
        t->leaves.push_back(std::move(all[i]));
    }
    if (off != shots) {
        delete t;
        return fail(TUSQ_ERR_INTERNAL, "shot conservation violated in pruning");
    }
    *out = t;
    return TUSQ_OK;
}

}  // namespace tq
