/*
 * oracle/tusq_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the TUSQ hot path
 * (arXiv 2508.04880, /root/reference/PAPER.md, cited as P:<line>).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.  It shares no code, header, table or helper with the
 * CUDA path in paper_2508_04880_b200/ and never includes anything from it;
 * the only shared things are the op-list inputs from workloads/ and the
 * documented record layouts (24-byte op, serialized tree bytes).
 *
 * Everything is step by step in the paper's order:
 *   sites + thresholds          (readings #1-#4, #9)
 *   ER sampling, Philox4x32-10  (reading #9)
 *   ER tallying                 (Fig. P:163)
 *   ER commutation with literal per-qubit STACKS (rules 1-6 of
 *                                P:213-220; readings #5-#7)
 *   pruning                     (reading #10)
 *   DFS order + shot offsets    (reading #12)
 *   per-leaf replay from |0..0> in complex128 (Eq. 1)
 *   inverse-CDF sampling over a compensated sequential sum (reading #9)
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without an independent
 * pin are marked "parity unpinned" (none at present).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC -o liboracle.so tusq_oracle.c -lm
 * (no FMA contraction; an OpenMP parallel-for over amplitude pairs is the only
 * concession to speed).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

enum { G_I, G_X, G_Y, G_Z, G_H, G_S, G_SDG, G_T, G_TDG, G_RX, G_RY, G_RZ, G_P, G_CX, G_CZ, G_CP, G_COUNT };
enum { PAULI_I = 0, PAULI_X = 1, PAULI_Y = 2, PAULI_Z = 3 };

typedef struct { uint32_t kind, q0, q1, pad; double theta; } or_op; /* 24 bytes, the input layout */

static int is_two_qubit(uint32_t k) { return k == G_CX || k == G_CZ || k == G_CP; }

/* ===================================================================== Philox
 * Philox4x32-10 (Salmon et al., SC'11), the generator curand calls
 * philox4x32_10: multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments
 * 0x9E3779B9 / 0xBB67AE85, ten rounds, key bumped before rounds 2..10.
 */
void or_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ===================================================================== sites
 * One independent single-qubit Pauli channel per (gate, acted qubit), placed
 * right after the gate ("after every gate", Fig. P:186 "II/XX" after the
 * CNOT; reading #1).  1q gates carry depolarizing p1, each qubit of a 2q gate
 * carries depolarizing p2 ((1-p, p/3, p/3, p/3); reading #2).
 * Measurement noise is an X flip before readout on every qubit (
 * reading #4), site position L.  A channel with p = 0 attaches no site.
 * Integer thresholds: t_P = round(p_P * 2^32), t_I = 2^32 - (t_X + t_Y + t_Z).
 */
typedef struct { uint32_t pos, q; uint64_t tI, tX, tY, tZ; } or_site;

static uint64_t thr(double p) { return (uint64_t)llround(p * 4294967296.0); }

/* A site's Pauli channel (pX, pY, pZ) as integer thresholds (reading #9): t_P = round(p_P 2^32),
 * t_I = 2^32 - (t_X + t_Y + t_Z); a channel summing to 1 may round past 2^32 -- the excess comes
 * off t_Y, then t_Z. */
static void set_channel(or_site *s, const double c[3])
{
    const uint64_t one = 4294967296ull;
    s->tX = thr(c[0]); if (s->tX > one) s->tX = one;
    s->tY = thr(c[1]);
    s->tZ = thr(c[2]);
    if (s->tX + s->tY > one) s->tY = one - s->tX;
    if (s->tX + s->tY + s->tZ > one) s->tZ = one - s->tX - s->tY;
    s->tI = one - (s->tX + s->tY + s->tZ);
}

/* depolarizing p (reading #2) -> (p/3, p/3, p/3); measurement bit flip p (P:137,
 * reading #4) -> (p, 0, 0) */
static void chan_depolarizing(double p, double c[3]) { c[0] = c[1] = c[2] = p / 3.0; }
static void chan_bitflip(double p, double c[3]) { c[0] = p; c[1] = 0.0; c[2] = 0.0; }
static int chan_live(const double c[3]) { return c[0] > 0.0 || c[1] > 0.0 || c[2] > 0.0; }

int or_validate(uint32_t n, const or_op *ops, uint64_t L)
{
    if (n == 0 || n > 62) return 1;
    for (uint64_t i = 0; i < L; i++) {
        if (ops[i].kind >= G_COUNT) return 1;
        if (ops[i].q0 >= n) return 1;
        if (is_two_qubit(ops[i].kind) && (ops[i].q1 >= n || ops[i].q1 == ops[i].q0)) return 1;
    }
    return 0;
}

/* Sites for general per-class Pauli channels chan[0..2] (1q gates), chan[3..5] (each qubit of a 2q
 * gate), chan[6..8] (readout); a class whose channel is all-zero attaches no site (reading #21).
 * Returns the number of sites; fills `out` when non-NULL. */
uint64_t or_site_table_chan(uint32_t n, const or_op *ops, uint64_t L, const double chan[9], or_site *out)
{
    uint64_t m = 0;
    for (uint64_t pos = 0; pos < L; pos++) {
        if (is_two_qubit(ops[pos].kind)) {
            if (chan_live(chan + 3)) {
                if (out) { out[m].pos = (uint32_t)pos; out[m].q = ops[pos].q0; set_channel(&out[m], chan + 3); }
                m++;
                if (out) { out[m].pos = (uint32_t)pos; out[m].q = ops[pos].q1; set_channel(&out[m], chan + 3); }
                m++;
            }
        } else if (chan_live(chan)) {
            if (out) { out[m].pos = (uint32_t)pos; out[m].q = ops[pos].q0; set_channel(&out[m], chan); }
            m++;
        }
    }
    if (chan_live(chan + 6)) {
        for (uint32_t q = 0; q < n; q++) {
            if (out) { out[m].pos = (uint32_t)L; out[m].q = q; set_channel(&out[m], chan + 6); }
            m++;
        }
    }
    return m;
}

static void chan_of(double p1, double p2, double pm, double chan[9])
{
    chan_depolarizing(p1, chan);
    chan_depolarizing(p2, chan + 3);
    chan_bitflip(pm, chan + 6);
}

/* depolarizing p1 / p2 + readout bit flip pm */
uint64_t or_site_table(uint32_t n, const or_op *ops, uint64_t L, double p1, double p2, double pm, or_site *out)
{
    double chan[9];
    chan_of(p1, p2, pm, chan);
    return or_site_table_chan(n, ops, L, chan, out);
}

/* ===================================================================== ER sampling
 * Shot s, site i: Philox counter (i >> 2, s_lo, s_hi, 0x45520000), key
 * (seed_lo, seed_hi); word w = out[i & 3]; I if w < t_I, X if w < t_I + t_X,
 * Y if w < t_I + t_X + t_Y, else Z ("sample from all error channels").
 */
static int draw_pauli(const or_site *s, uint32_t w)
{
    uint64_t x = w;
    if (x < s->tI) return PAULI_I;
    if (x < s->tI + s->tX) return PAULI_X;
    if (x < s->tI + s->tX + s->tY) return PAULI_Y;
    return PAULI_Z;
}

static int site_pauli(const or_site *sites, uint64_t i, uint64_t shot, uint64_t seed)
{
    uint32_t ctr[4] = { (uint32_t)(i >> 2), (uint32_t)shot, (uint32_t)(shot >> 32), 0x45520000u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t w[4];
    or_philox(ctr, key, w);
    return draw_pauli(&sites[i], w[i & 3]);
}

/* Raw ER of one shot as (site index, Pauli) pairs, site-ascending.  Returns the
 * Hamming weight; writes at most `cap` pairs. */
uint64_t or_sample_er(uint32_t n, const or_op *ops, uint64_t L, double p1, double p2, double pm,
                      uint64_t seed, uint64_t shot, uint32_t *out_pairs, uint64_t cap)
{
    uint64_t m = or_site_table(n, ops, L, p1, p2, pm, NULL);
    or_site *sites = (or_site *)malloc((m ? m : 1) * sizeof(or_site));
    or_site_table(n, ops, L, p1, p2, pm, sites);
    uint64_t hw = 0;
    for (uint64_t i = 0; i < m; i++) {
        int p = site_pauli(sites, i, shot, seed);
        if (p != PAULI_I) {
            if (hw < cap) { out_pairs[2 * hw] = (uint32_t)i; out_pairs[2 * hw + 1] = (uint32_t)p; }
            hw++;
        }
    }
    free(sites);
    return hw;
}

/* ===================================================================== ER commutation
 * The greedy algorithm of P:211-222 with literal per-qubit stacks.  A stack
 * entry is either a noiseless gate (its circuit position) or a noisy Pauli.
 * Rules:
 *   1. back-to-back noisy Paulis merge into their product (phase dropped);
 *   2. a noisy Pauli commutes through any noiseless Pauli (I, X, Y, Z gates);
 *   3. X/Y/Z commute through RX/RY/RZ respectively; reading #5 extends the
 *      Z rule to every Z-axis diagonal (S, Sdg, T, Tdg, P, RZ and CZ/CP per
 *      qubit); anything else on such a gate is blocked (Fig. P:193);
 *   4-6. CNOT: X_c -> X_c X_t, X_t -> X_t, Z_t -> Z_c Z_t, Z_c -> Z_c,
 *        Y_c -> Y_c X_t, Y_t -> Z_c Y_t;
 *   H conjugates X <-> Z and keeps Y (reading #5).
 * Blocked Paulis stay buried under the blocking gate (reading #6: the whole
 * Pauli), i.e. they are applied right before that gate.  At the end, Z before
 * measurement is dropped and a pending X or Y becomes a terminal X (reading #7).
 */
static const int PAULI_MUL[4][4] = {      /* phase-free Pauli product (rule 1) */
    { PAULI_I, PAULI_X, PAULI_Y, PAULI_Z },
    { PAULI_X, PAULI_I, PAULI_Z, PAULI_Y },
    { PAULI_Y, PAULI_Z, PAULI_I, PAULI_X },
    { PAULI_Z, PAULI_Y, PAULI_X, PAULI_I },
};

/* single-qubit gate: does noisy Pauli p pass, and what does it become? */
static int pass_1q(uint32_t kind, int p, int *p_out)
{
    switch (kind) {
    case G_I: case G_X: case G_Y: case G_Z:        /* rule 2 */
        *p_out = p; return 1;
    case G_H:
        *p_out = (p == PAULI_X) ? PAULI_Z : (p == PAULI_Z) ? PAULI_X : p; return 1;
    case G_S: case G_SDG: case G_T: case G_TDG: case G_P: case G_RZ:   /* rule 3, Z axis */
        *p_out = p; return p == PAULI_Z;
    case G_RX:
        *p_out = p; return p == PAULI_X;
    case G_RY:
        *p_out = p; return p == PAULI_Y;
    default:
        return 0;
    }
}

/* CNOT rules 4-6 for one Pauli on the control (role 0) or the target (role 1) */
static void push_cnot_single(int p, int role, int *pc, int *pt)
{
    *pc = PAULI_I; *pt = PAULI_I;
    if (p == PAULI_I) return;
    if (role == 0) {
        if (p == PAULI_X) { *pc = PAULI_X; *pt = PAULI_X; }      /* rule 4 */
        else if (p == PAULI_Z) { *pc = PAULI_Z; }                /* rule 5 */
        else { *pc = PAULI_Y; *pt = PAULI_X; }                   /* rule 6 */
    } else {
        if (p == PAULI_X) { *pt = PAULI_X; }                     /* rule 4 */
        else if (p == PAULI_Z) { *pc = PAULI_Z; *pt = PAULI_Z; } /* rule 5 */
        else { *pc = PAULI_Z; *pt = PAULI_Y; }                   /* rule 6 */
    }
}

typedef struct { int noisy; int pauli; uint32_t gate_pos; } st_entry;
typedef struct { st_entry *e; uint64_t size, cap; } pstack;

static void st_push(pstack *s, int noisy, int pauli, uint32_t gate_pos)
{
    if (s->size == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 16;
        s->e = (st_entry *)realloc(s->e, s->cap * sizeof(st_entry));
    }
    s->e[s->size].noisy = noisy; s->e[s->size].pauli = pauli; s->e[s->size].gate_pos = gate_pos;
    s->size++;
}

static int st_top_noisy(const pstack *s) { return s->size > 0 && s->e[s->size - 1].noisy; }

static int st_pop_noisy(pstack *s)          /* pops a noisy top, I otherwise */
{
    if (!st_top_noisy(s)) return PAULI_I;
    s->size--;
    return s->e[s->size].pauli;
}

static void push_noisy_candidate(pstack *s, int p)
{
    if (p == PAULI_I) return;
    if (st_top_noisy(s)) {                         /* rule 1: merge */
        int m = PAULI_MUL[s->e[s->size - 1].pauli][p];
        if (m == PAULI_I) s->size--;
        else s->e[s->size - 1].pauli = m;
    } else {
        st_push(s, 1, p, 0);
    }
}

static int cmp_pos_q(const void *a, const void *b)
{
    const uint32_t *x = (const uint32_t *)a, *y = (const uint32_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/*
 * in:  noise insertions (pos, q, P) meaning "Pauli P right AFTER gate pos"
 *      (pos = L: before readout), sorted by pos.
 * out: canonical key, (pos, q, P) triples meaning "P right BEFORE gate pos"
 *      (pos = L: a terminal X), sorted by (pos, q).  Returns the count (may
 *      exceed cap; only cap triples are written).
 */
uint32_t or_canonicalize(uint32_t n, const or_op *ops, uint64_t L,
                         const uint32_t *ins, uint32_t n_ins, uint32_t *out, uint32_t cap)
{
    pstack *st = (pstack *)calloc(n, sizeof(pstack));
    uint32_t k = 0;  /* cursor in the insertion list */
    for (uint64_t pos = 0; pos <= L; pos++) {
        if (pos < L) {
            const or_op *g = &ops[pos];
            if (g->kind == G_CX) {
                int pc = st_pop_noisy(&st[g->q0]);
                int pt = st_pop_noisy(&st[g->q1]);
                st_push(&st[g->q0], 0, 0, (uint32_t)pos);
                st_push(&st[g->q1], 0, 0, (uint32_t)pos);
                int c1, t1, c2, t2;
                push_cnot_single(pc, 0, &c1, &t1);
                push_cnot_single(pt, 1, &c2, &t2);
                push_noisy_candidate(&st[g->q0], PAULI_MUL[c1][c2]);
                push_noisy_candidate(&st[g->q1], PAULI_MUL[t1][t2]);
            } else if (g->kind == G_CZ || g->kind == G_CP) {
                uint32_t qs[2] = { g->q0, g->q1 };
                int passing[2] = { PAULI_I, PAULI_I };
                for (int j = 0; j < 2; j++) {
                    pstack *s = &st[qs[j]];
                    if (st_top_noisy(s) && s->e[s->size - 1].pauli == PAULI_Z) passing[j] = st_pop_noisy(s);
                }
                for (int j = 0; j < 2; j++) st_push(&st[qs[j]], 0, 0, (uint32_t)pos);
                for (int j = 0; j < 2; j++) push_noisy_candidate(&st[qs[j]], passing[j]);
            } else {
                pstack *s = &st[g->q0];
                int p_new;
                if (st_top_noisy(s) && pass_1q(g->kind, s->e[s->size - 1].pauli, &p_new)) {
                    st_pop_noisy(s);
                    st_push(s, 0, 0, (uint32_t)pos);
                    push_noisy_candidate(s, p_new);
                } else {
                    st_push(s, 0, 0, (uint32_t)pos);   /* blocked noisy gate stays buried */
                }
            }
        }
        /* noisy candidates at this position: the channels after gate pos */
        while (k < n_ins && ins[3 * k] == pos) {
            push_noisy_candidate(&st[ins[3 * k + 1]], (int)ins[3 * k + 2]);
            k++;
        }
    }
    /* serialize each stack bottom -> top */
    uint32_t cnt = 0;
    for (uint32_t q = 0; q < n; q++) {
        pstack *s = &st[q];
        for (uint64_t i = 0; i < s->size; i++) {
            if (!s->e[i].noisy) continue;
            uint32_t pos, p = (uint32_t)s->e[i].pauli;
            if (i + 1 < s->size) {
                pos = s->e[i + 1].gate_pos;         /* buried right before that gate */
            } else {
                if (p == PAULI_Z) continue;         /* Z before measurement is dropped */
                pos = (uint32_t)L;
                p = PAULI_X;                        /* X or Y reads out as a flip */
            }
            if (cnt < cap && out) {
                out[3 * cnt] = pos; out[3 * cnt + 1] = q; out[3 * cnt + 2] = p;
            }
            cnt++;
        }
        free(s->e);
    }
    free(st);
    if (out && cnt <= cap) qsort(out, cnt, 3 * sizeof(uint32_t), cmp_pos_q);
    return cnt;
}

/* ===================================================================== tree records */
typedef struct {
    uint32_t *tr;      /* 3*n triples */
    uint32_t n;
    uint64_t count;
} or_leafrec;

typedef struct {
    uint32_t n_qubits;
    uint64_t n_ops, shots, seed;
    uint64_t S2, S3, p0, n_sig, n_insig, n_selected;
    uint64_t n_leaves;
    or_leafrec *leaves;     /* DFS order, after pruning */
    uint64_t *offsets;
} or_tree;

/* lexicographic order of raw ERs (site, pauli) sequences, used only to tally */
static int cmp_raw(const void *a, const void *b)
{
    const or_leafrec *x = (const or_leafrec *)a, *y = (const or_leafrec *)b;
    uint32_t m = x->n < y->n ? x->n : y->n;
    for (uint32_t i = 0; i < 2 * m; i++)
        if (x->tr[i] != y->tr[i]) return x->tr[i] < y->tr[i] ? -1 : 1;
    if (x->n != y->n) return x->n < y->n ? -1 : 1;
    return 0;
}

/* any total order on canonical keys, used only to merge equal keys */
static int cmp_key(const void *a, const void *b)
{
    const or_leafrec *x = (const or_leafrec *)a, *y = (const or_leafrec *)b;
    uint32_t m = x->n < y->n ? x->n : y->n;
    for (uint32_t i = 0; i < 3 * m; i++)
        if (x->tr[i] != y->tr[i]) return x->tr[i] < y->tr[i] ? -1 : 1;
    if (x->n != y->n) return x->n < y->n ? -1 : 1;
    return 0;
}

/*
 * DFS order of the execution tree (reading #12): children ordered
 * I < X < Y < Z over slots (pos, q).  Walking two keys triple by triple, the
 * first difference decides: a key that ends first carries I at the other's
 * next slot (comes first); a Pauli at an earlier slot means the other key has
 * I there (the other comes first); at the same slot the smaller Pauli comes first.
 */
int or_dfs_cmp(const uint32_t *a, uint32_t na, const uint32_t *b, uint32_t nb)
{
    for (uint32_t j = 0;; j++) {
        if (j == na && j == nb) return 0;
        if (j == na) return -1;
        if (j == nb) return 1;
        uint64_t sa = ((uint64_t)a[3 * j] << 32) | a[3 * j + 1];
        uint64_t sb = ((uint64_t)b[3 * j] << 32) | b[3 * j + 1];
        if (sa < sb) return 1;
        if (sa > sb) return -1;
        if (a[3 * j + 2] != b[3 * j + 2]) return a[3 * j + 2] < b[3 * j + 2] ? -1 : 1;
    }
}

static int cmp_dfs(const void *a, const void *b)
{
    const or_leafrec *x = (const or_leafrec *)a, *y = (const or_leafrec *)b;
    return or_dfs_cmp(x->tr, x->n, y->tr, y->n);
}

/* ===================================================================== pruning
 * p0 = max count; a circuit is significant iff count >= alpha*p0
 * (alpha = a_num/a_den, reading #10: count*a_den >= a_num*p0).  If the
 * insignificant set I holds more than beta circuits, beta of them are drawn
 * count-proportionally without replacement (draw j: Philox counter
 * (j, 0, 0, 0x50520000); x = w0 | w1<<32; r = x mod W_remaining; first remaining
 * insignificant circuit in DFS order whose cumulative weight exceeds r).  Each
 * selected circuit is sampled floor(p_insig * p_t / sum_K p) times (the
 * P:340 scale p_insig / sum p_t), residual to the largest p_t (ties: earliest).
 * counts[] are in DFS order.  out_class: 0 pruned, 1 significant, 2 kept insignificant.
 */
int or_prune(const uint64_t *counts, uint64_t m, uint32_t a_num, uint32_t a_den, uint32_t beta,
             int enabled, uint64_t seed, uint64_t *out_counts, uint8_t *out_class, uint64_t stats[4])
{
    uint64_t p0 = 0;
    for (uint64_t i = 0; i < m; i++) if (counts[i] > p0) p0 = counts[i];
    uint64_t n_sig = 0, n_insig = 0, p_insig = 0;
    for (uint64_t i = 0; i < m; i++) {
        out_counts[i] = counts[i];
        int sig = !enabled || (unsigned __int128)counts[i] * a_den >= (unsigned __int128)a_num * p0;
        out_class[i] = sig ? 1 : 2;
        if (sig) n_sig++; else { n_insig++; p_insig += counts[i]; }
    }
    uint64_t n_sel = n_insig;
    if (enabled && n_insig > beta) {
        uint8_t *chosen = (uint8_t *)calloc(m ? m : 1, 1);
        uint64_t w_rem = p_insig;
        uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
        for (uint64_t j = 0; j < beta; j++) {
            uint32_t ctr[4] = { (uint32_t)j, 0u, 0u, 0x50520000u }, w[4];
            or_philox(ctr, key, w);
            uint64_t x = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
            uint64_t r = x % w_rem, cum = 0;
            for (uint64_t i = 0; i < m; i++) {
                if (out_class[i] != 2 || chosen[i]) continue;
                cum += counts[i];
                if (cum > r) { chosen[i] = 1; w_rem -= counts[i]; break; }
            }
        }
        uint64_t wk = 0;
        for (uint64_t i = 0; i < m; i++) if (chosen[i]) wk += counts[i];
        uint64_t assigned = 0, best = UINT64_MAX;
        for (uint64_t i = 0; i < m; i++) {
            if (out_class[i] != 2) continue;
            if (!chosen[i]) { out_class[i] = 0; out_counts[i] = 0; continue; }
            out_counts[i] = (uint64_t)(((unsigned __int128)p_insig * counts[i]) / wk);
            assigned += out_counts[i];
            if (best == UINT64_MAX || counts[i] > counts[best]) best = i;
        }
        out_counts[best] += p_insig - assigned;
        n_sel = beta;
        free(chosen);
    }
    if (stats) { stats[0] = p0; stats[1] = n_sig; stats[2] = n_insig; stats[3] = n_sel; }
    return 0;
}

/* ===================================================================== build */
static void free_recs(or_leafrec *r, uint64_t m)
{
    for (uint64_t i = 0; i < m; i++) free(r[i].tr);
    free(r);
}

int or_build_chan(uint32_t n, const or_op *ops, uint64_t L, const double chan[9],
                  uint64_t shots, uint64_t seed, uint32_t a_num, uint32_t a_den, uint32_t beta,
                  int prune_enabled, void **out)
{
    *out = NULL;
    if (or_validate(n, ops, L) || shots == 0 || a_den == 0) return 1;
    if (prune_enabled && (beta == 0 || a_num > a_den)) return 1;   /* beta >= 1 keeps shots conserved */
    for (int c = 0; c < 3; c++) {
        const double *p = chan + 3 * c;
        if (!(p[0] >= 0 && p[0] <= 1) || !(p[1] >= 0 && p[1] <= 1) || !(p[2] >= 0 && p[2] <= 1) ||
            !(p[0] + p[1] + p[2] <= 1))
            return 1;
    }
    uint64_t m = or_site_table_chan(n, ops, L, chan, NULL);
    or_site *sites = (or_site *)malloc((m ? m : 1) * sizeof(or_site));
    or_site_table_chan(n, ops, L, chan, sites);

    /* S1 raw ERs, one per shot */
    or_leafrec *raw = (or_leafrec *)calloc(shots, sizeof(or_leafrec));
    uint32_t *buf = (uint32_t *)malloc((2 * m + 2) * sizeof(uint32_t));
    for (uint64_t s = 0; s < shots; s++) {
        uint32_t hw = 0;
        for (uint64_t i = 0; i < m; i++) {
            int p = site_pauli(sites, i, s, seed);
            if (p != PAULI_I) { buf[2 * hw] = (uint32_t)i; buf[2 * hw + 1] = (uint32_t)p; hw++; }
        }
        raw[s].n = hw; raw[s].count = 1;
        raw[s].tr = (uint32_t *)malloc((2 * hw + 1) * sizeof(uint32_t));
        memcpy(raw[s].tr, buf, 2 * hw * sizeof(uint32_t));
    }
    free(buf);

    /* ER tallying: identical ERs share one circuit; S2 unique */
    qsort(raw, shots, sizeof(or_leafrec), cmp_raw);
    uint64_t S2 = 0;
    for (uint64_t s = 0; s < shots; s++) {
        if (S2 > 0 && cmp_raw(&raw[S2 - 1], &raw[s]) == 0) {
            raw[S2 - 1].count += raw[s].count;
            free(raw[s].tr);
        } else {
            raw[S2++] = raw[s];
        }
    }

    /* ER commutation: canonical keys; S3 unique after merging */
    or_leafrec *can = (or_leafrec *)calloc(S2 ? S2 : 1, sizeof(or_leafrec));
    for (uint64_t u = 0; u < S2; u++) {
        uint32_t hw = raw[u].n;
        uint32_t *ins = (uint32_t *)malloc((3 * hw + 1) * sizeof(uint32_t));
        for (uint32_t j = 0; j < hw; j++) {
            const or_site *st = &sites[raw[u].tr[2 * j]];
            ins[3 * j] = st->pos; ins[3 * j + 1] = st->q; ins[3 * j + 2] = raw[u].tr[2 * j + 1];
        }
        uint32_t cap = 3 * n + hw + 8;
        uint32_t *key = (uint32_t *)malloc(3 * (size_t)cap * sizeof(uint32_t));
        uint32_t nk = or_canonicalize(n, ops, L, ins, hw, key, cap);
        if (nk > cap) {  /* cannot happen: at most one triple per (pos, q) occupied by a noise path */
            free(ins); free(key); free_recs(raw, S2); free_recs(can, u); free(sites);
            return 7;
        }
        can[u].tr = key; can[u].n = nk; can[u].count = raw[u].count;
        free(ins);
    }
    free_recs(raw, S2);
    free(sites);
    qsort(can, S2, sizeof(or_leafrec), cmp_key);
    uint64_t S3 = 0;
    for (uint64_t u = 0; u < S2; u++) {
        if (S3 > 0 && cmp_key(&can[S3 - 1], &can[u]) == 0) {
            can[S3 - 1].count += can[u].count;
            free(can[u].tr);
        } else {
            can[S3++] = can[u];
        }
    }

    /* DFS order (reading #12), then pruning in that order */
    qsort(can, S3, sizeof(or_leafrec), cmp_dfs);
    uint64_t *cin = (uint64_t *)malloc((S3 ? S3 : 1) * sizeof(uint64_t));
    uint64_t *cout = (uint64_t *)malloc((S3 ? S3 : 1) * sizeof(uint64_t));
    uint8_t *cls = (uint8_t *)malloc(S3 ? S3 : 1);
    for (uint64_t u = 0; u < S3; u++) cin[u] = can[u].count;
    uint64_t pst[4];
    or_prune(cin, S3, a_num, a_den, beta, prune_enabled, seed, cout, cls, pst);

    or_tree *t = (or_tree *)calloc(1, sizeof(or_tree));
    t->n_qubits = n; t->n_ops = L; t->shots = shots; t->seed = seed;
    t->S2 = S2; t->S3 = S3; t->p0 = pst[0]; t->n_sig = pst[1]; t->n_insig = pst[2]; t->n_selected = pst[3];
    t->leaves = (or_leafrec *)calloc(S3 ? S3 : 1, sizeof(or_leafrec));
    t->offsets = (uint64_t *)calloc(S3 ? S3 : 1, sizeof(uint64_t));
    uint64_t nl = 0, off = 0;
    for (uint64_t u = 0; u < S3; u++) {
        if (cls[u] == 0) { free(can[u].tr); continue; }
        t->leaves[nl] = can[u];
        t->leaves[nl].count = cout[u];
        t->offsets[nl] = off;           /* exclusive prefix sum of counts */
        off += cout[u];
        nl++;
    }
    t->n_leaves = nl;
    free(can); free(cin); free(cout); free(cls);
    *out = t;
    return 0;
}

int or_build(uint32_t n, const or_op *ops, uint64_t L, double p1, double p2, double pm,
             uint64_t shots, uint64_t seed, uint32_t a_num, uint32_t a_den, uint32_t beta,
             int prune_enabled, void **out)
{
    double chan[9];
    *out = NULL;
    if (!(p1 >= 0 && p1 <= 1) || !(p2 >= 0 && p2 <= 1) || !(pm >= 0 && pm <= 1)) return 1;
    chan_of(p1, p2, pm, chan);
    return or_build_chan(n, ops, L, chan, shots, seed, a_num, a_den, beta, prune_enabled, out);
}

/* Eq. 2: Pauli twirl of decoherence for an idle time t -> (pX, pY, pZ); 1 on bad input */
int or_twirl(double t, double T1, double T2, double out[3])
{
    if (!(t >= 0) || !(T1 > 0) || !(T2 > 0)) return 1;
    double px = (1.0 - exp(-t / T1)) / 4.0;
    double pz = (1.0 - exp(-t / T2)) / 2.0 - (1.0 - exp(-t / T1)) / 4.0;
    if (pz < 0) return 1;
    out[0] = px; out[1] = px; out[2] = pz;
    return 0;
}

void or_free(void *p)
{
    or_tree *t = (or_tree *)p;
    if (!t) return;
    for (uint64_t i = 0; i < t->n_leaves; i++) free(t->leaves[i].tr);
    free(t->leaves); free(t->offsets); free(t);
}

void or_stats(const void *p, uint64_t out[9])
{
    const or_tree *t = (const or_tree *)p;
    out[0] = t->shots; out[1] = t->S2; out[2] = t->S3; out[3] = t->p0; out[4] = t->n_sig;
    out[5] = t->n_insig; out[6] = t->n_selected; out[7] = t->n_leaves; out[8] = t->n_ops;
}

/* leaf record: returns the number of triples (writes at most cap) */
uint32_t or_leaf(const void *p, uint64_t l, uint64_t *count, uint64_t *offset, uint32_t *triples, uint32_t cap)
{
    const or_tree *t = (const or_tree *)p;
    const or_leafrec *r = &t->leaves[l];
    *count = r->count; *offset = t->offsets[l];
    for (uint32_t i = 0; i < r->n && i < cap; i++) {
        triples[3 * i] = r->tr[3 * i]; triples[3 * i + 1] = r->tr[3 * i + 1]; triples[3 * i + 2] = r->tr[3 * i + 2];
    }
    return r->n;
}

/*
 * Canonical serialization (little-endian), documented in include/tusq.h:
 *   "TUSQTRE1", u32 n_qubits, u32 0, u64 n_ops, u64 shots, u64 seed,
 *   u64 S2, S3, p0, n_sig, n_insig, n_selected, n_leaves,
 *   per leaf: u64 count, u64 offset, u32 n_triples, n_triples x (u32 pos, q, P)
 */
static uint64_t put(uint8_t *buf, uint64_t cap, uint64_t at, const void *src, uint64_t len)
{
    if (buf && at + len <= cap) memcpy(buf + at, src, len);
    return at + len;
}

uint64_t or_serialize(const void *p, uint8_t *buf, uint64_t cap)
{
    const or_tree *t = (const or_tree *)p;
    uint64_t at = 0;
    uint32_t zero = 0;
    at = put(buf, cap, at, "TUSQTRE1", 8);
    at = put(buf, cap, at, &t->n_qubits, 4);
    at = put(buf, cap, at, &zero, 4);
    uint64_t hdr[10] = { t->n_ops, t->shots, t->seed, t->S2, t->S3, t->p0, t->n_sig, t->n_insig,
                         t->n_selected, t->n_leaves };
    at = put(buf, cap, at, hdr, sizeof(hdr));
    for (uint64_t l = 0; l < t->n_leaves; l++) {
        at = put(buf, cap, at, &t->leaves[l].count, 8);
        at = put(buf, cap, at, &t->offsets[l], 8);
        at = put(buf, cap, at, &t->leaves[l].n, 4);
        at = put(buf, cap, at, t->leaves[l].tr, 12ull * t->leaves[l].n);
    }
    return at;
}

/* ===================================================================== state vector
 * Eq. 1: a k-qubit gate touches only its own amplitude pairs/quads.
 * Matrices (reading list):
 *   H = M_SQRT1_2 [[1,1],[1,-1]], T = diag(1, (1+i) M_SQRT1_2),
 *   RZ(t) = diag(e^{-it/2}, e^{it/2}), Y = [[0,-i],[i,0]], P(t) = diag(1, e^{it}),
 *   RX(t) = [[c, -is], [-is, c]], RY(t) = [[c, -s], [s, c]] (c = cos t/2, s = sin t/2),
 *   CP(t): e^{it} on |11>.  Inverses: H->H, T<->Tdg, S<->Sdg, R(t)->R(-t).
 */
static void gate_matrix(uint32_t kind, double th, cplx u[4])
{
    const cplx I1 = 1.0 * I;
    double c = cos(th / 2), s = sin(th / 2);
    switch (kind) {
    case G_I:   u[0] = 1; u[1] = 0; u[2] = 0; u[3] = 1; break;
    case G_X:   u[0] = 0; u[1] = 1; u[2] = 1; u[3] = 0; break;
    case G_Y:   u[0] = 0; u[1] = -I1; u[2] = I1; u[3] = 0; break;
    case G_Z:   u[0] = 1; u[1] = 0; u[2] = 0; u[3] = -1; break;
    case G_H:   u[0] = M_SQRT1_2; u[1] = M_SQRT1_2; u[2] = M_SQRT1_2; u[3] = -M_SQRT1_2; break;
    case G_S:   u[0] = 1; u[1] = 0; u[2] = 0; u[3] = I1; break;
    case G_SDG: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = -I1; break;
    case G_T:   u[0] = 1; u[1] = 0; u[2] = 0; u[3] = (1.0 + I1) * M_SQRT1_2; break;
    case G_TDG: u[0] = 1; u[1] = 0; u[2] = 0; u[3] = (1.0 - I1) * M_SQRT1_2; break;
    case G_RX:  u[0] = c; u[1] = -I1 * s; u[2] = -I1 * s; u[3] = c; break;
    case G_RY:  u[0] = c; u[1] = -s; u[2] = s; u[3] = c; break;
    case G_RZ:  u[0] = cexp(-I1 * th / 2); u[1] = 0; u[2] = 0; u[3] = cexp(I1 * th / 2); break;
    case G_P:   u[0] = 1; u[1] = 0; u[2] = 0; u[3] = cexp(I1 * th); break;
    default:    u[0] = 1; u[1] = 0; u[2] = 0; u[3] = 1; break;
    }
}

static void apply_1q(cplx *psi, uint32_t n, uint32_t q, const cplx u[4])
{
    int64_t N = (int64_t)1 << n, bit = (int64_t)1 << q;
#pragma omp parallel for if (n >= 16) schedule(static)
    for (int64_t i = 0; i < N; i++) {
        if (i & bit) continue;
        cplx a = psi[i], b = psi[i | bit];
        psi[i] = u[0] * a + u[1] * b;
        psi[i | bit] = u[2] * a + u[3] * b;
    }
}

static void apply_gate(cplx *psi, uint32_t n, const or_op *g, int inverse)
{
    int64_t N = (int64_t)1 << n;
    if (g->kind == G_CX) {
        int64_t c = (int64_t)1 << g->q0, t = (int64_t)1 << g->q1;
#pragma omp parallel for if (n >= 16) schedule(static)
        for (int64_t i = 0; i < N; i++) {
            if ((i & c) && !(i & t)) { cplx a = psi[i]; psi[i] = psi[i | t]; psi[i | t] = a; }
        }
        return;
    }
    if (g->kind == G_CZ || g->kind == G_CP) {
        int64_t c = (int64_t)1 << g->q0, t = (int64_t)1 << g->q1;
        cplx ph = (g->kind == G_CZ) ? -1.0 : cexp((inverse ? -1.0 : 1.0) * I * g->theta);
#pragma omp parallel for if (n >= 16) schedule(static)
        for (int64_t i = 0; i < N; i++)
            if ((i & c) && (i & t)) psi[i] = ph * psi[i];
        return;
    }
    cplx u[4];
    uint32_t kind = g->kind;
    double th = g->theta;
    if (inverse) {
        if (kind == G_S) kind = G_SDG; else if (kind == G_SDG) kind = G_S;
        else if (kind == G_T) kind = G_TDG; else if (kind == G_TDG) kind = G_T;
        th = -th;
    }
    gate_matrix(kind, th, u);
    apply_1q(psi, n, g->q0, u);
}

static void apply_pauli(cplx *psi, uint32_t n, uint32_t q, uint32_t p)
{
    or_op g = { p == PAULI_X ? G_X : p == PAULI_Y ? G_Y : p == PAULI_Z ? G_Z : G_I, q, 0, 0, 0.0 };
    apply_gate(psi, n, &g, 0);
}

/* Apply one gate (or its inverse) to a caller-owned state: for pin tests. */
int or_apply_gate(double *state, uint32_t n, const or_op *g, int inverse)
{
    if (or_validate(n, g, 1)) return 1;
    apply_gate((cplx *)state, n, g, inverse);
    return 0;
}

/*
 * Replay a noisy circuit on `state` (2^n complex, interleaved re/im).
 * before_gate = 1: triples are canonical ("P right before gate pos", pos = L at the end);
 * before_gate = 0: triples are raw noise insertions ("P right after gate pos").
 * init = 1: start from |0..0>.
 */
int or_replay(uint32_t n, const or_op *ops, uint64_t L, const uint32_t *tr, uint32_t ntr,
              int before_gate, int init, double *state)
{
    if (or_validate(n, ops, L)) return 1;
    cplx *psi = (cplx *)state;
    int64_t N = (int64_t)1 << n;
    if (init) { for (int64_t i = 0; i < N; i++) psi[i] = 0; psi[0] = 1; }
    uint32_t k = 0;
    for (uint64_t pos = 0; pos <= L; pos++) {
        if (before_gate) {
            while (k < ntr && tr[3 * k] == pos) { apply_pauli(psi, n, tr[3 * k + 1], tr[3 * k + 2]); k++; }
            if (pos < L) apply_gate(psi, n, &ops[pos], 0);
        } else {
            if (pos < L) apply_gate(psi, n, &ops[pos], 0);
            while (k < ntr && tr[3 * k] == pos) { apply_pauli(psi, n, tr[3 * k + 1], tr[3 * k + 2]); k++; }
        }
    }
    return 0;
}

int or_replay_leaf(const void *p, const or_op *ops, uint64_t leaf, double *state)
{
    const or_tree *t = (const or_tree *)p;
    if (leaf >= t->n_leaves) return 1;
    return or_replay(t->n_qubits, ops, t->n_ops, t->leaves[leaf].tr, t->leaves[leaf].n, 1, 1, state);
}

/*
 * The state a leaf is SAMPLED from (reading #7): the leaf's triples before the readout
 * (pos < L) only.  Its terminal triples (pos = L: X flips of the readout, "measurement noise
 * is modeled as stochastic injection of the X gate") do not touch the amplitudes; they flip
 * bits of every bitstring drawn for the leaf (or_terminal_mask).  Applying X before an ideal
 * measurement and flipping the measured bit are the same channel on the outcome distribution.
 */
int or_replay_leaf_core(const void *p, const or_op *ops, uint64_t leaf, double *state)
{
    const or_tree *t = (const or_tree *)p;
    if (leaf >= t->n_leaves) return 1;
    uint32_t m = 0;   /* triples are sorted by pos: the core is a prefix */
    while (m < t->leaves[leaf].n && t->leaves[leaf].tr[3 * m] < t->n_ops) m++;
    return or_replay(t->n_qubits, ops, t->n_ops, t->leaves[leaf].tr, m, 1, 1, state);
}

uint64_t or_terminal_mask(const void *p, uint64_t leaf)
{
    const or_tree *t = (const or_tree *)p;
    uint64_t mask = 0;
    if (leaf >= t->n_leaves) return 0;
    for (uint32_t i = 0; i < t->leaves[leaf].n; i++) {
        const uint32_t *x = t->leaves[leaf].tr + 3 * i;
        if (x[0] == t->n_ops && (x[2] == PAULI_X || x[2] == PAULI_Y)) mask ^= (uint64_t)1 << x[1];
    }
    return mask;
}

/* ===================================================================== sampling
 * p_k = re*re + im*im (no FMA).  C(k) is a compensated (Neumaier) sequential
 * sum, T = C(N-1).  Draw j of leaf l: Philox counter (j_lo, l_lo, l_hi,
 * 0x53000000); x = w0 | w1<<32; u = (x >> 11) * 2^-53; t = u*T; the outcome is
 * k = min{k : C(k) > t} (if none, the last k with p_k > 0).  The draw is an
 * edge draw if min(t - C(k-1), C(k) - t) < edge_eps.
 */
typedef struct { double t; uint64_t j; } draw_t;

static int cmp_draw(const void *a, const void *b)
{
    const draw_t *x = (const draw_t *)a, *y = (const draw_t *)b;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return x->j < y->j ? -1 : (x->j > y->j);
}

int or_sample_state(const double *state, uint32_t n, uint64_t seed, uint64_t leaf, uint64_t n_draws,
                    double edge_eps, uint64_t *out, uint8_t *edge)
{
    if (n_draws == 0) return 0;
    int64_t N = (int64_t)1 << n;
    double sum = 0.0, comp = 0.0;
    int64_t last_pos = -1;
    for (int64_t k = 0; k < N; k++) {
        double re = state[2 * k], im = state[2 * k + 1];
        double pk = re * re + im * im;
        double tt = sum + pk;
        if (fabs(sum) >= fabs(pk)) comp += (sum - tt) + pk; else comp += (pk - tt) + sum;
        sum = tt;
        if (pk > 0) last_pos = k;
    }
    double T = sum + comp;
    draw_t *d = (draw_t *)malloc(n_draws * sizeof(draw_t));
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (uint64_t j = 0; j < n_draws; j++) {
        uint32_t ctr[4] = { (uint32_t)j, (uint32_t)leaf, (uint32_t)(leaf >> 32), 0x53000000u }, w[4];
        or_philox(ctr, key, w);
        uint64_t x = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        double u = (double)(x >> 11) * 0x1.0p-53;
        d[j].t = u * T; d[j].j = j;
    }
    qsort(d, n_draws, sizeof(draw_t), cmp_draw);
    uint64_t next = 0;
    double prev_c = 0.0;
    sum = 0.0; comp = 0.0;
    for (int64_t k = 0; k < N && next < n_draws; k++) {
        double re = state[2 * k], im = state[2 * k + 1];
        double pk = re * re + im * im;
        double tt = sum + pk;
        if (fabs(sum) >= fabs(pk)) comp += (sum - tt) + pk; else comp += (pk - tt) + sum;
        sum = tt;
        double ck = sum + comp;
        while (next < n_draws && ck > d[next].t) {
            out[d[next].j] = (uint64_t)k;
            double gap = fmin(d[next].t - prev_c, ck - d[next].t);
            edge[d[next].j] = gap < edge_eps;
            next++;
        }
        prev_c = ck;
    }
    for (; next < n_draws; next++) { out[d[next].j] = (uint64_t)last_pos; edge[d[next].j] = 1; }
    free(d);
    return 0;
}

/* Full oracle run: every leaf's core replayed from |0..0>, sampled into its slots, and the
 * drawn bitstrings flipped by its terminal X mask (reading #7). */
int or_run(const void *p, const or_op *ops, double edge_eps, uint64_t *slots, uint8_t *edge)
{
    const or_tree *t = (const or_tree *)p;
    uint32_t n = t->n_qubits;
    double *st = (double *)malloc(sizeof(double) * 2 * ((size_t)1 << n));
    if (!st) return 3;
    for (uint64_t l = 0; l < t->n_leaves; l++) {
        or_replay_leaf_core(p, ops, l, st);
        uint64_t *out = slots + t->offsets[l];
        or_sample_state(st, n, t->seed, l, t->leaves[l].count, edge_eps, out, edge + t->offsets[l]);
        uint64_t mask = or_terminal_mask(p, l);
        for (uint64_t j = 0; j < t->leaves[l].count; j++) out[j] ^= mask;
    }
    free(st);
    return 0;
}
