// Device kernel launchers (sm_100a).  All take raw device pointers and a cudaStream_t.
#pragma once
#include <cuda_runtime.h>

#include "common.h"

namespace tq {

// ----- K1-K4: one kernel per gate (the unfused path) -------------------------------
// Returns the algorithmic HBM bytes the launch moves.
double launch_gate(void *psi, uint32_t n, int prec, const Op &op, cudaStream_t st);
// K4: a Pauli string P = prod_q P_q applied in one pass (x/z bit masks).
double launch_pauli_string(void *psi, uint32_t n, int prec, uint64_t xmask, uint64_t zmask, cudaStream_t st);
// K7: psi <- amp |index>
double launch_init_basis(void *psi, uint32_t n, int prec, uint64_t index, double re, double im, cudaStream_t st);
// zeros at the elements of {x : (x & ~sfree) == sfix} outside the valid set {x : (x & ~vfree) == vfix}
double launch_zero_outside(void *psi, uint32_t n, int prec, uint64_t sfree, uint64_t sfix, uint64_t vfree, uint64_t vfix,
                           cudaStream_t st);

// ----- K6: sampler ---------------------------------------------------------------------
// block sums of |amp|^2 over contiguous blocks of 2^block_bits amplitudes; blocks outside the valid
// set {x : (x & ~vfree) == vfix} (whole blocks) sum to 0 unread
double launch_block_sums(const void *psi, uint32_t n, int prec, uint32_t block_bits, double *d_blocks,
                         cudaStream_t st, uint64_t vfree = ~0ull, uint64_t vfix = 0);
// superblock (1024 logical blocks) sums of nb block sums given in PHYSICAL order (physical block =
// logical ^ mh), then their exclusive prefix: d_prefix[0..nsb] (nsb = ceil(nb/1024)); needs
// 2*nsb + 2 doubles of d_prefix
void launch_scan_blocks(const double *d_phys, double *d_prefix, uint64_t nb, uint64_t mh, cudaStream_t st);
// draws of one leaf (d_ltab = NULL: draw j -> d_out[j], outcome XOR omask) or of a group of nlt
// consecutive leaves sharing this state (d_ltab: nlt + 1 relative slot offsets, then nlt readout
// masks; leaf ids leaf .. leaf + nlt - 1); logical index i lives at physical i ^ xm
double launch_draws(const void *psi, uint32_t n, int prec, uint32_t block_bits, const double *d_phys,
                    const double *d_sprefix, uint64_t n_draws, uint64_t seed, uint64_t leaf, const uint64_t *d_ltab,
                    uint32_t nlt, uint64_t omask, double edge_eps, uint64_t xm, uint64_t *d_out, uint32_t *d_edges,
                    cudaStream_t st, uint64_t *d_blist = nullptr);   // d_blist: only write each draw's block
// sharded mode: the draws of one leaf that fall into this shard's CDF window [t_lo, t_hi)
double launch_draws_window(const void *psi, uint32_t n, int prec, uint32_t block_bits, const double *d_phys,
                           const double *d_sprefix, uint64_t n_draws, uint64_t seed, uint64_t leaf, uint64_t omask,
                           double edge_eps, uint64_t *d_out, uint32_t *d_edges, double t_total, double t_lo,
                           double t_hi, uint64_t ohi, cudaStream_t st);

// slots of leaves whose state is a basis state: ntrip (slot offset, count, value) triples (device)
void launch_fill_slots(const uint64_t *d_trip, uint64_t ntrip, uint64_t *d_slots, cudaStream_t st);

int device_sm_count();

}  // namespace tq
