/*
 * tusq.h -- C ABI of the B200-native TUSQ hot path (arXiv 2508.04880).
 *
 * Problem statement: circuit + noise model + shot count
 * in, output bitstring distribution out.  The calls below are the steps of
 * that path:
 *
 *   tusq_build_error_tree   ECM + TEM tree build and pruning
 *                           (P:310-340): host-only, integer-only, deterministic.
 *   tusq_run_tree           TEM depth-first tree traversal with rollback by
 *                           uncomputation on one 2^n state vector
 *                           in device memory, with leaf sampling.
 *   tusq_sample             |amp|^2 inverse-CDF sampler on a device state.
 *   tusq_apply_ops          state-vector gate application (Eq. 1)
 *                           on a device state (kernel-level entry).
 *   tusq_init_basis         reset a device state to a basis state.
 *
 * Conventions
 *   - Qubit 0 is the least-significant bit of the amplitude index; every qubit
 *     is measured at the end (bitstring bit q = qubit q).
 *   - State vectors are complex128 (interleaved re, im doubles; precision 128)
 *     or complex64 (interleaved floats; precision 64), 2^n entries, 16-byte
 *     aligned, in device memory owned by the CALLER (e.g. a torch tensor).  The
 *     library never frees caller memory.
 *   - Trees are library-owned opaque handles, freed with tusq_tree_free.
 *   - Device calls are ordered on the caller's cudaStream_t (NULL = legacy
 *     default stream).  tusq_run_tree synchronizes its stream before it returns.
 *   - No C++ exception crosses the ABI.  On error the call returns a non-zero
 *     tusq_status, writes no host output buffer, sets output handles to NULL,
 *     and tusq_last_error() (thread-local, valid until the next call on the same
 *     thread) says why.
 *   - There is no CPU fallback: every device step runs in this library's
 *     sm_100a kernels; calls that need a GPU fail with TUSQ_ERR_CUDA without one.
 *   - Thread safety: every call is reentrant.  Trees are immutable after
 *     tusq_build_error_tree and may be shared by threads (e.g. one host thread per
 *     GPU); a communicator and a caller-owned state buffer must be used by one
 *     call at a time.  The library keeps no mutable process-global state besides
 *     lazily initialised, thread-safe caches (device attributes, the NCCL entry
 *     points).
 */
#ifndef TUSQ_ABI_H_
#define TUSQ_ABI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TUSQ_OK = 0,
    TUSQ_ERR_INVALID_ARG = 1,   /* bad gate kind/arity/qubit, p outside [0,1], shots = 0, n > 62, ... */
    TUSQ_ERR_UNSUPPORTED = 2,   /* valid request this build does not implement */
    TUSQ_ERR_OOM = 3,           /* host or device allocation failed */
    TUSQ_ERR_CUDA = 4,          /* CUDA runtime error (incl. no device) */
    TUSQ_ERR_NCCL = 5,          /* NCCL missing or a collective failed (sharded mode) */
    TUSQ_ERR_CAPACITY = 6,      /* state buffer smaller than 2^n * bytes per amplitude */
    TUSQ_ERR_INTERNAL = 7
} tusq_status;

/* Gate kinds: the 1q + CNOT basis of P:211 plus P, CZ, CP. */
enum {
    TUSQ_I = 0, TUSQ_X = 1, TUSQ_Y = 2, TUSQ_Z = 3, TUSQ_H = 4, TUSQ_S = 5, TUSQ_SDG = 6,
    TUSQ_T = 7, TUSQ_TDG = 8, TUSQ_RX = 9, TUSQ_RY = 10, TUSQ_RZ = 11, TUSQ_P = 12,
    TUSQ_CX = 13, TUSQ_CZ = 14, TUSQ_CP = 15
};

/* Pauli codes used in canonical ER triples. */
enum { TUSQ_PAULI_I = 0, TUSQ_PAULI_X = 1, TUSQ_PAULI_Y = 2, TUSQ_PAULI_Z = 3 };

/* One gate, 24 bytes.  q0 = control for two-qubit gates, q1 = target; theta in
 * radians for RX/RY/RZ/P/CP (RZ(t) = diag(e^{-it/2}, e^{it/2}), P(t) = diag(1, e^{it}),
 * CP(t) = e^{it} on |11>). */
typedef struct { uint32_t kind, q0, q1, _pad; double theta; } tusq_op;

/* Noise model (readings #1-#4):
 *   p1     depolarizing (1-p, p/3, p/3, p/3) after every 1q gate on its qubit,
 *   p2     depolarizing after every 2q gate on EACH of its two qubits,
 *   p_meas X flip before readout on every qubit.
 * With flags & TUSQ_NOISE_PAULI the three site classes instead carry general Pauli channels
 * (Eq. 2: rho -> (1 - pX - pY - pZ) rho + pX X rho X + pY Y rho Y + pZ Z rho Z), given
 * as (pX, pY, pZ) in pauli1 / pauli2 / pauli_meas -- e.g. the Pauli-twirled decoherence of
 * tusq_twirl_decoherence, or a depolarizing channel composed with it.  Every p in [0, 1] and each
 * triple's sum <= 1, else TUSQ_ERR_INVALID_ARG.  A channel whose probabilities are all 0 attaches
 * no noise site.  Integer thresholds t_P = round(p_P 2^32), t_I = 2^32 - (t_X + t_Y + t_Z). */
#define TUSQ_NOISE_PAULI 0x1u
typedef struct {
    double p1, p2, p_meas;
    uint32_t flags, _pad;
    double pauli1[3];       /* TUSQ_NOISE_PAULI: (pX, pY, pZ) after every 1q gate */
    double pauli2[3];       /*                   on each qubit of every 2q gate */
    double pauli_meas[3];   /*                   right before readout, every qubit */
} tusq_noise;

/* Pauli-twirling approximation of decoherence for an idle time t (Eq. 2):
 *   pX = pY = (1 - e^{-t/T1}) / 4,  pZ = (1 - e^{-t/T2}) / 2 - (1 - e^{-t/T1}) / 4.
 * out: (pX, pY, pZ).  TUSQ_ERR_INVALID_ARG if t < 0, T1 <= 0, T2 <= 0 or pZ < 0 (T2 > 2 T1 is
 * unphysical). */
tusq_status tusq_twirl_decoherence(double t, double T1, double T2, double out[3]);

/* Pruning (reading #10): significant iff count*alpha_den >= alpha_num*p0;
 * beta >= 1 insignificant leaves kept count-proportionally.  NULL -> 1/100, 100, enabled. */
typedef struct { uint32_t alpha_num, alpha_den, beta, enabled; } tusq_prune;

typedef struct tusq_tree tusq_tree;
/* Communicator of the sharded mode: library-owned, freed with tusq_comm_free. */
typedef struct tusq_comm tusq_comm;

typedef struct {
    uint64_t S1, S2, S3;          /* shots, unique raw ERs (tallying), unique canonical ERs (commutation) */
    uint64_t p0, n_sig, n_insig, n_selected, n_leaves;
    uint64_t n_sites;             /* noise sites M */
    uint64_t n_ops;               /* circuit length L */
    uint64_t edges;               /* |E|: ops on the edges of the prefix trie of leaf op streams */
    uint64_t dftt_ops;            /* pure-uncompute DFTT gate applications = 2|E| - depth(last leaf) */
    uint64_t naive_ops;           /* per-leaf replay from the root: sum of leaf op-stream lengths */
} tusq_tree_info;

/* exec.flags */
#define TUSQ_EXEC_NO_FUSE     0x1u  /* one kernel per gate (K1-K4) instead of fused tiles (K5) */
#define TUSQ_EXEC_NO_RESET    0x2u  /* pure uncompute DFTT: never re-anchor except when the budget is hit */
#define TUSQ_EXEC_NO_SAMPLE   0x4u  /* skip leaf sampling (slots not written) */
#define TUSQ_EXEC_NO_FOLD     0x8u  /* do not fold the classical basis-state prefix into the reset */
#define TUSQ_EXEC_PLAN_ONLY   0x10u /* run the scheduler and planner only: fill stats, launch nothing */
#define TUSQ_EXEC_PROFILE     0x20u /* bracket every gate-kernel launch with CUDA events (stats.gate_kernel_*) */
#define TUSQ_EXEC_CONTINUE    0x40u /* d_state already holds the final state of leaf leaf_begin-1 (left by a
                                       previous call): continue the DFS from there instead of re-anchoring
                                       (a hint: the small-n batched path re-anchors every sub-range) */
#define TUSQ_EXEC_NO_LIVE     0x100u /* no live tiles / valid sets / sums-only sampling: after a re-anchor
                                         every fused sweep visits the whole state (the zeros are written
                                         by the reset), and every sampled state is stored -- the plain
                                         dense state-vector path, for A/B comparison */
#define TUSQ_EXEC_NO_BATCH    0x80u /* n <= 13 (c128) / 14 (c64): do not run the batched on-chip path (one
                                       launch, one DFS sub-range per CTA, state in shared memory) but one
                                       transition at a time like larger n */

/* exec.mode */
#define TUSQ_MODE_REPLICA 0u    /* the whole 2^n vector on this device (leaf ranges shard across replicas) */
#define TUSQ_MODE_SHARDED 1u    /* amplitudes split over comm->nranks shards by the high (global) qubits;
                                   every rank runs the same leaves; slots are summed over ranks */

typedef struct {
    uint32_t precision;         /* 128 (complex128) or 64 (complex64) */
    uint32_t mode;              /* TUSQ_MODE_REPLICA or TUSQ_MODE_SHARDED */
    int32_t  device;            /* CUDA device ordinal; -1 = current */
    uint32_t flags;             /* TUSQ_EXEC_* */
    void    *d_state;           /* caller-owned device buffer of >= 2^n * (precision/8) bytes, or NULL
                                   (library allocates and frees it inside the call).  Sharded mode: this
                                   process's shards, 2^(n-g) amplitudes each (g = log2 nranks): one shard
                                   (NCCL communicator) or all nranks back to back (local communicator);
                                   on return they hold the canonical layout (shard r = global bits r) */
    uint64_t state_bytes;       /* size of d_state */
    void    *stream;            /* cudaStream_t; NULL = legacy default stream */
    uint64_t leaf_begin;        /* DFS leaf range [leaf_begin, leaf_end) to run; */
    uint64_t leaf_end;          /*   leaf_end = 0 means all leaves */
    uint64_t reanchor_budget;   /* re-anchor (reset + replay) once this many gate applications have
                                   accumulated since the last anchor; 0 = default (1e6 c128, 2e4 c64) */
    uint32_t fuse_qubits;       /* tile qubits of the fused kernel: 0 or 12 (the only tile this build
                                   compiles); anything else -> TUSQ_ERR_UNSUPPORTED */
    uint32_t _pad;
    double   edge_eps;          /* edge-draw window (0 = 1e-9 for c128, 1e-5 for c64) */
    tusq_comm *comm;            /* TUSQ_MODE_SHARDED: the communicator (required).
                                   TUSQ_MODE_REPLICA: NULL (single process), or an NCCL communicator
                                   (tusq_comm_init) of the replica ranks: this rank runs its leaf range
                                   (leaf_begin = leaf_end = 0 -> its tusq_tree_partition range) and the
                                   slot arrays of all ranks are summed with ncclAllReduce on the device
                                   (they are disjoint, so the sum is exact); out_slots then receives all
                                   S1 slots on every rank.  A local communicator is rejected here. */
} tusq_exec;

typedef struct {
    uint64_t leaves;            /* leaves traversed */
    uint64_t resets;            /* re-anchors (K7) */
    uint64_t gate_apps;         /* gate applications (forward + inverse) */
    uint64_t launches;          /* kernel launches of this library */
    uint64_t sweeps;            /* full-vector passes by gate kernels (fused groups count once) */
    uint64_t draws;             /* shots drawn */
    uint64_t edge_draws;        /* draws within edge_eps of a CDF edge (GPU's own CDF) */
    double   hbm_bytes;         /* algorithmic HBM bytes of the gate/init kernels */
    double   sample_bytes;      /* algorithmic HBM bytes of the sampler */
    double   host_seconds;      /* host time inside tusq_run_tree (plan + launch + sync) */
    uint64_t gate_kernel_launches;  /* TUSQ_EXEC_PROFILE: gate-kernel launches timed */
    double   gate_kernel_seconds;   /* TUSQ_EXEC_PROFILE: summed CUDA-event durations of those launches */
    double   gate_kernel_bytes;     /* algorithmic HBM bytes of those launches */
    uint64_t fused_launches;        /* K5 launches among `launches` */
    uint64_t exchanges;             /* sharded mode: global<->local qubit swaps (NCCL send/recv of half shards) */
    double   sample_kernel_seconds; /* TUSQ_EXEC_PROFILE: summed CUDA-event durations of the sampler (K6) launches */
    double   device_seconds;        /* CUDA-event time from the first launch of the call to its last one */
    double   reduce_seconds;        /* replica mode with comm: CUDA-event time of the slot all-reduce */
    double   h2d_bytes;             /* host -> device bytes of the call (kernel parameter blocks, draw tables) */
    double   d2h_bytes;             /* device -> host bytes of the call (slots, counters) */
    uint64_t sampled_vectors;       /* state vectors sampled (leaves that share a vector under a terminal
                                       relabel count once) */
    uint64_t dense_sweep_launches;  /* TUSQ_EXEC_PROFILE: K5 launches among gate_kernel_launches that visit
                                       every tile of a fully valid state (no live-tile / valid-set pruning) */
    double   dense_sweep_seconds;   /* their summed CUDA-event durations */
    double   dense_sweep_bytes;     /* their algorithmic HBM bytes (2 x 2^n x amplitude bytes each) */
} tusq_run_stats;

/* ECM + tree.  ops: n_ops gates (host).  seed keys every Philox stream.
 * Returns a library-owned tree in *out (NULL on error). */
tusq_status tusq_build_error_tree(uint32_t n_qubits, const tusq_op *ops, uint64_t n_ops,
                                  const tusq_noise *noise, uint64_t shots, uint64_t seed,
                                  const tusq_prune *prune, tusq_tree **out);

tusq_status tusq_tree_get_info(const tusq_tree *tree, tusq_tree_info *out);

/* Canonical serialization (little-endian):
 *   "TUSQTRE1", u32 n_qubits, u32 0, u64 n_ops, u64 shots, u64 seed,
 *   u64 S2, S3, p0, n_sig, n_insig, n_selected, n_leaves,
 *   per leaf in DFS order: u64 count, u64 offset, u32 n_triples, n_triples x (u32 pos, q, P).
 * A triple (pos, q, P) applies Pauli P on qubit q right before gate pos (pos = n_ops: after the
 * last gate).  buf = NULL -> *inout_len = required size.  TUSQ_ERR_CAPACITY if too small. */
tusq_status tusq_tree_serialize(const tusq_tree *tree, uint8_t *buf, uint64_t *inout_len);

/* One leaf: shot count, shot offset and its canonical triples (*inout_n: capacity in triples
 * on input, number of triples on output). */
tusq_status tusq_tree_leaf(const tusq_tree *tree, uint64_t leaf, uint64_t *count, uint64_t *offset,
                           uint32_t *triples, uint32_t *inout_n);

/* Contiguous DFS leaf ranges for nranks replicas balanced by the host cost model
 * (SURVEY 8(e)): bounds[r]..bounds[r+1] for r < nranks (nranks + 1 entries).  The model replays
 * the default scheduler of tusq_run_tree for `precision` (64 or 128): hybrid reset-vs-uncompute
 * per transition (an uncompute only when the reset's replay is >= 16x longer: live tiles make
 * replays cheap), plus the precision's re-anchor budget (1e6 gate applications c128, 2e4 c64),
 * costed in gate applications.  (Device time tracks full sweeps more than gate counts, so callers
 * that can should interleave finer ranges over their ranks -- bench.py does.) */
tusq_status tusq_tree_partition(const tusq_tree *tree, uint32_t nranks, uint32_t precision, uint64_t *bounds);

void tusq_tree_free(tusq_tree *tree);

/* DFTT over leaves [leaf_begin, leaf_end).  out_slots: host array of length S1;
 * slot i receives the bitstring of shot i for the shots of the leaves run (other slots untouched).
 * On return d_state holds the final state of the last leaf run.  stats may be NULL. */
tusq_status tusq_run_tree(const tusq_tree *tree, const tusq_exec *exec, uint64_t *out_slots,
                          tusq_run_stats *stats);

/* Sharded mode communicators (34q QFT at c128 = 256 GiB over 8 B200s).
 *   tusq_comm_unique_id  ncclGetUniqueId on one rank; broadcast the 128 bytes to the others.
 *   tusq_comm_init       one process per GPU: ncclCommInitRank(nranks, id, rank) on `device`.
 *   tusq_comm_init_local all nshards shards in THIS process on one device (exchanges are device
 *                        swaps): the same sharded logic, testable on one GPU.
 * nranks / nshards must be a power of two >= 2.  NCCL is loaded at run time (libnccl.so.2);
 * TUSQ_ERR_NCCL if it is missing or a collective fails. */
tusq_status tusq_comm_unique_id(uint8_t out[128]);
tusq_status tusq_comm_init(const uint8_t id[128], int nranks, int rank, int device, tusq_comm **out);
tusq_status tusq_comm_init_local(int nshards, int device, tusq_comm **out);
void tusq_comm_free(tusq_comm *comm);

/* Replica mode, one process per GPU (SURVEY 8(e), P:316 parallel sub-trees): every rank ran its
 * own DFS leaf ranges into its own host slot array (zeros elsewhere); this sums the arrays of all
 * ranks in place with one ncclAllReduce on the device (u64, exact: the ranks' slots are
 * disjoint), so every rank ends with all n slots.  slots: host array of n u64 (in/out).
 * comm: an NCCL communicator (tusq_comm_init); TUSQ_ERR_INVALID_ARG for a local one.
 * Synchronizes `stream` before returning. */
tusq_status tusq_reduce_slots(tusq_comm *comm, uint64_t *slots, uint64_t n, void *stream);

/* Inverse-CDF draws from |amp|^2 of a device state: draw j uses Philox counter
 * (j, leaf_lo, leaf_hi, 0x53000000) keyed by seed, u = (x >> 11) 2^-53, t = u * sum|amp|^2,
 * outcome min{k : C(k) > t}.  d_out: device array of n_draws u64. */
tusq_status tusq_sample(const void *d_state, uint32_t n_qubits, uint32_t precision, uint64_t n_draws,
                        uint64_t seed, uint64_t leaf_id, uint64_t *d_out, void *stream);

/* Apply n_ops gates (host array) to a device state in order; flags: TUSQ_APPLY_INVERSE applies
 * the inverse circuit (inverse gates in reverse order); TUSQ_APPLY_UNFUSED forces one kernel per gate. */
#define TUSQ_APPLY_INVERSE   0x1u
#define TUSQ_APPLY_UNFUSED   0x2u
/* TUSQ_APPLY_PLAN_ONLY: run the host planner only (no device access; d_state may be any non-NULL
 * value); with TUSQ_DEBUG_PLAN=2 in the environment the K5 group plans are printed to stderr. */
#define TUSQ_APPLY_PLAN_ONLY 0x4u
tusq_status tusq_apply_ops(void *d_state, uint32_t n_qubits, uint32_t precision, const tusq_op *ops,
                           uint64_t n_ops, uint32_t flags, void *stream);

/* d_state <- amp * |index> (amp = re + i im). */
tusq_status tusq_init_basis(void *d_state, uint32_t n_qubits, uint32_t precision, uint64_t index,
                            double re, double im, void *stream);

const char *tusq_last_error(void);
const char *tusq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TUSQ_ABI_H_ */
