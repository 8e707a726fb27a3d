// Execution context, gate-kernel timing and the K5 fused-tile planner interface.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "common.h"

namespace tq {

// CUDA-event brackets around kernel launches (TUSQ_EXEC_PROFILE): category 0 = gate kernels
// (K1-K5, K7), 1 = sampler kernels (K6).  Read once by flush() at the end of a call.
class GateTimer {
public:
    explicit GateTimer(bool on) : on_(on) {}
    ~GateTimer();
    bool on() const { return on_; }
    void begin(cudaStream_t st);
    void end(cudaStream_t st, double bytes, int cat = 0);
    void flush();                 // synchronizes the recorded events and accumulates
    size_t pending() const { return used_; }
    uint64_t launches = 0, dense_launches = 0;
    double seconds = 0.0, bytes = 0.0, sample_seconds = 0.0, dense_seconds = 0.0, dense_bytes = 0.0;

private:
    bool on_;
    std::vector<cudaEvent_t> a_, b_;
    std::vector<double> by_;
    std::vector<uint8_t> cat_;
    size_t used_ = 0;
};

struct Ctx {
    void *psi = nullptr;
    uint32_t n = 0;
    int prec = 128;
    cudaStream_t st = nullptr;
    bool dry = false;             // TUSQ_EXEC_PLAN_ONLY: count, launch nothing
    tusq_run_stats *stats = nullptr;
    GateTimer *timer = nullptr;
};

// Fused-tile planner (K5).  Splits an op stream into groups whose qubits fit a tile of 2^tile_bits
// amplitudes and applies each group in one HBM sweep; keeps a pending X-relabel mask between
// sweeps (physical index = logical index XOR mask).
struct InitState { uint64_t index; double re, im; };   // reset target (K7 fused into the first sweep)

struct PlanScratch;   // the K5 parameter block under construction (fused.cu), one per planner

// Thread safety: a planner is used by one host thread at a time; distinct planners (and so
// concurrent tusq_run_tree / tusq_apply_ops calls) share no mutable state.
class FusedPlanner {
public:
    FusedPlanner(uint32_t n, int prec);
    uint32_t tile_bits() const { return tile_bits_; }
    bool enabled() const { return enabled_; }
    void execute(const std::vector<Op> &ops, Ctx &ctx);
    // init: the state is first reset to init (no load); d_sums: if the last sweep's tile is the
    // contiguous block {0..11}, it writes per-block |amp|^2 sums (physical block order) there.
    // sums_only: the caller samples this state and then discards it (the next transition resets):
    // the last sweep writes only the block sums (if it produces them) and replay_tiles() then
    // computes and stores just the tiles the sampler's draws land in
    bool execute_ex(const std::vector<Op> &ops, Ctx &ctx, const InitState *init, double *d_sums,
                    bool *sums_written, bool sums_only = false);
    bool pending_tiles() const { return pending_tiles_; }
    // d_blist: n logical block indices (the sampler's chosen blocks, repeats allowed); mh: the
    // sampler's physical-block XOR (xmask() >> 12)
    void replay_tiles(Ctx &ctx, const uint64_t *d_blist, uint64_t n, uint64_t mh);
    // the logical state may be stored XOR-relabelled; materialize() clears the mask
    uint64_t xmask() const { return xmask_; }
    // a second device buffer of the state's size: enables the layout-changing (out-of-place) sweeps
    // whose tile reads are contiguous; NULL = every sweep in place
    void set_alt(void *alt) { alt_ = alt; }
    // or: allocate it (stream-ordered, `bytes`) only when a call has >= 2 groups; release() frees it
    void set_alt_lazy(uint64_t bytes) { alt_lazy_ = bytes; }
    // live tiles / valid sets off (TUSQ_EXEC_NO_LIVE): every sweep visits the whole state
    void set_live(bool on) { live_ = on; }
    void release(cudaStream_t st)
    {
        if (alt_owned_ && alt_) cudaFreeAsync(alt_, st);
        if (alt_owned_) alt_ = nullptr;
        alt_owned_ = false;
    }
    void materialize(Ctx &ctx);
    void reset_mask() { xmask_ = 0; }
    // the caller wrote the basis state |index> (K7) into the state: the known support is one element
    // and the whole buffer is valid
    void note_basis(uint64_t index) { xmask_ = 0; dfree_ = 0; dfix_ = index; vfree_ = ~0ull; vfix_ = 0; stale_ = false; }
    // The buffer may hold the state only on a valid set V = {x : (x & ~vfree) == vfix} (physical,
    // identity layout; outside it the state is zero and the buffer stale).  Readers outside K5:
    // close_blocks() makes V a union of whole 2^12-element blocks (zeros written inside the blocks
    // V touches) before the sampler's block sums, which skip the blocks outside V; finish() writes
    // the zeros outside V so the caller's buffer holds the whole state.
    void valid_set(uint64_t *vfree, uint64_t *vfix) const { *vfree = vfree_; *vfix = vfix_; }
    void close_blocks(Ctx &ctx, uint32_t block_bits);
    void finish(Ctx &ctx);

private:
    uint32_t n_;
    int prec_;
    uint32_t tile_bits_;
    bool enabled_;
    uint64_t xmask_ = 0;
    // known support of the state in ctx.psi (physical positions, identity layout): every nonzero
    // amplitude has (index & ~dfree_) == dfix_; dfree_ = ~0 when unknown
    uint64_t dfree_ = ~0ull, dfix_ = 0;
    uint64_t vfree_ = ~0ull, vfix_ = 0;   // the valid set V (see valid_set)
    bool pending_tiles_ = false, stale_ = false, live_ = true;
    void *alt_ = nullptr;
    uint64_t alt_lazy_ = 0;
    bool alt_owned_ = false;
    std::shared_ptr<PlanScratch> scratch_;
};

// one kernel per gate (K1-K4); consecutive Paulis on distinct qubits merge into one K4 pass
void execute_unfused(const std::vector<Op> &ops, Ctx &ctx);

// communicators (sharded.cu)
bool comm_is_local(const tusq_comm *c);
int comm_rank(const tusq_comm *c);
int comm_nranks(const tusq_comm *c);
tusq_status comm_allreduce_u64(tusq_comm *c, uint64_t *d, uint64_t n, cudaStream_t st, std::string &err);

// batched sub-trees with on-chip state for small n (smallsim.cu): the leaf range [lb, le) in one
// launch; draws go to d_slots (slot index - off0); the final state of leaf le-1 to psi
uint32_t small_max_qubits(int prec);
tusq_status run_tree_small(const tusq_tree *t, const tusq_exec *ex, uint64_t lb, uint64_t le, void *psi,
                           uint64_t *d_slots, uint64_t off0, uint32_t *d_edges, double eps, tusq_run_stats &stats);

// tusq_run_tree in TUSQ_MODE_SHARDED (sharded.cu)
tusq_status run_tree_sharded(const tusq_tree *t, const tusq_exec *ex, uint64_t *out_slots, tusq_run_stats *stats);

}  // namespace tq
