// Sharded mode: above one GPU's HBM the 2^n amplitudes are split over R = 2^g shards
// by the g high-order ("global") qubit positions; each shard holds 2^(n-g) amplitudes.
//
//   - gates on local qubits run on every shard with the fused / per-gate kernels (K1-K5);
//   - diagonal gates and Z on a global qubit are per-shard phases (no data touched; applied lazily
//     before the next exchange -- |amp|^2 sampling never needs them);
//   - X on a global qubit, and CX between global qubits, relabel which shard holds which
//     global pattern (zero communication);
//   - CX / CZ / CP with a global control become a shard-conditional local X / Z / P;
//   - a dense gate (H, RX, RY) on a global qubit, or CX with a global target and local control,
//     first swaps that qubit with the top local qubit (the "slot", position n-g-1): shard pairs
//     exchange contiguous halves -- NCCL send/recv over NVLink between ranks, or an in-place
//     swap kernel when all shards live on one device (the "local" communicator used to test the
//     same logic on one GPU).
// Because only the slot ever trades places with global positions, the logical qubits at
// {slot, globals} are always {n-g-1, ..., n-1}: restoring the canonical layout before sampling is a
// cycle sort through the slot (<= g+1 exchanges).  Sampling then walks the shards in logical
// order: per-shard |amp|^2 totals (all-reduced across ranks) give every draw's owning shard, which
// searches locally (K6 with a shard window).  Shot slots are disjoint and summed once at the end.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "fused.h"
#include "kernels.h"

// ---------------------------------------------------------------- NCCL (loaded at run time)
namespace tq {
namespace nccl {
struct Api {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
// libnccl.so.2 is resolved at first use (the one torch already loaded, if any): the library itself
// loads and runs replica mode on machines without NCCL.  Thread-safe (std::call_once).
static Api &api()
{
    static Api a;
    static std::once_flag once;
    std::call_once(once, []() {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define TQ_SYM(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f)); if (!a.f) return;
        TQ_SYM(GetUniqueId) TQ_SYM(CommInitRank) TQ_SYM(CommDestroy) TQ_SYM(GroupStart) TQ_SYM(GroupEnd)
        TQ_SYM(Send) TQ_SYM(Recv) TQ_SYM(AllReduce) TQ_SYM(GetErrorString)
#undef TQ_SYM
        a.ok = true;
    });
    return a;
}
}  // namespace nccl
}  // namespace tq

struct tusq_comm {
    int nranks = 1;          // R shards (power of two)
    int rank = 0;            // this process's shard (NCCL mode)
    bool local = false;      // all R shards in this process, on one device
    int device = -1;
    ncclComm_t nc = nullptr;
};

namespace tq {

bool comm_is_local(const tusq_comm *c) { return c->local; }
int comm_rank(const tusq_comm *c) { return c->rank; }
int comm_nranks(const tusq_comm *c) { return c->nranks; }

// replica mode: sum the ranks' (disjoint) u64 slot arrays in place on the device
tusq_status comm_allreduce_u64(tusq_comm *c, uint64_t *d, uint64_t n, cudaStream_t st, std::string &err)
{
    auto &a = nccl::api();
    if (!a.ok) { err = "libnccl.so.2 not available"; return TUSQ_ERR_NCCL; }
    ncclResult_t r = a.AllReduce(d, d, n, ncclUint64, ncclSum, c->nc, st);
    if (r != ncclSuccess) { err = std::string("ncclAllReduce: ") + a.GetErrorString(r); return TUSQ_ERR_NCCL; }
    return TUSQ_OK;
}

// ---------------------------------------------------------------- device helpers
template <typename V>
__global__ void k_swap(V *__restrict__ a, V *__restrict__ b, uint64_t n)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        V x = a[i], y = b[i];
        a[i] = y;
        b[i] = x;
    }
}

template <typename V, typename R>
__global__ void k_scale(V *__restrict__ a, uint64_t n, R cr, R ci)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        V x = a[i];
        a[i].x = x.x * cr - x.y * ci;
        a[i].y = x.x * ci + x.y * cr;
    }
}

static unsigned grid_for(uint64_t n)
{
    const uint64_t cap = (uint64_t)device_sm_count() * 8;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cap, (n + 255) / 256));
}

// values of a one-qubit diagonal gate on |0>, |1>
static void diag_vals(const Op &o, std::complex<double> &d0, std::complex<double> &d1)
{
    using C = std::complex<double>;
    const double r = M_SQRT1_2;
    d0 = 1.0;
    switch (o.kind) {
    case Z: d1 = -1.0; break;
    case S: d1 = C(0, 1); break;
    case SDG: d1 = C(0, -1); break;
    case T: d1 = C(r, r); break;
    case TDG: d1 = C(r, -r); break;
    case RZ: d0 = std::polar(1.0, -o.theta / 2); d1 = std::polar(1.0, o.theta / 2); break;
    case P: d1 = std::polar(1.0, o.theta); break;
    default: d1 = 1.0; break;
    }
}

namespace {

struct ShardRun {
    uint32_t n = 0, g = 0, nl = 0;
    int prec = 128;
    uint64_t R = 1, half = 0;                  // shards; amplitudes per half shard
    size_t esz = 16;
    tusq_comm *comm = nullptr;
    cudaStream_t st = nullptr;
    bool dry = false, fuse = true;
    std::vector<int> mine;                     // physical shards driven by this process
    std::vector<void *> buf;                   // device buffer per physical shard (nullptr if not mine)
    std::vector<uint32_t> pos, lq;             // logical qubit -> physical position, inverse
    std::vector<uint64_t> shard_of, v_of;      // global pattern -> physical shard, inverse
    std::vector<std::complex<double>> ph;      // pending phase per physical shard
    std::vector<std::vector<Op>> ops;          // pending local ops per physical shard
    std::vector<FusedPlanner> planners;        // per physical shard (own X-relabel mask)
    void *stage = nullptr;                     // NCCL exchange staging: two halves, alternating chunks
    uint64_t stage_amps = 0;
    cudaStream_t st2 = nullptr;                // copy-back stream of the exchange pipeline
    cudaEvent_t ev_recv[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr}, ev_done = nullptr;
    tusq_run_stats *stats = nullptr;
    GateTimer *timer = nullptr;

    bool glob(uint32_t q) const { return pos[q] >= nl; }
    uint32_t gb(uint32_t q) const { return pos[q] - nl; }
    uint64_t vbit(uint64_t s, uint32_t q) const { return (v_of[s] >> gb(q)) & 1; }

    Ctx ctx_for(int s)
    {
        Ctx c;
        c.psi = buf[s];
        c.n = nl;
        c.prec = prec;
        c.st = st;
        c.dry = dry;
        c.stats = stats;
        c.timer = timer;
        return c;
    }

    void flush()
    {
        for (int s : mine) {
            Ctx c = ctx_for(s);
            if (!ops[s].empty()) {
                if (fuse) planners[s].execute(ops[s], c);
                else execute_unfused(ops[s], c);
                ops[s].clear();
            }
            if (fuse) planners[s].materialize(c);
        }
    }

    void apply_phases()
    {
        for (int s : mine) {
            if (ph[s] == std::complex<double>(1.0, 0.0)) continue;
            if (!dry) {
                const uint64_t na = 2 * half;
                if (prec == 128)
                    k_scale<double2, double><<<grid_for(na), 256, 0, st>>>((double2 *)buf[s], na, ph[s].real(), ph[s].imag());
                else
                    k_scale<float2, float><<<grid_for(na), 256, 0, st>>>((float2 *)buf[s], na, (float)ph[s].real(),
                                                                         (float)ph[s].imag());
            }
            stats->launches++;
            stats->hbm_bytes += 2.0 * (double)(2 * half) * (double)esz;
            ph[s] = 1.0;
        }
    }

    // swap the qubit at global bit k with the slot (local position nl-1)
    void exchange(uint32_t k)
    {
        flush();
        apply_phases();
        const uint64_t bitk = 1ull << k;
        for (uint64_t v0 = 0; v0 < R; ++v0) {
            if (v0 & bitk) continue;
            const uint64_t A = shard_of[v0], Bs = shard_of[v0 | bitk];
            // A's upper half (slot = 1) <-> B's lower half (slot = 0)
            if (comm->local) {
                if (!dry) {
                    char *a = (char *)buf[A] + half * esz, *b = (char *)buf[Bs];
                    if (prec == 128) k_swap<double2><<<grid_for(half), 256, 0, st>>>((double2 *)a, (double2 *)b, half);
                    else k_swap<float2><<<grid_for(half), 256, 0, st>>>((float2 *)a, (float2 *)b, half);
                }
                stats->launches++;
            } else if ((int)A == comm->rank || (int)Bs == comm->rank) {
                const bool am_a = (int)A == comm->rank;
                const int peer = (int)(am_a ? Bs : A);
                char *mine_half = (char *)buf[comm->rank] + (am_a ? half * esz : 0);
                if (!dry) nccl_swap(mine_half, peer);
            }
            stats->hbm_bytes += 4.0 * (double)half * (double)esz;
        }
        stats->sweeps++;
        const uint32_t pg = nl + k, pl = nl - 1;
        std::swap(lq[pg], lq[pl]);
        pos[lq[pg]] = pg;
        pos[lq[pl]] = pl;
        exchanges++;
    }

    // Swap `region` (half a shard) with the peer's matching half: chunk i is sent from the region
    // and received into staging half i % 2 on the main stream, then copied back into the region on
    // st2 while chunk i + 1 is on the wire (NVLink ~0.9 TB/s vs the ~6.5 TB/s copy: the copy-back
    // hides behind the transfer).  Chunk i + 2 reuses staging half i % 2 after its copy-back.
    void nccl_swap(char *region, int peer)
    {
        auto &a = nccl::api();
        const uint64_t bytes = half * esz, chunk = (stage_amps / 2) * esz;
        char *stg[2] = {(char *)stage, (char *)stage + chunk};
        auto cu = [](cudaError_t e, const char *what) {
            if (e != cudaSuccess) throw std::runtime_error(std::string("exchange: ") + what + ": " + cudaGetErrorString(e));
        };
        uint64_t i = 0;
        for (uint64_t off = 0; off < bytes; off += chunk, ++i) {
            const uint64_t len = std::min(chunk, bytes - off);
            const int b = (int)(i & 1);
            if (i >= 2) cu(cudaStreamWaitEvent(st, ev_copied[b], 0), "wait copy-back");
            check(a.GroupStart());
            check(a.Send(region + off, len, ncclUint8, peer, comm->nc, st));
            check(a.Recv(stg[b], len, ncclUint8, peer, comm->nc, st));
            check(a.GroupEnd());
            cu(cudaEventRecord(ev_recv[b], st), "record");
            cu(cudaStreamWaitEvent(st2, ev_recv[b], 0), "wait recv");
            cu(cudaMemcpyAsync(region + off, stg[b], len, cudaMemcpyDeviceToDevice, st2), "copy-back");
            cu(cudaEventRecord(ev_copied[b], st2), "record");
        }
        cu(cudaEventRecord(ev_done, st2), "record");
        cu(cudaStreamWaitEvent(st, ev_done, 0), "join");
    }

    void check(ncclResult_t r)
    {
        if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + nccl::api().GetErrorString(r));
    }

    void relabel(const std::vector<uint64_t> &src)   // new shard_of[v] = shard_of[src[v]]
    {
        std::vector<uint64_t> ns(R);
        for (uint64_t v = 0; v < R; ++v) ns[v] = shard_of[src[v]];
        shard_of = ns;
        for (uint64_t v = 0; v < R; ++v) v_of[shard_of[v]] = v;
    }

    void local_op(const Op &o, uint64_t s) { ops[s].push_back(o); }

    void apply(const Op &o0)
    {
        Op o = o0;
        if (o.kind == I) return;
        const bool two = two_qubit(o.kind);
        if (!glob(o.q0) && (!two || !glob(o.q1))) {   // all local
            Op p = o;
            p.q0 = pos[o.q0];
            if (two) p.q1 = pos[o.q1];
            for (int s : mine) local_op(p, s);
            return;
        }
        using C = std::complex<double>;
        if (!two) {
            const uint32_t k = gb(o.q0);
            if (is_diag1(o.kind)) {
                C d0, d1;
                diag_vals(o, d0, d1);
                for (uint64_t s = 0; s < R; ++s) ph[s] *= vbit(s, o.q0) ? d1 : d0;
                return;
            }
            if (o.kind == X || o.kind == Y) {
                if (o.kind == Y)   // (Y psi)(b) = -i psi(1) for b = 0, +i psi(0) for b = 1
                    for (uint64_t s = 0; s < R; ++s) ph[s] *= vbit(s, o.q0) ? C(0, -1) : C(0, 1);
                std::vector<uint64_t> src(R);
                for (uint64_t v = 0; v < R; ++v) src[v] = v ^ (1ull << k);
                relabel(src);
                return;
            }
            exchange(k);   // dense: bring the qubit to the slot
            Op p = o;
            p.q0 = pos[o.q0];
            for (int s : mine) local_op(p, s);
            return;
        }
        const uint32_t c = o.q0, t = o.q1;
        if (o.kind == CX) {
            if (glob(c) && glob(t)) {
                const uint32_t kc = gb(c), kt = gb(t);
                std::vector<uint64_t> src(R);
                for (uint64_t v = 0; v < R; ++v) src[v] = ((v >> kc) & 1) ? v ^ (1ull << kt) : v;
                relabel(src);
                return;
            }
            if (glob(t)) {              // local control, global target: the target moves to the slot
                exchange(gb(t));
                if (glob(c)) { apply(o); return; }   // the control sat in the slot: now global
                Op p = o;
                p.q0 = pos[c];
                p.q1 = pos[t];
                for (int s : mine) local_op(p, s);
                return;
            }
            // global control, local target: X on the shards whose control bit is 1
            for (int s : mine)
                if (vbit(s, c)) local_op(Op{X, pos[t], 0, 0.0}, s);
            return;
        }
        // CZ / CP: symmetric diagonals
        const C e = o.kind == CZ ? C(-1.0, 0.0) : std::polar(1.0, o.theta);
        if (glob(c) && glob(t)) {
            for (uint64_t s = 0; s < R; ++s)
                if (vbit(s, c) && vbit(s, t)) ph[s] *= e;
            return;
        }
        const uint32_t gq = glob(c) ? c : t, lqb = glob(c) ? t : c;
        for (int s : mine)
            if (vbit(s, gq)) local_op(o.kind == CZ ? Op{Z, pos[lqb], 0, 0.0} : Op{P, pos[lqb], 0, o.theta}, s);
    }

    // reset to amp |index> in the canonical layout
    void reset(uint64_t index, double re, double im)
    {
        for (int s : mine) ops[s].clear();
        for (uint32_t q = 0; q < n; ++q) pos[q] = lq[q] = q;
        for (uint64_t v = 0; v < R; ++v) shard_of[v] = v_of[v] = v;
        for (auto &x : ph) x = 1.0;
        const uint64_t vi = index >> nl, li = index & ((1ull << nl) - 1);
        for (int s : mine) {
            if (fuse) planners[s].reset_mask();
            if (!dry) {
                if ((uint64_t)s == vi) launch_init_basis(buf[s], nl, prec, li, re, im, st);
                else if (cudaMemsetAsync(buf[s], 0, 2 * half * esz, st) != cudaSuccess)
                    throw std::runtime_error("cudaMemsetAsync failed");
            }
            stats->launches++;
            stats->hbm_bytes += (double)(2 * half * esz);
        }
        stats->resets++;
    }

    // canonical layout: cycle sort of {slot, globals} through the slot, then shard data back in place
    void canonical_positions()
    {
        for (;;) {
            const uint32_t ql = lq[nl - 1];
            if (ql != nl - 1) { exchange(ql - nl); continue; }   // put the slot's qubit home
            uint32_t k = g;
            for (uint32_t j = 0; j < g; ++j)
                if (lq[nl + j] != nl + j) { k = j; break; }
            if (k == g) break;
            exchange(k);                                         // park a misplaced global in the slot
        }
    }

    void canonical_shards()   // physical shard s holds pattern s (data moves)
    {
        flush();
        apply_phases();
        for (uint64_t v = 0; v < R; ++v) {
            const uint64_t s = shard_of[v];
            if (s == v) continue;
            // swap the contents of shards v and s, then fix the maps
            if (comm->local) {
                if (!dry) {
                    if (prec == 128) k_swap<double2><<<grid_for(2 * half), 256, 0, st>>>((double2 *)buf[v], (double2 *)buf[s], 2 * half);
                    else k_swap<float2><<<grid_for(2 * half), 256, 0, st>>>((float2 *)buf[v], (float2 *)buf[s], 2 * half);
                }
            } else if ((uint64_t)comm->rank == v || (uint64_t)comm->rank == s) {
                const int peer = (int)((uint64_t)comm->rank == v ? s : v);
                if (!dry) {
                    nccl_swap((char *)buf[comm->rank], peer);
                    nccl_swap((char *)buf[comm->rank] + half * esz, peer);
                }
            }
            stats->hbm_bytes += 4.0 * (double)(2 * half) * (double)esz;
            const uint64_t w = v_of[v];   // the pattern shard v held
            shard_of[w] = s;
            v_of[s] = w;
            shard_of[v] = v;
            v_of[v] = v;
        }
    }

    uint64_t exchanges = 0;
};

}  // namespace


tusq_status run_tree_sharded(const tusq_tree *t, const tusq_exec *ex, uint64_t *out_slots, tusq_run_stats *stats_out)
{
    auto t0 = std::chrono::steady_clock::now();
    tusq_comm *comm = reinterpret_cast<tusq_comm *>(ex->comm);
    if (!comm) return fail(TUSQ_ERR_INVALID_ARG, "sharded mode needs a communicator (tusq_comm_init*)");
    const uint64_t R = (uint64_t)comm->nranks;
    if (R < 2 || (R & (R - 1))) return fail(TUSQ_ERR_INVALID_ARG, "sharded mode: nranks must be a power of two >= 2");
    const uint32_t n = t->n;
    uint32_t g = 0;
    while ((1ull << g) < R) ++g;
    if (n < g + 2) return fail(TUSQ_ERR_INVALID_ARG, "sharded mode: n must exceed log2(nranks) + 1");
    const bool dry = ex->flags & TUSQ_EXEC_PLAN_ONLY;
    const bool sample = !(ex->flags & TUSQ_EXEC_NO_SAMPLE);
    if (sample && !dry && !out_slots) return fail(TUSQ_ERR_INVALID_ARG, "out_slots is NULL");
    ShardRun S;
    S.n = n; S.g = g; S.nl = n - g; S.prec = (int)ex->precision; S.R = R;
    S.esz = S.prec == 128 ? 16 : 8;
    S.half = 1ull << (S.nl - 1);
    S.comm = comm; S.st = (cudaStream_t)ex->stream; S.dry = dry;
    const uint64_t shard_bytes = (2 * S.half) * S.esz;
    const uint64_t nleaf = t->leaves.size();
    const uint64_t lb = ex->leaf_begin, le = ex->leaf_end ? ex->leaf_end : nleaf;
    if (lb > le || le > nleaf) return fail(TUSQ_ERR_INVALID_ARG, "leaf range out of bounds");
    if (!dry) {
        const int dev = ex->device >= 0 ? ex->device : comm->device;
        if (dev >= 0 && cudaSetDevice(dev) != cudaSuccess) return fail(TUSQ_ERR_CUDA, "cudaSetDevice failed");
    }
    if (comm->local) for (uint64_t s = 0; s < R; ++s) S.mine.push_back((int)s);
    else S.mine.push_back(comm->rank);
    const uint64_t need = shard_bytes * S.mine.size();
    S.buf.assign(R, nullptr);
    bool own = false;
    char *base = (char *)ex->d_state;
    std::vector<void *> allocs;
    if (base) {
        if (ex->state_bytes < need) return fail(TUSQ_ERR_CAPACITY, "state buffer smaller than this process's shards");
    } else if (!dry) {
        if (cudaMalloc((void **)&base, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(TUSQ_ERR_CAPACITY, "cannot allocate the shard buffers on this device");
        }
        own = true;
    }
    for (size_t i = 0; i < S.mine.size(); ++i)
        S.buf[S.mine[i]] = dry ? reinterpret_cast<void *>(16 + i) : base + i * shard_bytes;
    tusq_run_stats stats{};
    S.stats = &stats;
    GateTimer timer(!dry && (ex->flags & TUSQ_EXEC_PROFILE));
    S.timer = timer.on() ? &timer : nullptr;
    S.pos.resize(n); S.lq.resize(n);
    S.shard_of.resize(R); S.v_of.resize(R);
    S.ph.assign(R, 1.0);
    S.ops.resize(R);
    for (uint64_t s = 0; s < R; ++s) S.planners.emplace_back(S.nl, S.prec);
    S.fuse = !(ex->flags & TUSQ_EXEC_NO_FUSE) && S.planners[0].enabled();
    const uint32_t bb = S.nl < 12 ? S.nl : 12;
    const uint64_t nb = 1ull << (S.nl - bb);
    const uint64_t off0 = lb < le ? t->leaves[lb].offset : 0;
    const uint64_t off1 = lb < le ? t->leaves[le - 1].offset + t->leaves[le - 1].count : 0;
    uint64_t *d_slots = nullptr;
    double *d_blocks = nullptr, *d_tot = nullptr;
    uint32_t *d_edges = nullptr;
    auto cleanup = [&]() {
        if (d_slots) cudaFree(d_slots);
        if (d_blocks) cudaFree(d_blocks);
        if (d_tot) cudaFree(d_tot);
        if (d_edges) cudaFree(d_edges);
        if (S.stage) cudaFree(S.stage);
        for (cudaEvent_t e : {S.ev_recv[0], S.ev_recv[1], S.ev_copied[0], S.ev_copied[1], S.ev_done})
            if (e) cudaEventDestroy(e);
        if (S.st2) cudaStreamDestroy(S.st2);
        if (own) cudaFree(base);
    };
#define TQ_SH_CUDA(call)                                                                             \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) { cleanup(); return fail(TUSQ_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); } \
    } while (0)
    const size_t nsb = (nb + 1023) / 1024;
    const size_t blk_stride = 2 * nb + 2 * nsb + 16;   // per shard: block sums + superblock prefix
    if (!dry) {
        const uint64_t nslots = std::max<uint64_t>(1, off1 - off0);
        TQ_SH_CUDA(cudaMalloc((void **)&d_slots, nslots * sizeof(uint64_t)));
        TQ_SH_CUDA(cudaMemsetAsync(d_slots, 0, nslots * sizeof(uint64_t), S.st));
        TQ_SH_CUDA(cudaMalloc((void **)&d_blocks, S.mine.size() * blk_stride * sizeof(double)));
        TQ_SH_CUDA(cudaMalloc((void **)&d_tot, R * sizeof(double)));
        TQ_SH_CUDA(cudaMalloc((void **)&d_edges, sizeof(uint32_t)));
        TQ_SH_CUDA(cudaMemsetAsync(d_edges, 0, sizeof(uint32_t), S.st));
        if (!comm->local) {
            if (!nccl::api().ok) { cleanup(); return fail(TUSQ_ERR_NCCL, "libnccl.so.2 not available"); }
            // 2 x 128 MiB staging (even element count: two equal halves)
            S.stage_amps = std::min<uint64_t>(2 * S.half, (256ull << 20) / S.esz) & ~1ull;
            TQ_SH_CUDA(cudaMalloc(&S.stage, S.stage_amps * S.esz));
            TQ_SH_CUDA(cudaStreamCreateWithFlags(&S.st2, cudaStreamNonBlocking));
            for (cudaEvent_t *e : {&S.ev_recv[0], &S.ev_recv[1], &S.ev_copied[0], &S.ev_copied[1], &S.ev_done})
                TQ_SH_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
    }
    const double eps = ex->edge_eps > 0 ? ex->edge_eps : (S.prec == 128 ? 1e-9 : 1e-5);
    const bool hybrid = !(ex->flags & TUSQ_EXEC_NO_RESET);
    const uint64_t budget = ex->reanchor_budget ? ex->reanchor_budget : (S.prec == 128 ? 1000000ull : 20000ull);
    std::vector<Op> seq;
    uint64_t since_anchor = 0;
    try {
        const uint32_t L = (uint32_t)t->gates.size();
        Leaf prev_core;
        for (uint64_t li = lb; li < le; ++li) {
            // executed part of the leaf; terminal X flips relabel its draws (reading #7)
            uint64_t omask = 0;
            const Leaf l = core_of(t->leaves[li], L, &omask);
            const Leaf *prev = li > lb ? &prev_core : nullptr;
            seq.clear();
            uint64_t idx = 0;
            double re = 1.0, im = 0.0;
            Cursor cf = fold_prefix(*t, l, &idx, &re, &im);
            const uint64_t reset_cost = suffix_len(*t, l, cf);
            bool rst = prev == nullptr;
            if (!rst) {
                Cursor c = common_prefix(*t, *prev, l);
                const uint64_t up = suffix_len(*t, *prev, c), down = suffix_len(*t, l, c);
                if ((hybrid && reset_cost < up + down) || since_anchor + up + down > budget) {
                    rst = true;
                } else {
                    append_inverse(*t, *prev, c, seq);
                    append_forward(*t, l, c, seq);
                    since_anchor += up + down;
                }
            }
            if (rst) {
                S.reset(idx, re, im);
                append_forward(*t, l, cf, seq);
                since_anchor = seq.size();
            }
            stats.gate_apps += seq.size();
            for (const Op &o : seq) S.apply(o);
            if (sample && l.count) {
                S.canonical_positions();
                S.flush();
                // per-shard block sums + prefix; shard totals to every rank
                std::vector<double> tot(R, 0.0);
                for (size_t i = 0; i < S.mine.size(); ++i) {
                    const int s = S.mine[i];
                    double *bl = d_blocks + i * blk_stride;
                    if (!dry) {
                        launch_block_sums(S.buf[s], S.nl, S.prec, bb, bl, S.st);
                        launch_scan_blocks(bl, bl + nb, nb, 0, S.st);
                        TQ_SH_CUDA(cudaMemcpyAsync(d_tot + s, bl + nb + nsb, sizeof(double), cudaMemcpyDeviceToDevice, S.st));
                    }
                    stats.launches += 2;
                    stats.sample_bytes += (double)shard_bytes;
                }
                if (!dry) {
                    if (!comm->local) {
                        // every rank zeroes the others' entries, then one sum all-reduce
                        for (uint64_t s = 0; s < R; ++s)
                            if ((int)s != comm->rank) TQ_SH_CUDA(cudaMemsetAsync(d_tot + s, 0, sizeof(double), S.st));
                        S.check(nccl::api().AllReduce(d_tot, d_tot, R, ncclFloat64, ncclSum, comm->nc, S.st));
                    }
                    TQ_SH_CUDA(cudaMemcpyAsync(tot.data(), d_tot, R * sizeof(double), cudaMemcpyDeviceToHost, S.st));
                    TQ_SH_CUDA(cudaStreamSynchronize(S.st));
                }
                // logical order: pattern v lives in physical shard shard_of[v]
                double T = 0.0;
                for (uint64_t v = 0; v < R; ++v) T += tot[S.shard_of[v]];
                double lo = 0.0;
                uint64_t last_nz = 0;
                for (uint64_t v = 0; v < R; ++v)
                    if (tot[S.shard_of[v]] > 0) last_nz = v;
                for (uint64_t v = 0; v < R; ++v) {
                    const uint64_t s = S.shard_of[v];
                    const double hi = v == last_nz ? INFINITY : lo + tot[s];
                    auto it = std::find(S.mine.begin(), S.mine.end(), (int)s);
                    if (it != S.mine.end() && tot[s] > 0) {
                        const size_t i = it - S.mine.begin();
                        double *bl = d_blocks + i * blk_stride;
                        if (!dry)
                            stats.sample_bytes += launch_draws_window(S.buf[s], S.nl, S.prec, bb, bl, bl + nb, l.count,
                                                                      t->seed, li, omask, eps, d_slots + (l.offset - off0),
                                                                      d_edges, T, lo, hi, v << S.nl, S.st);
                        stats.launches++;
                    }
                    lo += tot[s];
                }
                stats.draws += l.count;
                stats.sampled_vectors++;
            }
            stats.leaves++;
            prev_core = l;
            if (!dry) {
                cudaError_t e = cudaPeekAtLastError();
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    cleanup();
                    return fail(TUSQ_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
                }
            }
        }
        // leave the caller's buffers in the canonical layout: shard r = pattern r, logical order
        S.canonical_positions();
        S.canonical_shards();
        if (!dry) {
            if (sample && off1 > off0) {
                if (!comm->local)
                    S.check(nccl::api().AllReduce(d_slots, d_slots, off1 - off0, ncclUint64, ncclSum, comm->nc, S.st));
                TQ_SH_CUDA(cudaMemcpyAsync(out_slots + off0, d_slots, (off1 - off0) * sizeof(uint64_t),
                                           cudaMemcpyDeviceToHost, S.st));
            }
            uint32_t h_edges = 0;
            TQ_SH_CUDA(cudaMemcpyAsync(&h_edges, d_edges, sizeof(uint32_t), cudaMemcpyDeviceToHost, S.st));
            TQ_SH_CUDA(cudaStreamSynchronize(S.st));
            stats.edge_draws = h_edges;
            timer.flush();
            stats.gate_kernel_launches = timer.launches;
            stats.gate_kernel_seconds = timer.seconds;
            stats.gate_kernel_bytes = timer.bytes;
        }
    } catch (const std::exception &e) {
        cleanup();
        return fail(TUSQ_ERR_INTERNAL, e.what());
    }
    stats.exchanges = S.exchanges;
    cleanup();
    stats.host_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats_out) *stats_out = stats;
    return TUSQ_OK;
#undef TQ_SH_CUDA
}

}  // namespace tq

using namespace tq;

extern "C" {

tusq_status tusq_comm_unique_id(uint8_t out[128])
{
    if (!out) return fail(TUSQ_ERR_INVALID_ARG, "out is NULL");
    auto &a = nccl::api();
    if (!a.ok) return fail(TUSQ_ERR_NCCL, "libnccl.so.2 not available");
    ncclUniqueId id;
    ncclResult_t r = a.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(TUSQ_ERR_NCCL, std::string("ncclGetUniqueId: ") + a.GetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, 128);
    return TUSQ_OK;
}

tusq_status tusq_comm_init(const uint8_t id[128], int nranks, int rank, int device, tusq_comm **out)
{
    if (!out) return fail(TUSQ_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!id || nranks < 2 || (nranks & (nranks - 1)) || rank < 0 || rank >= nranks)
        return fail(TUSQ_ERR_INVALID_ARG, "nranks must be a power of two >= 2 and 0 <= rank < nranks");
    auto &a = nccl::api();
    if (!a.ok) return fail(TUSQ_ERR_NCCL, "libnccl.so.2 not available");
    if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return fail(TUSQ_ERR_CUDA, "cudaSetDevice failed");
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = a.CommInitRank(&c, nranks, uid, rank);
    if (r != ncclSuccess) return fail(TUSQ_ERR_NCCL, std::string("ncclCommInitRank: ") + a.GetErrorString(r));
    tusq_comm *m = new (std::nothrow) tusq_comm;
    if (!m) { a.CommDestroy(c); return fail(TUSQ_ERR_OOM, "host allocation failed"); }
    m->nranks = nranks; m->rank = rank; m->local = false; m->device = device; m->nc = c;
    *out = m;
    return TUSQ_OK;
}

tusq_status tusq_comm_init_local(int nshards, int device, tusq_comm **out)
{
    if (!out) return fail(TUSQ_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (nshards < 2 || (nshards & (nshards - 1))) return fail(TUSQ_ERR_INVALID_ARG, "nshards must be a power of two >= 2");
    tusq_comm *m = new (std::nothrow) tusq_comm;
    if (!m) return fail(TUSQ_ERR_OOM, "host allocation failed");
    m->nranks = nshards; m->rank = 0; m->local = true; m->device = device;
    *out = m;
    return TUSQ_OK;
}

tusq_status tusq_reduce_slots(tusq_comm *comm, uint64_t *slots, uint64_t n, void *stream)
{
    if (!comm || (!slots && n)) return fail(TUSQ_ERR_INVALID_ARG, "NULL argument");
    if (comm->local) return fail(TUSQ_ERR_INVALID_ARG, "a local communicator has no ranks to reduce over");
    if (!n) return TUSQ_OK;
    auto &a = nccl::api();
    if (!a.ok) return fail(TUSQ_ERR_NCCL, "libnccl.so.2 not available");
    if (comm->device >= 0 && cudaSetDevice(comm->device) != cudaSuccess) return fail(TUSQ_ERR_CUDA, "cudaSetDevice failed");
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t *d = nullptr;
    if (cudaMallocAsync((void **)&d, n * sizeof(uint64_t), st) != cudaSuccess) return fail(TUSQ_ERR_OOM, "cudaMallocAsync failed");
    tusq_status rc = TUSQ_OK;
    std::string err;
    if (cudaMemcpyAsync(d, slots, n * sizeof(uint64_t), cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = fail(TUSQ_ERR_CUDA, "cudaMemcpyAsync (slots in) failed");
    else if (comm_allreduce_u64(comm, d, n, st, err) != TUSQ_OK)
        rc = fail(TUSQ_ERR_NCCL, err);
    else if (cudaMemcpyAsync(slots, d, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(TUSQ_ERR_CUDA, "cudaMemcpyAsync (slots out) failed");
    cudaFreeAsync(d, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == TUSQ_OK) rc = fail(TUSQ_ERR_CUDA, "cudaStreamSynchronize failed");
    return rc;
}

void tusq_comm_free(tusq_comm *c)
{
    if (!c) return;
    if (c->nc && nccl::api().ok) nccl::api().CommDestroy(c->nc);
    delete c;
}

}  // extern "C"
