// cwc_internal.h -- host/device shared layouts of the product path.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "cwc.h"

namespace cwc {

// Sets cwc_last_error() of the calling thread (cwc_api.cpp).
void set_last_error(const std::string &msg);

// Thread path limits: cells and reactions live in registers, net change of a
// reaction is packed as one int8 per cell into a 64-bit word.
constexpr int kThreadMaxCells = 8;
constexpr int kThreadMaxReactions = 32;
constexpr int kThreadMaxObs = 8;
constexpr int kOpWords = 4;  // operand-state chain for M <= 16

// Reaction encoding shared by both kernels (built by the host compiler):
// h = xa * (xb - sub) >> shr with xa = x[ia], xb = x[ib] and index
// "one" (= n_cells, or the padded cell count in the thread path) reading 1.
struct ReactionDesc {
    int32_t ia, ib;
    int32_t kind;   // sub | (shr << 1)
    int32_t rule;
};

// Statistics accumulator layout (device_common.cuh "limb accumulators").  A
// part holds, per cell, one count word, sl limb words of the sum and ql limb
// words of the sum of squares, as word arrays of n cells each (n a multiple
// of 4 so every part is 16-byte sized).  Shared-memory parts use 32-bit words
// with 16-bit limbs (<= 2^16 adds per word: one CTA); global parts use 64-bit
// words with 32-bit limbs (<= 2^32 adds per word).  Limb adds never carry, so
// every update is a fire-and-forget atomic (RED), never a dependent
// read-modify-write chain.
struct StatLayout {
    int32_t wb;   // word bytes: 4 (16-bit limbs) or 8 (32-bit limbs)
    int32_t sl;   // sum limbs
    int32_t ql;   // sum-of-squares limbs
    int32_t pad_;
};
__host__ __device__ __forceinline__ int stat_limb_bits(const StatLayout &l) { return l.wb == 4 ? 16 : 32; }
__host__ __device__ __forceinline__ int stat_words(const StatLayout &l) { return 1 + l.sl + l.ql; }
__host__ __device__ __forceinline__ long long stat_bytes(const StatLayout &l, long long n) {
    return (long long)l.wb * stat_words(l) * n;
}
// warp-specialised thread path (ssa_thread_ws.cuh): draws in flight per
// trajectory and the ring + hand-off counters' shared-memory bytes per CTA
// CWC_WS_STRESS (test builds only, tests/test_gpu_ws_stress.py): the
// smallest legal ring and pseudo-random sleeps in producer and consumer, so
// the hand-off runs in every interleaving order the timing can produce
#ifndef CWC_WS_STRESS
#define CWC_WS_STRESS 0
#endif
constexpr int kWsRing = CWC_WS_STRESS ? 8 : 32;
#ifndef CWC_WS_PRODUCERS
#define CWC_WS_PRODUCERS 1
#endif
constexpr int kWsProducers = CWC_WS_PRODUCERS;  // producer warps per group
#ifndef CWC_WS_GROUPS
#define CWC_WS_GROUPS 1
#endif
constexpr int kWsGroups = CWC_WS_GROUPS;  // 32-trajectory groups (consumer + producer warp pairs) per CTA
constexpr int kWsStage = 64;     // staged sample records of a consumer warp
constexpr size_t kWsGroupBytes = (size_t)2 * kWsRing * 32 * sizeof(double) +
                                 (size_t)(kWsProducers + 2) * 32 * sizeof(unsigned) +
                                 (size_t)kWsStage * (2 + kThreadMaxCells / 2) * sizeof(long long);
// staging longs per warp: per record its first cell, its dump row, its counts (int32)
constexpr long long kStageLL = (long long)kWsStage * (2 + kThreadMaxCells / 2);
constexpr size_t kWsRingBytes = kWsGroups * ((kWsGroupBytes + 15) & ~(size_t)15);  // per CTA
// two trajectories per consumer lane (ssa_thread_ws2.cuh), served by 1
// producer warp (both trajectories of each lane) or 2 (one slot each)
#ifndef CWC_WS2_PRODUCERS
#define CWC_WS2_PRODUCERS 2
#endif
constexpr int kWs2Producers = CWC_WS2_PRODUCERS;
// rings of 64
// trajectories, per-trajectory counters, the staging of one consumer warp
constexpr size_t kWs2RingBytes = (((size_t)2 * kWsRing * 64 * sizeof(double) + (size_t)3 * 64 * sizeof(unsigned) +
                                   (size_t)kWsStage * (2 + kThreadMaxCells / 2) * sizeof(long long)) + 15) & ~(size_t)15;
// shared-memory copy of the -log reduction table (device_common.cuh,
// neglog_table.h) in the thread kernels: {T, L_hi} pairs then L_lo
struct NegLogSmem {
    double2 tl[129];
    double lo[129];
};
constexpr size_t kNegLogSmemBytes = (sizeof(NegLogSmem) + 15) & ~(size_t)15;
constexpr long long kSmemPartMaxTraj = 1ll << 16;  // trajectories per shared-memory part (16-bit limbs)
__host__ __device__ __forceinline__ long long stat_cells_round(long long n) { return (n + 3) & ~3ll; }
// Layout for observables of at most vbits bits (v < 2^vbits, v^2 < 2^(2 vbits)).
__host__ __device__ __forceinline__ StatLayout stat_layout(bool smem, int vbits) {
    StatLayout l;
    l.wb = smem ? 4 : 8;
    const int lb = smem ? 16 : 32;
    l.sl = (vbits + lb - 1) / lb;
    l.ql = (2 * vbits + lb - 1) / lb;
    l.pad_ = 0;
    return l;
}

// RNG key of local trajectory g: point * R_total + r_off + replica.
__host__ __device__ __forceinline__ int64_t global_traj(int64_t g, int64_t R, int64_t R_total, int64_t r_off) {
    const int64_t p = g / R;
    return p * R_total + r_off + (g - p * R);
}

// Per-launch run description (both kernels).
struct RunParams {
    int64_t G;              // trajectories
    int64_t R;              // replicas per point in this call
    int64_t R_total;        // replicas per point of the whole (sharded) run
    int64_t r_off;          // first replica of this call
    int32_t P;              // points
    int32_t J;              // last sample index
    double dt;
    uint64_t seed;
    uint32_t rk[20];        // Philox4x32-10 round keys of seed (round r: rk[2r], rk[2r+1]; set_round_keys)
    const double *rates;    // [P][M] flat per-reaction rate constants
    const double *rates_h;  // [P][M] the same with A + A entries halved (k / 2: segment kernel)
    // statistics: accumulator parts (see stats.cu)
    void *parts;            // n_parts x stat_bytes(st, cells_per_part)
    StatLayout st;          // word / limb layout of the parts (shared- or global-memory form)
    int64_t cells_per_part;
    int32_t stats_smem;     // 1: block accumulators in shared memory, flushed to parts[blockIdx]
    int32_t ws;             // thread path: warp-specialised producer/consumer kernel (ssa_thread_ws.cuh)
    int32_t thread_nt;      // thread path, single-warp kernel: trajectories per lane (1 or 2)
    const int32_t *cta_order;  // thread path: CTA slot -> trajectory group (NULL = identity)
    unsigned *sm_ctr;          // warp-specialised kernel: per-SM CTA arrival counters (zeroed per call)
    int32_t part_stride_blocks;  // GLOBAL mode: block b accumulates into part (b % n_parts)
    int32_t n_parts;
    int64_t traj_per_part;  // static mapping: part b covers g in [b*T, (b+1)*T); 0 = all points
    // optional outputs
    int64_t *out_traj;
    int64_t *out_firings;
    int32_t *out_status;
    // trace
    const int64_t *trace_g; // device [n_trace]
    int32_t n_trace;
    int64_t trace_cap;
    double *trace_buf;
    int64_t *trace_len;
    // warp path dynamic scheduling
    unsigned long long *next_traj;
    // debug: consumer cycle accounting of the warp-specialised kernel (NULL = off)
    unsigned long long *prof;
    // launch slots and resumable runs (cwc_run_*).  Slot i
    // < n_launch runs trajectory rs_live[i] (i itself when rs_live is NULL).
    // With rs_x set, every trajectory starts from and ends by saving its state
    // (x [G][n_cells], t, n = applied firings = Philox counter, j = next
    // sample; j = J+1: finished) and is suspended after `quantum` further
    // firings (0 = no bound; checked per batch / per 32-draw window) or on
    // reaching sample j_stop (J+1 = no bound).  One-shot runs: rs_* NULL,
    // n_launch = G, quantum = 0, j_stop = J+1.
    int64_t n_launch;
    const int64_t *rs_live;
    int32_t *rs_x;
    double *rs_t;
    int64_t *rs_n;
    int32_t *rs_j;
    int64_t quantum;
    int64_t j_stop;
};

// Philox4x32-10 key schedule of seed: round r uses (seed_lo + r W0, seed_hi + r W1).
inline void set_round_keys(RunParams &rp) {
    for (int r = 0; r < 10; ++r) {
        rp.rk[2 * r] = (uint32_t)rp.seed + (uint32_t)r * 0x9E3779B9u;
        rp.rk[2 * r + 1] = (uint32_t)(rp.seed >> 32) + (uint32_t)r * 0xBB67AE85u;
    }
}

__host__ __device__ __forceinline__ long long launch_traj(const RunParams &rp, long long slot) {
    return rp.rs_live ? (long long)rp.rs_live[slot] : slot;
}

// Thread path tables (kernel parameter, constant bank).
struct ThreadTables {
    int32_t n_cells, M, O, pad_;
    int32_t ia[kThreadMaxReactions], ib[kThreadMaxReactions];
    int32_t sub[kThreadMaxReactions], shr[kThreadMaxReactions];
    uint64_t nu_pack[kThreadMaxReactions];   // int8 delta per cell
    // M <= 4 * kOpWords: int8 delta of every reaction operand (reaction m:
    // bytes 2(m mod 4) and 2(m mod 4)+1 of word m / 4 = x[ia_m], x[ib_m]; 0
    // for an absent reactant) -- the kernel then keeps the operands
    // themselves as state instead of gathering them from x
    uint64_t op_pack[kThreadMaxReactions][kOpWords];
    // nu_pack and op_pack word 0 in ONE word when 8 S_pad + 16 M_pad <= 64
    // (C1, C2): net change bytes 0 .. S_pad-1, operand deltas from byte
    // S_pad on -- the selection then moves one word per compare
    uint64_t comb_pack[kThreadMaxReactions];
    int32_t obs_of[kThreadMaxCells];
    int32_t init[kThreadMaxCells];
};

// Warp path tables (device pointers, read through L1).
// Reaction m lives in lane chunk l = m / B at position k = m % B; its
// propensity is stored at shared-memory slot l * Bp + k (Bp = B | 1: odd, so a
// lane-strided access and a chunk-contiguous access are both bank-conflict
// free).
struct WarpTables {
    int32_t n_cells, M, O, B;     // B = reactions per lane chunk = ceil(M / 32)
    int32_t Bp;                   // chunk stride (odd)
    int32_t B16, Bp16;            // the same for 16-lane segments (ssa_warp2.cu)
    int32_t B4;                   // entries per lane of the 4-lane groups (ssa_warp8.cu): ceil(M / 4)
    const ReactionDesc *rx;       // [M]
    const int32_t *nu_ptr;        // [M+1]
    const int2 *nu;               // (cell, delta)
    const int32_t *dep_ptr;       // [M+1]
    const int2 *dep;              // (m, slot | owner lane << 24) of every m in D(mu)
    const int2 *dep16;            // the same slots for the 16-lane segment layout
    const int4 *dep4;             // warp layout with the reactants inline: (m, slot | owner << 24, ia, ib | kind << 24)
    const int4 *dep16_4;          // the same for the 16-lane segment layout
    const int32_t *obs_ptr;       // [O+1]
    const int32_t *obs_cells;
    const int32_t *init;          // [n_cells]
    // per-mu header (nu offset, nu count, dependency offset, dependency
    // count: one 16-byte load); net change entries (x byte offset, delta);
    // dependency entries for the 16- and 32-lane chunk layouts (a slot byte
    // offset, x_a byte offset, x_b byte offset, m * 8 | owner lane << 26 |
    // sub << 31), read with the A + A-halved rates (RunParams.rates_h)
    const int4 *hdr;
    const int2 *nuw;
    const int4 *depw16;
    const int4 *depw32;
    // 4-lane group layout (ssa_warp8.cu): net change (cell * 32, delta) and
    // dependency entries (a byte offset (k * 32 + (owner ^ ((k >> 2) & 3))) * 8,
    // x_a * 32, x_b * 32, m * 8 | (owner * 4 + k / 16) << 26 | sub << 31);
    // the kernel adds its group's column / cell offsets
    const int2 *nuw8;
    const int4 *depw4;
    const int4 *depw8;            // the same for 8-lane groups: (k * 32 + (owner ^ ((k >> 1) & 7))) * 8, owner * 2 + k / 16
};

// Launchers (ssa_thread.cu, ssa_warp.cu, stats.cu); return cudaError_t.
cudaError_t launch_ssa_thread(int s_pad, int m_pad, const RunParams &rp, const ThreadTables &tt, int threads,
                              size_t smem_bytes, cudaStream_t stream);
bool thread_variant_exists(int s_pad, int m_pad);
int thread_pad_cells(int n_cells);
int thread_pad_reactions(int M);

cudaError_t launch_ssa_warp(const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                            size_t smem_bytes, cudaStream_t stream);
size_t warp_smem_per_warp(const WarpTables &wt);
cudaError_t launch_ssa_warp2(const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                             size_t smem_bytes, cudaStream_t stream);
size_t warp2_smem_per_warp(const WarpTables &wt);
// LG-lane groups (ssa_warp8.cu): LG = 4 (eight trajectories per warp) or 8 (four)
cudaError_t launch_ssa_group(int LG, const RunParams &rp, const WarpTables &wt, int blocks, int warps_per_block,
                             size_t smem_bytes, cudaStream_t stream);
size_t group_smem_per_warp(const WarpTables &wt, int LG);


cudaError_t launch_stats_stage2(const RunParams &rp, int64_t O, int64_t *count, int64_t *sum, uint64_t *sumsq,
                                cudaStream_t stream);
cudaError_t launch_stats_finalize(const int64_t *count, const int64_t *sum, const uint64_t *sumsq, int64_t n,
                                  double *mean, double *var, double *ci90, cudaStream_t stream);
cudaError_t launch_philox_blocks(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, uint32_t *out,
                                 cudaStream_t stream);
cudaError_t launch_draws(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, double *E, double *u2,
                         cudaStream_t stream);
cudaError_t launch_tau_div(const double *e, const double *a, int64_t count, double *q, cudaStream_t stream);
cudaError_t launch_block_draws(const uint32_t *w, int64_t count, double *u1, double *u2, double *E, cudaStream_t stream);

// resume.cu: resumable runs (state initialisation, live-list compaction)
cudaError_t launch_state_init(long long G, int n_cells, const int32_t *init, int32_t *x, double *t, int64_t *n,
                              int32_t *j, int64_t *live, cudaStream_t stream);
size_t compact_temp_bytes(long long G);
cudaError_t launch_compact(const int64_t *live_in, long long n_in, int64_t *live_out, int64_t *n_out,
                           const int32_t *j, int32_t J, void *temp, size_t temp_bytes, cudaStream_t stream);
cudaError_t launch_count_below(const int64_t *live, long long n, const int32_t *j, int32_t j_stop,
                               unsigned long long *out, cudaStream_t stream);

}  // namespace cwc
