// dyn_internal.h -- host/device layouts of the dynamic-topology path
// (include/cwc_dyn.h).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "cwc_dyn.h"
#include "cwc_internal.h"

namespace cwc {
namespace dyn {

// Physical slots of one term buffer (compartment 0 = the top level); a
// lane owns slots lane and lane + 32, and entry positions 2 lane, 2 lane + 1.
constexpr int kSlots = 64;
static_assert(kSlots == CWC_DYN_MAX_CAP, "slot count");
constexpr int kLevels = CWC_DYN_MAX_DEPTH + 1;  // depth 0 .. CWC_DYN_MAX_DEPTH
constexpr int kSegs = 8 + 2 * CWC_DYN_MAX_CTORS;

// Rule descriptor word x: label | (comp label + 1) << 8 | n factors << 16 |
// flags (CWC_DYN_KEEP_X ...) << 20 | structural << 24 | singleton << 25
// (a TOP rule without a child pattern: its only entry is the top level).  Factors (y, z): side
// | atom << 4 | mult << 12 (at most two: reaction order <= 2).  w: the
// non-structural rule's dependency mask (rules to re-evaluate after it
// fires).
__host__ __device__ __forceinline__ int rd_label(int x) { return x & 0xff; }
__host__ __device__ __forceinline__ int rd_comp(int x) { return ((x >> 8) & 0xff) - 1; }
__host__ __device__ __forceinline__ int rd_nfac(int x) { return (x >> 16) & 0xf; }
__host__ __device__ __forceinline__ int rd_flags(int x) { return (x >> 20) & 0xf; }
__host__ __device__ __forceinline__ bool rd_structural(int x) { return (x >> 24) & 1; }
__host__ __device__ __forceinline__ bool rd_singleton(int x) { return (x >> 25) & 1; }

// Device tables of a compiled model (one blob per device; pointers into it).
struct DynTables {
    int32_t A, R, O, n0;           // atoms, rules, observables, initial compartments
    int32_t max_keys, pad0, pad1, pad2;
    const int4 *rule;              // [R] descriptor (above)
    const double *rate;            // [R]
    const int32_t *lhs;            // [R][3][A] pattern multiplicities: context, wrap, content
    const int32_t *rhs;            // [R][A] atoms O adds to the context
    const int32_t *dctx;           // [R][A] non-structural: context net change
    const int32_t *dwrap;          // [R][A] non-structural: matched child's wrap net change
    const int32_t *dcont;          // [R][A] non-structural: matched child's content net change
    const int4 *ctor_hdr;          // [R] (first constructor, count, in-place constructor or -1, 0)
    const int4 *ctor;              // [n_ctors] (label, flags, 0, 0)
    const int32_t *ctor_atoms;     // [n_ctors][2][A] wrap, content
    const int32_t *init_label;     // [n0]
    const int32_t *init_depth;     // [n0]
    const int32_t *init_wrap;      // [n0][A]
    const int32_t *init_cont;      // [n0][A]
    const int32_t *obs_ptr;        // [O + 1]
    const int4 *obs_key;           // (kind, label, atom, 0)
};

struct DynParams {
    int64_t G;                     // trajectories of this call
    int64_t r_off;                 // RNG id of local trajectory g = r_off + g
    int32_t J, cap;
    double dt;
    uint64_t seed;
    void *part;                    // one global statistics part (limb words, StatLayout st)
    StatLayout st;
    int64_t cells;                 // (J + 1) * O rounded (stat_cells_round)
    int64_t *out_traj;
    int64_t *out_firings;
    int32_t *out_status;
    unsigned long long *next_traj;
};

// Shared memory of one warp (bytes, 16-aligned): the first entry of each
// lane pair ax [R][32] (double), lane prefixes pre [R][32], the positive-entry
// masks xm / ym [R] (bit l: entry 2l / 2l+1 > 0), two term buffers (wrap,
// content [A][64] int32, label, depth [64] int8), then the children
// histogram [64] int32, rebuild segments, depth masks, parent / corder [64],
// the per-position structure words pinfo [64] (uint2).
__host__ __device__ __forceinline__ size_t dyn_ax_off() { return 0; }
__host__ __device__ __forceinline__ size_t dyn_pre_off(int R) { return (size_t)R * 32 * 8; }
__host__ __device__ __forceinline__ size_t dyn_mask_off(int R) { return dyn_pre_off(R) + (size_t)R * 32 * 8; }
__host__ __device__ __forceinline__ size_t dyn_term_off(int R) {
    return (dyn_mask_off(R) + (size_t)R * 8 + 15) & ~(size_t)15;
}
__host__ __device__ __forceinline__ size_t dyn_term_bytes(int A) { return (size_t)2 * A * kSlots * 4 + 2 * kSlots; }
__host__ __device__ __forceinline__ size_t dyn_misc_off(int A, int R) { return dyn_term_off(R) + 2 * dyn_term_bytes(A); }
__host__ __device__ __forceinline__ size_t dyn_smem_per_warp(int A, int R) {
    const size_t misc = (size_t)kSlots * 4 + (size_t)kSegs * 16 + (size_t)kLevels * 8 + 2 * kSlots + (size_t)kSlots * 8;
    return (dyn_misc_off(A, R) + misc + 15) & ~(size_t)15;
}

cudaError_t launch_dyn_ssa(const DynParams &dp, const DynTables &dt, int blocks, int warps_per_block, size_t smem,
                           cudaStream_t stream);
const void *dyn_kernel_fn();

}  // namespace dyn
}  // namespace cwc
