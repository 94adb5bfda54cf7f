// stats.cu -- second stage of the on-line reduction, finalize, Philox hook.
//
// Stage 1 (inside the SSA kernels) leaves one partial moment set per part
// (per CTA, or per CTA slice) in limb form (cwc_internal.h StatLayout: count
// word, sum limbs, sum-of-squares limbs).  Stage 2 sums, for every (point,
// sample, observable) cell, the parts that cover its point, recombines the
// limbs and writes count / sum / sumsq(128)
// -- exact integer addition, so the result does not depend on how
// trajectories were spread over CTAs (SPEC S:513 determinism).
#include <cuda_runtime.h>

#include "cwc_internal.h"
#include "device_common.cuh"

namespace cwc {

__global__ void stats_stage2_kernel(const RunParams rp, long long O, long long n_cells, int64_t *count, int64_t *sum,
                                    uint64_t *sumsq) {
    const long long JO = (long long)(rp.J + 1) * O;
    const StatLayout L = rp.st;
    const int lb = stat_limb_bits(L);
    const long long pb = stat_bytes(L, rp.cells_per_part);
    const long long n = rp.cells_per_part;
    const bool sq16 = (reinterpret_cast<unsigned long long>(sumsq) & 15ull) == 0ull;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n_cells;
         c += (long long)gridDim.x * blockDim.x) {
        const long long p = c / JO;
        const long long rest = c - p * JO;
        long long b0, b1;
        if (rp.traj_per_part > 0) {
            b0 = (p * rp.R) / rp.traj_per_part;
            b1 = ((p + 1) * rp.R - 1) / rp.traj_per_part;
            if (b1 > rp.n_parts - 1) b1 = rp.n_parts - 1;
        } else {
            b0 = 0;
            b1 = rp.n_parts - 1;
        }
        // the parts' limb words summed straight into the recombined 128-bit
        // totals: sum_b sum_i (u[b][i] << lb i) (arithmetic mod 2^128, so the
        // order of the two sums does not matter; the true totals fit by the
        // planner's bound).  No per-thread word array (it lived in local memory).
        unsigned __int128 cnt = 0, s1 = 0, s2 = 0;
        for (long long b = b0; b <= b1; ++b) {
            long long local = c;
            if (rp.traj_per_part > 0) local = (p - (b * rp.traj_per_part) / rp.R) * JO + rest;
            const unsigned char *base = (const unsigned char *)rp.parts + b * pb;
            if (L.wb == 4) {
                const unsigned int *u = (const unsigned int *)base + local;
                cnt += u[0];
                for (int i = 0; i < L.sl; ++i) s1 += (unsigned __int128)u[(long long)(1 + i) * n] << (lb * i);
                for (int i = 0; i < L.ql; ++i) s2 += (unsigned __int128)u[(long long)(1 + L.sl + i) * n] << (lb * i);
            } else {
                const unsigned long long *u = (const unsigned long long *)base + local;
                cnt += u[0];
                for (int i = 0; i < L.sl; ++i) s1 += (unsigned __int128)u[(long long)(1 + i) * n] << (lb * i);
                for (int i = 0; i < L.ql; ++i) s2 += (unsigned __int128)u[(long long)(1 + L.sl + i) * n] << (lb * i);
            }
        }
        count[c] = (int64_t)cnt;
        sum[c] = (int64_t)s1;
        if (sq16) {  // one 16-byte store per cell (coalesced, vectorised) when the array is 16-byte aligned
            reinterpret_cast<ulonglong2 *>(sumsq)[c] = make_ulonglong2((unsigned long long)s2, (unsigned long long)(s2 >> 64));
        } else {
            sumsq[2 * c] = (uint64_t)s2;
            sumsq[2 * c + 1] = (uint64_t)(s2 >> 64);
        }
    }
}

cudaError_t launch_stats_stage2(const RunParams &rp, int64_t O, int64_t *count, int64_t *sum, uint64_t *sumsq,
                                cudaStream_t stream) {
    const long long n_cells = (long long)rp.P * (rp.J + 1) * O;
    if (n_cells == 0) return cudaSuccess;
    long long blocks = (n_cells + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    stats_stage2_kernel<<<(unsigned)blocks, 256, 0, stream>>>(rp, O, n_cells, count, sum, sumsq);
    return cudaGetLastError();
}

// ---- finalize ---------------------------------------------------------------
// 192-bit unsigned helpers for n * S2 - S1^2 (n < 2^63, S2 < 2^128, S1 < 2^64).
struct U192 {
    unsigned long long w[3];
};

__device__ __forceinline__ U192 mul_64x128(unsigned long long a, unsigned __int128 b) {
    const unsigned long long b0 = (unsigned long long)b, b1 = (unsigned long long)(b >> 64);
    const unsigned __int128 p0 = (unsigned __int128)a * b0;
    const unsigned __int128 p1 = (unsigned __int128)a * b1 + (p0 >> 64);
    U192 r;
    r.w[0] = (unsigned long long)p0;
    r.w[1] = (unsigned long long)p1;
    r.w[2] = (unsigned long long)(p1 >> 64);
    return r;
}

__device__ __forceinline__ U192 sub_192_128(U192 a, unsigned __int128 b) {
    const unsigned long long b0 = (unsigned long long)b, b1 = (unsigned long long)(b >> 64);
    U192 r;
    r.w[0] = a.w[0] - b0;
    unsigned long long br = (a.w[0] < b0) ? 1ull : 0ull;
    const unsigned long long t1 = a.w[1] - b1;
    const unsigned long long br1 = (a.w[1] < b1) ? 1ull : 0ull;
    r.w[1] = t1 - br;
    br = br1 | ((t1 < br) ? 1ull : 0ull);
    r.w[2] = a.w[2] - br;
    return r;
}

// RN(N / D) for 0 <= N < 2^192, 0 < D < 2^126: the quotient's binary expansion
// by restoring division, one bit per step from N's most significant set bit
// on.  The first 64 significant quotient bits are kept, every later bit and
// the final remainder fold into a sticky bit below them (11 bits under the
// rounding position), so the single conversion rounds the exact quotient to
// nearest-even once; the power-of-two scaling is exact (|result| >= 2^-126).
__device__ double div_rn_u192(U192 N, unsigned __int128 D) {
    int top = -1;
    for (int w = 2; w >= 0 && top < 0; --w)
        if (N.w[w]) top = 64 * w + 63 - __clzll((long long)N.w[w]);
    if (top < 0) return 0.0;
    unsigned __int128 rem = 0;  // < D < 2^126, so (rem << 1) | bit fits
    unsigned long long mant = 0;
    int nbits = 0, e_first = 0;  // kept bits; weight exponent of the first significant quotient bit
    bool sticky = false;
    // quotient bits at weights 2^pos: every integer position (pos >= 0), then
    // fractional ones while fewer than 64 bits are kept and the remainder is non-zero
    for (int pos = top;; --pos) {
        if (pos < 0 && (nbits >= 64 || rem == 0)) break;
        const unsigned long long bit = (pos >= 0) ? ((N.w[pos >> 6] >> (pos & 63)) & 1ull) : 0ull;
        rem = (rem << 1) | bit;
        const bool q = rem >= D;
        if (q) rem -= D;
        if (nbits < 64) {
            if (nbits > 0 || q) {
                if (nbits == 0) e_first = pos;
                mant = (mant << 1) | (q ? 1ull : 0ull);
                ++nbits;
            }
        } else if (q) {
            sticky = true;
        }
    }
    if (rem != 0) sticky = true;
    mant <<= (64 - nbits);  // N > 0, so 1 <= nbits <= 64
    const int last = e_first - 63;  // weight exponent of mant's bit 0
    if (sticky) mant |= 1ull;
    return scalbn(__ull2double_rn(mant), last);
}

__global__ void stats_finalize_kernel(const int64_t *count, const int64_t *sum, const uint64_t *sumsq, long long n,
                                      double *mean, double *var, double *ci90) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
        const long long cnt = count[c];
        const unsigned long long s1 = (unsigned long long)sum[c];
        const unsigned __int128 s2 = (unsigned __int128)sumsq[2 * c] | ((unsigned __int128)sumsq[2 * c + 1] << 64);
        double m = __longlong_as_double(0x7ff8000000000000ll), v = m, ci = m;
        if (cnt > 0) {
            U192 s;
            s.w[0] = s1;
            s.w[1] = s.w[2] = 0;
            m = div_rn_u192(s, (unsigned __int128)cnt);
            if (cnt == 1) {
                v = 0.0;
                ci = 0.0;
            } else {
                const U192 num = sub_192_128(mul_64x128((unsigned long long)cnt, s2), (unsigned __int128)s1 * s1);
                v = div_rn_u192(num, (unsigned __int128)cnt * (unsigned long long)(cnt - 1));
                ci = __dmul_rn(1.6449, __dsqrt_rn(__ddiv_rn(v, __ll2double_rn(cnt))));
            }
        }
        if (mean) mean[c] = m;
        if (var) var[c] = v;
        if (ci90) ci90[c] = ci;
    }
}

cudaError_t launch_stats_finalize(const int64_t *count, const int64_t *sum, const uint64_t *sumsq, int64_t n,
                                  double *mean, double *var, double *ci90, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    stats_finalize_kernel<<<(unsigned)blocks, 256, 0, stream>>>(count, sum, sumsq, n, mean, var, ci90);
    return cudaGetLastError();
}

// ---- Philox hook -------------------------------------------------------------
__global__ void philox_blocks_kernel(uint64_t seed, const int64_t *g, const int64_t *n, long long count, uint32_t *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        const uint4 w = philox_block(seed, (uint64_t)g[i], (uint64_t)n[i]);
        reinterpret_cast<uint4 *>(out)[i] = w;
    }
}

cudaError_t launch_philox_blocks(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, uint32_t *out,
                                 cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    philox_blocks_kernel<<<(unsigned)blocks, 256, 0, stream>>>(seed, g, n, count, out);
    return cudaGetLastError();
}

// ---- draw / division hooks (the SSA kernels' own device functions) ------------
// the thread kernels' draw pipeline (shared-memory table, four phases)
__global__ void draws_kernel(uint64_t seed, const int64_t *g, const int64_t *n, long long count, double *E,
                             double *u2) {
    __shared__ NegLogSmem tab;
    neglog_smem_fill(&tab, threadIdx.x, blockDim.x);
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        DrawPipe<1> pipe;
        double e[1], u[1];
        pipe.start((uint64_t)g[i], (uint64_t)n[i]);
#pragma unroll
        for (int ph = 0; ph < 4; ++ph) pipe.phase(ph, seed, &tab, e, u);
        E[i] = e[0];
        u2[i] = u[0];
    }
}

__global__ void block_draws_kernel(const uint32_t *w, long long count, double *u1, double *u2, double *E) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        double a, b;
        block_uniforms(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3], a, b);
        u1[i] = a;
        u2[i] = b;
        E[i] = neg_log_v(block_v1(w[4 * i], w[4 * i + 1]));  // the warp kernels' refill path (table through L1)
    }
}

cudaError_t launch_block_draws(const uint32_t *w, int64_t count, double *u1, double *u2, double *E, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    block_draws_kernel<<<(unsigned)blocks, 256, 0, stream>>>(w, count, u1, u2, E);
    return cudaGetLastError();
}

__global__ void tau_div_kernel(const double *e, const double *a, long long count, double *q) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        const double x = e[i], y = a[i];
        q[i] = div_fast_ok(x, y) ? div_fast(x, y) : __ddiv_rn(x, y);
    }
}

cudaError_t launch_draws(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, double *E, double *u2,
                         cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    draws_kernel<<<(unsigned)blocks, 256, 0, stream>>>(seed, g, n, count, E, u2);
    return cudaGetLastError();
}

cudaError_t launch_tau_div(const double *e, const double *a, int64_t count, double *q, cudaStream_t stream) {
    if (count == 0) return cudaSuccess;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    tau_div_kernel<<<(unsigned)blocks, 256, 0, stream>>>(e, a, count, q);
    return cudaGetLastError();
}

}  // namespace cwc
