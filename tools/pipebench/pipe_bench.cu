// pipe_bench.cu -- per-pipe issue microbenchmark for the roofline denominators
// of the SSA kernels (VERDICT r1 "measured per-pipe peaks").
//
// For each instruction class the SSA kernels lean on (fp64 FMA/ADD/MUL, the
// MUFU fp64 reciprocal seed, int->fp64 conversion, 32-bit IMAD / IMAD.HI /
// LOP3 / IADD3, fp32 FFMA as the issue reference, shuffles, shared loads):
//   throughput: one CTA of 1024 threads per SM (32 warps), 8 independent
//     dependency chains per thread, unrolled; warp instructions per SM per
//     cycle = 32 warps * iterations * 8 / SM cycles (clock64 on the SM, so
//     the number is clock-independent);
//   latency: one warp, one dependent chain: cycles per instruction.
// Output: one JSON object on stdout.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;

enum Op { DFMA, DADD, DMUL, RCP64, I2F64, IMAD, IMADHI, LOP3, IADD3, FFMA, SHFL, LDS, IMADW, FLO, I2F64S32, N_OPS };
static const char *names[N_OPS] = {"dfma", "dadd", "dmul", "mufu_rcp64h", "i2f_f64_u64", "imad", "imad_hi", "lop3",
                                   "iadd3", "ffma", "shfl", "lds", "imad_wide_u32", "flo_clz", "i2f_f64_s32"};

template <int OP, int C>
__device__ __forceinline__ void body(double (&d)[C], uint32_t (&u)[C], float (&f)[C], double a, double b,
                                     uint32_t ia, uint32_t ib, const volatile double *sm) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (OP == DFMA) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(a), "d"(b));
        if (OP == DADD) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(a));
        if (OP == DMUL) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(a));
        if (OP == RCP64) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d[c]));
        if (OP == I2F64) {
            uint64_t v = ((uint64_t)u[c] << 21) + ib;
            asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(d[c]) : "l"(v));
            u[c] = (uint32_t)__double2loint(d[c]);
        }
        if (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[c]) : "r"(ia), "r"(ib));
        if (OP == IMADHI) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(ia));
        if (OP == LOP3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(ia), "r"(ib));
        if (OP == IADD3) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(u[c]) : "r"(ia), "r"(ib));
        if (OP == FFMA) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"((float)a), "f"((float)b));
        if (OP == SHFL) u[c] = __shfl_xor_sync(0xffffffffu, u[c], 1 + (c & 3));
        if (OP == LDS) d[c] = sm[(__double2loint(d[c]) & 255) + c];
        if (OP == IMADW) {
            unsigned long long p;
            asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(u[c]), "r"(ia));
            u[c] = (uint32_t)(p >> 32) ^ (uint32_t)p;
        }
        if (OP == FLO) u[c] = __clz(u[c]) + ia;
        if (OP == I2F64S32) {
            asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(d[c]) : "r"(u[c]));
            u[c] = (uint32_t)__double2hiint(d[c]);
        }
    }
}

template <int OP, int C>
__global__ void kern(double a, double b, uint32_t ia, uint32_t ib, long long *cyc, double *sink) {
    __shared__ double sm[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) sm[i] = 0.0;
    __syncthreads();
    double d[C];
    uint32_t u[C];
    float f[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        d[c] = 1.0 + c * 1e-3 + threadIdx.x * 1e-6;
        u[c] = threadIdx.x * 7 + c;
        f[c] = 1.0f + c;
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) body<OP, C>(d, u, f, a, b, ia, ib, sm);
    __syncthreads();
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += d[c] + u[c] + f[c];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
int run(int nsm, long long *cyc, double *sink, double &tput, double &lat) {
    long long h[512];
    // throughput: 1024 threads per SM, CH chains each
    kern<OP, CH><<<nsm, 1024>>>(1.0000001, 1e-9, 3u, 5u, cyc, sink);
    CK(cudaDeviceSynchronize());
    kern<OP, CH><<<nsm, 1024>>>(1.0000001, 1e-9, 3u, 5u, cyc, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    tput = 32.0 * ITERS * CH / (double)mx;  // warp instructions per SM per cycle
    // latency: one warp, one chain
    kern<OP, 1><<<1, 32>>>(1.0000001, 1e-9, 3u, 5u, cyc, sink);
    CK(cudaDeviceSynchronize());
    kern<OP, 1><<<1, 32>>>(1.0000001, 1e-9, 3u, 5u, cyc, sink);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost));
    lat = (double)h[0] / ITERS;
    return 0;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    long long *cyc;
    double *sink;
    CK(cudaMalloc(&cyc, sizeof(long long) * 512));
    CK(cudaMalloc(&sink, 64));
    double tp[N_OPS], lt[N_OPS];
    if (run<DFMA>(nsm, cyc, sink, tp[DFMA], lt[DFMA])) return 1;
    if (run<DADD>(nsm, cyc, sink, tp[DADD], lt[DADD])) return 1;
    if (run<DMUL>(nsm, cyc, sink, tp[DMUL], lt[DMUL])) return 1;
    if (run<RCP64>(nsm, cyc, sink, tp[RCP64], lt[RCP64])) return 1;
    if (run<I2F64>(nsm, cyc, sink, tp[I2F64], lt[I2F64])) return 1;
    if (run<IMAD>(nsm, cyc, sink, tp[IMAD], lt[IMAD])) return 1;
    if (run<IMADHI>(nsm, cyc, sink, tp[IMADHI], lt[IMADHI])) return 1;
    if (run<LOP3>(nsm, cyc, sink, tp[LOP3], lt[LOP3])) return 1;
    if (run<IADD3>(nsm, cyc, sink, tp[IADD3], lt[IADD3])) return 1;
    if (run<FFMA>(nsm, cyc, sink, tp[FFMA], lt[FFMA])) return 1;
    if (run<SHFL>(nsm, cyc, sink, tp[SHFL], lt[SHFL])) return 1;
    if (run<LDS>(nsm, cyc, sink, tp[LDS], lt[LDS])) return 1;
    if (run<IMADW>(nsm, cyc, sink, tp[IMADW], lt[IMADW])) return 1;
    if (run<FLO>(nsm, cyc, sink, tp[FLO], lt[FLO])) return 1;
    if (run<I2F64S32>(nsm, cyc, sink, tp[I2F64S32], lt[I2F64S32])) return 1;
    printf("{\"sms\": %d, \"clock_rate_khz\": %d, \"unit\": \"warp instructions per SM per cycle (throughput); "
           "cycles per dependent instruction (latency)\", \"ops\": {", nsm, clk);
    for (int i = 0; i < N_OPS; ++i)
        printf("%s\"%s\": {\"warp_inst_per_sm_cycle\": %.4f, \"lanes_per_sm_cycle\": %.2f, \"latency_cycles\": %.2f}",
               i ? ", " : "", names[i], tp[i], 32.0 * tp[i], lt[i]);
    printf("}}\n");
    return 0;
}
