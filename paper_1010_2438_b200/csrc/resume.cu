// resume.cu -- resumable runs (cwc_run_*): state
// initialisation and live-list compaction.
//
// The paper's schema (ii) represents every simulation instance
// as an object holding its progress, so that a scheduler can stop and restart
// it and run it in slices; schema (iii) reduces a running window
// of the trajectories while they are still produced.  Here a trajectory's
// whole progress is (x, t, n, j): the counter-based RNG needs nothing but the
// firing index n to continue the stream, so a suspended trajectory resumes
// bit-exactly, on any SM, in any later launch.  Between launches the
// finished trajectories (j = J+1) are dropped from the live list, so the next
// launch packs only unfinished ones into dense warps.
#include <cuda_runtime.h>

#include <cub/device/device_select.cuh>

#include "cwc_internal.h"

namespace cwc {

namespace {

__global__ void state_init_kernel(long long G, int n_cells, const int32_t *init, int32_t *x, double *t, int64_t *n,
                                  int32_t *j, int64_t *live) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G * n_cells; i += stride)
        x[i] = __ldg(init + i % n_cells);
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G; g += stride) {
        t[g] = 0.0;
        n[g] = 0;
        j[g] = 0;
        if (live) live[g] = g;
    }
}

struct Unfinished {
    const int32_t *j;
    int32_t J;
    __device__ __forceinline__ bool operator()(const int64_t g) const { return j[g] <= J; }
};

__global__ void count_below_kernel(const int64_t *live, long long n, const int32_t *j, int32_t j_stop,
                                   unsigned long long *out) {
    unsigned c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        c += (j[live[i]] < j_stop) ? 1u : 0u;
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

}  // namespace

// *out (zeroed here) = |{i < n : j[live[i]] < j_stop}|
cudaError_t launch_count_below(const int64_t *live, long long n, const int32_t *j, int32_t j_stop,
                               unsigned long long *out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess || n == 0) return e;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    count_below_kernel<<<(unsigned)blocks, 256, 0, stream>>>(live, n, j, j_stop, out);
    return cudaGetLastError();
}

cudaError_t launch_state_init(long long G, int n_cells, const int32_t *init, int32_t *x, double *t, int64_t *n,
                              int32_t *j, int64_t *live, cudaStream_t stream) {
    if (G == 0) return cudaSuccess;
    long long blocks = (G * (n_cells > 0 ? n_cells : 1) + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    state_init_kernel<<<(unsigned)blocks, 256, 0, stream>>>(G, n_cells, init, x, t, n, j, live);
    return cudaGetLastError();
}

size_t compact_temp_bytes(long long G) {
    size_t bytes = 0;
    cub::DeviceSelect::If(nullptr, bytes, (const int64_t *)nullptr, (int64_t *)nullptr, (int64_t *)nullptr, G,
                          Unfinished{nullptr, 0});
    return bytes;
}

// Order-preserving: live_out = [g in live_in : j[g] <= J], *n_out = its length.
cudaError_t launch_compact(const int64_t *live_in, long long n_in, int64_t *live_out, int64_t *n_out,
                           const int32_t *j, int32_t J, void *temp, size_t temp_bytes, cudaStream_t stream) {
    return cub::DeviceSelect::If(temp, temp_bytes, live_in, live_out, n_out, n_in, Unfinished{j, J}, stream);
}

}  // namespace cwc
