// ssa_thread.cu -- dispatch over the compile-time padded thread-path variants
// (kernel: ssa_thread_impl.cuh; instantiations: ssa_thread_s{1,2,4,8}.cu).
#include <cuda_runtime.h>

#include "cwc_internal.h"

namespace cwc {

template <int S>
cudaError_t launch_s(int m_pad, const RunParams &rp, const ThreadTables &tt, int threads, size_t smem, cudaStream_t st,
                     bool trace);
extern template cudaError_t launch_s<1>(int, const RunParams &, const ThreadTables &, int, size_t, cudaStream_t, bool);
extern template cudaError_t launch_s<2>(int, const RunParams &, const ThreadTables &, int, size_t, cudaStream_t, bool);
extern template cudaError_t launch_s<4>(int, const RunParams &, const ThreadTables &, int, size_t, cudaStream_t, bool);
extern template cudaError_t launch_s<8>(int, const RunParams &, const ThreadTables &, int, size_t, cudaStream_t, bool);

static const int kSPads[] = {1, 2, 4, 8};
static const int kMPads[] = {2, 3, 4, 6, 8, 12, 16, 24, 32};

int thread_pad_cells(int n) {
    for (int s : kSPads)
        if (n <= s) return s;
    return -1;
}
int thread_pad_reactions(int M) {
    for (int m : kMPads)
        if (M <= m) return m;
    return -1;
}
bool thread_variant_exists(int s_pad, int m_pad) {
    return thread_pad_cells(s_pad) == s_pad && thread_pad_reactions(m_pad) == m_pad;
}

cudaError_t launch_ssa_thread(int s_pad, int m_pad, const RunParams &rp, const ThreadTables &tt, int threads,
                              size_t smem_bytes, cudaStream_t stream) {
    const bool trace = rp.n_trace > 0;
    switch (s_pad) {
        case 1: return launch_s<1>(m_pad, rp, tt, threads, smem_bytes, stream, trace);
        case 2: return launch_s<2>(m_pad, rp, tt, threads, smem_bytes, stream, trace);
        case 4: return launch_s<4>(m_pad, rp, tt, threads, smem_bytes, stream, trace);
        case 8: return launch_s<8>(m_pad, rp, tt, threads, smem_bytes, stream, trace);
    }
    return cudaErrorInvalidValue;
}

}  // namespace cwc
