// ssa_thread_s8.cu -- thread-path instantiations for 8 padded cell(s)
// (split per cell count so the variants compile in parallel).
#include "ssa_thread_impl.cuh"
#include "ssa_thread_ws.cuh"
#include "ssa_thread_ws2.cuh"

namespace cwc {
template cudaError_t launch_s<8>(int, const RunParams &, const ThreadTables &, int, size_t, cudaStream_t, bool);
}  // namespace cwc
