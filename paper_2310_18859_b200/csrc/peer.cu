// Peer-memory plumbing for expert parallelism without collectives
// (SURVEY §8(f) row 3): CUDA IPC handles to map every rank's receive buffers
// and flag words into every other rank (peer mappings over NVLink on a
// multi-GPU box; the same device in the two-process test), release/acquire
// flag signalling between the producing epilogue and the consuming kernel, and
// the segmented-arange kernel that builds the (rank, row) destination maps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>

#include "common.cuh"

namespace sida {
namespace peer {

// One thread per peer q: publish `epoch` in flags_q[me] after this stream's
// previous kernels (their peer stores) are complete and visible system-wide.
__global__ void signal_kernel(int32_t* const* peer_flags, int world, int me, int epoch) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  int32_t* f = peer_flags[q] + me;
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

// Wait until every rank has published `epoch` into this rank's flags.
__global__ void wait_kernel(const int32_t* flags, int world, int epoch) {
  const int q = threadIdx.x;
  if (q < world) {
    int v;
    while (true) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
      if (v >= epoch) break;
      __nanosleep(200);
    }
  }
  __syncthreads();
  __threadfence_system();
}

// out[i] = seg_val[b] + (p - seg_start[b]), p = index ? index[i] : i, b the
// segment holding p (seg_start ascending, n_seg + 1 entries).
__global__ void segment_map_kernel(const int32_t* __restrict__ seg_start,
                                   const int32_t* __restrict__ seg_val, int n_seg,
                                   const int32_t* __restrict__ index, int n,
                                   int32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = index ? index[i] : i;
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_start[mid] <= p) lo = mid; else hi = mid - 1;
  }
  out[i] = seg_val[lo] + (p - seg_start[lo]);
}

}  // namespace peer
}  // namespace sida

using namespace sida;

extern "C" size_t sida_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

// Handle of the allocation holding dev_ptr, plus dev_ptr's offset in it (a
// caching allocator hands out interior pointers; IPC maps whole allocations).
extern "C" int sida_ipc_handle(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  SIDA_REQUIRE(dev_ptr && handle_out && offset_out, SIDA_ERR_CONTRACT,
               "null pointer in sida_ipc_handle");
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    SIDA_REQUIRE(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) ==
                         cudaSuccess &&
                     q == cudaDriverEntryPointSuccess,
                 SIDA_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  SIDA_REQUIRE(range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) == CUDA_SUCCESS,
               SIDA_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  SIDA_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uintptr_t>(dev_ptr) - static_cast<uintptr_t>(base);
  return SIDA_OK;
}

// Map another process's allocation: base_out (for sida_ipc_close) and
// ptr_out = base + offset.
extern "C" int sida_ipc_open(const void* handle, size_t offset, void** base_out, void** ptr_out) {
  SIDA_REQUIRE(handle && base_out && ptr_out, SIDA_ERR_CONTRACT, "null pointer in sida_ipc_open");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SIDA_CUDA(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = static_cast<char*>(*base_out) + offset;
  return SIDA_OK;
}

extern "C" int sida_ipc_close(void* base) {
  SIDA_CUDA(cudaIpcCloseMemHandle(base));
  return SIDA_OK;
}

extern "C" int sida_peer_signal(int32_t* const* peer_flags, int world, int me, int epoch,
                                void* stream) {
  SIDA_REQUIRE(peer_flags && world >= 1 && world <= 1024 && me >= 0 && me < world,
               SIDA_ERR_CONTRACT, "bad peer signal (world=%d me=%d)", world, me);
  peer::signal_kernel<<<1, 32 * ceil_div(world, 32), 0, as_stream(stream)>>>(peer_flags, world,
                                                                            me, epoch);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_peer_wait(const int32_t* flags, int world, int epoch, void* stream) {
  SIDA_REQUIRE(flags && world >= 1 && world <= 1024, SIDA_ERR_CONTRACT, "bad peer wait");
  peer::wait_kernel<<<1, 32 * ceil_div(world, 32), 0, as_stream(stream)>>>(flags, world, epoch);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

extern "C" int sida_segment_map(const int32_t* seg_start, const int32_t* seg_val, int n_seg,
                                const int32_t* index, int n, int32_t* out, void* stream) {
  SIDA_REQUIRE(seg_start && seg_val && out && n_seg >= 1 && n >= 0, SIDA_ERR_CONTRACT,
               "bad segment map");
  if (n == 0) return SIDA_OK;
  peer::segment_map_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(seg_start, seg_val,
                                                                           n_seg, index, n, out);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
