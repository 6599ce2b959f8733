// Status plumbing, device check, expert streaming and host-side slot packing.
//
// sida_expert_copy is the B200 replacement of the simulated transfer in
// ref offload.py:207-222 + pipeline.py:141-146 (a sleep): a real
// cudaMemcpyAsync from pinned host DRAM into an HBM slot on the dedicated copy
// stream, ordered after the slot's last reader and followed by a done event
// the compute stream waits on.
#include <stdarg.h>
#include <string.h>

#include <atomic>

#include "common.cuh"

namespace sida {

static thread_local char g_err[512] = {0};
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace sida

extern "C" int sida_abi_version(void) { return 1; }

extern "C" const char* sida_last_error(void) { return sida::g_err; }

extern "C" unsigned long long sida_launch_count(void) {
  return sida::g_launches.load(std::memory_order_relaxed);
}

extern "C" int sida_device_check(int device) {
  cudaDeviceProp prop;
  SIDA_CUDA(cudaGetDeviceProperties(&prop, device));
  SIDA_REQUIRE(prop.major == 10 && prop.minor == 0, SIDA_ERR_UNSUPPORTED,
               "device %d is sm_%d%d (%s); this library is built for sm_100a only", device,
               prop.major, prop.minor, prop.name);
  return SIDA_OK;
}

extern "C" size_t sida_slot_bytes(int d, int h) {
  size_t raw = (2ull * d * h + h + d) * 2ull;
  return sida::align_up(raw, 256);
}

extern "C" int sida_expert_copy(void* dst_slot, const void* src_pinned, size_t bytes,
                                void* copy_stream, void* wait_event, void* done_event) {
  SIDA_REQUIRE(dst_slot && src_pinned, SIDA_ERR_CONTRACT, "null copy endpoint");
  cudaStream_t s = sida::as_stream(copy_stream);
  if (wait_event) SIDA_CUDA(cudaStreamWaitEvent(s, reinterpret_cast<cudaEvent_t>(wait_event), 0));
  SIDA_CUDA(cudaMemcpyAsync(dst_slot, src_pinned, bytes, cudaMemcpyHostToDevice, s));
  if (done_event) SIDA_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), s));
  return SIDA_OK;
}

static inline uint16_t host_bf16(double v) {
  float f = static_cast<float>(v);  // RNE double -> float
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

extern "C" int sida_pack_expert_host(const double* w1, const double* b1, const double* w2,
                                     const double* b2, int d, int h, void* dst) {
  SIDA_REQUIRE(w1 && b1 && w2 && b2 && dst, SIDA_ERR_CONTRACT, "null pointer in pack");
  uint16_t* out = static_cast<uint16_t*>(dst);
  uint16_t* w1t = out;                    // (h, d): w1t[n][k] = w1[k][n]
  uint16_t* w2t = out + (size_t)h * d;    // (d, h): w2t[n][k] = w2[k][n]
  uint16_t* ob1 = out + 2ull * h * d;
  uint16_t* ob2 = ob1 + h;
  for (int k = 0; k < d; ++k)
    for (int n = 0; n < h; ++n) w1t[(size_t)n * d + k] = host_bf16(w1[(size_t)k * h + n]);
  for (int k = 0; k < h; ++k)
    for (int n = 0; n < d; ++n) w2t[(size_t)n * h + k] = host_bf16(w2[(size_t)k * d + n]);
  for (int n = 0; n < h; ++n) ob1[n] = host_bf16(b1[n]);
  for (int n = 0; n < d; ++n) ob2[n] = host_bf16(b2[n]);
  size_t used = (2ull * d * h + h + d) * 2ull;
  memset(static_cast<char*>(dst) + used, 0, sida_slot_bytes(d, h) - used);
  return SIDA_OK;
}

// ---------------------------------------------------------------------------
// k > 1 rank combine: out[t] = resid[t] + sum_r y[t*k + r], ranks in order
// (ref moe.py:252-262 accumulates rank outputs in order then adds x).
__global__ void combine_ranks_kernel(const float4* __restrict__ y, const float4* __restrict__ resid,
                                     int n_tokens, int k, int d4, float4* __restrict__ out,
                                     uint2* __restrict__ out_bf16) {
  long total = (long)n_tokens * d4;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    long t = i / d4;
    int c = static_cast<int>(i - t * d4);
    float4 acc = y[(t * k) * d4 + c];
    for (int r = 1; r < k; ++r) {
      float4 v = y[(t * k + r) * d4 + c];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (resid) {
      float4 x = resid[t * d4 + c];
      acc.x = x.x + acc.x; acc.y = x.y + acc.y; acc.z = x.z + acc.z; acc.w = x.w + acc.w;
    }
    out[t * d4 + c] = acc;
    if (out_bf16) out_bf16[t * d4 + c] = make_uint2(sida::pack_bf16x2(acc.x, acc.y),
                                                   sida::pack_bf16x2(acc.z, acc.w));
  }
}

extern "C" int sida_combine_ranks(const float* y, const float* resid, int n_tokens, int k, int d,
                                  float* out, uint16_t* out_bf16, void* stream) {
  SIDA_REQUIRE(d % 4 == 0 && k >= 1 && n_tokens >= 0, SIDA_ERR_UNSUPPORTED,
               "combine needs d %% 4 == 0 (d=%d) and k >= 1", d);
  if (n_tokens == 0) return SIDA_OK;
  long total = (long)n_tokens * (d / 4);
  int blocks = (int)std::min<long>((total + 255) / 256, sida::kNumSMs * 8);
  combine_ranks_kernel<<<blocks, 256, 0, sida::as_stream(stream)>>>(
      reinterpret_cast<const float4*>(y), reinterpret_cast<const float4*>(resid), n_tokens, k,
      d / 4, reinterpret_cast<float4*>(out), reinterpret_cast<uint2*>(out_bf16));
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}

// Small int32 rows (expert -> slot maps, sequence offsets) host -> HBM as
// kernel parameters instead of an H2D memcpy: a memcpy on the compute or hash
// stream shares the copy engines with the multi-MB expert copies in flight
// on the copy stream and can wait behind them for milliseconds; a launch
// carrying the values in its parameter block does not touch the copy engines.
namespace {
constexpr int kPokeMax = 1000;  // 4 KB parameter block
struct PokeArgs {
  int n;
  int32_t v[kPokeMax];
};
__global__ void poke_i32_kernel(int32_t* __restrict__ dst, const PokeArgs a) {
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) dst[i] = a.v[i];
}
}  // namespace

extern "C" int sida_poke_i32(int32_t* dst, const int32_t* src, int n, void* stream) {
  SIDA_REQUIRE(n >= 0 && (n == 0 || (dst && src)), SIDA_ERR_CONTRACT,
               "bad sida_poke_i32 arguments (n=%d)", n);
  for (int off = 0; off < n; off += kPokeMax) {
    PokeArgs a;
    a.n = n - off < kPokeMax ? n - off : kPokeMax;
    memcpy(a.v, src + off, sizeof(int32_t) * a.n);
    poke_i32_kernel<<<1, 256, 0, sida::as_stream(stream)>>>(dst + off, a);
    SIDA_LAUNCH_CHECK();
  }
  return SIDA_OK;
}

// Byte copy by the SMs between device memory and pinned (mapped, UVA) host
// memory: for the per-batch token rows up and the logits down, which as
// cudaMemcpyAsync on the hash / compute stream would queue on the copy
// engines behind the expert copies the planner has already enqueued.
namespace {
__global__ void copy_sm_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                               size_t bytes) {
  const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (vec) {
    const size_t n16 = bytes / 16;
    for (size_t i = t; i < n16; i += stride)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = n16 * 16 + t; i < bytes; i += stride) dst[i] = src[i];
  } else {
    for (size_t i = t; i < bytes; i += stride) dst[i] = src[i];
  }
}
}  // namespace

extern "C" int sida_copy_sm(void* dst, const void* src, size_t bytes, void* stream) {
  SIDA_REQUIRE(bytes == 0 || (dst && src), SIDA_ERR_CONTRACT, "null pointer passed to sida_copy_sm");
  if (bytes == 0) return SIDA_OK;
  const size_t chunks = (bytes + 16 * 256 - 1) / (16 * 256);
  const int blocks = static_cast<int>(chunks < 148 ? chunks : 148);
  copy_sm_kernel<<<blocks, 256, 0, sida::as_stream(stream)>>>(static_cast<uint8_t*>(dst),
                                                              static_cast<const uint8_t*>(src), bytes);
  SIDA_LAUNCH_CHECK();
  return SIDA_OK;
}
