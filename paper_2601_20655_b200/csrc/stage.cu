// stage.cu — a synthetic stage kernel with a fused put epilogue (SURVEY.md §8
// f2): out = bf16(in * scale), computed and written by the same threads
// directly into the next entry of the peer ring (ring_stage.cuh), so the
// stage's output never round-trips through its own HBM and no separate put
// launch runs.  Stand-in for the last kernel of a model stage (e.g. a VAE
// decoder writing frames).
#include <cuda_bf16.h>

#include "ring_internal.h"
#include "../../include/b200ring_device.cuh"

namespace b200ring {

struct StageArgs {
  ring_dev_peer_t peer;
  ring_hdr_t hdr;
  const __nv_bfloat16* in;
  uint64_t n;
  uint32_t* status;
  uint64_t timeout_ns;
  float scale;
  uint32_t flags;
};

template <bool SYS>
__global__ void __launch_bounds__(256) stage_scale_put_kernel(const StageArgs a) {
  using namespace stage;
  StageCtl* ctl = reinterpret_cast<StageCtl*>(a.peer.ctl);
  const uint64_t len = 2 * a.n;
  const uint64_t P = grid_reserve<SYS>(a.peer, ctl, len, a.timeout_ns);
  if (P) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(payload_ptr(a.peer, P));   // 16-B aligned (R11)
    const uint64_t n8 = a.n / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(a.in) & 15) == 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
      __nv_bfloat162 v[4];
      if (aligned) {
        const int4 x = __ldcs(reinterpret_cast<const int4*>(a.in) + i);
        memcpy(v, &x, 16);
      } else {
        for (int j = 0; j < 4; ++j) v[j] = __halves2bfloat162(a.in[8 * i + 2 * j], a.in[8 * i + 2 * j + 1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 fv = __bfloat1622float2(v[j]);
        v[j] = __floats2bfloat162_rn(fv.x * a.scale, fv.y * a.scale);   // round to nearest even
      }
      int4 y;
      memcpy(&y, v, 16);
      st16(out + 8 * i, y);
    }
    for (uint64_t i = 8 * n8 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride)
      out[i] = __float2bfloat16_rn(__bfloat162float(a.in[i]) * a.scale);
  }
  grid_commit<SYS>(a.peer, ctl, P, len, a.hdr, a.flags, a.status);
}

cudaError_t preload_stage() {
  cudaError_t e = preload_kernel(stage_scale_put_kernel<true>);
  if (e == cudaSuccess) e = preload_kernel(stage_scale_put_kernel<false>);
  return e;
}

cudaError_t launch_stage_scale_put(const ring_dev_peer_t& peer, const void* in, uint64_t n, float scale,
                                   const ring_hdr_t& hdr, uint32_t flags, uint32_t* status, uint64_t timeout_ns,
                                   uint32_t ctas, cudaStream_t s) {
  StageArgs a{};
  a.peer = peer;
  a.hdr = hdr;
  a.in = static_cast<const __nv_bfloat16*>(in);
  a.n = n;
  a.status = status;
  a.timeout_ns = timeout_ns;
  a.scale = scale;
  a.flags = flags;
  if (peer.sys) stage_scale_put_kernel<true><<<ctas, 256, 0, s>>>(a);
  else stage_scale_put_kernel<false><<<ctas, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace b200ring
