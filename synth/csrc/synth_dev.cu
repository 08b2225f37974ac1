// synth_dev.cu — the seeded payload generator of synth/streams.py on the GPU,
// plus an exact compare against it (test / bench infrastructure, built as its
// own library libb200synth.so; it shares no code with libb200ring.so and holds
// none of the ring's arithmetic).
//
// Payload bytes of message (seed, channel, seq), as synth.payload_bytes:
//   key  = sm(sm(sm(seed) ^ (channel mod 2^32)) ^ (seq mod 2^48))
//   word i = sm(key + i)  (splitmix64 finaliser `sm`, wrapping arithmetic)
//   bytes = the words little-endian, truncated to the length.
// Messages of any size can thus be produced and checked on the device without
// a host copy (C4's 447,897,600-B frames, C5's 256 MiB sweep point).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t msg_key(uint64_t seed, uint32_t channel, uint64_t seq) {
  uint64_t k = sm64(seed);
  k = sm64(k ^ (uint64_t)channel);
  return sm64(k ^ (seq & 0xFFFFFFFFFFFFull));
}

constexpr uint32_t kTile = 16384;   // bytes per work tile

// Global tile g of the batch -> (message, tile): each block walks its tiles in
// increasing order with a running prefix over the message lengths.
struct Walker {
  const uint64_t* len;
  uint32_t n;
  uint32_t m = 0;
  uint64_t before = 0;   // tiles of messages [0, m)
  __device__ bool seek(uint64_t g, uint64_t& tile) {
    while (m < n) {
      const uint64_t t = (len[m] + kTile - 1) / kTile;
      if (g < before + t) { tile = g - before; return true; }
      before += t;
      ++m;
    }
    return false;
  }
};

template <bool VERIFY>
__global__ void __launch_bounds__(256) synth_kernel(const uint64_t* __restrict__ ptr, const uint64_t* __restrict__ len,
                                                    const uint32_t* __restrict__ chan,
                                                    const uint64_t* __restrict__ seq, uint32_t n, uint64_t seed,
                                                    unsigned long long* bad) {
  Walker w{len, n};
  uint64_t tile = 0;
  for (uint64_t g = blockIdx.x;; g += gridDim.x) {
    if (!w.seek(g, tile)) return;
    const uint32_t i = w.m;
    const uint64_t L = len[i];
    const uint64_t key = msg_key(seed, chan[i], seq[i]);
    uint8_t* p = reinterpret_cast<uint8_t*>(ptr[i]);
    const uint64_t lo = tile * kTile, hi = lo + kTile < L ? lo + kTile : L;
    const bool al = ((uintptr_t)p & 15) == 0;
    for (uint64_t o = lo + 16ull * threadIdx.x; o < hi; o += 16ull * blockDim.x) {
      const uint64_t w0 = sm64(key + o / 8), w1 = sm64(key + o / 8 + 1);
      if (al && o + 16 <= hi) {
        if (VERIFY) {
          const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(p + o));
          if (v.x != w0 || v.y != w1) {
            uint64_t d = v.x != w0 ? v.x ^ w0 : v.y ^ w1;
            const uint64_t at = o + (v.x != w0 ? 0 : 8) + (__ffsll((long long)d) - 1) / 8;
            atomicMin(bad + i, (unsigned long long)at);
          }
        } else {
          *reinterpret_cast<ulonglong2*>(p + o) = make_ulonglong2(w0, w1);
        }
      } else {
        for (uint32_t b = 0; b < 16 && o + b < hi; ++b) {
          const uint8_t e = (uint8_t)((b < 8 ? w0 >> (8 * b) : w1 >> (8 * (b - 8))) & 0xFF);
          if (VERIFY) {
            if (__ldcg(p + o + b) != e) atomicMin(bad + i, (unsigned long long)(o + b));
          } else {
            p[o + b] = e;
          }
        }
      }
    }
  }
}

__global__ void init_bad(unsigned long long* bad, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) bad[i] = ~0ull;
}

// View records (include/b200ring.h ring_view_t, 128 B: payload offset at byte 0,
// length at byte 8, entry header at byte 64 with producer_id at header[44,48)
// and seq at header[48,52)) -> the verify arguments.  Keys come from the header
// unless `chan` / `seq` are given; `lut` (optional) maps (producer_id, seq) to
// the generator's seq: lut[producer_id * lut_stride + seq].
__global__ void views_to_args(const uint8_t* __restrict__ views, uint32_t n, uint64_t data_base,
                              const uint32_t* __restrict__ chan, const uint64_t* __restrict__ seq,
                              const uint64_t* __restrict__ lut, uint64_t lut_stride, uint64_t* o_ptr, uint64_t* o_len,
                              uint32_t* o_chan, uint64_t* o_seq) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint8_t* v = views + 128ull * i;
    const uint64_t off = *reinterpret_cast<const uint64_t*>(v);
    const uint64_t len = *reinterpret_cast<const uint64_t*>(v + 8);
    const uint32_t pid = *reinterpret_cast<const uint32_t*>(v + 64 + 44);
    const uint32_t hseq = *reinterpret_cast<const uint32_t*>(v + 64 + 48);
    o_ptr[i] = data_base + off;
    o_len[i] = len;
    o_chan[i] = chan ? chan[i] : pid;
    uint64_t q = seq ? seq[i] : hseq;
    if (lut) q = lut[(uint64_t)o_chan[i] * lut_stride + q];
    o_seq[i] = q;
  }
}

// Test scaffolding (no payload arithmetic): CTA i occupies its SM -- all of
// its shared memory, so no other kernel's CTA can start there -- until
// base_ns + i * step_ns after the kernel started, so SMs become free one at a
// time (the late-CTA regression test of the ring's put).
__global__ void hold_sms(uint64_t base_ns, uint64_t step_ns) {
  extern __shared__ uint8_t hold_smem[];
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) hold_smem[0] = 1;
  const uint64_t until = t0 + base_ns + (uint64_t)blockIdx.x * step_ns;
  uint64_t t = t0;
  while (t < until) {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
}

// Kernels are loaded when a device is first used: a lazily loaded module waits
// for the kernels already running, and the ring tests launch these next to
// producer / consumer kernels that spin on each other.
void preload() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  // Same shared-memory carveout as the ring kernels (8 %: a 32 KB split): a CTA is
  // only placed on an SM whose L1/shared split matches its kernel's, and these
  // kernels must start next to a put that waits for the consumer they serve.
  auto load = [](auto* k) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 8);
  };
  load(synth_kernel<false>);
  load(synth_kernel<true>);
  load(init_bad);
  load(views_to_args);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, hold_sms);
  cudaFuncSetAttribute(hold_sms, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(hold_sms, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  done[dev] = true;
}

int grid_for(int device) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  return nsm * 8;
}

}  // namespace

extern "C" {

// Fill n payloads: d_ptr[i] (device address), d_len[i] bytes, keyed by
// (seed, d_chan[i], d_seq[i]).  All four arrays are DEVICE arrays of n.
// Returns a cudaError_t (0 = launched).
int synth_fill(const uint64_t* d_ptr, const uint64_t* d_len, const uint32_t* d_chan, const uint64_t* d_seq,
               uint32_t n, uint64_t seed, void* stream) {
  preload();
  if (n == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  synth_kernel<false><<<grid_for(dev), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_ptr, d_len, d_chan, d_seq, n,
                                                                                      seed, nullptr);
  return (int)cudaGetLastError();
}

// Compare n byte ranges with the generator: d_bad[i] (device, n u64) =
// offset of the first byte of message i that differs, or UINT64_MAX.
int synth_verify(const uint64_t* d_ptr, const uint64_t* d_len, const uint32_t* d_chan, const uint64_t* d_seq,
                 uint32_t n, uint64_t seed, uint64_t* d_bad, void* stream) {
  preload();
  if (n == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* bad = reinterpret_cast<unsigned long long*>(d_bad);
  init_bad<<<(n + 255) / 256, 256, 0, s>>>(bad, n);
  synth_kernel<true><<<grid_for(dev), 256, 0, s>>>(d_ptr, d_len, d_chan, d_seq, n, seed, bad);
  return (int)cudaGetLastError();
}

// synth_verify of the payloads n view records point at (inside the ring, base
// address `data_base` of its buffer region).  d_chan / d_seq / d_lut may be
// NULL (see views_to_args).  d_work: device scratch of 32 * n bytes.
int synth_verify_views(const void* d_views, uint32_t n, uint64_t data_base, const uint32_t* d_chan,
                       const uint64_t* d_seq, const uint64_t* d_lut, uint64_t lut_stride, uint64_t seed, void* d_work,
                       uint64_t* d_bad, void* stream) {
  preload();
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* w = static_cast<uint64_t*>(d_work);
  uint64_t *p = w, *l = w + n, *q = w + 2ull * n;
  auto* c = reinterpret_cast<uint32_t*>(w + 3ull * n);
  views_to_args<<<(n + 255) / 256, 256, 0, s>>>(static_cast<const uint8_t*>(d_views), n, data_base, d_chan, d_seq,
                                                d_lut, lut_stride, p, l, c, q);
  if (cudaError_t e = cudaGetLastError()) return (int)e;
  return synth_verify(p, l, c, q, n, seed, d_bad, stream);
}

// Occupy every SM of the current device (one CTA each, all shared memory),
// releasing them one at a time: CTA i exits base_ns + i * step_ns after start.
int synth_hold_sms(uint64_t base_ns, uint64_t step_ns, cudaStream_t stream) {
  preload();
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  hold_sms<<<nsm, 32, 200 << 10, stream>>>(base_ns, step_ns);
  return (int)cudaGetLastError();
}

// Host reference of one word (a check that both sides agree on the formula).
uint64_t synth_word(uint64_t seed, uint32_t channel, uint64_t seq, uint64_t i) {
  return sm64(msg_key(seed, channel, seq) + i);
}

}  // extern "C"
