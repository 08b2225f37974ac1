// clock.cu — measurement support (not on the data path): read a GPU's
// %globaltimer from the host, so that per-message latencies t_visible - t_put
// stamped on two different GPUs can be put on one time base.  The host brackets
// each sample with its own monotonic clock; the narrowest bracket gives the
// offset between the GPU's globaltimer and the host clock.
#include "ring_internal.h"

namespace b200ring {

// Publishes the GPU's globaltimer into mapped pinned host memory continuously
// for `duration_ns`; the host reads it in a loop (see ring_clock_offset_ns).
__global__ void clock_publish_kernel(unsigned long long* host, unsigned long long duration_ns) {
  const uint64_t t0 = globaltimer();
  uint64_t t = t0;
  while (t - t0 < duration_ns) {
    t = globaltimer();
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(host), "l"((unsigned long long)t) : "memory");
  }
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(host + 1), "l"(1ull) : "memory");
}

cudaError_t launch_clock_publish(unsigned long long* mapped_host, unsigned long long duration_ns, cudaStream_t s) {
  clock_publish_kernel<<<1, 1, 0, s>>>(mapped_host, duration_ns);
  return cudaGetLastError();
}

cudaError_t preload_clock() {
  return preload_kernel(clock_publish_kernel);
}

}  // namespace b200ring
