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

// Flag ping-pong: one thread on each side; each side
// polls a word in its OWN memory and stores into the other side's (the ring's
// pattern: remote store, local poll).  System-scope release / acquire, as the
// tail / head words.  Per round the ping side records its send time and the
// round trip, the pong side the time it saw the ping.
__global__ void probe_ping_kernel(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_send,
                                  uint64_t* rtt, uint64_t timeout_ns) {
  if (threadIdx.x) return;
  for (uint32_t i = 1; i <= iters; ++i) {
    const uint64_t t0 = globaltimer();
    st_release<true>(remote, (uint64_t)i);
    while (ld_acquire<true>(local) != i)
      if (globaltimer() - t0 > timeout_ns) return;
    const uint64_t t1 = globaltimer();
    t_send[i - 1] = t0;
    rtt[i - 1] = t1 - t0;
  }
}
__global__ void probe_pong_kernel(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_seen,
                                  uint64_t timeout_ns) {
  if (threadIdx.x) return;
  const uint64_t t0 = globaltimer();
  for (uint32_t i = 1; i <= iters; ++i) {
    while (ld_acquire<true>(local) != i)
      if (globaltimer() - t0 > timeout_ns) return;
    t_seen[i - 1] = globaltimer();
    st_release<true>(remote, (uint64_t)i);
  }
}

cudaError_t launch_probe_ping(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_send,
                              uint64_t* rtt, uint64_t timeout_ns, cudaStream_t s) {
  probe_ping_kernel<<<1, 32, 0, s>>>(remote, local, iters, t_send, rtt, timeout_ns);
  return cudaGetLastError();
}
cudaError_t launch_probe_pong(uint64_t* remote, const uint64_t* local, uint32_t iters, uint64_t* t_seen,
                              uint64_t timeout_ns, cudaStream_t s) {
  probe_pong_kernel<<<1, 32, 0, s>>>(remote, local, iters, t_seen, timeout_ns);
  return cudaGetLastError();
}

cudaError_t preload_clock() {
  cudaError_t e = preload_kernel(clock_publish_kernel);
  if (e == cudaSuccess) e = preload_kernel(probe_ping_kernel);
  if (e == cudaSuccess) e = preload_kernel(probe_pong_kernel);
  return e;
}

}  // namespace b200ring
