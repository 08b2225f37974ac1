// host.cu — the C ABI of include/b200ring.h: ring lifetime, IPC handles,
// attachment of producers, launch configuration of the put / get / release
// kernels and the stage router.  No protocol step runs here: the host only
// validates arguments, allocates, maps and launches ("no CPU
// intervention" on the data path).
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <cstring>
#include <mutex>
#include <vector>

#include "ring_internal.h"
#include "../../include/b200ring_device.cuh"

using namespace b200ring;

namespace {

thread_local char g_cuda_err[512] = "";
std::atomic<uint64_t> g_timeout_ns{2000000000ull};
std::atomic<uint64_t> g_lock_timeout_ns{200000ull};   // TL of fault-tolerant rings
std::atomic<uint64_t> g_hole_timeout_ns{50000000ull}; // reserve-then-commit hole timeout (50 ms)
std::atomic<uint64_t> g_launches{0};
std::mutex g_mu;
const uint32_t g_token = 0x9e3779b9u ^ (uint32_t)getpid() ^ (uint32_t)((uintptr_t)&g_mu & 0xffffffffu);

constexpr uint32_t kMagicRing = 0x52494e47;    // "RING"
constexpr uint32_t kMagicMirror = 0x4d495252;  // "MIRR"

struct HandleBlob {
  uint32_t magic;
  int32_t device;
  int32_t pid;
  uint32_t token;
  uint64_t ptr;          // device pointer in the exporting process
  uint64_t R;
  uint32_t N;
  uint32_t max_producers;
  uint32_t flags;
  uint32_t producer_id;  // mirror handles
  cudaIpcMemHandle_t ipc;
  // split placement (ring_create_split): the buffer region is a second allocation
  uint64_t data_ptr;     // 0 = the buffer region follows the control words in `ptr`
  int32_t data_device;
  uint32_t _d;
  cudaIpcMemHandle_t data_ipc;
};
static_assert(sizeof(HandleBlob) <= sizeof(ring_handle_t), "handle too large");

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
               __FILE__, __LINE__);                                                          \
      return RING_ECUDA;                                                                     \
    }                                                                                        \
  } while (0)

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---- CRC-32 slicing-by-4 tables (R10) ---------------------------------------
// Table 0 is the standard 256-entry table of the reflected CRC-32
// (0xEDB88320), built from this file's own shift-register step; table k
// advances table k-1 by one more zero byte.  Kernels consume 4 bytes per step.
// Slicing-by-4 tables (kCrcTableWords), then kCrcPowWords powers
// x^(2^n) mod P (reflected) for combining CRCs of adjacent byte ranges.
// The GF(2) multiply and the x^(2^n) table follow zlib's crc32_combine
// construction (multmodp / x2nmodp, zlib 1.2.12+, (C) 1995-2022 Jean-loup
// Gailly and Mark Adler, zlib license; an independent rewrite of that
// canonical routine).
static uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return p;
}
std::vector<uint32_t> build_crc_table() {
  std::vector<uint32_t> t(kCrcTableWords + kCrcPowWords);
  uint32_t* pw = t.data() + kCrcTableWords;
  pw[0] = 1u << 30;   // x^1
  for (int n = 1; n < kCrcPowWords; ++n) pw[n] = gf2_mulmod(pw[n - 1], pw[n - 1]);
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t reg = i;
    for (int b = 0; b < 8; ++b) reg = (reg & 1) ? (reg >> 1) ^ 0xEDB88320u : reg >> 1;
    t[i] = reg;
  }
  for (int k = 1; k < 4; ++k)
    for (uint32_t i = 0; i < 256; ++i) t[k * 256 + i] = (t[(k - 1) * 256 + i] >> 8) ^ t[t[(k - 1) * 256 + i] & 0xFFu];
  return t;
}
uint32_t* g_crc_dev[64] = {};
// Put engines running per device: a resident engine never exits on its own, so
// while one runs, host calls that would synchronise the whole device
// synchronise the legacy default stream instead (quiesce).
std::atomic<int> g_engines[64];
cudaError_t quiesce() {
  int device = -1;
  cudaGetDevice(&device);
  if (device >= 0 && device < 64 && g_engines[device].load() > 0) return cudaStreamSynchronize(cudaStreamLegacy);
  return cudaDeviceSynchronize();
}
ring_status_t crc_table_dev(int device, const uint32_t** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (device < 0 || device >= 64) return RING_EINVAL;
  if (!g_crc_dev[device]) {
    DevGuard g(device);
    static const std::vector<uint32_t> host = build_crc_table();
    uint32_t* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, host.size() * 4));
    CUDA_TRY(cudaMemcpy(d, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
    // Load every kernel on this device now (lazy loading would otherwise wait
    // for a running consumer kernel at the producer's first launch).
    CUDA_TRY(preload_put());
    CUDA_TRY(preload_get());
    CUDA_TRY(preload_clock());
    CUDA_TRY(preload_stage());
    CUDA_TRY(preload_fanin());
    g_crc_dev[device] = d;
  }
  *out = g_crc_dev[device];
  return RING_OK;
}

ring_status_t enable_peer(int from, int to) {
  if (from == to) return RING_OK;
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, from, to));
  if (!can) return RING_EPEER;
  DevGuard g(from);
  cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RING_OK;
  }
  CUDA_TRY(e);
  return RING_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr uint32_t kTraceWords = 2048;   // debug timeline of one put launch

}  // namespace

int b200ring::ring_carveout_percent() {
  static const int pct = [] {
    const char* e = getenv("B200RING_CARVEOUT");
    const int v = e ? atoi(e) : 8;
    return v >= 0 && v <= 100 ? v : 8;
  }();
  return pct;
}

// ---------------------------------------------------------------------------
struct ring_s {
  int device = 0;
  uint8_t* base = nullptr;
  uint64_t R = 0, data_off = 0, alloc = 0;
  uint32_t N = 0, max_producers = 0, flags = 0;
  uint64_t** mirrors_dev = nullptr;          // [max_producers] pointers into producer mirrors
  std::vector<void*> opened;                 // IPC mappings of mirrors to close
  LaunchCtx* ctx = nullptr;
  uint32_t launches = 0;                     // selects the LaunchSet of each get launch
  uint32_t copy_ctas = 0, threads = 0, chunk = 0;
  const uint32_t* crc = nullptr;
  uint32_t sys = 1;
  bool owner = true;                         // false: ring_open of a ring owned elsewhere (pull placement)
  bool ipc_opened = false;                   // base is an IPC mapping of another process's ring
  uint8_t* data = nullptr;                   // buffer region (base + data_off, or the split allocation)
  uint8_t* hdrs = nullptr;                   // split placement: header copies in the control allocation
  int data_device = -1;                      // split placement: the GPU holding the buffer region
  bool remote_data = false;                  // split / pull placement: the buffer region is on another GPU
  uint64_t* trace = nullptr;                 // debug timeline of the get kernels (B200RING_TRACE=1)
};

struct ring_peer_s {
  int device = 0;
  int ring_device = 0;
  int data_device = 0;                       // where the buffer region lives (the ring's GPU unless split)
  uint8_t* ring = nullptr;
  bool ipc_opened = false;
  DestState* st = nullptr;
  DestDesc* desc_dev = nullptr;
  DestDesc desc{};
  LaunchCtx* ctx = nullptr;
  uint64_t base = 0;                         // messages submitted
  uint32_t launches = 0;
  uint32_t copy_ctas = 0, threads = 0, chunk = 0, copy_mode = 0;
  uint64_t* trace = nullptr;                 // debug timeline (B200RING_TRACE=1)
  const uint32_t* crc = nullptr;
  uint8_t* data_opened = nullptr;            // split placement: IPC mapping of the buffer region
  FaultSpec fault;                           // test-only fault injection (fault-tolerant rings)
  void* stage_ctl = nullptr;                 // grid-coordination block of fused puts (ring_stage.cuh)
  uint32_t launches_stage = 0;
  // persistent put engine (ring_peer_engine_start)
  EngineQueue* eq = nullptr;
  EngineHost* eh = nullptr;                  // pinned, mapped: lease / alive
  cudaStream_t eng_stream = nullptr;
  cudaEvent_t eng_exit = nullptr;
  cudaEvent_t eng_ready = nullptr;
  bool engine_on = false;
  uint64_t posted = 0;                       // batches submitted to the engine
};

struct router_s {
  int device = 0;
  uint32_t max_routes = 0;
  Route* routes_dev = nullptr;
  std::vector<Route> routes;                 // host shadow (rr excluded)
  DestDesc* dests_dev = nullptr;             // [kMaxRouterDests]
  std::vector<ring_peer_t> dests;
  LaunchCtx* ctx = nullptr;
  uint64_t base = 0;
  uint32_t launches = 0;
  uint32_t copy_ctas = 0, threads = 0, chunk = 0;
  const uint32_t* crc = nullptr;
};

extern "C" {

const char* ring_strerror(ring_status_t s) {
  switch (s) {
    case RING_OK: return "ok";
    case RING_EINVAL: return "invalid argument";
    case RING_ENOMEM: return "out of device memory";
    case RING_EMSGSIZE: return "message larger than the ring (or the copy-out buffer)";
    case RING_FULL: return "ring full (try mode)";
    case RING_EMPTY: return "ring empty (try mode)";
    case RING_ETIMEDOUT: return "device spin timed out";
    case RING_ECORRUPT: return "entry header checksum mismatch";
    case RING_ECUDA: return "CUDA error";
    case RING_EPEER: return "no peer access / IPC failure";
    case RING_EPENDING: return "pending";
    case RING_EDROPPED: return "dropped: size slot taken after a lock take-over";
    case RING_EREJECTED: return "rejected by admission control";
  }
  return "unknown";
}
const char* ring_last_cuda_error(void) { return g_cuda_err; }
ring_status_t ring_set_hole_timeout_ns(uint64_t ns) {
  if (ns == 0) return RING_EINVAL;
  g_hole_timeout_ns = ns;
  return RING_OK;
}
ring_status_t ring_set_lock_timeout_ns(uint64_t ns) {
  if (ns == 0) return RING_EINVAL;
  g_lock_timeout_ns = ns;
  return RING_OK;
}
ring_status_t ring_set_timeout_ns(uint64_t ns) {
  if (ns == 0) return RING_EINVAL;
  g_timeout_ns = ns;
  return RING_OK;
}
uint64_t ring_launch_count(void) { return g_launches.load(); }

ring_status_t ring_clock_offset_ns(int device, int64_t* offset_ns) {
  if (!offset_ns) return RING_EINVAL;
  const uint32_t* unused = nullptr;
  ring_status_t s = crc_table_dev(device, &unused);   // loads the kernels on this device
  if (s != RING_OK) return s;
  DevGuard g(device);
  unsigned long long* host = nullptr;
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&host), 64, cudaHostAllocMapped));
  volatile unsigned long long* vh = host;
  vh[0] = 0;
  vh[1] = 0;
  unsigned long long* dev = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), host, 0));
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CUDA_TRY(launch_clock_publish(dev, 3000000ull, st));
  // gpu(t_after) >= g for every sample, so offset >= g - t_after; the max over
  // samples is within one PCIe write latency of the true offset.
  int64_t best = INT64_MIN;
  timespec ts;
  while (vh[1] == 0) {
    const unsigned long long gv = vh[0];
    clock_gettime(CLOCK_MONOTONIC, &ts);
    const int64_t t_after = (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
    if (gv) best = std::max(best, (int64_t)gv - t_after);
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  cudaStreamDestroy(st);
  cudaFreeHost(host);
  if (best == INT64_MIN) return RING_ECUDA;
  *offset_ns = best;
  g_launches++;
  return RING_OK;
}
ring_status_t ring_probe_rtt(int dev_a, int dev_b, uint32_t iters, uint64_t* rtt_min_ns, uint64_t* rtt_p50_ns,
                            int64_t* offset_b_minus_a_ns) {
  if (!rtt_min_ns || !rtt_p50_ns || iters == 0 || iters > (1u << 20)) return RING_EINVAL;
  const uint32_t* unused = nullptr;
  ring_status_t s = crc_table_dev(dev_a, &unused);   // loads the kernels
  if (s == RING_OK) s = crc_table_dev(dev_b, &unused);
  if (s != RING_OK) return s;
  s = enable_peer(dev_a, dev_b);
  if (s == RING_OK) s = enable_peer(dev_b, dev_a);
  if (s != RING_OK) return s;
  uint64_t *fa = nullptr, *fb = nullptr, *ta = nullptr, *rt = nullptr, *tb = nullptr;
  cudaStream_t sa = nullptr, sb = nullptr;
  {
    DevGuard g(dev_a);
    CUDA_TRY(cudaMalloc(&fa, 256));
    CUDA_TRY(cudaMemset(fa, 0, 256));
    CUDA_TRY(cudaMalloc(&ta, 16ull * iters));
    rt = ta + iters;
    CUDA_TRY(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  }
  {
    DevGuard g(dev_b);
    CUDA_TRY(cudaMalloc(&fb, 256));
    CUDA_TRY(cudaMemset(fb, 0, 256));
    CUDA_TRY(cudaMalloc(&tb, 8ull * iters));
    CUDA_TRY(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    CUDA_TRY(quiesce());                                                   // the flags are zero
  }
  {
    DevGuard g(dev_a);
    CUDA_TRY(quiesce());
    CUDA_TRY(cudaMemset(ta, 0, 16ull * iters));
    CUDA_TRY(quiesce());
  }
  {
    DevGuard g(dev_b);
    CUDA_TRY(launch_probe_pong(fa, fb, iters, tb, 2000000000ull, sb));   // pong first: it waits
  }
  {
    DevGuard g(dev_a);
    CUDA_TRY(launch_probe_ping(fb, fa, iters, ta, rt, 2000000000ull, sa));
    CUDA_TRY(cudaStreamSynchronize(sa));
  }
  {
    DevGuard g(dev_b);
    CUDA_TRY(cudaStreamSynchronize(sb));
  }
  std::vector<uint64_t> hs(iters), hr(iters), hb(iters);
  CUDA_TRY(cudaMemcpy(hs.data(), ta, 8ull * iters, cudaMemcpyDefault));
  CUDA_TRY(cudaMemcpy(hr.data(), rt, 8ull * iters, cudaMemcpyDefault));
  CUDA_TRY(cudaMemcpy(hb.data(), tb, 8ull * iters, cudaMemcpyDefault));
  { DevGuard g(dev_a); cudaFree(fa); cudaFree(ta); cudaStreamDestroy(sa); }
  { DevGuard g(dev_b); cudaFree(fb); cudaFree(tb); cudaStreamDestroy(sb); }
  g_launches += 2;
  // the first 10 % are warm-up; NTP-style offset from the minimum-RTT round
  const uint32_t w = iters / 10;
  std::vector<uint64_t> r(hr.begin() + w, hr.end());
  if (r.empty() || *std::min_element(r.begin(), r.end()) == 0) return RING_ETIMEDOUT;
  uint32_t best = w;
  for (uint32_t i = w; i < iters; ++i)
    if (hr[i] < hr[best]) best = i;
  std::sort(r.begin(), r.end());
  *rtt_min_ns = r.front();
  *rtt_p50_ns = r[r.size() / 2];
  if (offset_b_minus_a_ns)
    *offset_b_minus_a_ns = (int64_t)hb[best] - (int64_t)(hs[best] + hr[best] / 2);
  return RING_OK;
}

uint64_t ring_footprint(uint64_t len) { return footprint(len); }

// ---- lifetime ------------------------------------------------------------------
ring_status_t ring_create(int device, uint64_t data_bytes, uint32_t n_slots, uint32_t max_producers,
                          uint32_t flags, ring_t* out) {
  if (!out || data_bytes == 0 || data_bytes % kAlign || data_bytes >= (1ull << 39) || n_slots == 0 ||
      (n_slots & (n_slots - 1)) || n_slots > RING_MAX_SLOTS || max_producers == 0 ||
      max_producers > RING_MAX_PRODUCERS)
    return RING_EINVAL;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return RING_EINVAL;
  DevGuard g(device);
  ring_s* r = new ring_s;
  r->device = device;
  r->R = data_bytes;
  r->N = n_slots;
  r->max_producers = max_producers;
  r->flags = flags;
  r->sys = (flags & RING_CREATE_LOCAL) ? 0u : 1u;
  r->data_off = data_offset(n_slots);
  r->alloc = r->data_off + data_bytes;
  cudaError_t e = cudaMalloc(&r->base, r->alloc);
  r->data = r->base + r->data_off;
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete r;
    return RING_ENOMEM;
  }
  // Only the control words and the size region need zeroing: entries are
  // always written before they are published.
  CUDA_TRY(cudaMemset(r->base, 0, r->data_off));
  CUDA_TRY(cudaMalloc(&r->mirrors_dev, sizeof(uint64_t*) * max_producers));
  CUDA_TRY(cudaMemset(r->mirrors_dev, 0, sizeof(uint64_t*) * max_producers));
  CUDA_TRY(cudaMalloc(&r->ctx, sizeof(LaunchCtx)));
  CUDA_TRY(cudaMemset(r->ctx, 0, sizeof(LaunchCtx)));
  CUDA_TRY(quiesce());
  ring_status_t s = crc_table_dev(device, &r->crc);
  if (s != RING_OK) return s;
  *out = r;
  return RING_OK;
}

ring_status_t ring_create_split(int device, int data_device, uint64_t data_bytes, uint32_t n_slots,
                                uint32_t max_producers, uint32_t flags, ring_t* out) {
  if (!out || data_bytes == 0 || data_bytes % kAlign || data_bytes >= (1ull << 39) || n_slots == 0 ||
      (n_slots & (n_slots - 1)) || n_slots > RING_MAX_SLOTS || max_producers == 0 ||
      max_producers > RING_MAX_PRODUCERS ||
      (flags & (RING_CREATE_LOCAL | RING_CREATE_FAULT_TOLERANT | RING_CREATE_RESERVE_COMMIT)))
    return RING_EINVAL;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev || data_device < 0 || data_device >= ndev) return RING_EINVAL;
  ring_status_t s = enable_peer(device, data_device);
  if (s == RING_OK) s = enable_peer(data_device, device);
  if (s != RING_OK) return s;
  ring_s* r = new ring_s;
  r->device = device;
  r->data_device = data_device;
  r->remote_data = data_device != device;
  r->R = data_bytes;
  r->N = n_slots;
  r->max_producers = max_producers;
  r->flags = flags;
  r->sys = 1;
  r->data_off = split_control_bytes(n_slots);   // (ring_get_info: no buffer region in this allocation)
  r->alloc = r->data_off;
  {
    DevGuard gd(data_device);
    cudaError_t e = cudaMalloc(&r->data, data_bytes);
    if (e != cudaSuccess) { cudaGetLastError(); delete r; return RING_ENOMEM; }
  }
  DevGuard g(device);
  cudaError_t e = cudaMalloc(&r->base, r->alloc);
  if (e != cudaSuccess) {
    cudaGetLastError();
    DevGuard gd(data_device);
    cudaFree(r->data);
    delete r;
    return RING_ENOMEM;
  }
  r->hdrs = r->base + hdr_mirror_offset(n_slots);
  CUDA_TRY(cudaMemset(r->base, 0, r->alloc));
  CUDA_TRY(cudaMalloc(&r->mirrors_dev, sizeof(uint64_t*) * max_producers));
  CUDA_TRY(cudaMemset(r->mirrors_dev, 0, sizeof(uint64_t*) * max_producers));
  CUDA_TRY(cudaMalloc(&r->ctx, sizeof(LaunchCtx)));
  CUDA_TRY(cudaMemset(r->ctx, 0, sizeof(LaunchCtx)));
  CUDA_TRY(quiesce());
  s = crc_table_dev(device, &r->crc);
  if (s != RING_OK) return s;
  *out = r;
  return RING_OK;
}

ring_status_t ring_destroy(ring_t r) {
  if (!r) return RING_EINVAL;
  DevGuard g(r->device);
  quiesce();
  for (void* p : r->opened) cudaIpcCloseMemHandle(p);
  cudaFree(r->ctx);
  cudaFree(r->mirrors_dev);
  if (r->trace) cudaFree(r->trace);
  if (r->owner) cudaFree(r->base);
  else if (r->ipc_opened) cudaIpcCloseMemHandle(r->base);
  if (r->owner && r->data_device >= 0) {
    DevGuard gd(r->data_device);
    cudaFree(r->data);
  }
  delete r;
  return RING_OK;
}

// Pull placement: the consumer on `device` takes a ring that lives in another
// GPU's memory (created there with ring_create, usually by its producer).  The
// protocol is unchanged -- same words, same steps, same oracle -- only the
// placement of the ring moves: the producer's WB becomes a local HBM write and
// the consumer's copy-out get reads the payload over NVLink (the paper's
// one-sided READ, in place of the one-sided WRITE).
ring_status_t ring_open(const ring_handle_t* h, int device, ring_t* out) {
  if (!h || !out) return RING_EINVAL;
  HandleBlob b;
  memcpy(&b, h->bytes, sizeof b);
  if (b.magic != kMagicRing) return RING_EINVAL;
  if (b.flags & (RING_CREATE_LOCAL | RING_CREATE_FAULT_TOLERANT | RING_CREATE_RESERVE_COMMIT)) return RING_EINVAL;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return RING_EINVAL;
  const bool same_process = b.pid == (int32_t)getpid() && b.token == g_token;
  ring_s* r = new ring_s;
  r->device = device;
  r->R = b.R;
  r->N = b.N;
  r->max_producers = b.max_producers;
  r->flags = b.flags;
  r->sys = 1;
  r->owner = false;
  r->remote_data = b.device != device;
  if (b.data_ptr) { delete r; return RING_EINVAL; }   // split rings are consumed where their control words live
  r->data_off = data_offset(b.N);
  r->alloc = r->data_off + b.R;
  if (same_process) {
    ring_status_t s = enable_peer(device, b.device);
    if (s != RING_OK) { delete r; return s; }
    r->base = reinterpret_cast<uint8_t*>(b.ptr);
  } else {
    DevGuard g(device);
    void* m = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&m, b.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      snprintf(g_cuda_err, sizeof g_cuda_err, "cudaIpcOpenMemHandle(ring): %s", cudaGetErrorString(e));
      cudaGetLastError();
      delete r;
      return RING_EPEER;
    }
    r->base = static_cast<uint8_t*>(m);
    r->ipc_opened = true;
  }
  r->data = r->base + r->data_off;
  DevGuard g(device);
  CUDA_TRY(cudaMalloc(&r->mirrors_dev, sizeof(uint64_t*) * r->max_producers));
  CUDA_TRY(cudaMemset(r->mirrors_dev, 0, sizeof(uint64_t*) * r->max_producers));
  CUDA_TRY(cudaMalloc(&r->ctx, sizeof(LaunchCtx)));
  CUDA_TRY(cudaMemset(r->ctx, 0, sizeof(LaunchCtx)));
  CUDA_TRY(quiesce());
  ring_status_t s = crc_table_dev(device, &r->crc);
  if (s != RING_OK) return s;
  *out = r;
  return RING_OK;
}

ring_status_t ring_get_info(ring_t r, ring_info_t* out) {
  if (!r || !out) return RING_EINVAL;
  out->device = r->device;
  out->n_slots = r->N;
  out->max_producers = r->max_producers;
  out->data_bytes = r->R;
  out->base = reinterpret_cast<uint64_t>(r->base);
  out->data = reinterpret_cast<uint64_t>(r->data);
  out->data_offset = r->data_off;
  out->alloc_bytes = r->alloc;
  return RING_OK;
}

ring_status_t ring_export(ring_t r, ring_handle_t* out) {
  if (!r || !out) return RING_EINVAL;
  HandleBlob b{};
  b.magic = kMagicRing;
  b.device = r->device;
  b.pid = (int32_t)getpid();
  b.token = g_token;
  b.ptr = reinterpret_cast<uint64_t>(r->base);
  b.R = r->R;
  b.N = r->N;
  b.max_producers = r->max_producers;
  b.flags = r->flags;
  DevGuard g(r->device);
  CUDA_TRY(cudaIpcGetMemHandle(&b.ipc, r->base));
  if (r->data_device >= 0) {
    b.data_ptr = reinterpret_cast<uint64_t>(r->data);
    b.data_device = r->data_device;
    DevGuard gd(r->data_device);
    CUDA_TRY(cudaIpcGetMemHandle(&b.data_ipc, r->data));
  }
  memset(out, 0, sizeof *out);
  memcpy(out->bytes, &b, sizeof b);
  return RING_OK;
}

ring_status_t ring_attach_peer(const ring_handle_t* h, int producer_device, uint32_t producer_id, ring_peer_t* out,
                               ring_handle_t* mirror_out) {
  if (!h || !out) return RING_EINVAL;
  HandleBlob b;
  memcpy(&b, h->bytes, sizeof b);
  if (b.magic != kMagicRing || producer_id >= b.max_producers) return RING_EINVAL;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (producer_device < 0 || producer_device >= ndev) return RING_EINVAL;
  const bool same_process = b.pid == (int32_t)getpid() && b.token == g_token;
  if ((b.flags & RING_CREATE_LOCAL) && producer_device != b.device) return RING_EINVAL;
  ring_peer_s* p = new ring_peer_s;
  p->device = producer_device;
  p->ring_device = b.device;
  p->data_device = b.data_ptr ? b.data_device : b.device;
  if (same_process) {
    ring_status_t s = enable_peer(producer_device, b.device);
    if (s != RING_OK) { delete p; return s; }
    p->ring = reinterpret_cast<uint8_t*>(b.ptr);
  } else {
    DevGuard g(producer_device);
    void* m = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&m, b.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      snprintf(g_cuda_err, sizeof g_cuda_err, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
      cudaGetLastError();
      delete p;
      return RING_EPEER;
    }
    p->ring = static_cast<uint8_t*>(m);
    p->ipc_opened = true;
  }
  DevGuard g(producer_device);
  CUDA_TRY(cudaMalloc(&p->st, sizeof(DestState)));
  CUDA_TRY(cudaMemset(p->st, 0, sizeof(DestState)));
  // The channel starts where the ring is now (a ring may outlive producers).
  uint64_t tail = 0;
  CUDA_TRY(cudaMemcpy(&tail, p->ring + kTailOff, 8, cudaMemcpyDefault));
  CUDA_TRY(cudaMemcpy(&p->st->tail_cache, &tail, 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMalloc(&p->ctx, sizeof(LaunchCtx)));
  CUDA_TRY(cudaMemset(p->ctx, 0, sizeof(LaunchCtx)));
  p->desc.ring = p->ring;
  p->desc.data = p->ring + data_offset(b.N);
  if (b.data_ptr) {   // split placement: the buffer region is its own allocation (usually on this GPU)
    if (same_process) {
      ring_status_t s2 = enable_peer(producer_device, b.data_device);
      if (s2 != RING_OK) return s2;
      p->desc.data = reinterpret_cast<uint8_t*>(b.data_ptr);
    } else {
      DevGuard gd(producer_device);
      void* m = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&m, b.data_ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        snprintf(g_cuda_err, sizeof g_cuda_err, "cudaIpcOpenMemHandle(data): %s", cudaGetErrorString(e));
        cudaGetLastError();
        return RING_EPEER;
      }
      p->data_opened = static_cast<uint8_t*>(m);
      p->desc.data = p->data_opened;
    }
    p->desc.hdrs = p->ring + hdr_mirror_offset(b.N);
  }
  p->desc.st = p->st;
  p->desc.R = b.R;
  p->desc.N = b.N;
  p->desc.ft = (b.flags & RING_CREATE_FAULT_TOLERANT) ? 1u : 0u;
  p->desc.mpsc = (b.max_producers > 1 || p->desc.ft) ? 1u : 0u;   // fault tolerance needs the lock
  p->desc.rc = ((b.flags & RING_CREATE_RESERVE_COMMIT) && p->desc.mpsc && !p->desc.ft) ? 1u : 0u;
  p->desc.producer_id = producer_id;
  p->desc.has_mirror = 0;
  // Scope follows the ring: a ring created without RING_CREATE_LOCAL is a
  // system-scope ring for every producer, including one on its own GPU (the
  // lock, tail and slot words must be accessed with one scope by all of them:
  // a .gpu atomic next to a peer's .sys atomic is not morally strong).
  p->desc.sys = (b.flags & RING_CREATE_LOCAL) ? 0u : 1u;
  CUDA_TRY(cudaMalloc(&p->desc_dev, sizeof(DestDesc)));
  CUDA_TRY(cudaMemcpy(p->desc_dev, &p->desc, sizeof(DestDesc), cudaMemcpyHostToDevice));
  ring_status_t s = crc_table_dev(producer_device, &p->crc);
  if (s != RING_OK) return s;
  if (mirror_out) {
    HandleBlob mb{};
    mb.magic = kMagicMirror;
    mb.device = producer_device;
    mb.pid = (int32_t)getpid();
    mb.token = g_token;
    mb.ptr = reinterpret_cast<uint64_t>(p->st);
    mb.producer_id = producer_id;
    CUDA_TRY(cudaIpcGetMemHandle(&mb.ipc, p->st));
    memset(mirror_out, 0, sizeof *mirror_out);
    memcpy(mirror_out->bytes, &mb, sizeof mb);
  }
  *out = p;
  return RING_OK;
}

ring_status_t ring_bind_mirror(ring_t r, uint32_t producer_id, const ring_handle_t* mh) {
  if (!r || !mh || producer_id >= r->max_producers) return RING_EINVAL;
  HandleBlob b;
  memcpy(&b, mh->bytes, sizeof b);
  if (b.magic != kMagicMirror || b.producer_id != producer_id) return RING_EINVAL;
  const bool same_process = b.pid == (int32_t)getpid() && b.token == g_token;
  uint64_t* mirror = nullptr;
  if (same_process) {
    ring_status_t s = enable_peer(r->device, b.device);
    if (s != RING_OK) return s;
    mirror = reinterpret_cast<uint64_t*>(b.ptr);   // DestState::mirror_head is at offset 0
  } else {
    DevGuard g(r->device);
    void* m = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&m, b.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      snprintf(g_cuda_err, sizeof g_cuda_err, "cudaIpcOpenMemHandle(mirror): %s", cudaGetErrorString(e));
      cudaGetLastError();
      return RING_EPEER;
    }
    r->opened.push_back(m);
    mirror = static_cast<uint64_t*>(m);
  }
  DevGuard g(r->device);
  CUDA_TRY(quiesce());
  uint64_t head = 0;
  CUDA_TRY(cudaMemcpy(&head, r->base + kHeadOff, 8, cudaMemcpyDeviceToHost));
  head |= kMirrorValid;
  CUDA_TRY(cudaMemcpy(mirror, &head, 8, cudaMemcpyDefault));
  CUDA_TRY(cudaMemcpy(r->mirrors_dev + producer_id, &mirror, sizeof mirror, cudaMemcpyHostToDevice));
  CUDA_TRY(quiesce());
  return RING_OK;
}

ring_status_t ring_detach(ring_peer_t p) {
  if (!p) return RING_EINVAL;
  DevGuard g(p->device);
  if (p->engine_on) ring_peer_engine_stop(p, nullptr);
  quiesce();
  if (p->eq) cudaFree(p->eq);
  if (p->eh) cudaFreeHost(p->eh);
  if (p->eng_exit) cudaEventDestroy(p->eng_exit);
  if (p->eng_ready) cudaEventDestroy(p->eng_ready);
  if (p->eng_stream) cudaStreamDestroy(p->eng_stream);
  if (p->ipc_opened) cudaIpcCloseMemHandle(p->ring);
  if (p->data_opened) cudaIpcCloseMemHandle(p->data_opened);
  cudaFree(p->desc_dev);
  cudaFree(p->ctx);
  cudaFree(p->st);
  if (p->stage_ctl) cudaFree(p->stage_ctl);
  delete p;
  return RING_OK;
}

// ---- producer ----------------------------------------------------------------------
ring_status_t ring_peer_config(ring_peer_t p, uint32_t copy_ctas, uint32_t threads, uint32_t copy_mode) {
  if (!p || copy_ctas > 1023 || (threads && (threads % 32 || threads > 512 || threads < 64)) || copy_mode > 1)
    return RING_EINVAL;
  // CTA 0 holds the leader and publisher warps: a one-CTA LSU grid needs a third warp to copy
  if (copy_mode == 0 && copy_ctas == 1 && threads && threads < 96) return RING_EINVAL;
  p->copy_ctas = copy_ctas;
  p->threads = threads;
  p->copy_mode = copy_mode;
  return RING_OK;
}

uint64_t ring_peer_submitted(ring_peer_t p) { return p ? p->base : 0; }

// ---- lock-free fan-in set (fanin.cu) -----------------------------------------------
struct SetRingHost {                         // layout of fanin.cu's SetRing
  uint8_t* ring;
  uint8_t* data;
  uint64_t** mirrors;
  uint64_t R;
  uint32_t N;
  uint32_t _p;
};
struct ring_set_s {
  int device = 0;
  uint32_t k = 0;
  bool sys = false;
  void* rings_dev = nullptr;
  const uint32_t* crc = nullptr;
  uint32_t rr = 0;
};

ring_status_t ring_set_create(const ring_t* rings, uint32_t n, ring_set_t* out) {
  if (!rings || !out || n == 0 || n > 32) return RING_EINVAL;
  std::vector<SetRingHost> h(n);
  for (uint32_t i = 0; i < n; ++i) {
    ring_t r = rings[i];
    if (!r || r->device != rings[0]->device) return RING_EINVAL;
    h[i] = SetRingHost{r->base, r->data, r->mirrors_dev, r->R, r->N, 0};
  }
  ring_set_s* s = new ring_set_s;
  s->device = rings[0]->device;
  s->k = n;
  for (uint32_t i = 0; i < n; ++i) s->sys = s->sys || rings[i]->sys;
  DevGuard g(s->device);
  CUDA_TRY(cudaMalloc(&s->rings_dev, sizeof(SetRingHost) * n));
  CUDA_TRY(cudaMemcpy(s->rings_dev, h.data(), sizeof(SetRingHost) * n, cudaMemcpyHostToDevice));
  ring_status_t st = crc_table_dev(s->device, &s->crc);
  if (st != RING_OK) return st;
  *out = s;
  return RING_OK;
}

ring_status_t ring_set_destroy(ring_set_t s) {
  if (!s) return RING_EINVAL;
  DevGuard g(s->device);
  quiesce();
  cudaFree(s->rings_dev);
  delete s;
  return RING_OK;
}

ring_status_t ring_set_consume(ring_set_t s, uint32_t n, ring_view_t* d_views, uint32_t* d_ring_idx, uint32_t flags,
                               void* stream) {
  if (!s || !d_views || n == 0) return RING_EINVAL;
  DevGuard g(s->device);
  CUDA_TRY(launch_set_consume(static_cast<const SetRing*>(s->rings_dev), s->k, d_views, d_ring_idx, n, s->crc, flags,
                              g_timeout_ns, s->rr, s->sys, as_stream(stream)));
  s->rr = (s->rr + 1) % s->k;
  g_launches++;
  return RING_OK;
}

ring_status_t ring_peer_device_view(ring_peer_t p, ring_dev_peer_t* out) {
  if (!p || !out || p->desc.mpsc || p->engine_on || p->desc.hdrs) return RING_EINVAL;
  DevGuard g(p->device);
  if (!p->stage_ctl) {
    CUDA_TRY(cudaMalloc(&p->stage_ctl, sizeof(stage::StageCtl)));
    CUDA_TRY(cudaMemset(p->stage_ctl, 0, sizeof(stage::StageCtl)));
    CUDA_TRY(quiesce());
  }
  memset(out, 0, sizeof *out);
  out->ring = reinterpret_cast<uint64_t>(p->desc.ring);
  out->data = reinterpret_cast<uint64_t>(p->desc.data);
  out->state = reinterpret_cast<uint64_t>(p->st);
  out->ctl = reinterpret_cast<uint64_t>(p->stage_ctl);
  out->crc_table = reinterpret_cast<uint64_t>(p->crc);
  out->R = p->desc.R;
  out->N = p->desc.N;
  out->producer_id = p->desc.producer_id;
  out->sys = p->desc.sys;
  return RING_OK;
}

ring_status_t ring_stage_scale_bf16_put(ring_peer_t p, const void* d_in, uint64_t n_elems, float scale,
                                        const ring_hdr_t* hdr, uint32_t flags, uint32_t* d_status, void* stream) {
  if (!p || !d_in || !hdr || !d_status || hdr->reserved) return RING_EINVAL;
  ring_dev_peer_t v;
  ring_status_t s = ring_peer_device_view(p, &v);
  if (s != RING_OK) return s;
  DevGuard g(p->device);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
  const uint64_t work = (n_elems + 7) / 8;
  const uint32_t ctas = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)nsm * 2, (work + 255) / 256));
  CUDA_TRY(launch_stage_scale_put(v, d_in, n_elems, scale, *hdr, flags, d_status, g_timeout_ns, ctas,
                                  as_stream(stream)));
  p->launches_stage++;
  p->base += 1;
  g_launches++;
  return RING_OK;
}

ring_status_t ring_peer_set_fault(ring_peer_t p, const ring_fault_t* f) {
  if (!p || !(p->desc.ft || p->desc.rc)) return RING_EINVAL;
  if (!f) {
    p->fault = FaultSpec{};
    return RING_OK;
  }
  if (f->die_after > RING_AT_UH || (f->pause_mask & ~0x3Eu) || (f->pause_mask && (!f->arrived || !f->go)))
    return RING_EINVAL;
  p->fault.die_after = f->die_after;
  p->fault.pause_mask = f->pause_mask;
  p->fault.msg = f->msg;
  p->fault.arrived = f->arrived;
  p->fault.go = f->go;
  return RING_OK;
}

ring_status_t ring_get_trace(ring_t r, uint64_t* host_out, uint32_t n) {
  if (!r || !host_out || !r->trace || n > 1024) return RING_EINVAL;
  DevGuard g(r->device);
  CUDA_TRY(quiesce());
  CUDA_TRY(cudaMemcpy(host_out, r->trace, 8ull * n, cudaMemcpyDeviceToHost));
  return RING_OK;
}

ring_status_t ring_peer_trace(ring_peer_t p, uint64_t* host_out, uint32_t n) {
  if (!p || !host_out) return RING_EINVAL;
  if (!p->trace) return RING_EINVAL;
  DevGuard g(p->device);
  CUDA_TRY(quiesce());
  // two halves (launch parity): the last launch first, then the one before it
  const uint32_t last = (p->launches + 1) & 1;
  const uint32_t n0 = std::min<uint32_t>(n, kTraceWords), n1 = std::min<uint32_t>(n - n0, kTraceWords);
  CUDA_TRY(cudaMemcpy(host_out, p->trace + last * kTraceWords, 8ull * n0, cudaMemcpyDeviceToHost));
  if (n1) CUDA_TRY(cudaMemcpy(host_out + n0, p->trace + (last ^ 1) * kTraceWords, 8ull * n1, cudaMemcpyDeviceToHost));
  return RING_OK;
}

// Grid of a put / copy-out launch: CTA 0 holds the control warps, every other
// warp of the grid copies.  NVLink: ~32 SMs of 16-B stores saturate one peer
// link (profiles/r01_probe*.txt: 678-695 GB/s from 32 CTAs up); HBM->HBM
// (same-GPU ring): one CTA per SM.
// `remote`: the destination ring sits on another GPU (NVLink); a system-scope
// ring on the producer's own GPU takes the HBM grid (its CTAs must also fit next
// to the consumer's: 512-thread put CTAs do not fit beside a copy-out get CTA).
static void default_grid(int device, bool remote, uint32_t* ctas, uint32_t* threads, uint32_t* chunk) {
  const bool sys = remote;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  if (!*ctas) *ctas = sys ? 33u : (uint32_t)nsm;
  // Local (HBM -> HBM): 8 warps per SM already keep ~10 MB in flight, enough
  // for HBM (Little's law at ~1.5 us loaded latency); more warps only queue,
  // every unit then completes at the very end of the launch and the consumer
  // cannot release (and the next put cannot place) anything earlier.  With 8
  // warps units complete in waves, in order, and the streaming C2 step is ~10%
  // faster (profiles/r01_threads_sweep.txt).  7 warps rather than 8: the C2
  // launch's 2,048 units of 32 KiB then take almost exactly two rounds of the
  // 1,034 copy warps instead of 1.7 rounds of 1,182, and the streaming step is
  // ~5 % faster (profiles/r01_c2_grid_sweep.txt).  NVLink (sys) needs more in
  // flight.
  if (!*threads) *threads = sys ? 512u : 224u;
  if (!*chunk) {
    // NVLink: 33 CTAs x 15 copy warps x 16 KiB keeps ~8 MB in flight -- the
    // link's bandwidth x latency with room to spare; more in flight only
    // spreads every message's units over a longer window, so messages complete
    // (and free ring space) later: 32 KiB units lose ~6 % on the 64 MiB C3
    // ring, 64-256 KiB up to 30 % (profiles/r01_nvlink_sweep.txt).
    *chunk = sys ? 16u << 10 : 32u << 10;
    // tuning knob (power of two, 4 KiB .. 1 MiB)
    if (const char* e = getenv("B200RING_CHUNK")) {
      const unsigned long v = strtoul(e, nullptr, 0);
      if (v >= 4096 && v <= (1u << 20) && !(v & (v - 1))) *chunk = (uint32_t)v;
    }
  }
}

static ring_status_t engine_launch(ring_peer_t p, void* stream);

static ring_status_t put_common(ring_peer_t p, const ring_msg_t* d_msgs, const ring_msg_t* inline_msg, uint32_t n,
                                uint32_t flags, uint32_t* d_status, void* stream) {
  if (!p || !d_status || n == 0 || (!d_msgs && !inline_msg)) return RING_EINVAL;
  if (p->engine_on) {
    // the resident engine takes the batch: one doorbell thread on `stream`
    if (!d_msgs) return RING_EINVAL;   // the engine reads descriptors from device memory
    DevGuard g(p->device);
    p->eh->lease = p->eh->lease + 1;
    if (p->eh->alive == 0u) {          // it closed itself while idle: a new session
      ring_status_t s = engine_launch(p, stream);
      if (s != RING_OK) return s;
    }
    CUDA_TRY(launch_engine_doorbell(p->eq, p->posted, d_msgs, d_status, n, flags & ~RING_ASYNC,
                                    !(flags & RING_ASYNC), g_timeout_ns, as_stream(stream)));
    p->posted++;
    p->base += n;
    g_launches++;
    return RING_OK;
  }
  if (flags & RING_ASYNC) return RING_EINVAL;
  PutArgs a{};
  if (inline_msg) a.inline_msg = *inline_msg;
  a.msgs = d_msgs;
  a.status = d_status;
  a.ctx = p->ctx;
  a.dests = p->desc_dev;
  a.dest0 = p->desc;
  a.n_dests = 1;
  a.lock_timeout_ns = g_lock_timeout_ns;
  a.hole_timeout_ns = g_hole_timeout_ns;
  a.fault = p->fault;
  a.crc_table = p->crc;
  a.timeout_ns = g_timeout_ns;
  a.n = n;
  a.flags = flags;
  uint32_t ctas = p->copy_ctas, thr = p->threads, chunk = p->chunk;
  DevGuard g(p->device);
  default_grid(p->device, p->device != p->data_device, &ctas, &thr, &chunk);
  a.copy_mode = p->copy_mode;
  // engine stages live in shared memory: the largest power of two that fits
  while (a.copy_mode == 1 && chunk > 4096 && (uint64_t)chunk * kEngineStages * kMaxEngineWarps > kEngineSmem)
    chunk >>= 1;
  a.chunk = chunk;
  a.launch = p->launches;
  if (getenv("B200RING_TRACE")) {
    if (!p->trace) {
      CUDA_TRY(cudaMalloc(&p->trace, 2 * kTraceWords * 8));
      CUDA_TRY(cudaMemset(p->trace, 0, 2 * kTraceWords * 8));
    }
    a.trace = p->trace + (p->launches & 1) * kTraceWords;
    CUDA_TRY(cudaMemsetAsync(a.trace, 0, kTraceWords * 8, as_stream(stream)));
  }
  CUDA_TRY(launch_put(a, ctas, thr, as_stream(stream)));
  p->launches++;
  p->base += n;
  g_launches++;
  return RING_OK;
}

// ---- persistent put engine -----------------------------------------------------
// Launch an engine session on the attachment's own stream, after the work
// queued on `stream` (and after the previous session's kernel); later work on
// `stream` comes after the queue reset, never after the engine.
static ring_status_t engine_launch(ring_peer_t p, void* stream) {
  DevGuard g(p->device);
  // each resource on its own: a failed first start leaves nothing half-made behind
  if (!p->eq) CUDA_TRY(cudaMalloc(&p->eq, sizeof(EngineQueue)));
  if (!p->eh) {
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&p->eh), sizeof(EngineHost), cudaHostAllocMapped));
    p->eh->lease = 0;
    p->eh->alive = 0;
  }
  if (!p->eng_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->eng_stream, cudaStreamNonBlocking));
  if (!p->eng_exit) CUDA_TRY(cudaEventCreateWithFlags(&p->eng_exit, cudaEventDisableTiming));
  if (!p->eng_ready) CUDA_TRY(cudaEventCreateWithFlags(&p->eng_ready, cudaEventDisableTiming));
  p->eh->lease = p->eh->lease + 1;
  p->eh->alive = 1u;
  CUDA_TRY(cudaEventRecord(p->eng_ready, as_stream(stream)));
  CUDA_TRY(cudaStreamWaitEvent(p->eng_stream, p->eng_ready, 0));
  CUDA_TRY(cudaMemsetAsync(p->eq, 0, sizeof(EngineQueue), p->eng_stream));
  CUDA_TRY(cudaEventRecord(p->eng_ready, p->eng_stream));
  CUDA_TRY(cudaStreamWaitEvent(as_stream(stream), p->eng_ready, 0));
  EngineHost* eh_dev = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&eh_dev), p->eh, 0));
  PutArgs a{};
  a.ctx = p->ctx;
  a.dests = p->desc_dev;
  a.dest0 = p->desc;
  a.n_dests = 1;
  a.lock_timeout_ns = g_lock_timeout_ns;
  a.hole_timeout_ns = g_hole_timeout_ns;
  a.crc_table = p->crc;
  a.timeout_ns = g_timeout_ns;
  a.engine = p->eq;
  a.engine_host = eh_dev;
  a.engine_idle_ns = std::max<uint64_t>(1000000000ull, g_timeout_ns);
  if (getenv("B200RING_TRACE")) {
    if (!p->trace) {
      CUDA_TRY(cudaMalloc(&p->trace, 2 * kTraceWords * 8));
      CUDA_TRY(cudaMemset(p->trace, 0, 2 * kTraceWords * 8));
    }
    a.trace = p->trace + (p->launches & 1) * kTraceWords;
    CUDA_TRY(cudaMemsetAsync(a.trace, 0, kTraceWords * 8, p->eng_stream));
  }
  uint32_t ctas = p->copy_ctas, thr = p->threads, chunk = p->chunk;
  if (!ctas && p->device == p->data_device) {
    // a resident grid on every SM would leave no SM for kernels with another
    // shared-memory split (they only start next to CTAs of the same split)
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
    ctas = (uint32_t)std::max(1, nsm - 8);
  }
  default_grid(p->device, p->device != p->data_device, &ctas, &thr, &chunk);
  a.chunk = chunk;
  a.launch = p->launches;
  CUDA_TRY(launch_put(a, ctas, thr, p->eng_stream));
  CUDA_TRY(cudaEventRecord(p->eng_exit, p->eng_stream));
  p->launches++;
  g_launches++;
  p->posted = 0;
  return RING_OK;
}

ring_status_t ring_peer_engine_start(ring_peer_t p, void* stream) {
  if (!p || p->engine_on || p->desc.ft || p->desc.rc || p->copy_mode != 0) return RING_EINVAL;
  ring_status_t s = engine_launch(p, stream);
  if (s != RING_OK) return s;
  p->engine_on = true;
  if (p->device >= 0 && p->device < 64) g_engines[p->device]++;
  return RING_OK;
}

ring_status_t ring_peer_engine_state(ring_peer_t p, uint64_t* out4) {
  if (!p || !out4 || !p->eq) return RING_EINVAL;
  DevGuard g(p->device);
  cudaStream_t s = nullptr;   // a private non-blocking stream: never waits for the engine or the user's streams
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint64_t v[64];
  cudaError_t e = cudaMemcpyAsync(v, p->eq, sizeof v, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  CUDA_TRY(e);
  out4[0] = v[0] & ~kEngineClosed;   // posted
  out4[1] = v[16];                   // planned_batches
  out4[2] = v[32];                   // done
  out4[3] = v[0] >> 63;              // closed
  return RING_OK;
}

ring_status_t ring_peer_engine_wait(ring_peer_t p, void* stream) {
  if (!p || !p->engine_on) return RING_EINVAL;
  DevGuard g(p->device);
  p->eh->lease = p->eh->lease + 1;
  CUDA_TRY(launch_engine_wait(p->eq, p->posted, 2 * g_timeout_ns, as_stream(stream)));
  g_launches++;
  return RING_OK;
}

ring_status_t ring_peer_engine_stop(ring_peer_t p, void* stream) {
  if (!p || !p->engine_on) return RING_EINVAL;
  DevGuard g(p->device);
  p->eh->lease = p->eh->lease + 1;
  CUDA_TRY(launch_engine_stop(p->eq, as_stream(stream)));
  CUDA_TRY(cudaStreamWaitEvent(as_stream(stream), p->eng_exit, 0));   // the engine has drained and exited
  g_launches++;
  p->engine_on = false;
  if (p->device >= 0 && p->device < 64) g_engines[p->device]--;
  return RING_OK;
}

ring_status_t ring_put_batch(ring_peer_t p, const ring_msg_t* d_msgs, uint32_t n, uint32_t flags, uint32_t* d_status,
                             void* stream) {
  return put_common(p, d_msgs, nullptr, n, flags, d_status, stream);
}

ring_status_t ring_put(ring_peer_t p, const void* d_payload, uint64_t len, const ring_hdr_t* hdr, uint32_t flags,
                       uint32_t* d_status, void* stream) {
  if (!hdr || (!d_payload && len)) return RING_EINVAL;
  ring_msg_t m{};
  m.src = reinterpret_cast<uint64_t>(d_payload);
  m.len = len;
  m.hdr = *hdr;
  return put_common(p, nullptr, &m, 1, flags, d_status, stream);
}

// ---- consumer ----------------------------------------------------------------------
ring_status_t ring_config(ring_t r, uint32_t copy_ctas, uint32_t threads) {
  // get_kernel is __launch_bounds__(512, 1); CTA 0 holds the control and
  // finisher warps, so a one-CTA grid needs a third warp to copy
  if (!r || copy_ctas > 1023 || (threads && (threads % 32 || threads > 512 || threads < 64))) return RING_EINVAL;
  if (copy_ctas == 1 && threads && threads < 96) return RING_EINVAL;
  r->copy_ctas = copy_ctas;
  r->threads = threads;
  return RING_OK;
}

static ring_status_t get_common(ring_t r, uint32_t n, ring_view_t* d_views, void* d_dst, uint64_t dst_stride,
                                uint32_t flags, uint32_t consume, void* stream) {
  if (!r || !d_views || n == 0 || (d_dst && dst_stride == 0)) return RING_EINVAL;
  GetArgs a{};
  a.ring = r->base;
  a.data = r->data;
  a.hdrs = r->hdrs;
  if (getenv("B200RING_TRACE")) {
    if (!r->trace) {
      CUDA_TRY(cudaMalloc(&r->trace, 1024 * 8));
      CUDA_TRY(cudaMemset(r->trace, 0, 1024 * 8));
    }
    a.trace = r->trace;
  }
  a.views = d_views;
  a.dst = static_cast<uint8_t*>(d_dst);
  a.mirrors = r->mirrors_dev;
  a.ctx = r->ctx;
  a.crc_table = r->crc;
  a.R = r->R;
  a.dst_stride = dst_stride;
  a.timeout_ns = g_timeout_ns;
  a.N = r->N;
  a.n = n;
  a.flags = flags;
  a.consume = consume;
  a.sys = r->sys;
  a.n_mirrors = r->max_producers;
  a.remote_data = r->remote_data;
  // B200RING_COPYOUT_ALIGN=1 / 0 forces the line-aligned copy-out loads on / off
  // (tests exercise the remote path on one GPU; A/B measurements)
  if (const char* e = getenv("B200RING_COPYOUT_ALIGN")) a.remote_data = e[0] == '1';
  DevGuard g(r->device);
  uint32_t ctas = r->copy_ctas, thr = r->threads, chunk = r->chunk;
  default_grid(r->device, false, &ctas, &thr, &chunk);
  a.chunk = chunk;
  a.launch = r->launches;
  CUDA_TRY(launch_get(a, ctas, thr, as_stream(stream)));
  r->launches++;
  g_launches++;
  return RING_OK;
}

ring_status_t ring_get(ring_t r, uint32_t n, ring_view_t* d_views, void* d_dst, uint64_t dst_stride, uint32_t flags,
                       void* stream) {
  return get_common(r, n, d_views, d_dst, dst_stride, flags, 0, stream);
}

ring_status_t ring_consume(ring_t r, uint32_t n, ring_view_t* d_views, void* d_dst, uint64_t dst_stride,
                           uint32_t flags, void* stream) {
  return get_common(r, n, d_views, d_dst, dst_stride, flags, 1, stream);
}

ring_status_t ring_release(ring_t r, uint32_t count, void* stream) {
  if (!r) return RING_EINVAL;
  ReleaseArgs a{};
  a.ring = r->base;
  a.mirrors = r->mirrors_dev;
  a.R = r->R;
  a.N = r->N;
  a.count = count;
  a.sys = r->sys;
  a.n_mirrors = r->max_producers;
  DevGuard g(r->device);
  CUDA_TRY(launch_release(a, as_stream(stream)));
  g_launches++;
  return RING_OK;
}

ring_status_t ring_read_image(ring_t r, uint64_t* lock, uint64_t* tail, uint64_t* head, uint64_t* cursor,
                              uint64_t* slots) {
  if (!r) return RING_EINVAL;
  DevGuard g(r->device);
  CUDA_TRY(quiesce());
  uint64_t w[4];
  CUDA_TRY(cudaMemcpy(&w[0], r->base + kLockOff, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&w[1], r->base + kTailOff, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&w[2], r->base + kHeadOff, 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&w[3], r->base + kCursorOff, 8, cudaMemcpyDeviceToHost));
  if (lock) *lock = w[0];
  if (tail) *tail = w[1];
  if (head) *head = w[2];
  if (cursor) *cursor = w[3];
  if (slots) CUDA_TRY(cudaMemcpy(slots, r->base + kSlotsOff, 8ull * r->N, cudaMemcpyDeviceToHost));
  return RING_OK;
}

ring_status_t ring_read_data(ring_t r, uint64_t offset, uint64_t len, void* host_dst) {
  if (!r || (len && !host_dst) || offset > r->R || len > r->R - offset) return RING_EINVAL;
  DevGuard g(r->device);
  CUDA_TRY(quiesce());
  if (len) CUDA_TRY(cudaMemcpy(host_dst, r->data + offset, len, cudaMemcpyDefault));
  return RING_OK;
}

ring_status_t ring_write_data(ring_t r, uint64_t offset, uint64_t len, const void* host_src) {
  if (!r || (len && !host_src) || offset > r->R || len > r->R - offset) return RING_EINVAL;
  DevGuard g(r->device);
  CUDA_TRY(quiesce());
  if (len) CUDA_TRY(cudaMemcpy(r->data + offset, host_src, len, cudaMemcpyDefault));
  CUDA_TRY(quiesce());
  return RING_OK;
}

// ---- router ------------------------------------------------------------------------
ring_status_t router_create(int device, uint32_t max_routes, router_t* out) {
  if (!out || max_routes == 0 || max_routes > 4096) return RING_EINVAL;
  DevGuard g(device);
  router_s* r = new router_s;
  r->device = device;
  r->max_routes = max_routes;
  r->routes.resize(max_routes);
  memset(r->routes.data(), 0, sizeof(Route) * max_routes);
  CUDA_TRY(cudaMalloc(&r->routes_dev, sizeof(Route) * max_routes));
  CUDA_TRY(cudaMemset(r->routes_dev, 0, sizeof(Route) * max_routes));
  CUDA_TRY(cudaMalloc(&r->dests_dev, sizeof(DestDesc) * kMaxRouterDests));
  CUDA_TRY(cudaMemset(r->dests_dev, 0, sizeof(DestDesc) * kMaxRouterDests));
  CUDA_TRY(cudaMalloc(&r->ctx, sizeof(LaunchCtx)));
  CUDA_TRY(cudaMemset(r->ctx, 0, sizeof(LaunchCtx)));
  ring_status_t s = crc_table_dev(device, &r->crc);
  if (s != RING_OK) return s;
  *out = r;
  return RING_OK;
}

ring_status_t router_destroy(router_t r) {
  if (!r) return RING_EINVAL;
  DevGuard g(r->device);
  quiesce();
  cudaFree(r->ctx);
  cudaFree(r->dests_dev);
  cudaFree(r->routes_dev);
  delete r;
  return RING_OK;
}

ring_status_t router_set_route(router_t r, uint32_t app_id, uint16_t stage, const ring_peer_t* dests, uint32_t n,
                               void* stream) {
  if (!r || n > kMaxDests || (n && !dests)) return RING_EINVAL;
  DevGuard g(r->device);
  Route nr{};
  nr.app_id = app_id;
  nr.stage = stage;
  nr.n = (uint16_t)n;
  std::vector<uint32_t> added;   // destinations new to this router: their descriptors go up first
  for (uint32_t i = 0; i < n; ++i) {
    ring_peer_t p = dests[i];
    // A routed put runs the batched (non-fault-tolerant) sender: it must never
    // write untagged slots or hold a plain lock on a fault-tolerant ring.
    if (!p || p->device != r->device || p->desc.ft) return RING_EINVAL;
    uint32_t idx = 0;
    while (idx < r->dests.size() && r->dests[idx] != p) ++idx;
    if (idx == r->dests.size()) {
      if (idx >= (uint32_t)kMaxRouterDests) return RING_EINVAL;
      r->dests.push_back(p);
      added.push_back(idx);
    }
    nr.dests[i] = idx;
  }
  uint32_t slot = r->max_routes;
  for (uint32_t i = 0; i < r->max_routes; ++i)
    if (r->routes[i].n && r->routes[i].app_id == app_id && r->routes[i].stage == stage) { slot = i; break; }
  if (slot == r->max_routes)
    for (uint32_t i = 0; i < r->max_routes; ++i)
      if (!r->routes[i].n) { slot = i; break; }
  if (slot == r->max_routes) return RING_EINVAL;
  nr.epoch = r->routes[slot].epoch + 1;     // epoch flip (NodeManager reassignment)
  r->routes[slot] = nr;
  // Device-side, in stream order with the caller's puts (launched puts finish
  // to the old destinations), no host synchronisation.
  Route* d = r->routes_dev + slot;
  for (size_t k = 0; k + 1 < added.size(); ++k)
    CUDA_TRY(launch_route_update(d, r->routes[slot], r->dests_dev + added[k], &r->dests[added[k]]->desc,
                                 as_stream(stream)));
  CUDA_TRY(launch_route_update(d, nr, added.empty() ? nullptr : r->dests_dev + added.back(),
                               added.empty() ? nullptr : &r->dests[added.back()]->desc, as_stream(stream)));
  g_launches += added.size() > 1 ? added.size() : 1;
  return RING_OK;
}

ring_status_t router_set_admission(router_t r, uint32_t app_id, uint16_t stage, uint64_t t_x, uint32_t k,
                                   void* stream) {
  if (!r || (k && t_x == 0)) return RING_EINVAL;
  uint32_t slot = r->max_routes;
  for (uint32_t i = 0; i < r->max_routes; ++i)
    if (r->routes[i].n && r->routes[i].app_id == app_id && r->routes[i].stage == stage) { slot = i; break; }
  if (slot == r->max_routes) return RING_EINVAL;
  DevGuard g(r->device);
  static thread_local Route staged;
  staged.adm_tx = t_x;
  staged.adm_k = k;
  staged._ra = 0;
  staged.adm_next = 0;
  Route* d = r->routes_dev + slot;
  const size_t off = offsetof(Route, adm_tx);
  CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(d) + off, reinterpret_cast<uint8_t*>(&staged) + off,
                           sizeof(Route) - off, cudaMemcpyHostToDevice, as_stream(stream)));
  CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  return RING_OK;
}

uint64_t ring_required_instances(uint64_t t_x, uint64_t t_y, uint32_t k) {
  if (t_x == 0 || t_y == 0 || k == 0) return 0;
  const unsigned __int128 num = (unsigned __int128)k * t_y;
  return (uint64_t)((num + t_x - 1) / t_x);
}

ring_status_t router_size_route(router_t r, uint32_t app_id, uint16_t stage, uint64_t t_x, uint64_t t_y, uint32_t k,
                                const ring_peer_t* pool, uint32_t n_pool, uint32_t* m_out, void* stream) {
  const uint64_t m = ring_required_instances(t_x, t_y, k);
  if (!r || !pool || m == 0 || m > n_pool || m > kMaxDests) return RING_EINVAL;
  ring_status_t s = router_set_route(r, app_id, stage, pool, (uint32_t)m, stream);
  if (s != RING_OK) return s;
  s = router_set_admission(r, app_id, stage, t_x, k, stream);
  if (s == RING_OK && m_out) *m_out = (uint32_t)m;
  return s;
}

ring_status_t ring_put_routed(router_t r, const ring_msg_t* d_msgs, uint32_t n, uint32_t flags, uint32_t* d_status,
                              uint32_t* d_dest, void* stream) {
  if (!r || !d_msgs || !d_status || n == 0 || (flags & RING_ASYNC)) return RING_EINVAL;
  if (r->dests.empty()) return RING_EINVAL;
  for (auto* p : r->dests)
    if (p->engine_on) return RING_EINVAL;   // the attachment's state belongs to its engine
  PutArgs a{};
  a.msgs = d_msgs;
  a.status = d_status;
  a.dest_out = d_dest;
  a.ctx = r->ctx;
  a.dests = r->dests_dev;
  a.dest0 = r->dests[0]->desc;
  a.n_dests = (uint32_t)r->dests.size();
  a.lock_timeout_ns = g_lock_timeout_ns;
  a.hole_timeout_ns = g_hole_timeout_ns;
  a.routes = r->routes_dev;
  a.n_routes = r->max_routes;
  a.crc_table = r->crc;
  a.timeout_ns = g_timeout_ns;
  a.n = n;
  a.flags = flags;
  bool remote = false;
  for (auto* p : r->dests) remote = remote || p->data_device != r->device;
  uint32_t ctas = r->copy_ctas, thr = r->threads, chunk = r->chunk;
  DevGuard g(r->device);
  default_grid(r->device, remote, &ctas, &thr, &chunk);
  a.chunk = chunk;
  a.launch = r->launches;
  CUDA_TRY(launch_put(a, ctas, thr, as_stream(stream)));
  r->launches++;
  r->base += n;
  g_launches++;
  return RING_OK;
}

}  // extern "C"
