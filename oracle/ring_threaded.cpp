// ring_threaded.cpp — the paper's double-ring buffer run by host threads over
// host memory: the CPU baseline the GPU path is reported next to (BASELINE.md
// §6).  TEST / BENCH INFRASTRUCTURE ONLY: only tests/,
// bench.py's cpu_baseline leg and __graft_entry__ may build or run it; it
// shares no code with the product library (paper_2601_20655_b200/).
//
// Same protocol as oracle/ring.py (PAPER.md:693-747 with the readings of
// DESIGN.md §2), written plainly: one std::thread per producer plus one
// consumer, pinned to cores with sched_setaffinity; control words are
// std::atomic with acquire / release; payloads move with memcpy.
//   sender, per message:
//     1 Lock (MPSC only: CAS 0 -> pid+1, acquire; R14 elides it for SPSC)
//     2 read the tail (acquire)
//     3 space check (R4: the bytes [P_b, P_b+f) must not meet the live range;
//       R5: at most N entries), PAD entry over [P_b, R) when the entry would
//       straddle R (R3); insufficient space -> release the lock, wait for the
//       head to move, start over (R12, blocking mode)
//     5 WB: 64-B header (R11, CRC-32 of bytes [4,56), R10) + payload memcpy
//     6 WL: size slot = busy | f (release)
//     7 UH: tail = advance(P) (release)
//     8 Unlock (release)
//   receiver: poll the tail (acquire); per entry read the
//     size slot (PAD: step over), header (CRC check), payload (memcpy out);
//     then clear the busy bit and move the head (release).
// Word formats (R8/R9): pointer = (offset << 24) | (seq mod 2^24); slot =
// busy << 63 | pad << 62 | footprint.
//
// Payload bytes: synth.payload_bytes (splitmix64 keyed by (seed, channel,
// seq)), generated here by the producers and re-derived by the consumer,
// which checks every byte it copies out (exactly-once, in order per channel).
//
// Usage: ring_threaded R N producers msgs_per_producer len_lo len_hi seed
//        [mode] [core0]
//   mode "place": SPSC only, prints "start f seq" per delivered message (for
//   the pin against oracle/ring.py); otherwise one JSON line of results.
#include <sched.h>
#include <pthread.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kBusy = 1ull << 63, kPad = 1ull << 62, kMask24 = (1u << 24) - 1;
constexpr uint64_t kHdr = 64, kAlign = 128;

uint64_t pack(uint64_t b, uint64_t q) { return (b << 24) | (q & kMask24); }
uint64_t off(uint64_t w) { return w >> 24; }
uint64_t seq(uint64_t w) { return w & kMask24; }
uint64_t footprint(uint64_t len) { return (kHdr + len + kAlign - 1) / kAlign * kAlign; }

// ---- CRC-32/IEEE (reflected 0xEDB88320), bitwise table ----
uint32_t g_crc[256];
void crc_init() {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
    g_crc[i] = c;
  }
}
uint32_t crc32(const uint8_t* p, size_t n) {
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = g_crc[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return ~c;
}

// ---- synth.payload_bytes ----
uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void payload(uint64_t seed, uint32_t ch, uint64_t q, uint8_t* out, uint64_t len) {
  const uint64_t key = sm64(sm64(sm64(seed) ^ ch) ^ (q & 0xFFFFFFFFFFFFull));
  uint64_t i = 0;
  for (; i + 8 <= len; i += 8) {
    const uint64_t w = sm64(key + i / 8);
    memcpy(out + i, &w, 8);
  }
  if (i < len) {
    const uint64_t w = sm64(key + i / 8);
    memcpy(out + i, &w, len - i);
  }
}

// message lengths of channel `ch`: U[lo, hi] from splitmix64 (independent of numpy)
uint64_t msg_len(uint64_t seed, uint32_t ch, uint64_t k, uint64_t lo, uint64_t hi) {
  if (lo == hi) return lo;
  return lo + sm64(sm64(seed ^ 0x5151) ^ ((uint64_t)ch << 32) ^ k) % (hi - lo + 1);
}

uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void pin(int core) {
  const int n = (int)std::thread::hardware_concurrency();
  if (n <= 0) return;
  cpu_set_t s;
  CPU_ZERO(&s);
  CPU_SET(core % n, &s);
  sched_setaffinity(0, sizeof s, &s);
}

// ---- the ring in host memory ----
struct Ring {
  uint64_t R;
  uint32_t N;
  bool mpsc;
  alignas(64) std::atomic<uint64_t> lock{0};
  alignas(64) std::atomic<uint64_t> tail{0};
  alignas(64) std::atomic<uint64_t> head{0};
  std::vector<std::atomic<uint64_t>> slots;
  std::vector<uint8_t> data;
  Ring(uint64_t r, uint32_t n, bool m) : R(r), N(n), mpsc(m), slots(n), data(r) {
    for (auto& s : slots) s.store(0);
  }
  uint64_t advance(uint64_t b, uint64_t f) const { return b + f < R ? b + f : 0; }
  bool interval_free(uint64_t pb, uint64_t pq, uint64_t hb, uint64_t hq, uint64_t f) const {   // R4
    if (pq == hq) return true;
    if (pb > hb) return true;
    if (pb < hb) return pb + f <= hb;
    return false;
  }
};

struct Args {
  uint64_t R, lo, hi, seed;
  uint32_t N, producers, per;
  bool place;
  int core0;
};

// Sender steps 1-8 for every message of channel `pid`.
void producer(Ring& ring, const Args& A, uint32_t pid, std::vector<uint8_t>& buf) {
  pin(A.core0 + 1 + (int)pid);
  uint64_t local_tail = 0;   // SPSC: the producer owns the tail (R14)
  for (uint64_t k = 0; k < A.per; ++k) {
    const uint64_t len = msg_len(A.seed, pid, k, A.lo, A.hi);
    if (buf.size() < len) buf.resize(len);
    payload(A.seed, pid, k, buf.data(), len);
    const uint64_t f = footprint(len);
    const uint64_t t_put = now_ns();
    bool locked = false;
    uint64_t P = 0, pb = 0, pq = 0;
    while (true) {
      if (ring.mpsc && !locked) {                                         // 1 Lock
        uint64_t z = 0;
        while (!ring.lock.compare_exchange_weak(z, pid + 1, std::memory_order_acquire)) z = 0;
        locked = true;
      }
      P = ring.mpsc ? ring.tail.load(std::memory_order_acquire) : local_tail;   // 2 read the tail
      const uint64_t H = ring.head.load(std::memory_order_acquire);
      pb = off(P);
      pq = seq(P);
      const uint64_t hb = off(H), hq = seq(H);
      bool ok = ((pq - hq) & kMask24) < ring.N;                           // 3 (R5: a free slot)
      if (ok && pb + f > ring.R) {                                        // R3: PAD over [P_b, R) first
        if (ring.interval_free(pb, pq, hb, hq, ring.R - pb)) {
          ring.slots[pq % ring.N].store(kBusy | kPad | (ring.R - pb), std::memory_order_release);
          local_tail = pack(0, pq + 1);
          ring.tail.store(local_tail, std::memory_order_release);
          continue;                                                       // the message, from P = (0, q+1)
        }
        ok = false;
      }
      if (ok) ok = ring.interval_free(pb, pq, hb, hq, f);
      if (!ok) {                                                          // R12: unlock, wait, start over
        if (ring.mpsc) {
          ring.lock.store(0, std::memory_order_release);
          locked = false;
        }
        while (ring.head.load(std::memory_order_acquire) == H) std::this_thread::yield();
        continue;
      }
      break;
    }
    {
      uint8_t* e = ring.data.data() + pb;                                 // 5 WB
      uint8_t h[64] = {};
      const uint32_t app = 7, len32 = (uint32_t)len, ch = pid, q = (uint32_t)k;
      const uint16_t stage = 1;
      memcpy(h + 28, &app, 4);
      memcpy(h + 32, &stage, 2);
      memcpy(h + 34, &len32, 4);
      memcpy(h + 44, &ch, 4);
      memcpy(h + 48, &q, 4);
      const uint32_t c = crc32(h + 4, 52);
      memcpy(h, &c, 4);
      memcpy(h + 56, &t_put, 8);
      memcpy(e, h, 64);
      memcpy(e + kHdr, buf.data(), len);
      ring.slots[pq % ring.N].store(kBusy | f, std::memory_order_release);   // 6 WL
      P = pack(ring.advance(pb, f), pq + 1);
      ring.tail.store(P, std::memory_order_release);                      // 7 UH
      local_tail = P;
      if (ring.mpsc) ring.lock.store(0, std::memory_order_release);       // 8 Unlock
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 8) {
    fprintf(stderr, "usage: %s R N producers msgs_per_producer len_lo len_hi seed [place|run] [core0]\n", argv[0]);
    return 2;
  }
  crc_init();
  Args A{};
  A.R = strtoull(argv[1], nullptr, 0);
  A.N = (uint32_t)strtoul(argv[2], nullptr, 0);
  A.producers = (uint32_t)strtoul(argv[3], nullptr, 0);
  A.per = (uint32_t)strtoul(argv[4], nullptr, 0);
  A.lo = strtoull(argv[5], nullptr, 0);
  A.hi = strtoull(argv[6], nullptr, 0);
  A.seed = strtoull(argv[7], nullptr, 0);
  A.place = argc > 8 && std::string(argv[8]) == "place";
  A.core0 = argc > 9 ? atoi(argv[9]) : 0;
  if (A.R % kAlign || footprint(A.hi) > A.R || !A.N || !A.producers) return 2;
  Ring ring(A.R, A.N, A.producers > 1);
  const uint64_t total = (uint64_t)A.producers * A.per;
  std::vector<uint64_t> next(A.producers, 0), lat;
  lat.reserve(total);
  std::vector<std::vector<uint8_t>> bufs(A.producers);
  std::vector<uint8_t> out, expect;
  uint64_t bytes = 0, bad = 0;
  std::vector<std::thread> th;
  const uint64_t t0 = now_ns();
  for (uint32_t p = 0; p < A.producers; ++p) th.emplace_back(producer, std::ref(ring), std::cref(A), p, std::ref(bufs[p]));
  // receiver on this thread
  pin(A.core0);
  uint64_t G = 0, got = 0;
  while (got < total) {
    const uint64_t T = ring.tail.load(std::memory_order_acquire);            // 1-2 poll
    while (seq(G) != seq(T) && got < total) {
      const uint64_t w = ring.slots[seq(G) % ring.N].load(std::memory_order_acquire);
      const uint64_t f = w & ((1ull << 62) - 1);
      if (!(w & kPad)) {                                                       // 3 header + payload
        const uint8_t* e = ring.data.data() + off(G);
        uint32_t c, len32, ch, q;
        uint64_t t_put;
        memcpy(&c, e, 4);
        memcpy(&len32, e + 34, 4);
        memcpy(&ch, e + 44, 4);
        memcpy(&q, e + 48, 4);
        memcpy(&t_put, e + 56, 8);
        const uint64_t t_vis = now_ns();
        if (c != crc32(e + 4, 52) || ch >= A.producers || q != next[ch]) ++bad;
        if (out.size() < len32) { out.resize(len32); expect.resize(len32); }
        memcpy(out.data(), e + kHdr, len32);
        payload(A.seed, ch, q, expect.data(), len32);
        if (memcmp(out.data(), expect.data(), len32)) ++bad;
        if (ch < A.producers) next[ch] = q + 1;
        bytes += len32;
        lat.push_back(t_vis - t_put);
        ++got;
        if (A.place) printf("%llu %llu %llu\n", (unsigned long long)off(G), (unsigned long long)f,
                            (unsigned long long)seq(G));
      }
      ring.slots[seq(G) % ring.N].store(0, std::memory_order_relaxed);         // 4 clear busy
      G = pack(ring.advance(off(G), f), seq(G) + 1);
      ring.head.store(G, std::memory_order_release);                          // 5 move the head
    }
  }
  for (auto& t : th) t.join();
  const double dt = (double)(now_ns() - t0) / 1e9;
  if (A.place) return bad ? 1 : 0;
  std::sort(lat.begin(), lat.end());
  auto pct = [&](double q) { return lat.empty() ? 0.0 : (double)lat[(size_t)(q * (lat.size() - 1))] / 1e3; };
  std::string model = "unknown";
  std::ifstream ci("/proc/cpuinfo");
  for (std::string line; std::getline(ci, line);)
    if (line.rfind("model name", 0) == 0) { model = line.substr(line.find(':') + 2); break; }
  printf("{\"gbs\": %.4f, \"msgs_per_s\": %.1f, \"p50_us\": %.2f, \"p99_us\": %.2f, \"messages\": %llu, "
         "\"bytes\": %llu, \"seconds\": %.4f, \"threads\": %u, \"bad\": %llu, \"cpu_model\": \"%s\", "
         "\"host_cpus\": %u}\n",
         bytes / dt / 1e9, got / dt, pct(0.5), pct(0.99), (unsigned long long)got, (unsigned long long)bytes, dt,
         A.producers + 1, (unsigned long long)bad, model.c_str(), std::thread::hardware_concurrency());
  return bad ? 1 : 0;
}
