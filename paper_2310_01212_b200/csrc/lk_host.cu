// lk_host.cu -- host side of the LK runtime behind the C ABI in include/lk.h.
//
// Owns the CUDA context use, the pinned mapped mailboxes, the device
// descriptor table and the persistent kernel's stream.  All spinning happens
// here, outside Python (ctypes releases the GIL for every call).
//
// Host rules follow persistkern.native.NativeSession
// (/root/reference/pkg/src/persistkern/native.py:82-299): trigger validates
// mask / busy / slot lock / idle (208-231), writes 16+slot ascending; wait spins
// to FINISHED, acks with NOP ascending and spins to NOP (250-275); dispose
// refuses while pending, writes EXIT, joins (277-295).
#include <cuda.h>            // driver types only: entry points come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <errno.h>
#include <pthread.h>
#include <sched.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#define LK_PAUSE() _mm_pause()
#else
#define LK_PAUSE() asm volatile("" ::: "memory")
#endif

#include "lk_internal.h"
#include "lk_protocol.cuh"

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define LK_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(LK_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                               \
  } while (0)

static inline uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return uint64_t(ts.tv_sec) * 1000000000ull + uint64_t(ts.tv_nsec);
}

// ------------------------------------------------------------------ driver entry points
// Green contexts (SM partitions) are driver-API only.  liblk.so does not link
// libcuda: the functions are fetched through the runtime, so the library still
// loads (and its CPU tests run) on machines without a driver.
struct Drv {
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetDevResource) DeviceGetDevResource = nullptr;
  decltype(&cuDevSmResourceSplitByCount) DevSmResourceSplitByCount = nullptr;
  decltype(&cuDevResourceGenerateDesc) DevResourceGenerateDesc = nullptr;
  decltype(&cuGreenCtxCreate) GreenCtxCreate = nullptr;
  decltype(&cuGreenCtxDestroy) GreenCtxDestroy = nullptr;
  decltype(&cuCtxFromGreenCtx) CtxFromGreenCtx = nullptr;
  decltype(&cuCtxPushCurrent) CtxPushCurrent = nullptr;
  decltype(&cuCtxPopCurrent) CtxPopCurrent = nullptr;
  bool ok = false;
};

static Drv* drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    auto get = [&](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !*fn)
        ok = false;
    };
    get("cuDeviceGet", reinterpret_cast<void**>(&d.DeviceGet));
    get("cuDeviceGetDevResource", reinterpret_cast<void**>(&d.DeviceGetDevResource));
    get("cuDevSmResourceSplitByCount", reinterpret_cast<void**>(&d.DevSmResourceSplitByCount));
    get("cuDevResourceGenerateDesc", reinterpret_cast<void**>(&d.DevResourceGenerateDesc));
    get("cuGreenCtxCreate", reinterpret_cast<void**>(&d.GreenCtxCreate));
    get("cuGreenCtxDestroy", reinterpret_cast<void**>(&d.GreenCtxDestroy));
    get("cuCtxFromGreenCtx", reinterpret_cast<void**>(&d.CtxFromGreenCtx));
    get("cuCtxPushCurrent", reinterpret_cast<void**>(&d.CtxPushCurrent));
    get("cuCtxPopCurrent", reinterpret_cast<void**>(&d.CtxPopCurrent));
    d.ok = ok;
  });
  return &d;
}

// Makes a (green) context current for a scope; no-op for nullptr.
struct CtxScope {
  CUcontext c;
  explicit CtxScope(CUcontext ctx) : c(ctx) {
    if (c) drv()->CtxPushCurrent(c);
  }
  ~CtxScope() {
    if (c) {
      CUcontext prev;
      drv()->CtxPopCurrent(&prev);
    }
  }
};

// An SM partition: green context A (>= `sms` SMs, rounded up by the driver to
// its granularity, 8 on sm_90+) for the persistent kernel, and green context B
// holding every remaining SM for ordinary kernels that run beside it.
struct Partition {
  CUgreenCtx ga = nullptr, gb = nullptr;
  CUcontext ca = nullptr, cb = nullptr;
  uint32_t a_sms = 0, b_sms = 0;
};

static void free_partition(Partition* p);

static int make_partition(int device, uint32_t sms, Partition* p) {
  Drv* d = drv();
  if (!d->ok) return fail(LK_E_INIT, "green-context driver entry points unavailable");
  CUdevice dev;
  CUresult r = d->DeviceGet(&dev, device);
  CUdevResource all, part, rest;
  unsigned groups = 1;
  if (r == CUDA_SUCCESS) r = d->DeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  if (r == CUDA_SUCCESS) r = d->DevSmResourceSplitByCount(&part, &groups, &all, &rest, 0, sms);
  if (r != CUDA_SUCCESS || groups != 1)
    return fail(LK_E_CONFIG, "cannot split %u SMs off device %d (driver error %d)", sms, device, int(r));
  CUdevResourceDesc da, db;
  r = d->DevResourceGenerateDesc(&da, &part, 1);
  if (r == CUDA_SUCCESS) r = d->GreenCtxCreate(&p->ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM);
  if (r == CUDA_SUCCESS) r = d->CtxFromGreenCtx(&p->ca, p->ga);
  if (r == CUDA_SUCCESS && rest.sm.smCount) {
    r = d->DevResourceGenerateDesc(&db, &rest, 1);
    if (r == CUDA_SUCCESS) r = d->GreenCtxCreate(&p->gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r == CUDA_SUCCESS) r = d->CtxFromGreenCtx(&p->cb, p->gb);
  }
  if (r != CUDA_SUCCESS) {
    free_partition(p);
    return fail(LK_E_INIT, "green context creation failed (driver error %d)", int(r));
  }
  p->a_sms = part.sm.smCount;
  p->b_sms = rest.sm.smCount;
  return LK_OK;
}

static void free_partition(Partition* p) {
  if (p->ga) drv()->GreenCtxDestroy(p->ga);
  if (p->gb) drv()->GreenCtxDestroy(p->gb);
  *p = Partition{};
}

// ------------------------------------------------------------------ service stream
// Allocation, frees and staging copies never touch the legacy stream and never
// synchronize the device: a resident persistent kernel never "completes", so a
// device-wide sync (cudaDeviceSynchronize, cudaFree, cudaMemset) would block
// forever.  Stream-ordered allocation on a private non-blocking stream does not.
static std::mutex g_svc_mu;
static constexpr int kMaxDevices = 64;
static cudaStream_t g_svc[kMaxDevices];

static cudaStream_t svc_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return nullptr;   // create() refuses such devices first
  std::lock_guard<std::mutex> g(g_svc_mu);
  if (!g_svc[dev]) {
    cudaStreamCreateWithFlags(&g_svc[dev], cudaStreamNonBlocking);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;  // keep freed memory mapped: no unmap on sync
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  return g_svc[dev];
}

static cudaError_t dev_alloc(void** p, size_t bytes) {
  cudaStream_t st = svc_stream();
  cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 1, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

static cudaError_t dev_free(void* p) {
  if (!p) return cudaSuccess;
  cudaStream_t st = svc_stream();
  cudaError_t e = cudaFreeAsync(p, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

// ------------------------------------------------------------------ session
struct HostRec {
  uint32_t hseq;
  uint32_t word;
  uint64_t t_ns;
};

struct lk_session {
  lk_config cfg;
  uint32_t nw = 0, nwords = 0, threads = 0;
  int device = 0;
  size_t smem = 0;
  cudaStream_t stream = nullptr;   // persistent kernel (in part.ca when partitioned)
  Partition part;                  // sm_partition > 0: green contexts A (LK) and B (the rest)
  cudaStream_t copy_stream = nullptr;

  // pinned mapped host block
  uint8_t* host_block = nullptr;
  unsigned long long* to_gpu = nullptr;       // DIRECT: worker i replica k at [(i*replicas+k)*cell_u64]
  unsigned long long* ring = nullptr;         // GATEWAY: event ring replicas (8 u64 per entry)
  volatile unsigned long long* gw_tail = nullptr;   // GATEWAY: events consumed (device-written)
  uint32_t ring_entries = 256;
  uint32_t ev_head = 0;                       // GATEWAY: events appended
  uint32_t tail_seen = 0;                     // GATEWAY: the consumed count as last read
  std::vector<uint32_t> last_word;            // GATEWAY: shadow of each worker's to_gpu value
  std::mutex post_mu;
  std::vector<uint32_t> all_ids;
  bool gateway = false;                       // event ring in use (GATEWAY or HYBRID)
  bool hybrid = false;
  uint32_t dreps = 1;                         // replicas of each direct cell (HYBRID: 1)
  std::vector<uint32_t> host_dseq;            // writes that went to each worker's direct cell
  volatile unsigned long long* status = nullptr;  // stride status_u64
  volatile unsigned long long* err = nullptr;
  volatile uint32_t* err_any = nullptr;
  volatile uint32_t* smid = nullptr;
  uint32_t cell_u64 = 16, status_u64 = 16, replicas = 4;

  // device block
  uint8_t* dev_block = nullptr;
  lk_desc* d_desc = nullptr;
  unsigned long long* d_mask = nullptr;
  uint32_t* d_ctr = nullptr;
  unsigned long long* d_spans = nullptr;
  unsigned long long* d_dmb = nullptr;
  uint32_t* d_exited = nullptr;
  lk_dev_trace* d_trace = nullptr;
  uint32_t* d_tcnt = nullptr;
  uint32_t* d_fast = nullptr;      // per-worker fast-path counts (lk_fast_count)
  bool host_desc = false;          // LK_CF_HOST_DESC: d_desc / d_mask point into host_block

  // host bookkeeping (guarded by mu)
  std::mutex mu;
  std::vector<uint64_t> pending;                          // nwords
  // pending_by_slot (native.py:97): per-slot worker masks of un-waited
  // dispatches, flat (num_slots * nwords), plus the list of slots in flight.
  std::vector<uint64_t> slot_pend;
  std::vector<uint8_t> slot_busy;
  std::vector<uint32_t> inflight;
  std::vector<uint64_t> scratch;                          // nwords, under mu
  // LK_CF_LAZY_ACK: workers whose NOP ack was written but whose republished
  // NOP has not been seen yet; the next trigger/dispose touching them waits
  std::vector<uint64_t> ack_pending;                      // nwords, under mu
  // Workers whose NOP the host has observed since its last write to them: a
  // worker only changes its cell in answer to a host write (a failing one
  // raises err_any, which every call checks first), so trigger's idle check
  // need not re-read their cells (native.py:219-220).  Under mu.
  std::vector<uint64_t> idle_known;
  std::vector<uint8_t> registered;                        // per slot
  std::vector<lk_desc> reg_desc;                          // host copy per slot (as staged)
  std::vector<lk_desc> reg_in;                            // ... and as the caller passed it
  std::vector<uint64_t> stage_mask;                       // scratch for stage_locked
  // descriptor caching (LK_HINT_CACHED): a slot's stage version goes up with
  // every upload; each worker's last fetched (slot, version)
  std::vector<uint32_t> slot_ver;                         // per slot
  std::vector<uint32_t> wslot, wver;                      // per worker
  std::vector<std::vector<uint64_t>> reg_mask;            // per slot (nwords)
  bool disposed = false;
  bool kernel_done = false;
  // The cooperative launch is issued from this thread.  Normally it returns
  // at once; under a profiler that serialises launches (ncu) it returns only
  // when the kernel exits, so the session's API keeps running meanwhile.
  // launch_state: 0 launch call not returned yet, 1 launched, -1 failed.
  std::thread launcher;
  std::atomic<int> launch_state{0};
  cudaError_t launch_err = cudaSuccess;
  void join_launcher() {
    if (launcher.joinable()) launcher.join();
  }
  bool claimed = true;             // holds the device's one-session claim until the kernel retired
  void release_claim();
  uint64_t t_create = 0;

  // host half of the last dispatch per worker (lk_last_host_times)
  std::vector<uint64_t> host_times;                       // 3 per worker

  // tracing
  std::vector<uint32_t> host_seq;                         // per worker
  std::vector<std::vector<HostRec>> host_log;             // per worker

  // scratch
  std::vector<uint32_t> ids;

  inline uint32_t word(uint32_t i) const { return uint32_t(status[uint64_t(i) * status_u64]); }
  inline uint32_t phase(uint32_t i) const { return uint32_t(status[uint64_t(i) * status_u64] >> 32); }
  // One logical to_gpu write: {word, seq} into every replica (seq = this
  // worker's host write index; the device acts only on newer seqs, so the
  // replicas, written one after another, can never step it backwards).
  // DIRECT: one worker's cell value {word:32, seq:24, hint:8} (lk_kernels.cu:
  // accept).  seq counts the writes made through this cell (all of them in
  // DIRECT mode; in HYBRID the rest travel as ring events).
  inline void host_write(uint32_t i, uint32_t w, uint32_t hint = 0) {
    const uint32_t sq = ++host_seq[i];
    const uint32_t dq = ++host_dseq[i];
    last_word[i] = w;
    if (cfg.record_trace) host_log[i].push_back(HostRec{sq, w, now_ns()});
    const unsigned long long v = uint64_t(w) | (uint64_t(dq & 0xFFFFFFu) << 32) | (uint64_t(hint & 0xFFu) << 56);
    unsigned long long* c = to_gpu + uint64_t(i) * dreps * cell_u64;
    for (uint32_t k = 0; k < dreps; ++k) __atomic_store_n(c + k * cell_u64, v, __ATOMIC_RELEASE);
  }
  // LK_CF_FULL_BOARD (DIRECT): the paper's workaround for the driver that
  // deferred single-word mailbox transfers indefinitely (
  // P/link.py:104-122, workaround_full_board): every write ships the whole
  // board.  Ascending over all workers, the targets get their new value and
  // every other cell is stored again unchanged (same seq: the worker ignores
  // it), so the link carries the full mailbox each time.
  void full_board_write(const std::vector<uint32_t>& ids, uint32_t w, uint32_t hint) {
    size_t j = 0;
    for (uint32_t i = 0; i < nw; ++i) {
      if (j < ids.size() && ids[j] == i) {
        host_write(i, w, hint);
        ++j;
        continue;
      }
      unsigned long long* c = to_gpu + uint64_t(i) * dreps * cell_u64;
      const unsigned long long v = __atomic_load_n(c, __ATOMIC_RELAXED);
      for (uint32_t k = 0; k < dreps; ++k) __atomic_store_n(c + k * cell_u64, v, __ATOMIC_RELEASE);
    }
  }
  // One logical write of `w` to every worker in ids (ascending), i.e. the
  // reference's `for i in sm_ids: _host_write(i, word)` (native.py:224-225).
  // GATEWAY: a single ring event carries the word and the worker mask.
  // Returns false if the ring stayed full past the timeout.
  bool post(const std::vector<uint32_t>& ids, uint32_t w, uint32_t hint = 0) {
    if (!gateway || (hybrid && ids.size() <= LK_HYBRID_DIRECT_MAX)) {
      if (cfg.flags & LK_CF_FULL_BOARD) {
        full_board_write(ids, w, hint);
        return true;
      }
      for (uint32_t i : ids) host_write(i, w, hint);
      return true;
    }
    std::lock_guard<std::mutex> g(post_mu);   // trigger and wait may run on different host threads
    // flow control: the consumed count is re-read (a cache miss: the device
    // writes that line) only when the count seen last says the ring is full
    if (ev_head - tail_seen >= ring_entries - 1) {
      const uint64_t deadline = now_ns() + cfg.wait_timeout_ns;
      while (ev_head - (tail_seen = uint32_t(*gw_tail)) >= ring_entries - 1) {
        LK_PAUSE();
        if (now_ns() > deadline) return false;
      }
    }
    const uint32_t seq = ++ev_head;
    const uint64_t tag = uint64_t(seq & 0xFFFFu) << 48;
    uint64_t mw[4] = {0, 0, 0, 0};
    const uint64_t t = cfg.record_trace ? now_ns() : 0;
    for (uint32_t i : ids) {
      mw[i / 48] |= 1ull << (i % 48);
      const uint32_t sq = ++host_seq[i];
      last_word[i] = w;
      if (cfg.record_trace) host_log[i].push_back(HostRec{sq, w, t});
    }
    const uint32_t e = (seq - 1) % ring_entries;
    for (uint32_t k = 0; k < replicas; ++k) {
      unsigned long long* ent = ring + (uint64_t(k) * ring_entries + e) * 8;
      for (int j = 0; j < 4; ++j) __atomic_store_n(ent + 1 + j, mw[j] | tag, __ATOMIC_RELAXED);
      __atomic_store_n(ent + 5, uint64_t(hint & 0xFFu) | tag, __ATOMIC_RELAXED);
      __atomic_store_n(ent, uint64_t(seq) | (uint64_t(w) << 32), __ATOMIC_RELEASE);   // last: publishes the entry
    }
    return true;
  }
  inline uint32_t to_gpu_word(uint32_t i) const {
    if (gateway) return last_word[i];   // (HYBRID: whichever channel wrote last)
    return uint32_t(__atomic_load_n(to_gpu + uint64_t(i) * dreps * cell_u64, __ATOMIC_ACQUIRE));
  }
};

static bool mask_ids(const lk_session* s, const uint64_t* mask, uint32_t nwords, std::vector<uint32_t>& ids,
                     int* rc) {
  ids.clear();
  for (uint32_t k = 0; k < nwords; ++k) {
    uint64_t m = mask[k];
    while (m) {
      const uint32_t b = uint32_t(__builtin_ctzll(m));
      m &= m - 1;
      const uint64_t id = uint64_t(k) * 64 + b;
      if (id >= s->nw) {
        *rc = fail(LK_E_USAGE, "sm mask wider than %u clusters", s->nw);
        return false;
      }
      ids.push_back(uint32_t(id));
    }
  }
  if (ids.empty()) {
    *rc = fail(LK_E_USAGE, "sm mask must select at least one cluster");
    return false;
  }
  return true;
}

static std::string ids_str(const std::vector<uint32_t>& v) {
  std::string out = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) out += ", ";
    out += std::to_string(v[i]);
  }
  return out + "]";
}

// Worker errors surface on the next host call (native.py:128-131).
static int check_workers(lk_session* s) {
  if (*s->err_any == 0) return LK_OK;   // set (after err[i]) by any worker that records an error
  for (uint32_t i = 0; i < s->nw; ++i) {
    const unsigned long long e = s->err[i];
    if (e) return fail(LK_E_WORKER_DIED, "worker %u died: device error %u on word %u", i, uint32_t(e),
                       uint32_t(e >> 32));
  }
  return LK_OK;
}

static int require_live(lk_session* s) {
  if (!s) return fail(LK_E_USAGE, "null session");
  if (s->disposed) return fail(LK_E_USAGE, "session already disposed");
  return check_workers(s);
}

static int kernel_status(lk_session* s) {
  if (s->kernel_done) return 1;
  const int ls = s->launch_state.load(std::memory_order_acquire);
  if (ls == 0) return 0;     // launch call still inside the driver (or a profiler): resident
  if (ls < 0) {
    s->kernel_done = true;
    fail(LK_E_CUDA, "cooperative launch: %s", cudaGetErrorString(s->launch_err));
    return -1;
  }
  cudaSetDevice(s->device);
  CtxScope cs(s->part.ca);
  cudaError_t q = cudaStreamQuery(s->stream);
  if (q == cudaErrorNotReady) return 0;
  s->kernel_done = true;
  if (q != cudaSuccess) {
    fail(LK_E_CUDA, "persistent kernel failed: %s", cudaGetErrorString(q));
    return -1;
  }
  return 1;
}

// Host spin with the reference's timeout contract (native.py:233-248).  The
// clock is read every 256 spins and started lazily, and the slow checks
// (worker error words, cudaStreamQuery on the kernel -- a driver call of
// several microseconds) run only once a wait has lasted 200 us, so a normal
// microsecond-scale round trip never pays for them.
struct Spinner {
  static constexpr uint64_t kSlowEveryNs = 200000;
  const lk_session* s;
  uint64_t t0 = 0, next_slow = 0;
  uint32_t spins = 0, checks = 0;
  explicit Spinner(const lk_session* ss) : s(ss) {}
  enum { kGo = 0, kTimeout = 1, kSlowCheck = 2 };
  inline int step() {
    LK_PAUSE();
    if (s->cfg.spin_strategy == 1 && ++spins >= s->cfg.spin_yield_threshold) {
      spins = 0;
      sched_yield();
    }
    if ((++checks & 255u) == 0) {
      const uint64_t t = now_ns();
      if (!t0) {
        t0 = t;
        next_slow = t + kSlowEveryNs;
        return kGo;
      }
      if (t - t0 > s->cfg.wait_timeout_ns) return kTimeout;
      if (t >= next_slow) {
        next_slow = t + kSlowEveryNs;
        return kSlowCheck;
      }
    }
    return kGo;
  }
};

// Host-preemption probe (lk_bench_roundtrip_gaps): the largest gap between
// consecutive TSC reads of the calling thread's spin loops in a round.  A
// spinning iteration takes tens of ns, so a gap of microseconds means the
// thread was not running: an interrupt, a timer tick or a vCPU preemption.
struct GapProbe {
  uint64_t last = 0, max = 0;
};
static thread_local GapProbe* t_gap = nullptr;

static inline uint64_t tsc() {
#if defined(__x86_64__)
  return __rdtsc();
#else
  return now_ns();
#endif
}

static inline void gap_tick() {
  GapProbe* g = t_gap;
  if (!g) return;
  const uint64_t t = tsc();
  if (g->last && t - g->last > g->max) g->max = t - g->last;
  g->last = t;
}

// TSC ticks per ns, calibrated once against CLOCK_MONOTONIC over 20 ms.
static double tsc_per_ns() {
  static double r = 0.0;
  static std::once_flag once;
  std::call_once(once, [] {
    const uint64_t c0 = tsc(), n0 = now_ns();
    usleep(20000);
    const uint64_t c1 = tsc(), n1 = now_ns();
    r = n1 > n0 ? double(c1 - c0) / double(n1 - n0) : 1.0;
  });
  return r;
}

// Spin until word(i) == want for every id.  Returns LK_OK, LK_E_HANG or
// LK_E_WORKER_DIED.
static int spin_words(lk_session* s, const std::vector<uint32_t>& ids, uint32_t want, const char* what,
                      bool ack_each = false) {
  Spinner sp(s);
  size_t j = 0;
  while (j < ids.size()) {
    gap_tick();
    if (s->word(ids[j]) == want) {
      if (ack_each) s->host_write(ids[j], LK_NOP);
      ++j;
      continue;
    }
    const int st = sp.step();
    if (st == Spinner::kTimeout) {
      int rc = check_workers(s);
      if (rc) return rc;
      return fail(LK_E_HANG, "%s made no progress within %.3fs (workers %s)", what,
                  double(s->cfg.wait_timeout_ns) / 1e9, ids_str(ids).c_str());
    }
    if (st == Spinner::kSlowCheck) {
      int rc = check_workers(s);
      if (rc) return rc;
      if (kernel_status(s) != 0) return fail(LK_E_WORKER_DIED, "persistent kernel is no longer running");
    }
  }
  return LK_OK;
}

// ------------------------------------------------------------------ device claims
static std::mutex g_claim_mu;
static void release_device(int dev);
void lk_session::release_claim() {
  if (claimed) {
    release_device(device);
    claimed = false;
  }
}
static uint8_t g_claimed[kMaxDevices];
static int g_live = 0;                        // claimed devices
// cudaFreeHost synchronizes the device: with a persistent kernel resident it
// would wait for that kernel to exit -- forever when the caller is the thread
// that would dispose it (a garbage-collected session object of an earlier
// test, a HostBuffer dropped mid-session).  Pinned frees are therefore
// deferred while any session holds a device claim, and made once none does.
static std::vector<void*> g_pinned_graveyard;  // under g_claim_mu

static void free_pinned(void* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> g(g_claim_mu);
    if (g_live > 0) {
      g_pinned_graveyard.push_back(p);
      return;
    }
  }
  cudaFreeHost(p);
}

static bool claim_device(int dev) {
  std::lock_guard<std::mutex> g(g_claim_mu);
  if (dev < 0 || dev >= kMaxDevices || g_claimed[dev]) return false;
  g_claimed[dev] = 1;
  ++g_live;
  return true;
}
static void release_device(int dev) {
  std::vector<void*> drain;
  {
    std::lock_guard<std::mutex> g(g_claim_mu);
    if (dev >= 0 && dev < kMaxDevices && g_claimed[dev]) {
      g_claimed[dev] = 0;
      --g_live;
    }
    if (g_live == 0) drain.swap(g_pinned_graveyard);
  }
  for (void* p : drain) cudaFreeHost(p);
}

// ------------------------------------------------------------------ profile runs
// lk_profile_run: a session whose handshakes come from a host thread started
// before the kernel launch.  A profiler that serializes launches (ncu returns
// from the launch only when the kernel has exited) then sees a complete run.
// The thread makes no CUDA calls: it writes and reads the mapped mailboxes
// only (the descriptor is staged before the launch).
static int stage_locked(lk_session* s, uint32_t slot, const lk_desc* d, const uint64_t* mask, uint32_t nwords);

struct ProfileRun {
  const lk_desc* descs = nullptr;   // payload items, dispatched to every worker in turn (null: empty tasks)
  uint32_t ndesc = 0;
  uint64_t rounds = 0;
  uint64_t elapsed_ns = 0;
  int rc = LK_OK;
};
static thread_local ProfileRun* t_profile = nullptr;

static void profile_driver(lk_session* s, ProfileRun* pr) {
  auto spin = [&](uint32_t i, uint32_t want, uint64_t limit_ns) {
    const uint64_t dl = now_ns() + limit_ns;
    uint32_t k = 0;
    while (s->word(i) != want) {
      LK_PAUSE();
      if ((++k & 1023u) == 0 && now_ns() > dl) return false;
    }
    return true;
  };
  const uint64_t boot_dl = now_ns() + 60ull * 1000000000ull;   // profilers slow the boot down
  for (uint32_t i = 0; i < s->nw;) {
    if (s->word(i) == LK_NOP && s->phase(i) == LK_PHASE_IDLE) { ++i; continue; }
    if (now_ns() > boot_dl) { pr->rc = LK_E_INIT; break; }
    LK_PAUSE();
  }
  const uint64_t t0 = now_ns();
  for (uint64_t r = 0; r < pr->rounds && pr->rc == LK_OK; ++r) {
    if (pr->ndesc) {   // full-mask payload dispatch of slot 1 + r % ndesc, then the ack
      const uint32_t w = LK_WORK_BASE + 1 + uint32_t(r % pr->ndesc);
      for (uint32_t i = 0; i < s->nw; ++i) s->host_write(i, w);
      for (uint32_t i = 0; i < s->nw && pr->rc == LK_OK; ++i)
        if (!spin(i, LK_FINISHED, 10ull * 1000000000ull)) pr->rc = LK_E_HANG;
      for (uint32_t i = 0; i < s->nw; ++i) s->host_write(i, LK_NOP);
      for (uint32_t i = 0; i < s->nw && pr->rc == LK_OK; ++i)
        if (!spin(i, LK_NOP, 10ull * 1000000000ull)) pr->rc = LK_E_HANG;
      continue;
    }
    const uint32_t i = uint32_t(r % s->nw);
    s->host_write(i, LK_WORK_BASE, LK_HINT_EMPTY);
    if (!spin(i, LK_FINISHED, 10ull * 1000000000ull)) { pr->rc = LK_E_HANG; break; }
    s->host_write(i, LK_NOP);
    if (!spin(i, LK_NOP, 10ull * 1000000000ull)) { pr->rc = LK_E_HANG; break; }
  }
  pr->elapsed_ns = now_ns() - t0;
  for (uint32_t i = 0; i < s->nw; ++i) s->host_write(i, LK_EXIT);
}

// ------------------------------------------------------------------ create
extern "C" int lk_create(const lk_config* cfg_in, lk_session** out, uint64_t* init_ns) {
  if (!cfg_in || !out) return fail(LK_E_USAGE, "null argument");
  *out = nullptr;
  const uint64_t t0 = now_ns();
  lk_config cfg = *cfg_in;
  if (cfg.spin_strategy > 1) return fail(LK_E_USAGE, "unknown spin strategy %u", cfg.spin_strategy);
  if (cfg.spin_strategy == 1 && cfg.spin_yield_threshold == 0)
    return fail(LK_E_USAGE, "spin_yield_threshold must be positive");
  if (cfg.cell_stride == 0) cfg.cell_stride = 128;
  if (cfg.cell_stride != 8 && cfg.cell_stride != 16 && cfg.cell_stride != 32 && cfg.cell_stride != 64 &&
      cfg.cell_stride != 128)
    return fail(LK_E_CONFIG, "cell_stride must be 8, 16, 32, 64 or 128");
  // two workers per host cache line: the host's scan after a wide dispatch
  // reads 74 lines instead of 148 (-0.9 us gateway full mask, round robin
  // unchanged; tools/ab_status_stride2.py); four per line serialize the DMA
  // writes (tools/ab_status_wide.py)
  if (cfg.status_stride == 0) cfg.status_stride = 32;
  if (cfg.status_stride != 16 && cfg.status_stride != 32 && cfg.status_stride != 64 && cfg.status_stride != 128)
    return fail(LK_E_CONFIG, "status_stride must be 16, 32, 64 or 128");
  if (cfg.poll_mode > LK_POLL_HYBRID) return fail(LK_E_CONFIG, "unknown poll_mode %u", cfg.poll_mode);
  // Replicated cells / event rings and the ack window measured slower or
  // neutral in every mode and were removed; the fields
  // stay in the ABI and take their one remaining value.
  if (cfg.poll_replicas == 0) cfg.poll_replicas = 1;
  if (cfg.poll_replicas != 1)
    return fail(LK_E_CONFIG, "poll_replicas must be 1 (replicated cells were measured slower and removed)");
  if (cfg.flags & (LK_CF_ACK_WINDOW | LK_CF_DYNAMIC_TILES))
    return fail(LK_E_CONFIG, "LK_CF_ACK_WINDOW and LK_CF_DYNAMIC_TILES were measured neutral or slower and "
                "removed");
  if (cfg.ring_stages == 0) cfg.ring_stages = 6;
  if (cfg.ring_stages < 2 || cfg.ring_stages > lk_ring_max_stages())
    return fail(LK_E_CONFIG, "ring_stages must be 2..%u", lk_ring_max_stages());
  if (cfg.poll_spacing_ns == 0) cfg.poll_spacing_ns = 300;
  if (cfg.threads_per_worker == 0) cfg.threads_per_worker = 512;
  if (cfg.threads_per_worker % 32 || cfg.threads_per_worker > 544)
    return fail(LK_E_CONFIG, "threads_per_worker must be a multiple of 32 and <= 544");
  if (cfg.num_slots == 0) cfg.num_slots = 1024;
  if (cfg.trace_capacity == 0) cfg.trace_capacity = 65536;
  if (cfg.wait_timeout_ns == 0) cfg.wait_timeout_ns = 10ull * 1000000000ull;
  if (cfg.ack_delay_ns == 0) cfg.ack_delay_ns = 300;
  if (cfg.tma_min_workers == 0) cfg.tma_min_workers = 49;
  if ((cfg.flags & LK_CF_HOST_DESC) && cfg.poll_mode != LK_POLL_DIRECT)
    return fail(LK_E_CONFIG, "host-resident descriptors (LK_CF_HOST_DESC) need DIRECT polling");
  // polls are acquires (ld.acquire.sys: LDG.STRONG.SYS + CCTL.IVALL, no membar;
  // within noise of relaxed polls, tools/ab_acquire.py) unless the caller asks
  // for relaxed ones; host-written descriptors need the acquire
  if (cfg.flags & LK_CF_RELAXED_POLL) cfg.flags &= ~LK_CF_ACQUIRE_POLL;
  else cfg.flags |= LK_CF_ACQUIRE_POLL;
  if ((cfg.flags & LK_CF_HOST_DESC) && (cfg.flags & LK_CF_RELAXED_POLL))
    return fail(LK_E_CONFIG, "host-resident descriptors (LK_CF_HOST_DESC) need acquire polls");
  if (cfg.ack_delay_ns > 100000 || cfg.idle_delay_ns > 100000)
    return fail(LK_E_CONFIG, "ack_delay_ns and idle_delay_ns must be at most 100000");

  int ndev = 0;
  LK_CUDA(cudaGetDeviceCount(&ndev));
  if (cfg.device < 0 || cfg.device >= ndev) return fail(LK_E_CONFIG, "no CUDA device %d", cfg.device);
  if (cfg.device >= kMaxDevices) return fail(LK_E_CONFIG, "device %d beyond the %d supported", cfg.device, kMaxDevices);
  LK_CUDA(cudaSetDevice(cfg.device));
  cudaDeviceProp prop;
  LK_CUDA(cudaGetDeviceProperties(&prop, cfg.device));
  if (!prop.cooperativeLaunch) return fail(LK_E_INIT, "device lacks cooperative launch");
  if (!prop.canMapHostMemory) return fail(LK_E_INIT, "device cannot map host memory");
  svc_stream();   // created in the primary context, before any green context is pushed
  // One live session per device and process: a session's CTAs hold every SM
  // (or, partitioned, SMs split off the whole device), so a second one could
  // never become resident -- it would spin in boot, then run unbidden later.
  uint32_t nsm = uint32_t(prop.multiProcessorCount);
  if (cfg.sm_partition && cfg.sm_partition >= nsm)
    return fail(LK_E_CONFIG, "sm_partition %u must be below the %u SMs", cfg.sm_partition, nsm);
  if (!cfg.sm_partition && cfg.num_workers > nsm)
    return fail(LK_E_CONFIG, "num_workers %u exceeds the %u SMs (one worker per SM)", cfg.num_workers, nsm);
  if (cfg.num_workers > 256) return fail(LK_E_CONFIG, "at most 256 workers (4 mask words)");
  if (cfg.poll_mode != LK_POLL_DIRECT && (cfg.num_workers ? cfg.num_workers : nsm) > 192 && !cfg.sm_partition)
    return fail(LK_E_CONFIG, "gateway/hybrid modes support up to 192 workers (4 x 48-bit event masks)");
  if (!claim_device(cfg.device))
    return fail(LK_E_BUSY, "device %d already has a live LK session in this process", cfg.device);
  // from here on every failure path releases the claim (cleanup, or explicitly)
  Partition part;
  if (cfg.sm_partition) {
    int prc = make_partition(cfg.device, cfg.sm_partition, &part);
    if (prc) {
      release_device(cfg.device);
      return prc;
    }
    nsm = part.a_sms;
  }
  if (cfg.num_workers == 0) cfg.num_workers = nsm;
  if (cfg.num_workers > nsm) {
    free_partition(&part);
    release_device(cfg.device);
    return fail(LK_E_CONFIG, "num_workers %u exceeds the partition's %u SMs (one worker per SM)", cfg.num_workers,
                nsm);
  }

  auto* s = new lk_session();
  s->part = part;
  s->cfg = cfg;
  s->nw = cfg.num_workers;
  s->nwords = (s->nw + 63) / 64;
  s->threads = cfg.threads_per_worker;
  s->device = cfg.device;
  s->cell_u64 = cfg.cell_stride / 8;
  s->status_u64 = cfg.status_stride / 8;
  s->replicas = cfg.poll_replicas;
  s->gateway = cfg.poll_mode == LK_POLL_GATEWAY || cfg.poll_mode == LK_POLL_HYBRID;
  s->hybrid = cfg.poll_mode == LK_POLL_HYBRID;
  s->dreps = s->hybrid ? 1 : s->replicas;
  s->host_dseq.assign(s->nw, 0);
  s->last_word.assign(s->nw, LK_NOP);
  for (uint32_t i = 0; i < s->nw; ++i) s->all_ids.push_back(i);
  s->pending.assign(s->nwords, 0);
  s->registered.assign(cfg.num_slots, 0);
  s->slot_pend.assign(size_t(cfg.num_slots) * s->nwords, 0);
  s->slot_busy.assign(cfg.num_slots, 0);
  s->inflight.reserve(64);
  s->scratch.assign(s->nwords, 0);
  s->ack_pending.assign(s->nwords, 0);
  s->idle_known.assign(s->nwords, 0);
  s->reg_desc.resize(cfg.num_slots);
  s->reg_in.resize(cfg.num_slots);
  s->slot_ver.assign(cfg.num_slots, 0);
  s->wslot.assign(s->nw, 0xFFFFFFFFu);
  s->wver.assign(s->nw, 0);
  s->reg_mask.resize(cfg.num_slots);
  s->host_seq.assign(s->nw, 0);
  s->host_times.assign(3 * size_t(s->nw), 0);
  s->host_log.resize(s->nw);
  s->t_create = t0;

  auto cleanup = [&](int rc) {
    if (s->host_block) free_pinned(s->host_block);
    if (s->dev_block) dev_free(s->dev_block);
    if (s->stream) {
      CtxScope cs(s->part.ca);
      cudaStreamDestroy(s->stream);
    }
    if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
    free_partition(&s->part);
    release_device(s->device);
    delete s;
    return rc;
  };

  // --- pinned mapped mailboxes: to_gpu (DIRECT replicas | GATEWAY doorbell
  // replicas) | status | err | smid, 4 KiB aligned
  auto al = [](size_t x) { return (x + 4095) & ~size_t(4095); };
  // HYBRID: direct cells (1 replica) first, then the ring replicas + tail line
  const size_t directb = (!s->gateway || s->hybrid)
                             ? al(size_t(s->nw) * (s->hybrid ? 1 : s->replicas) * cfg.cell_stride) : 0;
  const size_t ringb = s->gateway ? al(size_t(s->replicas) * s->ring_entries * 64 + 128) : 0;
  const size_t tob = directb + ringb;
  const size_t cells = al(size_t(s->nw) * cfg.status_stride);
  const size_t err_words = (size_t(s->nw) + 15) / 16 * 16;   // err[] then err_any on its own line
  const size_t errb = al(err_words * 8 + 128), smidb = al(size_t(s->nw) * 4);
  const bool host_desc = (cfg.flags & LK_CF_HOST_DESC) != 0;
  const size_t hdescb = host_desc ? al(size_t(cfg.num_slots) * sizeof(lk_desc)) : 0;
  const size_t hmaskb = host_desc ? al(size_t(cfg.num_slots) * ((s->nw + 63) / 64) * 8) : 0;
  const size_t host_bytes = tob + cells + errb + smidb + hdescb + hmaskb;
  cudaError_t ce = cudaHostAlloc(reinterpret_cast<void**>(&s->host_block), host_bytes,
                                 cudaHostAllocMapped | cudaHostAllocPortable);
  if (ce != cudaSuccess) return cleanup(fail(LK_E_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(ce)));
  memset(s->host_block, 0, host_bytes);
  s->to_gpu = reinterpret_cast<unsigned long long*>(s->host_block);
  s->ring = s->to_gpu + directb / 8;
  s->gw_tail = s->ring + size_t(s->replicas) * s->ring_entries * 8;   // own line after the rings
  s->status = reinterpret_cast<volatile unsigned long long*>(s->host_block + tob);
  s->err = reinterpret_cast<volatile unsigned long long*>(s->host_block + tob + cells);
  s->smid = reinterpret_cast<volatile uint32_t*>(s->host_block + tob + cells + errb);
  s->err_any = reinterpret_cast<volatile uint32_t*>(s->err + err_words);
  if (host_desc) {   // mapped + UVA: the host pointer is the device pointer
    s->d_desc = reinterpret_cast<lk_desc*>(s->host_block + tob + cells + errb + smidb);
    s->d_mask = reinterpret_cast<unsigned long long*>(s->host_block + tob + cells + errb + smidb + hdescb);
    s->host_desc = true;
  }
  for (uint32_t i = 0; i < s->nw; ++i) {
    for (uint32_t k = 0; k < s->replicas; ++k) {
      if (k < s->dreps && (!s->gateway || s->hybrid))
        s->to_gpu[(uint64_t(i) * s->dreps + k) * s->cell_u64] = LK_NOP;   // {NOP, seq 0}
    }
    s->status[uint64_t(i) * s->status_u64] = uint64_t(LK_NOP) | (uint64_t(LK_PHASE_BOOTING) << 32);
    s->smid[i] = 0xFFFFFFFFu;
  }

  // --- device block: desc | masks | ctr | spans | dmb | exited | trace | tcnt
  const size_t descb = al(size_t(cfg.num_slots) * sizeof(lk_desc));
  const size_t maskb = al(size_t(cfg.num_slots) * s->nwords * 8);
  const size_t ctrb = al(size_t(cfg.num_slots) * 16);   // per slot: reduce counter, tile claim, done, spare
  const size_t spanb = al(size_t(s->nw) * 8 * LK_TIMELINE_WORDS);
  const size_t dmbb = al(size_t(s->nw) * 128);
  const size_t exb = al(4);
  const size_t traceb = cfg.record_trace ? al(size_t(s->nw) * cfg.trace_capacity * sizeof(lk_dev_trace)) : 0;
  const size_t tcntb = al(size_t(s->nw) * 4);
  const size_t fastb = al(size_t(s->nw) * 4);
  const size_t dev_bytes = descb + maskb + ctrb + spanb + dmbb + exb + traceb + tcntb + fastb;
  ce = dev_alloc(reinterpret_cast<void**>(&s->dev_block), dev_bytes);
  if (ce != cudaSuccess) return cleanup(fail(LK_E_CUDA, "device alloc: %s", cudaGetErrorString(ce)));
  ce = cudaMemsetAsync(s->dev_block, 0, dev_bytes, svc_stream());
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(svc_stream());  // zeroed before the kernel reads it
  if (ce != cudaSuccess) return cleanup(fail(LK_E_CUDA, "memset: %s", cudaGetErrorString(ce)));
  uint8_t* p = s->dev_block;
  if (!s->host_desc) {
    s->d_desc = reinterpret_cast<lk_desc*>(p);
    s->d_mask = reinterpret_cast<unsigned long long*>(p + descb);
  }
  p += descb + maskb;
  s->d_ctr = reinterpret_cast<uint32_t*>(p); p += ctrb;
  s->d_spans = reinterpret_cast<unsigned long long*>(p); p += spanb;
  s->d_dmb = reinterpret_cast<unsigned long long*>(p); p += dmbb;
  s->d_exited = reinterpret_cast<uint32_t*>(p); p += exb;
  s->d_trace = traceb ? reinterpret_cast<lk_dev_trace*>(p) : nullptr; p += traceb;
  s->d_tcnt = reinterpret_cast<uint32_t*>(p); p += tcntb;
  s->d_fast = reinterpret_cast<uint32_t*>(p);

  ce = cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) return cleanup(fail(LK_E_CUDA, "stream: %s", cudaGetErrorString(ce)));

  // --- one CTA per SM: dynamic smem above half the SM's capacity
  const bool use_tma = !(cfg.flags & LK_CF_LSU_PAYLOAD);
  s->smem = std::max(size_t(prop.sharedMemPerMultiprocessor) / 2 + 8192, use_tma ? lk_ring_bytes(cfg.ring_stages) : 0);
  if (s->smem > size_t(prop.sharedMemPerBlockOptin) - 1024)
    return cleanup(fail(LK_E_INIT, "payload ring needs %zu B of shared memory, the device offers %zu",
                        s->smem, size_t(prop.sharedMemPerBlockOptin) - 1024));
  // Kernel load, attributes, occupancy, the kernel's stream and the launch
  // happen in the partition's green context when there is one: its streams
  // run on its SMs only.  (Memory is shared with the primary context.)
  int bps = 0;
  // + three warps: host-cell poller and mailbox poller (HYBRID), gateway (CTA 0);
  // unused ones retire at once
  const uint32_t launch_threads = s->threads + 96;
  const char* what = "stream";
  {
    CtxScope cs(s->part.ca);
    ce = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (ce == cudaSuccess) { what = "kernel load"; ce = lk_preload_kernels(); }
    if (ce == cudaSuccess) { what = "smem attr"; ce = lk_persistent_configure(s->smem); }
    if (ce == cudaSuccess) { what = "occupancy"; ce = lk_persistent_occupancy(launch_threads, s->smem, &bps); }
  }
  if (ce != cudaSuccess) return cleanup(fail(LK_E_CUDA, "%s: %s", what, cudaGetErrorString(ce)));
  if (bps != 1) return cleanup(fail(LK_E_INIT, "expected exactly 1 resident worker per SM, got %d", bps));

  lk_dev_args a;
  memset(&a, 0, sizeof a);
  a.to_gpu = s->to_gpu;
  a.status = const_cast<unsigned long long*>(s->status);
  a.err = const_cast<unsigned long long*>(s->err);
  a.err_any = const_cast<uint32_t*>(s->err_any);
  a.smid = const_cast<uint32_t*>(s->smid);
  a.desc = s->d_desc;
  a.slot_mask = s->d_mask;
  a.reduce_ctr = s->d_ctr;
  a.spans = s->d_spans;
  a.trace = s->d_trace;
  a.trace_cnt = s->d_tcnt;
  a.fast_cnt = s->d_fast;
  a.cell_u64 = s->cell_u64;
  a.status_u64 = s->status_u64;
  a.replicas = s->replicas;
  a.spacing_ns = cfg.poll_spacing_ns;
  a.num_slots = cfg.num_slots;
  a.nwords = s->nwords;
  a.trace_cap = cfg.trace_capacity;
  a.record_trace = cfg.record_trace ? 1 : 0;
  a.backoff_ns = cfg.poll_backoff_ns;
  a.flags = cfg.flags;
  a.ring = s->ring;
  a.gw_tail = const_cast<unsigned long long*>(s->gw_tail);
  a.dmb = s->d_dmb;
  a.exited = s->d_exited;
  a.sink = s->d_exited + 64;   // same zeroed page, its own 128-B line
  a.ring_entries = s->ring_entries;
  a.dmb_u64 = 16;
  a.nw = s->nw;
  a.wthreads = s->threads;
  a.poll_mode = cfg.poll_mode;
  a.use_tma = use_tma ? 1 : 0;
  a.ring_stages = cfg.ring_stages;
  a.tma_min_workers = cfg.tma_min_workers;
  {   // block_reduce schedule (tuning overrides for tools/reduce_sizes.py)
    const char* e1 = getenv("LK_RED_SHARE8");
    const char* e2 = getenv("LK_RED_CLAIM");
    a.red_share8 = e1 ? uint32_t(atoi(e1)) : 2u;
    a.red_claim = e2 ? uint32_t(atoi(e2)) : 2u;
    if (a.red_share8 > 8) a.red_share8 = 8;
    if (a.red_claim < 1) a.red_claim = 1;
  }
  {
    int khz = 0;   // SM clock: the delay is spun on clock64
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, cfg.device) != cudaSuccess || khz <= 0) khz = 1965000;
    const bool off = (cfg.flags & LK_CF_NO_ACK_DELAY) != 0;
    a.ack_delay_cyc = off ? 0u : uint32_t(uint64_t(cfg.ack_delay_ns) * uint64_t(khz) / 1000000ull);
    a.idle_delay_cyc = uint32_t(uint64_t(cfg.idle_delay_ns) * uint64_t(khz) / 1000000ull);
  }
  ProfileRun* pr = t_profile;
  std::thread driver;
  if (pr) {
    lk_desc ed;
    memset(&ed, 0, sizeof ed);
    ed.kind = LK_KIND_EMPTY;
    int src = stage_locked(s, 0, &ed, nullptr, 0);
    std::vector<uint64_t> full(s->nwords, 0);
    for (uint32_t i = 0; i < s->nw; ++i) full[i >> 6] |= 1ull << (i & 63);
    for (uint32_t k = 0; k < pr->ndesc && !src; ++k) {
      if (pr->descs[k].kind >= LK_KIND_COUNT || k + 1 >= cfg.num_slots) src = fail(LK_E_USAGE, "bad profile descriptor");
      else src = stage_locked(s, k + 1, &pr->descs[k], full.data(), s->nwords);
    }
    if (src) return cleanup(src);
    driver = std::thread(profile_driver, s, pr);
  }
  if (!pr) {
    // the launch runs on its own thread (see lk_session::launcher); the boot
    // wait below watches both the workers and the launch's outcome
    s->launcher = std::thread([s, a, launch_threads] {
      cudaSetDevice(s->device);
      cudaError_t e;
      {
        CtxScope cs(s->part.ca);
        e = lk_launch_persistent(a, s->nw, launch_threads, s->smem, s->stream);
      }
      s->launch_err = e;
      s->launch_state.store(e == cudaSuccess ? 1 : -1, std::memory_order_release);
    });
  } else {
    CtxScope cs(s->part.ca);
    ce = lk_launch_persistent(a, s->nw, launch_threads, s->smem, s->stream);
  }
  if (pr) {
    // the driver thread ends every worker with EXIT, launch failure or not
    if (ce != cudaSuccess) pr->rc = LK_E_INIT;
    driver.join();
    if (ce == cudaSuccess) {
      CtxScope cs(s->part.ca);
      ce = cudaStreamSynchronize(s->stream);
    }
    s->kernel_done = true;
    const int rc = ce != cudaSuccess ? fail(LK_E_CUDA, "profile run: %s", cudaGetErrorString(ce))
                   : pr->rc       ? fail(pr->rc, "profile run: handshakes stalled")
                                  : LK_OK;
    const std::string msg = g_last_error;
    cleanup(rc);
    g_last_error = msg;
    return rc;
  }

  // --- boot: every worker publishes INIT then NOP (native.py:113-118)
  // A failed boot frees the session only once the kernel has retired (the
  // surviving workers are told EXIT first); a kernel that stays resident can
  // still touch the mailboxes, so then everything, the device claim included,
  // is deliberately leaked.
  auto boot_failed = [&](int rc) {
    if (kernel_status(s) == 0) {
      s->post(s->all_ids, LK_EXIT);
      const uint64_t until = now_ns() + std::min<uint64_t>(cfg.wait_timeout_ns, 2000000000ull);
      while (kernel_status(s) == 0 && now_ns() < until) usleep(50);
      if (kernel_status(s) == 0) {
        s->launcher.detach();   // still inside the launch call: leaked with the session
        return rc;
      }
    }
    s->join_launcher();
    return cleanup(rc);
  };
  const uint64_t deadline = now_ns() + cfg.wait_timeout_ns;
  for (uint32_t i = 0; i < s->nw;) {
    if (s->word(i) == LK_NOP && s->phase(i) == LK_PHASE_IDLE) { ++i; continue; }
    if (s->launch_state.load(std::memory_order_acquire) < 0) {
      const int rc = fail(LK_E_INIT, "cooperative launch: %s", cudaGetErrorString(s->launch_err));
      const std::string msg = g_last_error;
      s->join_launcher();
      cleanup(rc);
      g_last_error = msg;
      return rc;
    }
    if (s->err[i]) {
      const int rc = fail(LK_E_INIT, "worker %u failed during boot", i);
      const std::string msg = g_last_error;
      boot_failed(rc);
      g_last_error = msg;
      return rc;
    }
    if (now_ns() > deadline) {
      const int rc = fail(LK_E_INIT, "workers failed to reach idle (worker %u)", i);
      const std::string msg = g_last_error;
      boot_failed(rc);
      g_last_error = msg;
      return rc;
    }
    LK_PAUSE();
  }
  *out = s;
  if (init_ns) *init_ns = now_ns() - t0;
  return LK_OK;
}

extern "C" int lk_profile_run(const lk_config* cfg, const lk_desc* descs, uint32_t ndesc, uint64_t rounds,
                              uint64_t* elapsed_ns) {
  if (!cfg || (ndesc && !descs)) return fail(LK_E_USAGE, "null argument");
  if (cfg->poll_mode != LK_POLL_DIRECT || cfg->record_trace)
    return fail(LK_E_CONFIG, "profile runs use DIRECT polling without trace recording");
  ProfileRun pr;
  pr.descs = descs;
  pr.ndesc = ndesc;
  pr.rounds = rounds;
  t_profile = &pr;
  lk_session* s = nullptr;
  const int rc = lk_create(cfg, &s, nullptr);
  t_profile = nullptr;
  if (elapsed_ns) *elapsed_ns = pr.elapsed_ns;
  return rc;
}

// ------------------------------------------------------------------ descriptors
static int stage_locked(lk_session* s, uint32_t slot, const lk_desc* d, const uint64_t* mask, uint32_t nwords);

extern "C" int lk_register_desc(lk_session* s, uint32_t slot, const lk_desc* d, const uint64_t* mask,
                                uint32_t nwords) {
  int rc = require_live(s);
  if (rc) return rc;
  if (!d) return fail(LK_E_USAGE, "null descriptor");
  if (slot >= s->cfg.num_slots)
    return fail(LK_E_USAGE, "slot %u outside the %u-entry descriptor table", slot, s->cfg.num_slots);
  if (d->kind >= LK_KIND_COUNT) return fail(LK_E_USAGE, "unknown work kind %u", d->kind);
  std::lock_guard<std::mutex> g(s->mu);
  if (s->slot_busy[slot])
    return fail(LK_E_USAGE, "descriptor slot %u still referenced by an un-waited dispatch", slot);
  return stage_locked(s, slot, d, mask, nwords);
}

// ------------------------------------------------------------------ trigger / wait
static inline bool multi_worker_kind(uint32_t kind) {
  return kind != LK_KIND_EMPTY && kind != LK_KIND_BUSY_LOOP;
}

// Stage desc (+ the worker set that shards it) in the slot; a no-op when the
// device copy is already identical.  Caller holds s->mu.
// A C caller's descriptor is checked and normalised before it reaches the
// device: payload pointers must be 4-B aligned (element size) and non-null,
// pointers that are not 16-B aligned take the scalar path (cp.async.bulk and
// ld.global.v4 would fault on them), and the reduce's total is a double.
// Every payload pointer is classified with cudaPointerGetAttributes: device
// memory of the session's GPU, or host-mapped pinned memory (LK_DF_HOSTMEM:
// sys-scope loads, sys-scope release before FINISHED).  Anything else -- an
// unregistered host address, another GPU's memory -- would fault the resident
// kernel and with it the context, so it is refused here.
static int classify_ptr(uint64_t p, int device, const char* what, bool* host) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, reinterpret_cast<const void*>(p));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(LK_E_USAGE, "%s pointer 0x%llx: %s", what, (unsigned long long)p, cudaGetErrorString(e));
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (at.device != device)
      return fail(LK_E_USAGE, "%s pointer 0x%llx is memory of device %d, the session runs on device %d", what,
                  (unsigned long long)p, at.device, device);
    return LK_OK;
  }
  if (at.type == cudaMemoryTypeHost && at.devicePointer == reinterpret_cast<void*>(p)) {
    *host = true;
    return LK_OK;
  }
  return fail(LK_E_USAGE, "%s pointer 0x%llx is neither device memory nor mapped pinned host memory "
              "(lk_host_alloc)", what, (unsigned long long)p);
}

static int normalise_desc(int device, const lk_desc* in, lk_desc* out) {
  *out = *in;
  out->flags &= LK_DF_SCALAR;   // LK_DF_HOSTMEM is the runtime's to set
  if (!multi_worker_kind(in->kind)) return LK_OK;
  const bool two = in->kind == LK_KIND_VECTOR_ADD_I32 || in->kind == LK_KIND_SAXPY_F32;
  if (in->n && (!in->in0 || !in->out || (two && !in->in1)))
    return fail(LK_E_USAGE, "work kind %u needs non-null input and output pointers", in->kind);
  const uint64_t any = in->in0 | in->in1 | in->out;
  if (any & 3) return fail(LK_E_USAGE, "payload pointers must be 4-byte aligned");
  if (in->aux & 7) return fail(LK_E_USAGE, "the reduce total pointer must be 8-byte aligned");
  if (any & 15) out->flags |= LK_DF_SCALAR;
  if (in->n) {
    bool host = false, out_host = false;
    int rc = classify_ptr(in->in0, device, "input", &host);
    if (!rc && two) rc = classify_ptr(in->in1, device, "second input", &host);
    if (!rc) rc = classify_ptr(in->out, device, "output", &out_host);
    if (!rc && in->kind == LK_KIND_BLOCK_REDUCE_F32 && in->aux) rc = classify_ptr(in->aux, device, "total", &host);
    if (rc) return rc;
    if (out_host && in->kind == LK_KIND_BLOCK_REDUCE_F32)
      return fail(LK_E_USAGE, "block_reduce_f32 block partials (out) must be device memory; "
                  "the total (aux) may be host-mapped");
    if (host || out_host) out->flags |= LK_DF_HOSTMEM;
  }
  return LK_OK;
}

static int stage_locked(lk_session* s, uint32_t slot, const lk_desc* din, const uint64_t* mask, uint32_t nwords) {
  std::vector<uint64_t>& m = s->stage_mask;
  m.assign(s->nwords, 0);
  if (mask && multi_worker_kind(din->kind))
    for (uint32_t k = 0; k < nwords && k < s->nwords; ++k) m[k] = mask[k];
  // the caller's descriptor as last staged: re-staging the same one is free
  // (no pointer classification, no upload)
  if (s->registered[slot] && memcmp(&s->reg_in[slot], din, sizeof(lk_desc)) == 0 && s->reg_mask[slot] == m)
    return LK_OK;
  lk_desc dn;
  int nrc = normalise_desc(s->device, din, &dn);
  if (nrc) return nrc;
  const lk_desc* d = &dn;
  if (s->host_desc) {
    // plain stores into the mapped table; the WORK word that names the slot
    // is written later with release semantics, and the worker polls it with
    // an acquire load before fetching (LK_CF_HOST_DESC)
    memcpy(s->d_desc + slot, d, sizeof(lk_desc));
    memcpy(s->d_mask + uint64_t(slot) * s->nwords, m.data(), 8 * s->nwords);
    std::atomic_thread_fence(std::memory_order_release);
  } else {
    LK_CUDA(cudaSetDevice(s->device));
    LK_CUDA(cudaMemcpyAsync(s->d_desc + slot, d, sizeof(lk_desc), cudaMemcpyHostToDevice, s->copy_stream));
    LK_CUDA(cudaMemcpyAsync(s->d_mask + uint64_t(slot) * s->nwords, m.data(), 8 * s->nwords,
                            cudaMemcpyHostToDevice, s->copy_stream));
    LK_CUDA(cudaStreamSynchronize(s->copy_stream));  // in place before any WORK word names it
  }
  s->registered[slot] = 1;
  ++s->slot_ver[slot];   // workers' cached copies of this slot are stale now
  s->reg_desc[slot] = *d;
  s->reg_in[slot] = *din;
  s->reg_mask[slot] = m;
  return LK_OK;
}

// Checks in the reference's order (native.py:210-220): live, mask, busy
// workers, slot lock, idle cells; then stage the descriptor (when given) and
// write the WORK word to every masked worker, ascending.
// LK_CF_LAZY_ACK: before a worker is written again, its ack must have been
// consumed (the reference's wait spins for it, native.py:263-265; lazily it is
// spun for here instead).  Caller holds s->mu.
static int settle_acks(lk_session* s, const std::vector<uint32_t>& ids) {
  static thread_local std::vector<uint32_t> due;
  due.clear();
  for (uint32_t i : ids)
    if (s->ack_pending[i >> 6] >> (i & 63) & 1) due.push_back(i);
  if (due.empty()) return LK_OK;
  int rc = spin_words(s, due, LK_NOP, "wait for ack consumption");
  if (rc) return rc;
  for (uint32_t i : due) {
    s->ack_pending[i >> 6] &= ~(1ull << (i & 63));
    s->idle_known[i >> 6] |= 1ull << (i & 63);
  }
  return LK_OK;
}

static int trigger_locked(lk_session* s, const uint64_t* mask, uint32_t nwords, uint32_t slot,
                          const lk_desc* d, std::vector<uint32_t>& ids, uint64_t* elapsed_ns,
                          uint64_t t_call) {
  int rc = require_live(s);
  if (rc) return rc;
  if (!mask_ids(s, mask, nwords, ids, &rc)) return rc;
  std::vector<uint32_t> busy;
  for (uint32_t i : ids)
    if (s->pending[i >> 6] >> (i & 63) & 1) busy.push_back(i);
  if (!busy.empty()) return fail(LK_E_BUSY, "worker(s) %s still busy", ids_str(busy).c_str());
  if (slot < s->cfg.num_slots && s->slot_busy[slot])
    return fail(LK_E_USAGE, "descriptor slot %u still referenced by an un-waited dispatch", slot);
  if (slot >= s->cfg.num_slots)
    return fail(LK_E_USAGE, "slot %u outside the %u-entry descriptor table", slot, s->cfg.num_slots);
  rc = settle_acks(s, ids);
  if (rc) return rc;
  for (uint32_t i : ids) {
    if (s->idle_known[i >> 6] >> (i & 63) & 1) continue;
    const uint32_t w = s->word(i);
    if (w != LK_NOP) return fail(LK_E_BUSY, "worker %u not idle (from_gpu=%u)", i, w);
  }
  const uint64_t t0 = now_ns();
  if (d) {
    if (d->kind >= LK_KIND_COUNT) return fail(LK_E_USAGE, "unknown work kind %u", d->kind);
    rc = stage_locked(s, slot, d, mask, nwords);
    if (rc) return rc;
  } else if (!s->registered[slot]) {
    return fail(LK_E_USAGE, "descriptor slot %u not registered", slot);
  } else if (multi_worker_kind(s->reg_desc[slot].kind)) {
    // a payload shards by the trigger mask: workers derive rank and count
    // from the mask staged with the slot, so a different mask re-stages it
    // (else chunks would be skipped or done twice, and the reduce's arrival
    // count would never close)
    const std::vector<uint64_t>& rm = s->reg_mask[slot];
    bool same = true;
    for (uint32_t k = 0; k < s->nwords; ++k) same &= rm[k] == (k < nwords ? mask[k] : 0ull);
    if (!same) {
      const lk_desc cur = s->reg_in[slot];
      rc = stage_locked(s, slot, &cur, mask, nwords);
      if (rc) return rc;
    }
  }
  const uint32_t word = LK_WORK_BASE + slot;
  // a busy_loop of 0 iterations (the reference's default WorkDescriptor,
  // P/device.py:48-66) is an empty task: the worker may skip the fetch too
  const lk_desc& rd = s->reg_desc[slot];
  const bool no_work = rd.kind == LK_KIND_EMPTY || (rd.kind == LK_KIND_BUSY_LOOP && rd.iterations == 0);
  uint32_t hint = no_work ? LK_HINT_EMPTY : 0u;
  if (rd.flags & LK_DF_HOSTMEM) hint |= LK_HINT_SYSMEM;
  const uint32_t ver = s->slot_ver[slot];
  if (!no_work) {   // every masked worker fetched this slot version last: it may reuse its copy
    bool cached = true;
    for (uint32_t i : ids) cached &= s->wslot[i] == slot && s->wver[i] == ver;
    if (cached) hint |= LK_HINT_CACHED;
  }
  if (!s->post(ids, word, hint)) return fail(LK_E_HANG, "event ring full: gateway not consuming");
  const uint64_t t1 = now_ns();
  if (!no_work)
    for (uint32_t i : ids) {   // what each worker now holds (fetched, or reused)
      s->wslot[i] = slot;
      s->wver[i] = ver;
    }
  for (uint32_t i : ids) {
    s->host_times[3 * i] = t_call;
    s->host_times[3 * i + 1] = t1;
  }
  uint64_t* sp = s->slot_pend.data() + uint64_t(slot) * s->nwords;
  for (uint32_t i : ids) {
    s->pending[i >> 6] |= 1ull << (i & 63);
    sp[i >> 6] |= 1ull << (i & 63);
    s->idle_known[i >> 6] &= ~(1ull << (i & 63));
  }
  s->slot_busy[slot] = 1;
  s->inflight.push_back(slot);
  if (elapsed_ns) *elapsed_ns = t1 - t0;
  return LK_OK;
}

extern "C" int lk_trigger(lk_session* s, const uint64_t* mask, uint32_t nwords, uint32_t slot,
                          const lk_desc* d, uint64_t* elapsed_ns) {
  if (!s || !mask) return fail(LK_E_USAGE, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  static thread_local std::vector<uint32_t> ids;
  return trigger_locked(s, mask, nwords, slot, d, ids, elapsed_ns, now_ns());
}

static int wait_impl(lk_session* s, const uint64_t* mask, uint32_t nwords, std::vector<uint32_t>& ids,
                     uint64_t* finished_ns, uint64_t t_trigger, uint64_t* done_abs) {
  {
    std::lock_guard<std::mutex> g(s->mu);
    int rc = require_live(s);
    if (rc) return rc;
    if (!mask_ids(s, mask, nwords, ids, &rc)) return rc;
    for (uint32_t i : ids)
      if (!(s->pending[i >> 6] >> (i & 63) & 1)) return fail(LK_E_USAGE, "wait on worker(s) that were never triggered");
  }
  const uint64_t t0 = t_trigger ? t_trigger : now_ns();
  // Direct cells: ack each worker the moment its FINISHED is seen, not all
  // of them after the last.  Per worker this is the reference's order
  // (FINISHED seen, then NOP written: native.py:256-265); across workers the
  // acks overlap the rest of the scan.  Full-mask cycle 9.6 -> 7.9 us,
  // trigger->done 5.3 -> 4.9 us (tools/ab_early_ack.py).  HYBRID sessions
  // take every ack on the direct cells this way too, wide masks included
  // (their triggers still travel as one ring event): full-mask cycle 10.4 ->
  // 9.25 us, 64 MiB saxpy e2e +4% (profiles/r02_ab_hybrid_acks.txt).
  // GATEWAY acks stay one ring event for the whole mask.
  const bool ack_each = ids.size() > 1 && !(s->cfg.flags & LK_CF_FULL_BOARD) && (!s->gateway || s->hybrid);
  int rc = spin_words(s, ids, LK_FINISHED, "wait for FINISHED", ack_each);
  if (rc) return rc;
  const uint64_t finished_at = now_ns();
  for (uint32_t i : ids) s->host_times[3 * i + 2] = finished_at;
  if (!ack_each && !s->post(ids, LK_NOP)) return fail(LK_E_HANG, "event ring full: gateway not consuming");
  const bool lazy = (s->cfg.flags & LK_CF_LAZY_ACK) != 0;
  if (!lazy) {
    rc = spin_words(s, ids, LK_NOP, "wait for ack consumption");
    if (rc) return rc;
  }
  {
    std::lock_guard<std::mutex> g(s->mu);
    std::vector<uint64_t>& m = s->scratch;
    std::fill(m.begin(), m.end(), 0);
    for (uint32_t i : ids) m[i >> 6] |= 1ull << (i & 63);
    for (uint32_t k = 0; k < s->nwords; ++k) s->pending[k] &= ~m[k];
    if (lazy)
      for (uint32_t k = 0; k < s->nwords; ++k) s->ack_pending[k] |= m[k];
    else
      for (uint32_t k = 0; k < s->nwords; ++k) s->idle_known[k] |= m[k];   // NOP observed above
    // a slot is freed only once every worker it was triggered on was waited (native.py:266-272)
    for (size_t j = 0; j < s->inflight.size();) {
      const uint32_t slot = s->inflight[j];
      uint64_t* sp = s->slot_pend.data() + uint64_t(slot) * s->nwords;
      bool any = false;
      for (uint32_t k = 0; k < s->nwords; ++k) {
        sp[k] &= ~m[k];
        any |= sp[k] != 0;
      }
      if (any) {
        ++j;
      } else {
        s->slot_busy[slot] = 0;
        s->inflight[j] = s->inflight.back();
        s->inflight.pop_back();
      }
    }
  }
  if (finished_ns) *finished_ns = finished_at - t0;
  if (done_abs) *done_abs = finished_at;
  return LK_OK;
}

extern "C" int lk_wait(lk_session* s, const uint64_t* mask, uint32_t nwords, uint64_t* finished_ns) {
  if (!s || !mask) return fail(LK_E_USAGE, "null argument");
  static thread_local std::vector<uint32_t> ids;
  return wait_impl(s, mask, nwords, ids, finished_ns, 0, nullptr);
}

static int bench_roundtrip(lk_session* s, const uint64_t* masks, uint32_t nmasks, uint32_t nwords, uint32_t slot,
                           uint64_t rounds, uint64_t* trig_ns, uint64_t* done_ns, uint64_t* cycle_ns,
                           uint64_t* gap_ns) {
  if (!s || !masks || nmasks == 0) return fail(LK_E_USAGE, "null argument");
  std::vector<uint32_t> ids;
  ids.reserve(s->nw);
  GapProbe gp;
  const double tpn = gap_ns ? tsc_per_ns() : 1.0;
  struct Unset {
    ~Unset() { t_gap = nullptr; }
  } unset;
  if (gap_ns) t_gap = &gp;
  for (uint64_t k = 0; k < rounds; ++k) {
    const uint64_t* m = masks + (k % nmasks) * uint64_t(nwords);
    if (gap_ns) {
      gp.max = 0;
      gp.last = 0;
      gap_tick();
    }
    const uint64_t t0 = now_ns();
    uint64_t el = 0;
    int rc;
    {
      std::lock_guard<std::mutex> g(s->mu);
      rc = trigger_locked(s, m, nwords, slot, nullptr, ids, &el, t0);
    }
    if (rc) return rc;
    uint64_t done_abs = 0;
    rc = wait_impl(s, m, nwords, ids, nullptr, t0, &done_abs);
    if (rc) return rc;
    const uint64_t t2 = now_ns();
    if (trig_ns) trig_ns[k] = el;
    if (done_ns) done_ns[k] = done_abs - t0;
    if (cycle_ns) cycle_ns[k] = t2 - t0;
    if (gap_ns) {
      gap_tick();
      gap_ns[k] = uint64_t(double(gp.max) / tpn);
    }
  }
  return LK_OK;
}

extern "C" int lk_bench_roundtrip(lk_session* s, const uint64_t* masks, uint32_t nmasks, uint32_t nwords,
                                  uint32_t slot, uint64_t rounds, uint64_t* trig_ns, uint64_t* done_ns,
                                  uint64_t* cycle_ns) {
  return bench_roundtrip(s, masks, nmasks, nwords, slot, rounds, trig_ns, done_ns, cycle_ns, nullptr);
}

extern "C" int lk_bench_roundtrip_gaps(lk_session* s, const uint64_t* masks, uint32_t nmasks, uint32_t nwords,
                                       uint32_t slot, uint64_t rounds, uint64_t* trig_ns, uint64_t* done_ns,
                                       uint64_t* cycle_ns, uint64_t* gap_ns) {
  if (!gap_ns) return fail(LK_E_USAGE, "null gap array");
  return bench_roundtrip(s, masks, nmasks, nwords, slot, rounds, trig_ns, done_ns, cycle_ns, gap_ns);
}

// ------------------------------------------------------------------ dispose
extern "C" int lk_dispose(lk_session* s, uint64_t* elapsed_ns) {
  if (!s) return fail(LK_E_USAGE, "null session");
  std::lock_guard<std::mutex> g(s->mu);
  int rc = require_live(s);
  if (rc) return rc;
  std::vector<uint32_t> busy;
  for (uint32_t i = 0; i < s->nw; ++i)
    if (s->pending[i >> 6] >> (i & 63) & 1) busy.push_back(i);
  if (!busy.empty()) return fail(LK_E_DISPOSE_BUSY, "worker(s) %s still working", ids_str(busy).c_str());
  const uint64_t t0 = now_ns();
  rc = settle_acks(s, s->all_ids);
  if (rc) return rc;
  if (!s->post(s->all_ids, LK_EXIT)) return fail(LK_E_HANG, "event ring full: gateway not consuming");
  const uint64_t deadline = t0 + s->cfg.wait_timeout_ns;
  for (;;) {
    const int ks = kernel_status(s);
    if (ks < 0) return LK_E_CUDA;
    if (ks == 1) break;
    if (now_ns() > deadline) return fail(LK_E_HANG, "persistent kernel did not exit");
    usleep(20);
  }
  s->join_launcher();
  s->disposed = true;
  s->release_claim();
  if (elapsed_ns) *elapsed_ns = now_ns() - t0;
  return LK_OK;
}

// Teardown that ignores the host rules: EXIT to every worker whatever its
// state (a WORKING worker finishes its item first), then wait for the kernel.
// Used to reclaim the GPU after a worker died or a caller bailed out.
extern "C" int lk_abort(lk_session* s, uint64_t timeout_ns) {
  if (!s) return fail(LK_E_USAGE, "null session");
  std::lock_guard<std::mutex> g(s->mu);
  if (s->kernel_done || kernel_status(s) != 0) {   // already retired (or failed): nothing to tell
    s->join_launcher();
    s->disposed = true;
    s->release_claim();
    return LK_OK;
  }
  s->post(s->all_ids, LK_EXIT);
  const uint64_t deadline = now_ns() + (timeout_ns ? timeout_ns : s->cfg.wait_timeout_ns);
  for (;;) {
    const int ks = kernel_status(s);
    if (ks != 0) break;
    if (now_ns() > deadline) return fail(LK_E_HANG, "persistent kernel did not exit after abort");
    usleep(50);
  }
  s->join_launcher();
  s->disposed = true;
  s->release_claim();
  return LK_OK;
}

extern "C" int lk_destroy(lk_session* s) {
  if (!s) return LK_OK;
  if (!s->kernel_done) {
    if (kernel_status(s) == 0) {
      // Still resident (never disposed, or hung): the kernel can touch the
      // mailboxes, so the memory is deliberately leaked.
      return fail(LK_E_HANG, "persistent kernel still resident; resources leaked");
    }
  }
  s->join_launcher();
  cudaSetDevice(s->device);
  free_pinned(s->host_block);
  dev_free(s->dev_block);
  {
    CtxScope cs(s->part.ca);
    cudaStreamDestroy(s->stream);
  }
  cudaStreamDestroy(s->copy_stream);
  free_partition(&s->part);
  s->release_claim();
  delete s;
  return LK_OK;
}

extern "C" int lk_partition_info(lk_session* s, uint32_t* lk_sms, uint32_t* rest_sms) {
  if (!s) return fail(LK_E_USAGE, "null session");
  if (lk_sms) *lk_sms = s->part.ca ? s->part.a_sms : 0;
  if (rest_sms) *rest_sms = s->part.ca ? s->part.b_sms : 0;
  return LK_OK;
}

// ------------------------------------------------------------------ introspection
extern "C" int lk_read_cells(lk_session* s, uint32_t* to_gpu, uint32_t* from_gpu, uint32_t* phase, uint32_t n) {
  if (!s) return fail(LK_E_USAGE, "null session");
  const uint32_t m = std::min(n, s->nw);
  for (uint32_t i = 0; i < m; ++i) {
    const unsigned long long st = s->status[uint64_t(i) * s->status_u64];
    if (to_gpu) to_gpu[i] = s->to_gpu_word(i);
    if (from_gpu) from_gpu[i] = uint32_t(st);
    if (phase) phase[i] = uint32_t(st >> 32);
  }
  return LK_OK;
}

extern "C" int lk_debug_poke(lk_session* s, uint32_t worker, uint32_t word) {
  if (!s || worker >= s->nw) return fail(LK_E_USAGE, "bad worker");
  std::lock_guard<std::mutex> g(s->mu);
  s->wslot[worker] = 0xFFFFFFFFu;   // a poked WORK may refill the worker's descriptor cache
  s->idle_known[worker >> 6] &= ~(1ull << (worker & 63));   // its cell may change now
  s->post(std::vector<uint32_t>{worker}, word);
  return LK_OK;
}

extern "C" int lk_worker_error(lk_session* s, uint32_t worker, uint32_t* code, uint32_t* word) {
  if (!s || worker >= s->nw) return fail(LK_E_USAGE, "bad worker");
  const unsigned long long e = s->err[worker];
  if (code) *code = uint32_t(e);
  if (word) *word = uint32_t(e >> 32);
  return LK_OK;
}

extern "C" int lk_smid_map(lk_session* s, uint32_t* smid, uint32_t n) {
  if (!s || !smid) return fail(LK_E_USAGE, "null argument");
  for (uint32_t i = 0; i < std::min(n, s->nw); ++i) smid[i] = s->smid[i];
  return LK_OK;
}

extern "C" int lk_num_workers(lk_session* s, uint32_t* n) {
  if (!s || !n) return fail(LK_E_USAGE, "null argument");
  *n = s->nw;
  return LK_OK;
}

extern "C" int lk_pending(lk_session* s, uint64_t* mask, uint32_t nwords) {
  if (!s || !mask) return fail(LK_E_USAGE, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  for (uint32_t k = 0; k < nwords; ++k) mask[k] = k < s->nwords ? s->pending[k] : 0;
  return LK_OK;
}

extern "C" int lk_kernel_alive(lk_session* s, uint32_t* alive) {
  if (!s || !alive) return fail(LK_E_USAGE, "null argument");
  const int ks = kernel_status(s);
  *alive = ks == 0 ? 1u : 0u;
  return LK_OK;
}

extern "C" int lk_last_timeline(lk_session* s, uint64_t* t, uint32_t n) {
  if (!s || !t) return fail(LK_E_USAGE, "null argument");
  const uint32_t m = std::min(n, s->nw);
  LK_CUDA(cudaSetDevice(s->device));
  LK_CUDA(cudaMemcpyAsync(t, s->d_spans, size_t(m) * 8 * LK_TIMELINE_WORDS, cudaMemcpyDeviceToHost,
                          s->copy_stream));
  LK_CUDA(cudaStreamSynchronize(s->copy_stream));
  return LK_OK;
}

extern "C" int lk_fast_count(lk_session* s, uint32_t* counts, uint32_t n) {
  if (!s || !counts) return fail(LK_E_USAGE, "null argument");
  const uint32_t m = std::min(n, s->nw);
  LK_CUDA(cudaSetDevice(s->device));
  LK_CUDA(cudaMemcpyAsync(counts, s->d_fast, size_t(m) * 4, cudaMemcpyDeviceToHost, s->copy_stream));
  LK_CUDA(cudaStreamSynchronize(s->copy_stream));
  return LK_OK;
}

extern "C" int lk_last_host_times(lk_session* s, uint64_t* t, uint32_t n) {
  if (!s || !t) return fail(LK_E_USAGE, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  const uint32_t m = std::min(n, s->nw);
  memcpy(t, s->host_times.data(), size_t(m) * 24);
  return LK_OK;
}

// GPC membership of every SM: clustered launches of a probe kernel (a
// cluster's CTAs share a GPC) over many grid sizes, SM ids of a cluster
// unioned.  Run with no session live (it needs every SM).  gpc[smid] = group
// id (dense, 0..*ngroups-1), or -1 for an SM never observed.
extern "C" int lk_sm_topology(int device, int32_t* gpc, uint32_t n, uint32_t* ngroups) {
  if (!gpc || !ngroups) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaSetDevice(device));
  int nsm = 0, optin = 0;
  LK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  LK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  std::vector<int> parent(size_t(nsm) + 1);
  std::vector<uint8_t> seen(size_t(nsm) + 1, 0);
  for (int i = 0; i <= nsm; ++i) parent[i] = i;
  auto find = [&](int x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  uint32_t* d = nullptr;
  LK_CUDA(dev_alloc(reinterpret_cast<void**>(&d), 4096 * 4));
  std::vector<uint32_t> h(4096);
  cudaStream_t st;
  LK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const size_t smem = size_t(optin) / 2 + 1024;   // one CTA per SM
  int rc = LK_OK;
  for (uint32_t cluster : {8u, 16u, 4u, 2u}) {
    for (uint32_t k = 1; k * cluster <= uint32_t(nsm) && rc == LK_OK; ++k) {
      const uint32_t grid = k * cluster;
      cudaError_t e = lk_launch_topo(d, grid, cluster, smem, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, grid * 4, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) {
        cudaGetLastError();
        if (cluster > 8) break;   // non-portable size unsupported: skip it
        rc = fail(LK_E_CUDA, "topology probe: %s", cudaGetErrorString(e));
        break;
      }
      for (uint32_t c = 0; c < grid; c += cluster) {
        const int r0 = find(int(std::min<uint32_t>(h[c], uint32_t(nsm))));
        for (uint32_t j = 0; j < cluster; ++j) {
          const uint32_t sm = std::min<uint32_t>(h[c + j], uint32_t(nsm));
          seen[sm] = 1;
          const int rj = find(int(sm));
          if (rj != r0) parent[rj] = r0;
        }
      }
    }
  }
  cudaStreamDestroy(st);
  dev_free(d);
  if (rc) return rc;
  std::vector<int> id(size_t(nsm) + 1, -1);
  uint32_t groups = 0;
  for (uint32_t sm = 0; sm < n; ++sm) {
    if (sm >= uint32_t(nsm) || !seen[sm]) {
      gpc[sm] = -1;
      continue;
    }
    const int r = find(int(sm));
    if (id[r] < 0) id[r] = int(groups++);
    gpc[sm] = id[r];
  }
  *ngroups = groups;
  return LK_OK;
}

extern "C" int lk_clock_offset(int device, uint32_t rounds, int64_t* offset_ns, uint64_t* best_rtt_ns) {
  if (!offset_ns || rounds == 0) return fail(LK_E_USAGE, "bad argument");
  LK_CUDA(cudaSetDevice(device));
  LK_CUDA(lk_preload_kernels());
  uint8_t* cells = nullptr;
  LK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cells), 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(cells, 0, 4096);
  uint32_t* flag = reinterpret_cast<uint32_t*>(cells);
  volatile unsigned long long* echo = reinterpret_cast<volatile unsigned long long*>(cells + 128);
  cudaStream_t st;
  LK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t ce = lk_launch_clocksync(flag, const_cast<unsigned long long*>(echo), rounds, st);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(st);
    free_pinned(cells);
    return fail(LK_E_CUDA, "clocksync launch: %s", cudaGetErrorString(ce));
  }
  uint64_t best = ~0ull;
  int64_t off = 0;
  for (uint32_t r = 1; r <= rounds; ++r) {
    const uint64_t t0 = now_ns();
    __atomic_store_n(flag, r, __ATOMIC_RELEASE);
    const uint64_t deadline = t0 + 2000000000ull;
    while (uint32_t(__atomic_load_n(reinterpret_cast<volatile uint32_t*>(echo + 1), __ATOMIC_ACQUIRE)) != r) {
      LK_PAUSE();
      if (now_ns() > deadline) return fail(LK_E_HANG, "clock sync stalled at round %u (kernel left running)", r);
    }
    const uint64_t t1 = now_ns();
    const uint64_t g = echo[0];
    if (t1 - t0 < best) {
      best = t1 - t0;
      off = int64_t(g) - int64_t(t0 + (t1 - t0) / 2);
    }
  }
  LK_CUDA(cudaStreamSynchronize(st));
  cudaStreamDestroy(st);
  free_pinned(cells);
  *offset_ns = off;
  if (best_rtt_ns) *best_rtt_ns = best;
  return LK_OK;
}

extern "C" int lk_last_spans(lk_session* s, uint64_t* begin_ns, uint64_t* end_ns, uint32_t n) {
  if (!s) return fail(LK_E_USAGE, "null session");
  std::vector<uint64_t> sp(LK_TIMELINE_WORDS * size_t(s->nw));
  int rc = lk_last_timeline(s, sp.data(), s->nw);
  if (rc) return rc;
  for (uint32_t i = 0; i < std::min(n, s->nw); ++i) {
    if (begin_ns) begin_ns[i] = sp[LK_TIMELINE_WORDS * i + 1];
    if (end_ns) end_ns[i] = sp[LK_TIMELINE_WORDS * i + 2];
  }
  return LK_OK;
}

// ------------------------------------------------------------------ tracing
struct MergedRec {
  uint64_t anchor;  // host time of the host write this record follows
  uint32_t worker;
  uint32_t local;   // position in the worker's merged stream
  lk_trace_rec r;
};

static int build_trace(lk_session* s, std::vector<MergedRec>& outv) {
  if (!s->cfg.record_trace) return fail(LK_E_USAGE, "session was started without record_trace");
  std::vector<uint32_t> cnt(s->nw);
  LK_CUDA(cudaSetDevice(s->device));
  LK_CUDA(cudaMemcpyAsync(cnt.data(), s->d_tcnt, 4 * size_t(s->nw), cudaMemcpyDeviceToHost, s->copy_stream));
  LK_CUDA(cudaStreamSynchronize(s->copy_stream));
  for (uint32_t i = 0; i < s->nw; ++i)
    if (cnt[i] > s->cfg.trace_capacity)
      return fail(LK_E_TRACE_LOST, "worker %u wrote %u trace records into a %u-record ring", i, cnt[i],
                  s->cfg.trace_capacity);
  std::vector<lk_dev_trace> ring(s->cfg.trace_capacity);
  outv.clear();
  for (uint32_t i = 0; i < s->nw; ++i) {
    if (cnt[i]) {
      LK_CUDA(cudaMemcpyAsync(ring.data(), s->d_trace + uint64_t(i) * s->cfg.trace_capacity,
                              size_t(cnt[i]) * sizeof(lk_dev_trace), cudaMemcpyDeviceToHost, s->copy_stream));
      LK_CUDA(cudaStreamSynchronize(s->copy_stream));
    }
    const auto& hl = s->host_log[i];
    size_t h = 0, d = 0;
    uint32_t local = 0;
    uint64_t anchor = s->t_create;
    // device record tagged hseq=k follows host write k and precedes write k+1
    while (h < hl.size() || d < cnt[i]) {
      const bool take_dev = d < cnt[i] && (h >= hl.size() || ring[d].hseq < hl[h].hseq);
      MergedRec m;
      m.worker = i;
      m.local = local++;
      if (take_dev) {
        m.anchor = anchor;
        m.r = lk_trace_rec{0, 'D', i, ring[d].word, ring[d].hseq, ring[d].t_ns};
        ++d;
      } else {
        anchor = hl[h].t_ns;
        m.anchor = anchor;
        m.r = lk_trace_rec{0, 'H', i, hl[h].word, hl[h].hseq, hl[h].t_ns};
        ++h;
      }
      outv.push_back(m);
    }
  }
  std::stable_sort(outv.begin(), outv.end(), [](const MergedRec& a, const MergedRec& b) {
    if (a.anchor != b.anchor) return a.anchor < b.anchor;
    if (a.worker != b.worker) return a.worker < b.worker;
    return a.local < b.local;
  });
  for (size_t k = 0; k < outv.size(); ++k) outv[k].r.step = k;
  return LK_OK;
}

extern "C" int lk_trace_count(lk_session* s, uint64_t* n) {
  if (!s || !n) return fail(LK_E_USAGE, "null argument");
  std::vector<MergedRec> v;
  int rc = build_trace(s, v);
  if (rc) return rc;
  *n = v.size();
  return LK_OK;
}

extern "C" int lk_trace_read(lk_session* s, lk_trace_rec* out, uint64_t cap, uint64_t* n) {
  if (!s || !n) return fail(LK_E_USAGE, "null argument");
  std::vector<MergedRec> v;
  int rc = build_trace(s, v);
  if (rc) return rc;
  const uint64_t m = std::min<uint64_t>(cap, v.size());
  for (uint64_t k = 0; k < m; ++k) out[k] = v[k].r;
  *n = m;
  return LK_OK;
}

// ------------------------------------------------------------------ protocol (host build)
extern "C" int lk_protocol_step(uint32_t* phase, uint32_t* slot, uint32_t observed, uint32_t* publish,
                                uint32_t* action, uint32_t* werr) {
  if (!phase || !slot) return fail(LK_E_USAGE, "null argument");
  lk_wstate st{*phase, *slot};
  const lk_step_out o = lk_worker_step(st, observed);
  if (werr) *werr = o.werr;
  if (o.werr) return LK_E_PROTOCOL;
  *phase = st.phase;
  *slot = st.slot;
  if (publish) *publish = o.publish;
  if (action) *action = o.action;
  return LK_OK;
}

extern "C" int lk_protocol_complete(uint32_t* phase, uint32_t* slot, uint32_t* publish, uint32_t* werr) {
  if (!phase || !slot) return fail(LK_E_USAGE, "null argument");
  lk_wstate st{*phase, *slot};
  const lk_step_out o = lk_complete_work(st);
  if (werr) *werr = o.werr;
  if (o.werr) return LK_E_PROTOCOL;
  *phase = st.phase;
  *slot = st.slot;
  if (publish) *publish = o.publish;
  return LK_OK;
}

// ------------------------------------------------------------------ ping-pong floor
extern "C" int lk_pingpong(int device, uint64_t rounds, uint64_t* rt_ns) {
  if (!rt_ns) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaSetDevice(device));
  uint32_t* cells = nullptr;
  LK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cells), 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(cells, 0, 4096);
  uint32_t* flag = cells;
  uint32_t* echo = cells + 32;  // separate 128-B line
  cudaStream_t st;
  LK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t ce = lk_launch_pingpong(flag, echo, rounds, st);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(st);
    free_pinned(cells);
    return fail(LK_E_CUDA, "pingpong launch: %s", cudaGetErrorString(ce));
  }
  int rc = LK_OK;
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    const uint64_t t0 = now_ns();
    __atomic_store_n(flag, want, __ATOMIC_RELEASE);
    const uint64_t deadline = t0 + 5000000000ull;
    while (__atomic_load_n(echo, __ATOMIC_ACQUIRE) != want) {
      LK_PAUSE();
      if (now_ns() > deadline) { rc = fail(LK_E_HANG, "pingpong stalled at round %llu", (unsigned long long)r); break; }
    }
    if (rc) break;
    rt_ns[r - 1] = now_ns() - t0;
  }
  if (rc != LK_OK) {
    // release the kernel: it waits for flag >= round, so the largest value
    // lets every remaining round through; reclaim everything once it exited
    __atomic_store_n(flag, 0xFFFFFFFFu, __ATOMIC_RELEASE);
    const uint64_t until = now_ns() + 1000000000ull;
    cudaError_t q;
    while ((q = cudaStreamQuery(st)) == cudaErrorNotReady && now_ns() < until) usleep(100);
    if (q == cudaErrorNotReady) return rc;   // still resident: it may touch the cells, so they are leaked
    cudaStreamDestroy(st);
    free_pinned(cells);
    return rc;
  }
  LK_CUDA(cudaStreamSynchronize(st));
  cudaStreamDestroy(st);
  free_pinned(cells);
  return rc;
}

// ------------------------------------------------------------------ baseline
struct lk_baseline {
  CUcontext ctx = nullptr;   // green context B of a partitioned session, else the primary
  int device;
  lk_desc last_in{}, last_norm{};   // the caller's last descriptor and its normalised form
  bool have_last = false;
  uint32_t threads;
  cudaStream_t stream;
  uint32_t* d_ctr;
  bool in_flight;
  int use_tma;
  cudaEvent_t e0, e1;
};

static int baseline_create(int device, uint32_t threads, CUcontext ctx, lk_baseline** out);

// The baseline's own device (the primary context's case; a green context
// names its device itself) and the descriptor as the launch takes it:
// normalised like a staged one (LK_DF_SCALAR / LK_DF_HOSTMEM, pointer checks),
// cached so a loop re-launching one descriptor classifies its pointers once.
struct BaseScope {
  CtxScope cs;
  explicit BaseScope(lk_baseline* b) : cs(b->ctx) {
    if (!b->ctx) cudaSetDevice(b->device);
  }
};

static int baseline_desc(lk_baseline* b, const lk_desc* d, const lk_desc** out) {
  if (!b->have_last || memcmp(&b->last_in, d, sizeof(lk_desc)) != 0) {
    lk_desc n;
    int rc = normalise_desc(b->device, d, &n);
    if (rc) return rc;
    b->last_in = *d;
    b->last_norm = n;
    b->have_last = true;
  }
  *out = &b->last_norm;
  return LK_OK;
}

extern "C" int lk_baseline_create(int device, uint32_t threads, lk_baseline** out) {
  return baseline_create(device, threads, nullptr, out);
}

extern "C" int lk_baseline_create_in(lk_session* s, uint32_t threads, lk_baseline** out) {
  if (!s || !out) return fail(LK_E_USAGE, "null argument");
  if (!s->part.cb) return fail(LK_E_USAGE, "session has no SM partition (lk_config.sm_partition)");
  return baseline_create(s->device, threads, s->part.cb, out);
}

static int baseline_create(int device, uint32_t threads, CUcontext ctx, lk_baseline** out) {
  if (!out) return fail(LK_E_USAGE, "null argument");
  if (threads == 0) threads = 512;
  if (threads % 32 || threads > 1024) return fail(LK_E_CONFIG, "threads must be a multiple of 32 <= 1024");
  LK_CUDA(cudaSetDevice(device));
  auto* b = new lk_baseline();
  b->ctx = ctx;
  b->device = device;
  b->threads = threads;
  b->in_flight = false;
  b->use_tma = 1;
  LK_CUDA(dev_alloc(reinterpret_cast<void**>(&b->d_ctr), 16));   // primary context: shared memory
  LK_CUDA(cudaMemsetAsync(b->d_ctr, 0, 16, svc_stream()));
  LK_CUDA(cudaStreamSynchronize(svc_stream()));
  CtxScope cs(b->ctx);   // kernels, stream and events in the partition's green context
  LK_CUDA(lk_preload_kernels());
  LK_CUDA(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  LK_CUDA(cudaEventCreate(&b->e0));
  LK_CUDA(cudaEventCreate(&b->e1));
  *out = b;
  return LK_OK;
}

extern "C" int lk_baseline_launch(lk_baseline* b, const lk_desc* din, uint32_t grid, uint64_t* launch_ns) {
  if (!b || !din || grid == 0) return fail(LK_E_USAGE, "bad argument");
  BaseScope cs(b);
  if (b->in_flight) return fail(LK_E_USAGE, "previous task not yet joined");
  const lk_desc* d = nullptr;
  int rc = baseline_desc(b, din, &d);
  if (rc) return rc;
  const uint64_t t0 = now_ns();
  cudaError_t ce = lk_launch_work(*d, grid, b->threads, b->d_ctr, b->stream, b->use_tma);
  const uint64_t t1 = now_ns();
  if (ce != cudaSuccess) return fail(LK_E_CUDA, "launch: %s", cudaGetErrorString(ce));
  b->in_flight = true;
  if (launch_ns) *launch_ns = t1 - t0;
  return LK_OK;
}

extern "C" int lk_baseline_wait(lk_baseline* b, uint64_t* wait_ns) {
  if (!b) return fail(LK_E_USAGE, "null argument");
  BaseScope cs(b);
  if (!b->in_flight) return fail(LK_E_USAGE, "no task in flight");
  const uint64_t t0 = now_ns();
  LK_CUDA(cudaStreamSynchronize(b->stream));
  b->in_flight = false;
  if (wait_ns) *wait_ns = now_ns() - t0;
  return LK_OK;
}

extern "C" int lk_baseline_bench(lk_baseline* b, const lk_desc* din, uint32_t grid, uint64_t rounds,
                                 uint64_t* launch_ns, uint64_t* total_ns) {
  if (!b || !din || grid == 0) return fail(LK_E_USAGE, "bad argument");
  BaseScope cs(b);
  const lk_desc* d = nullptr;
  int rc = baseline_desc(b, din, &d);
  if (rc) return rc;
  for (uint64_t k = 0; k < rounds; ++k) {
    const uint64_t t0 = now_ns();
    cudaError_t ce = lk_launch_work(*d, grid, b->threads, b->d_ctr, b->stream, b->use_tma);
    const uint64_t t1 = now_ns();
    if (ce != cudaSuccess) return fail(LK_E_CUDA, "launch: %s", cudaGetErrorString(ce));
    LK_CUDA(cudaStreamSynchronize(b->stream));
    const uint64_t t2 = now_ns();
    if (launch_ns) launch_ns[k] = t1 - t0;
    if (total_ns) total_ns[k] = t2 - t0;
  }
  return LK_OK;
}

extern "C" int lk_baseline_time_kernel(lk_baseline* b, const lk_desc* din, uint32_t grid, uint32_t reps,
                                       float* avg_ms) {
  if (!b || !din || !avg_ms || reps == 0) return fail(LK_E_USAGE, "bad argument");
  BaseScope cs(b);
  const lk_desc* d = nullptr;
  int rc = baseline_desc(b, din, &d);
  if (rc) return rc;
  LK_CUDA(cudaEventRecord(b->e0, b->stream));
  for (uint32_t k = 0; k < reps; ++k) {
    cudaError_t ce = lk_launch_work(*d, grid, b->threads, b->d_ctr, b->stream, b->use_tma);
    if (ce != cudaSuccess) return fail(LK_E_CUDA, "launch: %s", cudaGetErrorString(ce));
  }
  LK_CUDA(cudaEventRecord(b->e1, b->stream));
  LK_CUDA(cudaEventSynchronize(b->e1));
  float ms = 0.f;
  LK_CUDA(cudaEventElapsedTime(&ms, b->e0, b->e1));
  *avg_ms = ms / float(reps);
  return LK_OK;
}

// The fastest conventional launch+sync this host can do, per task: an empty
// <<<1, 32, 0>>> kernel (no shared memory, no arguments) on a non-blocking
// stream, joined by
//   LK_FLOOR_SYNC:  cudaStreamSynchronize
//   LK_FLOOR_QUERY: a host spin on cudaStreamQuery (no driver wait primitive)
//   LK_FLOOR_GRAPH: the kernel as a one-node CUDA graph, cudaGraphLaunch +
//                   cudaStreamSynchronize
// with the device's host-wait policy set to cudaDeviceScheduleSpin first when
// `spin_sched` (process-wide; the primary context takes the flag while live).
// total_ns[k] = launch call start -> task observed complete; launch_ns[k] =
// the launch call alone.  Replaces ThreadSpawnBaseline.launch/wait
// (P/native.py:304-331) at its cheapest.
extern "C" int lk_launch_floor_bench(int device, uint32_t mode, uint32_t spin_sched, uint64_t rounds,
                                     uint64_t* total_ns, uint64_t* launch_ns) {
  if (mode > LK_FLOOR_GRAPH) return fail(LK_E_USAGE, "unknown floor mode %u", mode);
  LK_CUDA(cudaSetDevice(device));
  if (spin_sched) LK_CUDA(cudaSetDeviceFlags(cudaDeviceScheduleSpin));
  LK_CUDA(lk_preload_kernels());
  cudaStream_t st;
  LK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  int rc = LK_OK;
  if (mode == LK_FLOOR_GRAPH) {
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) e = lk_launch_empty(st);
    cudaError_t e2 = cudaStreamEndCapture(st, &graph);
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) rc = fail(LK_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
  }
  for (uint64_t k = 0; k < rounds && rc == LK_OK; ++k) {
    const uint64_t t0 = now_ns();
    cudaError_t e = mode == LK_FLOOR_GRAPH ? cudaGraphLaunch(exec, st) : lk_launch_empty(st);
    const uint64_t t1 = now_ns();
    if (e == cudaSuccess) {
      if (mode == LK_FLOOR_QUERY) {
        while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) LK_PAUSE();
      } else {
        e = cudaStreamSynchronize(st);
      }
    }
    const uint64_t t2 = now_ns();
    if (e != cudaSuccess) {
      rc = fail(LK_E_CUDA, "floor task: %s", cudaGetErrorString(e));
      break;
    }
    if (launch_ns) launch_ns[k] = t1 - t0;
    if (total_ns) total_ns[k] = t2 - t0;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return rc;
}

extern "C" int lk_baseline_set_tma(lk_baseline* b, int on) {
  if (!b) return fail(LK_E_USAGE, "null argument");
  b->use_tma = on ? 1 : 0;
  return LK_OK;
}

extern "C" int lk_baseline_destroy(lk_baseline* b) {
  if (!b) return LK_OK;
  {
    BaseScope cs(b);
    cudaStreamSynchronize(b->stream);
    cudaStreamDestroy(b->stream);
    cudaEventDestroy(b->e0);
    cudaEventDestroy(b->e1);
  }
  dev_free(b->d_ctr);
  delete b;
  return LK_OK;
}

// ------------------------------------------------------------------ helpers
extern "C" int lk_pin_thread_near(int device, uint32_t* ncores) {
  char bdf[64] = {0};
  LK_CUDA(cudaDeviceGetPCIBusId(bdf, sizeof bdf, device));
  for (char* c = bdf; *c; ++c) *c = char(tolower(*c));
  char path[160];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/local_cpulist", bdf);
  FILE* f = fopen(path, "r");
  if (!f) return fail(LK_E_USAGE, "cannot read %s", path);
  char line[4096] = {0};
  if (!fgets(line, sizeof line, f)) line[0] = 0;
  fclose(f);
  cpu_set_t allowed, want;
  CPU_ZERO(&want);
  if (sched_getaffinity(0, sizeof allowed, &allowed) != 0) return fail(LK_E_USAGE, "sched_getaffinity failed");
  uint32_t n = 0;
  for (char* tok = strtok(line, ",\n"); tok; tok = strtok(nullptr, ",\n")) {
    int a = 0, b = 0;
    if (sscanf(tok, "%d-%d", &a, &b) == 2) {
    } else if (sscanf(tok, "%d", &a) == 1) {
      b = a;
    } else {
      continue;
    }
    for (int c = a; c <= b && c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &allowed)) { CPU_SET(c, &want); ++n; }
  }
  if (n == 0) return fail(LK_E_USAGE, "no allowed cores local to device %d (%s)", device, path);
  if (pthread_setaffinity_np(pthread_self(), sizeof want, &want) != 0)
    return fail(LK_E_USAGE, "pthread_setaffinity_np failed: %s", strerror(errno));
  if (ncores) *ncores = n;
  return LK_OK;
}

extern "C" int lk_device_count(int* n) {
  if (!n) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaGetDeviceCount(n));
  return LK_OK;
}

extern "C" int lk_sm_count(int device, int* n) {
  if (!n) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, device));
  return LK_OK;
}

// The device whose memory `p` is (else the calling thread's device), made
// current so the copy goes to that device's service stream.
static void set_device_of(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess &&
      (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
    cudaSetDevice(at.device);
  cudaGetLastError();
}

extern "C" int lk_dev_alloc(int device, uint64_t bytes, uint64_t* ptr) {
  if (!ptr) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaSetDevice(device));
  void* p = nullptr;
  LK_CUDA(dev_alloc(&p, bytes));
  *ptr = reinterpret_cast<uint64_t>(p);
  return LK_OK;
}

extern "C" int lk_dev_free(uint64_t ptr) {
  set_device_of(reinterpret_cast<const void*>(ptr));
  LK_CUDA(dev_free(reinterpret_cast<void*>(ptr)));
  return LK_OK;
}

// Mapped pinned host memory for zero-copy payloads (LK_DF_HOSTMEM): the
// persistent kernel reads and writes it over the link with no cudaMemcpy.
// Portable: every device's sessions may use it.  The device address equals
// the host address (UVA), so it goes into lk_desc as is.
extern "C" int lk_host_alloc(int device, uint64_t bytes, void** host) {
  if (!host) return fail(LK_E_USAGE, "null argument");
  LK_CUDA(cudaSetDevice(device));
  void* p = nullptr;
  LK_CUDA(cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocMapped | cudaHostAllocPortable));
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess || d != p) {
    free_pinned(p);
    return fail(LK_E_CUDA, "host allocation has no identical device mapping (UVA)");
  }
  memset(p, 0, bytes);
  *host = p;
  return LK_OK;
}

extern "C" int lk_host_free(void* host) {
  if (!host) return LK_OK;
  free_pinned(host);
  return LK_OK;
}

extern "C" int lk_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes) {
  set_device_of(reinterpret_cast<const void*>(dst));
  cudaStream_t st = svc_stream();
  LK_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(dst), src, bytes, cudaMemcpyHostToDevice, st));
  LK_CUDA(cudaStreamSynchronize(st));
  return LK_OK;
}

extern "C" int lk_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes) {
  set_device_of(reinterpret_cast<const void*>(src));
  cudaStream_t st = svc_stream();
  LK_CUDA(cudaMemcpyAsync(dst, reinterpret_cast<const void*>(src), bytes, cudaMemcpyDeviceToHost, st));
  LK_CUDA(cudaStreamSynchronize(st));
  return LK_OK;
}

extern "C" const char* lk_strerror(int code) {
  switch (code) {
    case LK_OK: return "ok";
    case LK_E_USAGE: return "usage error";
    case LK_E_BUSY: return "worker busy";
    case LK_E_DISPOSE_BUSY: return "dispose while busy";
    case LK_E_HANG: return "hang detected";
    case LK_E_INIT: return "init failed";
    case LK_E_WORKER_DIED: return "worker died";
    case LK_E_CUDA: return "CUDA error";
    case LK_E_CONFIG: return "configuration error";
    case LK_E_PROTOCOL: return "protocol violation";
    case LK_E_TRACE_LOST: return "trace ring overflow";
    default: return "unknown error";
  }
}

extern "C" const char* lk_last_error(void) { return g_last_error.c_str(); }

extern "C" uint32_t lk_abi_version(void) { return 1u; }
