// lk_kernels.cu -- the sm_100a device side of the LK runtime.
//
//  * lk_persistent_kernel: one CTA per SM for the whole session (the paper's
//    persistent worker; reference loop native.py:149-199).
//    Thread 0 of each CTA is the elected worker thread: it runs the shared
//    state machine (lk_protocol.cuh) on every new to_gpu value and publishes
//    its from_gpu/status cell in pinned host memory with sys-scope stores.
//    The other worker threads park on a named barrier (no issue slots used)
//    and only wake for payload work items.
//    How to_gpu values reach thread 0 (lk_config.poll_mode):
//     - DIRECT (default): thread 0 polls its own host cell over PCIe, one
//       load in flight; after FINISHED it waits a per-worker adaptive delay
//       before polling for the ack (ack_wait), and after the closing NOP an
//       adaptive idle delay when the host re-triggers it back to back.
//     - GATEWAY: one extra warp in CTA 0 polls a ring of host events and
//       forwards each to the masked workers' mailbox lines in device memory;
//       workers poll L2.  One event reaches a full mask.
//     - HYBRID: direct cells for narrow writes, ring events for wide ones,
//       forwarded by two poller warps per CTA into shared memory.
//  * Payload work (run_multi): elementwise maps and a reduction streamed
//    through a TMA bulk-copy ring in shared memory, or 128-bit LSU loads for
//    dispatches to few workers (a lone SM streams faster that way).
//  * lk_work_kernel: the same work functions as an ordinary kernel, for the
//    cudaLaunchKernel+cudaStreamSynchronize baseline (ThreadSpawnBaseline
//    analogue, native.py:304-331).
//  * lk_pingpong_kernel: the raw host<->GPU round-trip floor.
//
// Work items are HBM-streaming element-wise maps / reductions: no tensor
// cores.  Payload loads use ld.global.cg (L2-coherent, no L1 allocation) since
// the persistent kernel re-reads buffers that DMA or other SMs rewrote between
// dispatches; 128-bit vectors, U independent loads per thread before use.
#include <cuda_runtime.h>
#include <stdint.h>
#include "lk_internal.h"
#include "lk_protocol.cuh"

namespace {

constexpr uint32_t kMaxThreads = 1024;
// Persistent CTA: up to 544 worker threads + three extra warps (channel
// pollers, gateway); the bound leaves ~96 registers per thread.
constexpr uint32_t kPersistMaxThreads = 640;
constexpr uint32_t kCmdWork = 1;
constexpr uint32_t kCmdExit = 2;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Named barrier 1 over the T worker threads of the CTA (the gateway warp of
// CTA 0 never joins it).
__device__ __forceinline__ void wsync(uint32_t T) { asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory"); }
__device__ __forceinline__ uint4 ld_cg4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_sys4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_cg1(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_cg64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// Payload load policies.  Device buffers: ld.global.cg (L2, the coherence
// point for every SM).  Host-mapped buffers (LK_DF_HOSTMEM): ld.relaxed.sys,
// which may not be served from a line the GPU cached on an earlier dispatch
// of the same buffer -- the host may have rewritten it since.
struct LdCg {
  static __device__ __forceinline__ uint4 v4(const uint4* p) { return ld_cg4(p); }
  static __device__ __forceinline__ uint32_t s1(const uint32_t* p) { return ld_cg1(p); }
};
struct LdSys {
  static __device__ __forceinline__ uint4 v4(const uint4* p) { return ld_sys4(p); }
  static __device__ __forceinline__ uint32_t s1(const uint32_t* p) { return ld_relaxed_sys(p); }
};
__device__ __forceinline__ void st4(uint4* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

// ---------------------------------------------------------------- TMA bulk ring
// Payload tiles stream HBM -> shared memory with cp.async.bulk (the TMA
// engine's 1-D bulk copy: no tensor map, no register staging), completion
// counted on an mbarrier by transaction bytes.  Up to `stages` tiles of
// kStageBytes are in flight per SM (6 x 16 KiB = 96 KiB by default: at
// ~44 GB/s per SM and a loaded HBM latency of ~1.5 us Little's law asks for
// ~66 KiB per SM; 6 measured best of 4/6/8/12, tools/ab_stages.py), issued
// by one elected thread while the other warps consume.  The ring persists
// across dispatches: `g` is the ring position (identical in every thread),
// kept modulo 2 x stages, so stage = g mod stages and the mbarrier phase
// parity = g / stages come from one compare (rp_* below).  A tile count
// would need two u32 divisions by the run-time stage count per tile (~100
// cycles each on the producer's path to the first copy) and would break
// the stage/phase mapping when it wrapped at 2^32 (2^32 mod 6 != 0).
constexpr uint32_t kStageBytes = 16384;
constexpr uint32_t kMaxStages = 12;
constexpr uint32_t kDefaultStages = 6;

__device__ __forceinline__ uint32_t rp_stage(uint32_t pos, uint32_t S) { return pos >= S ? pos - S : pos; }
__device__ __forceinline__ uint32_t rp_parity(uint32_t pos, uint32_t S) { return pos >= S ? 1u : 0u; }
__device__ __forceinline__ uint32_t rp_next(uint32_t pos, uint32_t S) { return pos + 1 == 2 * S ? 0u : pos + 1; }

struct Ring {
  uint8_t* buf;       // stages x kStageBytes, 128-B aligned, dynamic shared memory
  uint64_t* full;     // 2 x kMaxStages mbarriers: [0, stages) the shared-consumer ring (maps): 1 arrival
                      // (expect_tx) + tx bytes; [kMaxStages, +stages) the owner-warp ring (reduce)
  uint64_t* empty;    // same layout: one arrival per consumer warp (maps) / the stage's owner warp (reduce)
  uint32_t stages;    // <= kMaxStages
  uint32_t* tile;     // stages: global tile index a stage holds (dynamic schedule), shared memory
  uint32_t* gred;     // shared memory: the owner-warp ring's position, modulo 2 x stages (persists across dispatches)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "LK_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LK_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Generic-proxy writes (earlier dispatches' st.global outputs, ordered before
// this thread by the CTA barriers) made visible to the async proxy before this
// dispatch's cp.async.bulk reads: an in-place saxpy re-reads its own y.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint4 lds4(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ uint32_t ring_consumer_warps(uint32_t T) { return T >= 64 ? T / 32 - 1 : 1; }

// Called by every worker thread once, before the first dispatch.
__device__ __forceinline__ void ring_init(Ring& r, uint32_t T) {
  if (threadIdx.x == 0) {
    for (uint32_t k = 0; k < r.stages; ++k) {
      mbar_init(r.full + k, 1);
      mbar_init(r.empty + k, ring_consumer_warps(T));   // one arrival per consumer warp
      mbar_init(r.full + kMaxStages + k, 1);
      mbar_init(r.empty + kMaxStages + k, 1);           // the stage's owner warp
    }
    if (r.gred) *r.gred = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  wsync(T);
}

// Stream tiles [0, ntiles) of a chunk through the ring: thread 0 keeps up to
// kStages-1 tiles ahead; `load(i, stage_ptr, bar)` issues tile i's bulk copies
// (after arming the barrier with its byte count), `use(i, stage_ptr)` consumes
// it in every thread, and each warp releases the stage with one arrival.
// Warp 0 is the producer: its lane 0 issues every tile, running ahead until
// a stage it needs is still held, and never consumes (so a refill is never
// delayed by the producer's own share of a tile).  Warps 1.. consume;
// `use(i, stage, ci, nc)` gets the consumer's index and count.

template <class Load, class Use>
__device__ __forceinline__ void ring_stream(Ring& r, uint32_t& g, uint32_t ntiles, uint32_t T, const Load& load,
                                            const Use& use) {
  const uint32_t c0 = g, S = r.stages;
  uint32_t f = c0;                                  // the producer's position (tiles are filled in order)
  auto fill = [&](uint32_t i) {
    const uint32_t st = rp_stage(f, S);
    mbar_wait(r.empty + st, rp_parity(f, S) ^ 1u);  // previous use of this stage released
    load(i, r.buf + st * kStageBytes, r.full + st);
    f = rp_next(f, S);
  };
  const bool split = T >= 64;
  const uint32_t ci = split ? threadIdx.x - 32 : threadIdx.x, nc = split ? T - 32 : T;
  if (split && threadIdx.x < 32) {
    if (threadIdx.x == 0)
      for (uint32_t i = 0; i < ntiles; ++i) fill(i);
    g = __shfl_sync(0xffffffffu, f, 0);             // the producer's position after its last fill
  } else {
    if (!split && threadIdx.x == 0)
      for (uint32_t i = 0; i < ntiles && i < S - 1; ++i) fill(i);
    uint32_t c = c0;
    for (uint32_t i = 0; i < ntiles; ++i) {
      if (!split && threadIdx.x == 0 && i + S - 1 < ntiles) fill(i + S - 1);
      const uint32_t st = rp_stage(c, S);
      mbar_wait(r.full + st, rp_parity(c, S));
      use(i, r.buf + st * kStageBytes, ci, nc);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(r.empty + st);
      c = rp_next(c, S);
    }
    g = c;
  }
}

// ---------------------------------------------------------------- work items
// Shard [0, n) over `count` workers in 128-B (32-element) aligned chunks.
struct Part { uint64_t b, e; };
__device__ __forceinline__ Part partition(uint64_t n, uint32_t rank, uint32_t count) {
  uint64_t chunk = (n + count - 1) / count;
  chunk = (chunk + 31) & ~uint64_t(31);
  uint64_t b = min(n, uint64_t(rank) * chunk);
  return Part{b, min(n, b + chunk)};
}

struct OpAddI32 {  // int32 add with two's-complement wraparound
  __device__ __forceinline__ uint32_t s(uint32_t x, uint32_t y) const { return x + y; }
};
struct OpSaxpy {   // numpy float32: fl(fl(alpha*x) + y), no FMA contraction
  float alpha;
  __device__ __forceinline__ uint32_t s(uint32_t x, uint32_t y) const {
    return __float_as_uint(__fadd_rn(__fmul_rn(alpha, __uint_as_float(x)), __uint_as_float(y)));
  }
};
struct OpCopy {
  __device__ __forceinline__ uint32_t s(uint32_t x, uint32_t) const { return x; }
};

template <class Op>
__device__ __forceinline__ uint4 vop(const Op& op, uint4 x, uint4 y) {
  return make_uint4(op.s(x.x, y.x), op.s(x.y, y.y), op.s(x.z, y.z), op.s(x.w, y.w));
}

// out[i] = op(in0[i], in1[i]) over [p.b, p.e), all threads of the CTA (LSU path;
// Ld = LdSys for host-mapped buffers).
template <int U, bool kTwo, class Op, class Ld = LdCg>
__device__ __forceinline__ void map_chunk(const lk_desc& d, Part p, const Op& op, uint32_t T) {
  const uint32_t t = threadIdx.x;
  const uint32_t* a = reinterpret_cast<const uint32_t*>(d.in0);
  const uint32_t* c = reinterpret_cast<const uint32_t*>(d.in1);
  uint32_t* o = reinterpret_cast<uint32_t*>(d.out);
  if (d.flags & LK_DF_SCALAR) {
    for (uint64_t i = p.b + t; i < p.e; i += T) o[i] = op.s(Ld::s1(a + i), kTwo ? Ld::s1(c + i) : 0u);
    return;
  }
  const uint4* a4 = reinterpret_cast<const uint4*>(a);
  const uint4* c4 = reinterpret_cast<const uint4*>(c);
  uint4* o4 = reinterpret_cast<uint4*>(o);
  const uint64_t vb = p.b >> 2, ve = p.e >> 2;
  uint64_t v = vb + t;
  for (; v + uint64_t(U - 1) * T < ve; v += uint64_t(U) * T) {
    uint4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = Ld::v4(a4 + v + u * T);
      if (kTwo) y[u] = Ld::v4(c4 + v + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st4(o4 + v + u * T, vop(op, x[u], kTwo ? y[u] : x[u]));
  }
  for (; v < ve; v += T) st4(o4 + v, vop(op, Ld::v4(a4 + v), kTwo ? Ld::v4(c4 + v) : make_uint4(0, 0, 0, 0)));
  for (uint64_t i = max(p.b, ve << 2) + t; i < p.e; i += T) o[i] = op.s(Ld::s1(a + i), kTwo ? Ld::s1(c + i) : 0u);
}

// map_chunk through the TMA ring: tiles of kStageBytes/2 per input (2 inputs)
// or kStageBytes (1 input); each thread reads its 16-B lanes of the tile from
// shared memory and stores the result straight to global memory.
template <bool kTwo, class Op>
__device__ __forceinline__ void map_tma(const lk_desc& d, Part p, const Op& op, uint32_t T, Ring& r,
                                        uint32_t& g) {
  const uint32_t t = threadIdx.x;
  const uint4* a4 = reinterpret_cast<const uint4*>(d.in0);
  const uint4* c4 = reinterpret_cast<const uint4*>(d.in1);
  uint4* o4 = reinterpret_cast<uint4*>(d.out);
  const uint64_t vb = p.b >> 2, ve = p.e >> 2;
  constexpr uint32_t kTileV = kTwo ? kStageBytes / 32 : kStageBytes / 16;   // uint4 per input per tile
  const uint64_t nv = ve > vb ? ve - vb : 0;
  const uint32_t ntiles = uint32_t((nv + kTileV - 1) / kTileV);
  ring_stream(
      r, g, ntiles, T,
      [&](uint32_t i, uint8_t* stage, uint64_t* bar) {
        const uint64_t v0 = vb + uint64_t(i) * kTileV;
        const uint32_t bytes = uint32_t(min(uint64_t(kTileV), ve - v0)) * 16u;
        mbar_expect_tx(bar, kTwo ? 2 * bytes : bytes);
        bulk_g2s(stage, a4 + v0, bytes, bar);
        if (kTwo) bulk_g2s(stage + kStageBytes / 2, c4 + v0, bytes, bar);
      },
      [&](uint32_t i, const uint8_t* stage, uint32_t ci, uint32_t nc) {
        const uint64_t v0 = vb + uint64_t(i) * kTileV;
        const uint32_t nvt = uint32_t(min(uint64_t(kTileV), ve - v0));
        for (uint32_t v = ci; v < nvt; v += nc) {
          const uint4 x = lds4(stage + 16 * v);
          const uint4 y = kTwo ? lds4(stage + kStageBytes / 2 + 16 * v) : x;
          st4(o4 + v0 + v, vop(op, x, y));
        }
      });
  const uint32_t* a = reinterpret_cast<const uint32_t*>(d.in0);
  const uint32_t* c = reinterpret_cast<const uint32_t*>(d.in1);
  uint32_t* o = reinterpret_cast<uint32_t*>(d.out);
  for (uint64_t i = max(p.b, ve << 2) + t; i < p.e; i += T) o[i] = op.s(ld_cg1(a + i), kTwo ? ld_cg1(c + i) : 0u);
}

constexpr uint32_t kTileEnd = 0xFFFFFFFFu;   // ring end marker (reduce_dyn)

// ---------------------------------------------------------------- block reduce
// block_reduce_f32 is defined on fixed 4096-element blocks (oracle/work.py:
// block_reduce_partials / block_reduce_combine), independent of the mask,
// the worker count, the thread count, the schedule and the payload path:
//   out[b]  = sum of block b: lane l of one warp owns the float4 vectors
//             l + 32k (k ascending) into two fp32 accumulators per component
//             (even / odd k), a_c = even + odd, lane value (a0 + a1) + (a2 + a3)
//             in fp64, then a 32-lane fp64 xor butterfly;
//   *aux    = fp64 combine of out[0, nb): virtual lane j of 512 adds
//             out[j], out[j + 512], ... in order, then a 512-lane butterfly.
// So any worker may sum any block: blocks are handed out dynamically (a
// static share per worker, the rest claimed from a pool), which absorbs
// dispatch skew and slow SMs without changing a bit of the result.
constexpr uint32_t kRedBlock = 4096;              // elements per block = one 16-KiB ring stage
constexpr uint32_t kRedVecs = kRedBlock / 4;      // float4 vectors per block
constexpr uint32_t kRedVLanes = 512;              // virtual lanes of the combine
constexpr uint32_t kRedClaim = 2;                 // blocks per pool claim
static_assert(kRedBlock * 4 == kStageBytes, "a reduce block is one ring stage");

struct ReduceSmem {
  double comb[2 * kRedVLanes];   // the combine's two butterfly buffers
  uint32_t last;
};

__device__ __forceinline__ double butterfly32(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);   // lanes l, l^o: same sum
  return v;
}

// Lane accumulators are fp32, two per component -- even k and odd k, 16
// sequential adds each (short FADD chains, no conversions) -- folded as
// a_c = even_c + odd_c, then lane value (a0 + a1) + (a2 + a3) in fp64.
struct RedAcc {
  float e[4], o[4];
};

__device__ __forceinline__ void acc4(float (&a)[4], uint4 r) {
  a[0] = __fadd_rn(a[0], __uint_as_float(r.x));
  a[1] = __fadd_rn(a[1], __uint_as_float(r.y));
  a[2] = __fadd_rn(a[2], __uint_as_float(r.z));
  a[3] = __fadd_rn(a[3], __uint_as_float(r.w));
}

__device__ __forceinline__ void acc_k(RedAcc& a, uint32_t k, uint4 r) {
  if (k & 1) acc4(a.o, r); else acc4(a.e, r);
}

// The trailing n % 4 elements belong to vector `nvt` of the last block: the
// lane's last vector (k = nvt / 32), so they are added after its loop.
template <class Ld = LdCg>
__device__ __forceinline__ void acc_tail(RedAcc& a, uint32_t nvt, const float* x, uint64_t first, uint32_t tail) {
  float* h = ((nvt >> 5) & 1) ? a.o : a.e;
  for (uint32_t c = 0; c < tail; ++c)
    h[c] = __fadd_rn(h[c], __uint_as_float(Ld::s1(reinterpret_cast<const uint32_t*>(x) + first + c)));
}

__device__ __forceinline__ double block_fold(const RedAcc& a) {
  double v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = double(__fadd_rn(a.e[c], a.o[c]));
  return butterfly32((v[0] + v[1]) + (v[2] + v[3]));
}

// A block's lane sums from a ring stage (nvt full vectors in shared memory).
__device__ __forceinline__ RedAcc block_acc_smem(const uint8_t* stage, uint32_t nvt) {
  const uint32_t lane = threadIdx.x & 31;
  RedAcc a = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  if (nvt == kRedVecs) {
#pragma unroll 4
    for (uint32_t k = 0; k < 32; k += 2) {
      const uint4 r0 = lds4(stage + 16 * (lane + 32 * k)), r1 = lds4(stage + 16 * (lane + 32 * (k + 1)));
      acc4(a.e, r0);
      acc4(a.o, r1);
    }
  } else {
    for (uint32_t k = 0; k < 32; ++k) {
      const uint32_t v = lane + 32 * k;
      if (v < nvt) acc_k(a, k, lds4(stage + 16 * v));
    }
  }
  return a;
}

// One block straight from global memory (LSU path; `vec`: 16-B aligned x).
template <class Ld = LdCg>
__device__ __forceinline__ double block_sum_global(const float* x, uint64_t b, uint64_t n, bool vec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t e0 = b * kRedBlock;
  const uint64_t ne = min(uint64_t(kRedBlock), n - e0);
  const uint32_t nvt = uint32_t(ne >> 2), tail = uint32_t(ne & 3);
  RedAcc a = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const uint32_t* xu = reinterpret_cast<const uint32_t*>(x) + e0;
  if (vec && nvt == kRedVecs) {
    const uint4* x4 = reinterpret_cast<const uint4*>(xu);
#pragma unroll
    for (uint32_t k0 = 0; k0 < 32; k0 += 8) {
      uint4 r[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) r[u] = Ld::v4(x4 + lane + 32 * (k0 + u));
#pragma unroll
      for (uint32_t u = 0; u < 8; u += 2) {
        acc4(a.e, r[u]);
        acc4(a.o, r[u + 1]);
      }
    }
  } else {
    for (uint32_t k = 0; k < 32; ++k) {
      const uint32_t v = lane + 32 * k;
      if (v >= nvt) break;
      uint4 r;
      if (vec) {
        r = Ld::v4(reinterpret_cast<const uint4*>(xu) + v);
      } else {
        r = make_uint4(Ld::s1(xu + 4 * v), Ld::s1(xu + 4 * v + 1), Ld::s1(xu + 4 * v + 2), Ld::s1(xu + 4 * v + 3));
      }
      acc_k(a, k, r);
    }
  }
  if (tail && lane == (nvt & 31)) acc_tail<Ld>(a, nvt, x, e0 + 4ull * nvt, tail);
  return block_fold(a);
}

__device__ __forceinline__ void st_f64(double* p, double v) {
  asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_cg_f64(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Arrival count and, in the last worker to arrive, the combine of every
// block partial into *aux (all T threads of that CTA).  ctr[0] = arrivals,
// ctr[1] = pool claims; the last worker resets both for the slot's next
// dispatch (no worker claims or arrives any more by then).
__device__ __forceinline__ void reduce_finish(const lk_desc& d, uint32_t count, uint32_t* ctr, ReduceSmem& sm,
                                              uint32_t T, unsigned long long* tl = nullptr) {
  const uint32_t t = threadIdx.x;
  wsync(T);                 // every block partial of this worker stored
  if (t == 0) {
    // acq_rel RMW after the barrier: releases this CTA's partial stores,
    // and the last arrival acquires every other worker's
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
    sm.last = prev == count - 1;
    if (tl) tl[15] = globaltimer();
  }
  wsync(T);
  if (!sm.last) return;
  if (!d.aux) {             // partials only: just reset the slot's counters
    if (t == 0) {
      ctr[0] = 0;
      ctr[1] = 0;
    }
    return;
  }
  const double* part = reinterpret_cast<const double*>(d.out);
  const uint64_t nb = (d.n + kRedBlock - 1) / kRedBlock;
  double* s0 = sm.comb;
  for (uint32_t j = t; j < kRedVLanes; j += T) {
    double acc = 0.0;
    uint64_t i = j;
    for (; i + 7ull * kRedVLanes < nb; i += 8ull * kRedVLanes) {   // eight loads in flight, added in order
      double v[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) v[u] = ld_cg_f64(part + i + u * kRedVLanes);
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) acc += v[u];
    }
    for (; i < nb; i += kRedVLanes) acc += ld_cg_f64(part + i);
    s0[j] = acc;
  }
  wsync(T);
  // The 512-lane butterfly in warp 0 alone: lane l holds virtual lanes
  // l + 32m (m < 16), so each level o = 256..32 pairs the same operands as
  // the shared-memory form s1[t] = s0[t] + s0[t ^ o] (t ^ o = l + 32(m ^ o/32);
  // fp addition is commutative, so both lanes of a pair get the same bits),
  // and levels 16..1 are the shuffle butterfly.  No CTA barrier: -0.25 us on
  // the last worker's combine against four barrier-separated smem levels.
  if (t < 32) {
    double v[kRedVLanes / 32];
#pragma unroll
    for (uint32_t m = 0; m < kRedVLanes / 32; ++m) v[m] = s0[t + 32 * m];
#pragma unroll
    for (uint32_t k = kRedVLanes / 64; k >= 1; k >>= 1) {
#pragma unroll
      for (uint32_t m = 0; m < kRedVLanes / 32; ++m)
        if (!(m & k)) {
          const double x = v[m] + v[m | k];
          v[m] = x;
          v[m | k] = x;
        }
    }
    const double r = butterfly32(v[0]);
    if (t == 0) st_f64(reinterpret_cast<double*>(d.aux), r);
  }
  if (t == 0) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

// Dynamic blocks through the owner-warp ring (needs stages + 1 warps).  Lane
// 0 of warp 0 produces: a static share of blocks by rank first, then pool
// claims of `claim_n` blocks, the next claim in flight while the current
// one's copies are issued; then one end marker per stage.  Warp 1 + s owns
// ring stage s: it alone waits on that stage's barriers (its own phase
// sequence, count-1 release), reads the block, releases the stage, then folds
// and stores the block sum.  Other warps sit on the closing barrier.
__device__ __forceinline__ void reduce_dyn(const lk_desc& d, uint32_t rank, uint32_t count, uint32_t* ctr,
                                           ReduceSmem& sm, uint32_t T, Ring& r, uint32_t share8,
                                           uint32_t claim_n, unsigned long long* tl = nullptr) {
  const float* x = reinterpret_cast<const float*>(d.in0);
  const uint4* x4 = reinterpret_cast<const uint4*>(d.in0);
  double* part = reinterpret_cast<double*>(d.out);
  const uint64_t nv = d.n >> 2;                                   // full vectors, all blocks
  const uint32_t tail = uint32_t(d.n & 3);
  const uint32_t nb = uint32_t((d.n + kRedBlock - 1) / kRedBlock);
  // static share: share8/8 of a fair share when every worker has >= 4
  // blocks, else whatever divides evenly; the pool is the rest
  const uint32_t fair = nb / count;
  const uint32_t share = nb >= 4 * count ? (share8 * fair) / 8 : fair;
  const uint32_t pool0 = share * count;
  const uint32_t S = r.stages;
  uint64_t* const fullr = r.full + kMaxStages;
  uint64_t* const emptyr = r.empty + kMaxStages;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    uint32_t f = *r.gred;                                          // ring position, modulo 2S
    auto fill = [&](uint32_t b) {                                  // b = block or kTileEnd
      const uint32_t st = rp_stage(f, S);
      mbar_wait(emptyr + st, rp_parity(f, S) ^ 1u);
      r.tile[st] = b;
      if (b == kTileEnd) {
        mbar_arrive(fullr + st);                                   // wake the owner, no bytes
      } else {
        const uint64_t v0 = uint64_t(b) * kRedVecs;
        const uint32_t bytes = v0 < nv ? uint32_t(min(uint64_t(kRedVecs), nv - v0)) * 16u : 0u;
        mbar_expect_tx(fullr + st, bytes);                         // 0 bytes: a tail-only block
        if (bytes) bulk_g2s(r.buf + st * kStageBytes, x4 + v0, bytes, fullr + st);
      }
      f = rp_next(f, S);
    };
    // the first claim goes out right after the first static copy (before it
    // when there is no static share): its L2 round trip overlaps the copies,
    // and the first copy does not wait behind the atomic (-0.26 us to the
    // first issue, tools/reduce_phases.py)
    uint32_t claim = nb;
    if (share == 0) claim = pool0 < nb ? atomicAdd(ctr + 1, claim_n) : nb;
    if (tl) tl[12] = globaltimer();
    for (uint32_t i = 0; i < share; ++i) {
      fill(rank * share + i);
      if (i == 0) claim = pool0 < nb ? atomicAdd(ctr + 1, claim_n) : nb;
    }
    while (pool0 + claim < nb) {
      const uint32_t b = pool0 + claim;
      const uint32_t next = b + claim_n < nb ? atomicAdd(ctr + 1, claim_n) : nb;
      for (uint32_t k = 0; k < claim_n && b + k < nb; ++k) fill(b + k);
      claim = next;
    }
    if (tl) tl[13] = globaltimer();
    for (uint32_t k = 0; k < S; ++k) fill(kTileEnd);               // every owner sees one end marker
    *r.gred = f;                                                   // read by all after the closing barrier
  } else if (warp >= 1 && warp <= S) {
    const uint32_t st = warp - 1;
    const uint32_t c0 = *r.gred, s0 = rp_stage(c0, S);
    // parity of this stage's first position at or after c0 (the next lap
    // when the stage precedes c0's); every later use is S positions on
    uint32_t par = rp_parity(c0, S) ^ (st < s0 ? 1u : 0u);
    for (bool first = st == s0;; par ^= 1u, first = false) {
      mbar_wait(fullr + st, par);
      if (tl && first && lane == 0) tl[14] = globaltimer();        // the dispatch's first stage landed
      const uint32_t b = r.tile[st];
      if (b == kTileEnd) {
        __syncwarp();
        if (lane == 0) mbar_arrive(emptyr + st);
        break;
      }
      const uint64_t v0 = uint64_t(b) * kRedVecs;
      const uint32_t nvt = v0 < nv ? uint32_t(min(uint64_t(kRedVecs), nv - v0)) : 0u;
      RedAcc acc = block_acc_smem(r.buf + st * kStageBytes, nvt);
      __syncwarp();
      if (lane == 0) mbar_arrive(emptyr + st);                      // stage read: release it first
      if (b == nb - 1 && tail && lane == (nvt & 31)) acc_tail(acc, nvt, x, nv << 2, tail);
      const double ps = block_fold(acc);
      if (lane == 0) st_f64(part + b, ps);
    }
  }
  reduce_finish(d, count, ctr, sm, T, tl);                         // (its first barrier publishes *r.gred)
}

// Static blocks, 128-bit (or scalar) loads straight from global memory: the
// narrow-dispatch and misaligned path.  Worker rank r takes the r-th
// contiguous run of blocks; its warps take the run's blocks round robin.
template <class Ld = LdCg>
__device__ __forceinline__ void reduce_static(const lk_desc& d, uint32_t rank, uint32_t count, uint32_t* ctr,
                                              ReduceSmem& sm, uint32_t T) {
  const float* x = reinterpret_cast<const float*>(d.in0);
  double* part = reinterpret_cast<double*>(d.out);
  const uint64_t nb = (d.n + kRedBlock - 1) / kRedBlock;
  const uint64_t per = (nb + count - 1) / count;
  const uint64_t b0 = min(nb, uint64_t(rank) * per), b1 = min(nb, b0 + per);
  const bool vec = !(d.flags & LK_DF_SCALAR);
  const uint32_t warp = threadIdx.x >> 5, nwarps = T >> 5;
  for (uint64_t b = b0 + warp; b < b1; b += nwarps) {
    const double p = block_sum_global<Ld>(x, b, d.n, vec);
    if ((threadIdx.x & 31) == 0) st_f64(part + b, p);
  }
  reduce_finish(d, count, ctr, sm, T);
}

// native.py:63-67 counts to `iterations`.  Each iteration here reads %clock
// (a special-register read ptxas may neither fold nor hoist) and folds it into
// a value the caller stores to global memory (a.sink, the baseline's counter
// line), so the trip count is really executed: an unused result, or one only
// stored to shared memory, lets ptxas drop the loop.  One out-of-line copy
// serves every call site -- the persistent kernel's fast and general paths
// and the baseline kernel -- so an iteration costs the same everywhere and
// LK and launch+sync run the same work in the same time (table2).  Inlined
// copies were unrolled differently per site (2x apart in time per
// iteration).
__device__ __noinline__ uint32_t busy_loop(uint64_t iterations) {
  // One PTX loop (a dependent 32-bit LCG step per iteration) so that ptxas
  // emits the same SASS wherever it is compiled.  As C++ reading %clock, the
  // two kernels' copies were unrolled and scheduled differently and an
  // iteration cost 20 cycles in the persistent kernel against 26 in
  // lk_work_kernel; S2UR's latency also varied with its neighbours
  // (tools/busy_spans.py).  The caller stores the result, so the loop runs.
  // The counter runs from the lane id to iterations + lane id (the same trip
  // count), which keeps ptxas from moving the loop onto the uniform datapath
  // in one kernel and not the other.
  uint32_t acc = 0;
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      ".reg .u64 i, e;\n\t"
      ".reg .u32 l;\n\t"
      "mov.u32 l, %%laneid;\n\t"
      "cvt.u64.u32 i, l;\n\t"
      "add.u64 e, %1, i;\n"
      "LK_BUSY_%=:\n\t"
      "setp.ge.u64 p, i, e;\n\t"
      "@p bra.uni LK_BUSY_DONE_%=;\n\t"
      "mad.lo.u32 %0, %0, 1664525, 1013904223;\n\t"
      "add.u64 i, i, 1;\n\t"
      "bra.uni LK_BUSY_%=;\n"
      "LK_BUSY_DONE_%=:\n\t"
      "}"
      : "+r"(acc)
      : "l"(iterations)
      : "memory");
  return acc;
}

__device__ __forceinline__ bool single_thread_kind(uint32_t kind) {
  return kind == LK_KIND_EMPTY || kind == LK_KIND_BUSY_LOOP;
}

// Payload work shared by both kernels; every thread of the CTA calls it.
// !ring_on (or misaligned buffers): 128-bit LSU loads; else the TMA ring.
// The ring travels by reference with a flag, never as a pointer to the
// caller's local: a pointer would pin the Ring in local memory and turn
// every field access on the per-tile path into an LDL.
__device__ __forceinline__ void run_multi(const lk_desc& d, uint32_t rank, uint32_t count,
                                          uint32_t* ctr, ReduceSmem& rs, uint32_t T, Ring& ring, bool ring_on,
                                          uint32_t& g, uint32_t red_share8 = 2, uint32_t red_claim = kRedClaim,
                                          unsigned long long* tl = nullptr) {
  const Part p = partition(d.n, rank, count);
  // host-mapped buffers go through the LSU with sys-scope loads: bulk copies
  // would read them through L2 lines an earlier dispatch may have left behind
  const bool host = (d.flags & LK_DF_HOSTMEM) != 0;
  const bool tma = ring_on && !(d.flags & (LK_DF_SCALAR | LK_DF_HOSTMEM));
  if (tma && threadIdx.x == 0) fence_proxy_async();   // the producer issues every bulk copy
  switch (d.kind) {
    case LK_KIND_VECTOR_ADD_I32:
      if (tma) map_tma<true>(d, p, OpAddI32{}, T, ring, g);
      else if (host) map_chunk<4, true, OpAddI32, LdSys>(d, p, OpAddI32{}, T);
      else map_chunk<4, true>(d, p, OpAddI32{}, T);
      break;
    case LK_KIND_SAXPY_F32:
      if (tma) map_tma<true>(d, p, OpSaxpy{d.alpha}, T, ring, g);
      else if (host) map_chunk<4, true, OpSaxpy, LdSys>(d, p, OpSaxpy{d.alpha}, T);
      else map_chunk<4, true>(d, p, OpSaxpy{d.alpha}, T);
      break;
    case LK_KIND_HBM_STREAM: {
      const uint64_t passes = d.iterations ? d.iterations : 1;
      for (uint64_t k = 0; k < passes; ++k) {
        if (tma) {
          map_tma<false>(d, p, OpCopy{}, T, ring, g);
        } else if (host) {
          map_chunk<8, false, OpCopy, LdSys>(d, p, OpCopy{}, T);
        } else {
          map_chunk<8, false>(d, p, OpCopy{}, T);
        }
      }
      break;
    }
    case LK_KIND_BLOCK_REDUCE_F32:
      if (tma && T >= 32 * (ring.stages + 1) && ring.gred != nullptr)
        reduce_dyn(d, rank, count, ctr, rs, T, ring, red_share8, red_claim, tl);
      else if (host) reduce_static<LdSys>(d, rank, count, ctr, rs, T);
      else reduce_static(d, rank, count, ctr, rs, T);
      break;
    default: break;
  }
}

// ---------------------------------------------------------------- persistent
struct Elected {           // thread 0's private protocol state
  lk_wstate st;
  uint32_t pub;            // word currently in our from_gpu cell
  uint32_t seq;            // host write index of the current to_gpu word
  uint32_t cur;            // current to_gpu word
  uint32_t hint;           // host hint bits of the current value (LK_HINT_*)
  uint32_t dseq, rseq;     // HYBRID: writes seen on the direct cell / via the event ring
  uint32_t tcnt;
  uint32_t fhits;          // values settled by fast_step (mirrored to a.fast_cnt[wid])
  uint32_t nload;          // DIRECT: cell loads issued since the ack wait began
  uint32_t cslot;          // slot of the cached descriptor (sm.cdesc), or ~0
  uint32_t ckind;          // its kind and iterations, for the cached single-thread fast path
  uint64_t citer;
  uint32_t ack_cyc;        // DIRECT, 1 replica: this worker's current ack delay (adapted, see ack_adapt)
  bool dirty;              // cur not yet stepped to a fixed point
  bool idle_pub;           // just published NOP (ack consumed): the host may trigger this worker next
  bool idle_armed;         // the idle wait ran: the next WORK's load count adapts idle_cyc
  uint32_t idle_cyc;       // DIRECT, 1 replica: this worker's current idle delay (idle_adapt)
  uint64_t t_seen;         // globaltimer when the current to_gpu value arrived
  uint64_t c_seen;         // clock64 at the same point
  uint64_t t_fwd;          // GATEWAY + LK_CF_TIMELINE: globaltimer when the gateway forwarded it
};

// One device trace record: a value-changing from_gpu write, tagged with the
// host write index it answers (P/native.py:135-140).  Both the general path
// (publish) and the fast path (fast_step) record through here.
__device__ __forceinline__ void trace_rec(const lk_dev_args& a, uint32_t wid, Elected& e, uint32_t word) {
  lk_dev_trace* r = a.trace + uint64_t(wid) * a.trace_cap + (e.tcnt % a.trace_cap);
  r->word = word;
  r->hseq = e.seq;
  r->t_ns = globaltimer();
  ++e.tcnt;
  a.trace_cnt[wid] = e.tcnt;
  __threadfence();
}

__device__ __forceinline__ void publish(const lk_dev_args& a, uint32_t wid, Elected& e, uint32_t word,
                                        bool release) {
  if (a.record_trace && word != e.pub) trace_rec(a, wid, e, word);
  const unsigned long long v = uint64_t(word) | (uint64_t(e.st.phase) << 32);
  unsigned long long* cell = a.status + uint64_t(wid) * a.status_u64;
  if (release) st_release_sys(cell, v); else st_relaxed_sys(cell, v);
  e.pub = word;
}

__device__ __forceinline__ void report_error(const lk_dev_args& a, uint32_t wid, Elected& e, uint32_t werr,
                                             uint32_t word) {
  st_relaxed_sys(a.err + wid, uint64_t(werr) | (uint64_t(word) << 32));
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.err_any), "r"(1u) : "memory");
  e.st.phase = LK_PHASE_EXITED;
  publish(a, wid, e, e.pub, true);
}

__device__ __forceinline__ unsigned long long ld_cell(const unsigned long long* p, bool acquire) {
  unsigned long long v;
  if (acquire) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// The host wrote a host-mapped payload's inputs before the WORK value that
// names it (release on the host side).  A DIRECT poll with ld.acquire.sys
// (LK_CF_ACQUIRE_POLL, the default; LDG.STRONG.SYS + CCTL.IVALL, no membar)
// is already the acquire the payload's loads are ordered behind.  A relaxed
// poll or a channel poller's value gets a sys-scope fence after it instead,
// a value forwarded by the gateway (which fenced at sys scope) a gpu-scope
// one (LK_HINT_SYSMEM only: MEMBAR.SYS costs ~1.5 us).
__device__ __forceinline__ void acquire_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// A to_gpu value is {word:32, seq:24, hint:8}; seq is the host's per-worker
// write index mod 2^24 (serial-number compare: a worker is never 2^23 writes
// behind, every write waits on its handshake) and is widened back to 32 bits
// here, so trace records carry the host's full write index.
__device__ __forceinline__ bool accept(Elected& e, unsigned long long c, bool timeline, bool acquired = false,
                                       bool via_gateway = false) {
  const uint32_t sq = uint32_t(c >> 32) & 0xFFFFFFu;
  const uint32_t delta = (sq - e.seq) & 0xFFFFFFu;
  if (delta == 0 || delta >= 0x800000u) return false;
  e.seq += delta;
  e.cur = uint32_t(c);
  e.hint = uint32_t(c >> 56);
  if ((e.hint & LK_HINT_SYSMEM) && !acquired) {
    if (via_gateway) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    else acquire_sys();
  }
  e.dirty = true;
  e.c_seen = clock64();
  if (timeline) e.t_seen = globaltimer();
  return true;
}

// Fast-path publish: every call changes the cell's word (WORKING after NOP,
// FINISHED after WORKING, NOP after FINISHED), so with record_trace on each
// one is a trace record, exactly as publish() would write it.
__device__ __forceinline__ void publish_fast(const lk_dev_args& a, uint32_t wid, Elected& e, uint32_t word,
                                             uint32_t phase) {
  if (a.record_trace) trace_rec(a, wid, e, word);
  st_relaxed_sys(a.status + uint64_t(wid) * a.status_u64, uint64_t(word) | (uint64_t(phase) << 32));
}

// Per-worker count of values the fast path settled (lk_fast_count): the
// evidence that the benchmarked branches ran, and were trace-checked.
__device__ __forceinline__ void fast_hit(const lk_dev_args& a, uint32_t wid, Elected& e) {
  a.fast_cnt[wid] = ++e.fhits;
}

// The ack delay (see spin_cycles below) is per worker and adapts to the host:
// a host that needs longer than the delay to see FINISHED and write the NOP
// makes the delayed load miss, and the NOP arrives on the second load; the
// delay then grows by a quarter of its configured value.  Every ack seen on
// the first load shrinks it by 1/256, so it settles just above the host's
// answer time (boxes differ: 150-250 ns measured, tools/ab_ack.py) with a
// ~2% miss rate.  Acks that took more loads (wide masks: the host acks after
// the last worker finished) say nothing about that time and are ignored.
// Bounds: 1/4 to 4x the configured delay.
__device__ __forceinline__ void ack_adapt(const lk_dev_args& a, Elected& e) {
  if (!a.ack_delay_cyc || a.replicas != 1 || (a.flags & LK_CF_ACK_FIXED)) return;
  if (e.nload == 1) {
    const uint32_t lo = a.ack_delay_cyc >> 2;
    e.ack_cyc -= e.ack_cyc >> 8;
    if (e.ack_cyc < lo) e.ack_cyc = lo;
  } else if (e.nload == 2) {
    const uint32_t hi = a.ack_delay_cyc << 2;
    e.ack_cyc = min(e.ack_cyc + (a.ack_delay_cyc >> 2), hi);
  }
}

// The idle delay adapts the same way, from idle_delay_ns (default 0): a WORK
// that arrives on the second load after the closing NOP means the host
// re-triggers this worker right after each handshake, a little later than
// the delay; the delay grows by ~65 ns (cap ~1.5 us).  A WORK on the first
// load shrinks it by 1/256.  A WORK after more loads (the host triggered
// other workers in between: round robin) leaves it alone, so only loops
// that re-trigger one worker back to back get a delay (tools/ab_idle.py).
constexpr uint32_t kIdleStepCyc = 128, kIdleMaxCyc = 3000;
__device__ __forceinline__ void idle_adapt(const lk_dev_args& a, Elected& e) {
  if (!e.idle_armed) return;
  e.idle_armed = false;
  if (a.replicas != 1 || (a.flags & LK_CF_ACK_FIXED)) return;
  if (e.nload == 1) e.idle_cyc -= e.idle_cyc >> 8;
  else if (e.nload == 2) e.idle_cyc = min(e.idle_cyc + kIdleStepCyc, max(kIdleMaxCyc, a.idle_delay_cyc));
}

// The transitions of a short round trip, settled in place right where the
// new value was seen (no descriptor fetch, no trip through the general
// dispatch code and its cold instruction-cache lines):
//   IDLE x WORK(s), slot s cached (LK_HINT_CACHED) as busy_loop/empty -> publish
//      WORKING, run the loop, publish FINISHED;
//   IDLE x WORK(s), slot s holds no work (LK_HINT_EMPTY) -> publish WORKING,
//      FINISHED; re-stepping the same word in FINISHED publishes FINISHED
//      again (a no-op);
//   IDLE x WORK(s) of a payload kind -> publish WORKING and begin at once;
//   FINISHED x NOP -> publish NOP, IDLE; re-stepping NOP in IDLE is a no-op.
// Exactly lk_worker_step + lk_complete_work for these cases (protocol.py:151-206);
// anything else takes settle().  With record_trace on, every publish here
// appends the same trace record publish() would, so the recorded sessions
// replay the fast path itself (tests/test_gpu_fastpath.py).
// The fast path's part of the dispatch timeline (lk_last_timeline): clock64
// stamps always, globaltimer stamps under LK_CF_TIMELINE (same words as
// write_timeline, plus word 8 = FINISHED issued for the ack-phase breakdown).
__device__ __forceinline__ void fast_timeline(const lk_dev_args& a, uint32_t wid, const Elected& e,
                                              uint64_t c_begin, uint64_t c_fin, uint64_t t_b, uint64_t t_e,
                                              bool tlf) {
  unsigned long long* tl = a.spans + uint64_t(LK_TIMELINE_WORDS) * wid;
  tl[5] = e.c_seen; tl[6] = c_begin; tl[7] = c_fin;
  if (tlf) {
    const uint64_t t_f = globaltimer();
    tl[0] = e.t_seen; tl[1] = t_b; tl[2] = t_e; tl[3] = t_f; tl[4] = e.t_fwd; tl[8] = t_f;
  }
}

enum FastResult : uint32_t { kFastNone = 0, kFastSettled = 1, kFastBegin = 2 };

__device__ __forceinline__ uint32_t fast_step(const lk_dev_args& a, uint32_t wid, Elected& e) {
  if (a.flags & LK_CF_FENCE_ALWAYS) return kFastNone;   // every FINISHED is a sys-scope release: settle()
  const uint32_t w = e.cur;
  if (e.st.phase == LK_PHASE_IDLE && w >= LK_WORK_BASE && (e.hint & LK_HINT_CACHED) &&
      w - LK_WORK_BASE == e.cslot && single_thread_kind(e.ckind)) {
    // a cached busy_loop/empty item: run it right here, like an empty task
    const bool tlf = (a.flags & LK_CF_TIMELINE) != 0;
    const uint64_t c_begin = clock64();
    const uint64_t t_b = tlf ? globaltimer() : 0;
    publish_fast(a, wid, e, LK_WORKING, LK_PHASE_WORKING);
    if (e.ckind == LK_KIND_BUSY_LOOP) *a.sink = busy_loop(e.citer);   // stored: the loop must run
    const uint64_t t_e = tlf ? globaltimer() : 0;
    publish_fast(a, wid, e, LK_FINISHED, LK_PHASE_FINISHED);
    const uint64_t c_fin = clock64();
    e.st = lk_wstate{LK_PHASE_FINISHED, w - LK_WORK_BASE};
    e.pub = LK_FINISHED;
    e.dirty = false;
    idle_adapt(a, e);
    fast_timeline(a, wid, e, c_begin, c_fin, t_b, t_e, tlf);
    fast_hit(a, wid, e);
    return kFastSettled;
  }
  if (e.st.phase == LK_PHASE_IDLE && w >= LK_WORK_BASE && !(e.hint & LK_HINT_EMPTY) &&
      w - LK_WORK_BASE < a.num_slots) {
    // IDLE x WORK(s) of any other kind: publish WORKING and begin at once; the
    // word stays dirty so it is re-stepped after completion, as in settle().
    publish_fast(a, wid, e, LK_WORKING, LK_PHASE_WORKING);
    idle_adapt(a, e);
    e.st = lk_wstate{LK_PHASE_WORKING, w - LK_WORK_BASE};
    e.pub = LK_WORKING;
    e.dirty = true;
    fast_hit(a, wid, e);
    return kFastBegin;
  }
  if (e.st.phase == LK_PHASE_IDLE && w >= LK_WORK_BASE && (e.hint & LK_HINT_EMPTY) &&
      w - LK_WORK_BASE < a.num_slots) {
    const bool tlf = (a.flags & LK_CF_TIMELINE) != 0;
    const uint64_t c_begin = clock64();
    const uint64_t t_b = tlf ? globaltimer() : 0;
    publish_fast(a, wid, e, LK_WORKING, LK_PHASE_WORKING);
    publish_fast(a, wid, e, LK_FINISHED, LK_PHASE_FINISHED);
    const uint64_t c_fin = clock64();
    idle_adapt(a, e);
    e.st = lk_wstate{LK_PHASE_FINISHED, w - LK_WORK_BASE};
    e.pub = LK_FINISHED;
    e.dirty = false;
    fast_timeline(a, wid, e, c_begin, c_fin, t_b, t_b, tlf);
    fast_hit(a, wid, e);
    return kFastSettled;
  }
  if (e.st.phase == LK_PHASE_FINISHED && w == LK_NOP) {
    publish_fast(a, wid, e, LK_NOP, LK_PHASE_IDLE);
    e.idle_pub = true;
    ack_adapt(a, e);
    if (a.flags & LK_CF_TIMELINE) {
      unsigned long long* tl = a.spans + uint64_t(LK_TIMELINE_WORDS) * wid;
      tl[9] = e.t_seen; tl[10] = e.nload; tl[11] = e.c_seen;
    }
    e.st.phase = LK_PHASE_IDLE;
    e.pub = LK_NOP;
    e.dirty = false;
    fast_hit(a, wid, e);
    return kFastSettled;
  }
  return kFastNone;
}

// HYBRID: a value from one of two channels, each with its own 24-bit write
// count (`last`: the direct cell's or the ring's); the host's per-worker write
// index is their sum.  The host issues a worker's next write only after the
// device answered the previous one, so at most one channel holds an unseen
// value and the sum orders them.
__device__ __forceinline__ bool accept_chan(Elected& e, unsigned long long c, uint32_t& last, bool timeline) {
  const uint32_t sq = uint32_t(c >> 32) & 0xFFFFFFu;
  const uint32_t delta = (sq - last) & 0xFFFFFFu;
  if (delta == 0 || delta >= 0x800000u) return false;
  last += delta;
  e.seq = e.dseq + e.rseq;
  e.cur = uint32_t(c);
  e.hint = uint32_t(c >> 56);
  if (e.hint & LK_HINT_SYSMEM) acquire_sys();
  e.dirty = true;
  e.c_seen = clock64();
  if (timeline) e.t_seen = globaltimer();
  return true;
}

// Step the current word to a fixed point, exactly as the reference worker
// re-reads a level-triggered cell until it stops making progress
// (native.py:158-195).  Returns an action, or LK_ACT_NONE once settled.
__device__ __forceinline__ uint32_t settle(const lk_dev_args& a, uint32_t wid, Elected& e) {
  while (e.dirty) {
    const uint32_t before = e.st.phase;
    const lk_step_out o = lk_worker_step(e.st, e.cur);
    if (o.werr) {
      report_error(a, wid, e, o.werr, e.cur);
      return LK_ACT_EXIT;
    }
    bool progressed = e.st.phase != before;
    if (o.publish != LK_NO_PUBLISH && o.publish != e.pub) {
      publish(a, wid, e, o.publish, false);
      progressed = true;
    } else if (e.st.phase != before) {
      publish(a, wid, e, e.pub, false);  // phase-only update (EXIT): word unchanged
    }
    if (o.action != LK_ACT_NONE) return o.action;  // cur stays dirty: re-stepped after the work
    e.dirty = progressed;
  }
  return LK_ACT_NONE;
}

// A worker that has just published FINISHED expects the host's NOP ack about
// one link round trip later.  A cell load issued at once is ordered behind the
// FINISHED store on the link (reads do not pass posted writes), so it samples
// host memory the moment FINISHED lands -- before the host can have seen it
// and answered -- and the ack waits a whole extra round trip for the next
// load.  Waiting ack_delay_cyc (~200 ns: the host's detect-and-write time)
// first makes that one load the one that sees the ack: the empty-task cycle
// drops from 4.5 to 3.5 us (tools/ab_ack.py, tools/ack_breakdown.py).  The
// NOP that closes a handshake can be answered the same way when the host
// re-triggers the same worker at once: idle_delay_cyc (opt-in; the host's
// re-trigger time, ~300 ns from C, ~600 ns from Python) before the next
// load (tools/ab_idle.py).
__device__ __forceinline__ void spin_cycles(uint32_t cyc) {
  if (!cyc) return;
  const uint64_t c0 = clock64();
  while (clock64() - c0 < cyc) {
  }
}

__device__ __forceinline__ void ack_wait(Elected& e) {
  spin_cycles(e.ack_cyc);
  e.nload = 0;
}

__device__ __forceinline__ void idle_wait(Elected& e) {
  spin_cycles(e.idle_cyc);
  e.nload = 0;
  e.idle_armed = true;
}

// Spin until the state machine begins work or exits.  The to_gpu cell is K
// replicas {word, seq} on separate 128-B lines; one ld.relaxed.sys per replica
// is kept in flight, staggered by spacing_ns, so the host's write is sampled K
// times per PCIe round trip (same-line loads would merge in L1).  A value is
// accepted only when its seq is newer, so replicas written one after another
// never make the state machine go backwards.
template <int K>
__device__ __forceinline__ uint32_t poll_k(const lk_dev_args& a, uint32_t wid, Elected& e) {
  const unsigned long long* base = a.to_gpu + uint64_t(wid) * K * a.cell_u64;
  const uint32_t step = a.cell_u64;
  const bool acquire = (a.flags & LK_CF_ACQUIRE_POLL) != 0;
  const bool timeline = (a.flags & LK_CF_TIMELINE) != 0;
  for (;;) {
    const uint32_t act = settle(a, wid, e);
    if (act != LK_ACT_NONE) return act;
    if (K == 1 && e.st.phase == LK_PHASE_FINISHED) ack_wait(e);
    unsigned long long v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k] = ld_cell(base + k * step, acquire);
      if (K > 1) __nanosleep(a.spacing_ns);
    }
    for (bool fresh = false; !fresh;) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (accept(e, v[k], timeline, acquire)) {
          const uint32_t f = fast_step(a, wid, e);
          if (f == kFastBegin) return LK_ACT_BEGIN;
          fresh = f == kFastNone;          // settled in place: keep polling
          if (fresh) break;
          if (K == 1) {
            if (e.st.phase == LK_PHASE_FINISHED) ack_wait(e);
            else if (e.idle_pub) idle_wait(e);
          }
          e.idle_pub = false;
          v[k] = ld_cell(base + k * step, acquire);
          ++e.nload;
          continue;
        }
        if (K == 1 && a.backoff_ns) __nanosleep(a.backoff_ns);   // before the load: a real gap between polls
        v[k] = ld_cell(base + k * step, acquire);
        ++e.nload;
        if (K > 1) __nanosleep(a.spacing_ns);
      }
      if (!fresh && K > 1 && a.backoff_ns) __nanosleep(a.backoff_ns);
    }
  }
}

// GATEWAY mode: the worker's to_gpu value arrives in its device mailbox line
// (written by the gateway warp); poll it in L2, one load in flight.
__device__ __forceinline__ uint32_t poll_mailbox(const lk_dev_args& a, uint32_t wid, Elected& e) {
  const unsigned long long* mb = a.dmb + uint64_t(wid) * a.dmb_u64;
  const bool timeline = (a.flags & LK_CF_TIMELINE) != 0;
  for (;;) {
    const uint32_t act = settle(a, wid, e);
    if (act != LK_ACT_NONE) return act;
    for (;;) {
      if (accept(e, ld_relaxed_gpu64(mb), timeline, false, true)) {
        if (timeline) e.t_fwd = ld_relaxed_gpu64(mb + 1);
        const uint32_t f = fast_step(a, wid, e);
        if (f == kFastBegin) return LK_ACT_BEGIN;
        if (f == kFastNone) break;
        continue;
      }
      if (a.backoff_ns) __nanosleep(a.backoff_ns);
    }
  }
}

// Inlined into the worker loop so the protocol state stays in registers.
__device__ __forceinline__ unsigned long long lds_volatile64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_volatile64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}

// HYBRID mode, protocol thread: both channels arrive in shared memory (chan[0]
// from this CTA's host-cell poller warp, chan[1] from its mailbox poller
// warp), so the thread spins on two ~30-cycle shared loads and never holds a
// PCIe or L2 load in flight itself.
__device__ __forceinline__ uint32_t poll_hybrid(const lk_dev_args& a, uint32_t wid, Elected& e,
                                                const unsigned long long* chan) {
  const bool timeline = (a.flags & LK_CF_TIMELINE) != 0;
  for (;;) {
    const uint32_t act = settle(a, wid, e);
    if (act != LK_ACT_NONE) return act;
    for (;;) {
      bool got = accept_chan(e, lds_volatile64(chan), e.dseq, timeline);
      if (!got) got = accept_chan(e, lds_volatile64(chan + 1), e.rseq, timeline);
      if (!got) continue;
      const uint32_t f = fast_step(a, wid, e);
      if (f == kFastBegin) return LK_ACT_BEGIN;
      if (f == kFastNone) break;
    }
  }
}

// HYBRID mode, channel pollers (lane 0 of two extra warps per CTA): forward
// every new value of the host cell (one ld.relaxed.sys in flight) or of the
// device mailbox (L2) into the CTA's shared-memory channel slot.
__device__ __noinline__ void chan_poller(const unsigned long long* src, bool sys, unsigned long long* slot,
                                         const volatile uint32_t* stop) {
  uint32_t last = 0;
  while (!*stop) {
    const unsigned long long v = sys ? ld_cell(src, false) : ld_relaxed_gpu64(src);
    const uint32_t sq = uint32_t(v >> 32) & 0xFFFFFFu;
    if (sq != last) {
      last = sq;
      sts_volatile64(slot, v);
    }
  }
}

__device__ __forceinline__ uint32_t poll(const lk_dev_args& a, uint32_t wid, Elected& e,
                                         const unsigned long long* chan) {
  if (a.poll_mode == LK_POLL_HYBRID) return poll_hybrid(a, wid, e, chan);
  if (a.poll_mode == LK_POLL_GATEWAY) return poll_mailbox(a, wid, e);
  return poll_k<1>(a, wid, e);   // one cell per worker (replicas measured slower)
}

// ---------------------------------------------------------------- gateway
// GATEWAY mode.  The host does not write per-worker cells; it appends one
// event per logical write (a trigger, an ack, EXIT) to a ring in pinned host
// memory: entry = 8 u64 on one 64-B line,
//   w[0] = seq:32 | word:32           (written last: the "new event" signal)
//   w[1..4] = mask bits [48j, 48j+48) | tag:16 << 48
//   w[5] = hint | tag:16 << 48        (tag = seq & 0xFFFF: torn-read check)
// in K replica rings.  One warp of CTA 0 polls the entry it expects next on
// each replica, one load per lane (lanes 0..5) in flight per replica,
// staggered spacing_ns.  The PCIe link therefore carries ~6K small reads in
// flight instead of one per worker, which is what kept the per-read round
// trip long in DIRECT mode.  An accepted event is fanned out to every masked
// worker's mailbox line in device memory ({word, per-worker seq24, hint}, the
// same value DIRECT mode reads from host memory), and the consumed count is
// posted back to the host (ring flow control).  Exits once every worker has
// left its loop.
constexpr uint32_t kRingMaskBits = 48;
static_assert(4 * kRingMaskBits >= 148, "event masks cover every SM of a B200");   // host: <= 192 workers

template <int K>
__device__ __forceinline__ void gateway_k(const lk_dev_args& a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = a.nw, N = a.ring_entries;
  const bool timeline = (a.flags & LK_CF_TIMELINE) != 0;
  uint32_t wseq[6];                               // per-worker write counts, workers lane + 32q
#pragma unroll
  for (int q = 0; q < 6; ++q) wseq[q] = 0;
  uint32_t expect = 1;                            // next event seq
  unsigned long long v[K];
  auto issue = [&](int k) {
    if (lane < 6)
      v[k] = ld_cell(a.ring + (uint64_t(k) * N + (expect - 1) % N) * 8 + lane, false);
  };
#pragma unroll
  for (int k = 0; k < K; ++k) {
    issue(k);
    if (K > 1) __nanosleep(a.spacing_ns);
  }
  for (uint32_t it = 0;; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      // lanes 0..5 hold the 6 words of the entry this replica load saw
      const unsigned long long w = lane < 6 ? v[k] : 0ull;
      const unsigned long long w0 = __shfl_sync(0xffffffffu, w, 0);
      const uint32_t tag = expect & 0xFFFFu;
      const bool mine = lane == 0 ? uint32_t(w0) == expect
                                  : (lane < 6 ? uint32_t(w >> 48) == tag : true);
      if (__all_sync(0xffffffffu, mine)) {
        const uint32_t word = uint32_t(w0 >> 32);
        const uint32_t hint = uint32_t(__shfl_sync(0xffffffffu, w, 5)) & 0xFFu;
        // a host-mapped payload: the sys-scope fence makes the entry's load
        // the acquire of the host's release, and releases the forwarding
        // stores after it; the worker's gpu-scope fence completes the chain
        // (the ring is polled relaxed: acquire loads here and on the
        // mailboxes cost 1.2 us per full-mask dispatch, tools/ab_wide.py)
        if (hint & LK_HINT_SYSMEM) acquire_sys();
        // the four 48-bit mask words stay in registers: a runtime index into
        // an array would put it in local memory
        const unsigned long long mm = (1ull << kRingMaskBits) - 1;
        const unsigned long long m0 = __shfl_sync(0xffffffffu, w, 1) & mm, m1 = __shfl_sync(0xffffffffu, w, 2) & mm,
                                 m2 = __shfl_sync(0xffffffffu, w, 3) & mm, m3 = __shfl_sync(0xffffffffu, w, 4) & mm;
        const uint64_t t_fwd = timeline ? globaltimer() : 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const uint32_t i = lane + 32u * q;
          const uint32_t wi = i / kRingMaskBits;
          const unsigned long long mw = wi == 0 ? m0 : wi == 1 ? m1 : wi == 2 ? m2 : m3;
          if (i < nw && (mw >> (i % kRingMaskBits) & 1ull)) {
            ++wseq[q];
            unsigned long long* mb = a.dmb + uint64_t(i) * a.dmb_u64;
            if (timeline) st_relaxed_gpu64(mb + 1, t_fwd);
            st_relaxed_gpu64(mb, uint64_t(word) | (uint64_t(wseq[q] & 0xFFFFFFu) << 32) |
                                     (uint64_t(hint) << 56));
          }
        }
        if (lane == 0) st_relaxed_sys(a.gw_tail, expect);   // consumed: ring slot reusable
        ++expect;
      }
      issue(k);
      if (K > 1) __nanosleep(a.spacing_ns);
      else if (a.backoff_ns) __nanosleep(a.backoff_ns);
    }
    if ((it & 63u) == 0 && ld_relaxed_gpu32(a.exited) >= nw) return;
  }
}

__device__ __noinline__ void gateway(const lk_dev_args& a) { gateway_k<1>(a); }   // one event ring

// Per-worker record of the last dispatch (lk_last_timeline): globaltimer at
// value seen / work begin / work end / FINISHED issued, gateway forward time,
// and clock64 at seen / work begin / FINISHED issued.
// globaltimer reads cost a few hundred cycles each, so the single-thread
// (latency) kinds stamp clock64 only unless LK_CF_TIMELINE asks for both.
__device__ __forceinline__ void write_timeline(const lk_dev_args& a, uint32_t wid, const Elected& e,
                                               uint64_t t_begin, uint64_t t_end, uint64_t c_begin,
                                               uint64_t c_fin, bool globaltime) {
  unsigned long long* tl = a.spans + uint64_t(LK_TIMELINE_WORDS) * wid;
  tl[0] = e.t_seen; tl[1] = t_begin; tl[2] = t_end; tl[3] = globaltime ? globaltimer() : 0;
  tl[4] = e.t_fwd; tl[5] = e.c_seen; tl[6] = c_begin; tl[7] = c_fin;
}

struct PersistSmem {
  lk_desc desc;
  uint32_t cmd, rank, count, slot;
  ReduceSmem red;
  uint64_t full[2 * kMaxStages], empty[2 * kMaxStages];
  uint32_t tile[kMaxStages], ring_gr;
  unsigned long long chan[2];      // HYBRID: latest direct-cell value, latest mailbox value
  lk_desc cdesc;                   // this worker's last fetched descriptor (LK_HINT_CACHED)
  unsigned long long cmask[4];     // ... and its slot's trigger mask
  uint32_t stop;                   // HYBRID: the protocol thread left its loop
};

__global__ void __launch_bounds__(kPersistMaxThreads, 1) lk_persistent_kernel(const __grid_constant__ lk_dev_args a) {
  __shared__ PersistSmem sm;
  const uint32_t wid = blockIdx.x;
  const uint32_t T = a.wthreads;
  if (threadIdx.x == 0) {
    sm.chan[0] = 0ull;              // {NOP, count 0}: nothing new on either channel
    sm.chan[1] = 0ull;
    sm.stop = 0;
  }
  __syncthreads();                  // the only CTA-wide barrier: before the roles split
  if (threadIdx.x >= T) {           // three extra warps: host-cell poller, mailbox poller, gateway
    const uint32_t xw = (threadIdx.x - T) >> 5, lane = threadIdx.x & 31;
    const bool hybrid = a.poll_mode == LK_POLL_HYBRID;
    if (xw == 0) {
      if (hybrid && lane == 0)
        chan_poller(a.to_gpu + uint64_t(wid) * a.cell_u64, true, sm.chan, &sm.stop);   // 1 replica
    } else if (xw == 1) {
      if (hybrid && lane == 0) chan_poller(a.dmb + uint64_t(wid) * a.dmb_u64, false, sm.chan + 1, &sm.stop);
    } else if (wid == 0 && (hybrid || a.poll_mode == LK_POLL_GATEWAY)) {
      gateway(a);
    }
    return;
  }
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  Ring ring{dyn_smem, sm.full, sm.empty, a.ring_stages, sm.tile, &sm.ring_gr};
  const bool ring_ok = a.use_tma != 0;
  uint32_t g = 0;
  if (ring_ok) ring_init(ring, T);
  Elected e;
  e.st = lk_wstate{LK_PHASE_BOOTING, 0};
  e.pub = LK_NOP;  // cells start at the NOP sentinel (protocol.py:217-218)
  e.seq = 0;       // the host's initial {NOP, seq 0} value
  e.cur = LK_NOP;
  e.hint = 0;
  e.dseq = 0;
  e.rseq = 0;
  e.tcnt = 0;
  e.fhits = 0;
  e.nload = 0;
  e.cslot = 0xFFFFFFFFu;
  e.ckind = 0;
  e.citer = 0;
  e.ack_cyc = a.ack_delay_cyc;
  e.idle_pub = false;
  e.idle_armed = false;
  e.idle_cyc = a.idle_delay_cyc;
  e.dirty = true;  // boot: step NOP -> INIT, then NOP -> IDLE
  e.t_seen = 0;
  e.c_seen = 0;
  e.t_fwd = 0;
  uint64_t t_begin = 0, c_begin = 0;
  if (threadIdx.x == 0) st_relaxed_sys_u32(a.smid + wid, smid());

  for (;;) {
    if (threadIdx.x == 0) {
      for (;;) {
        const uint32_t act = poll(a, wid, e, sm.chan);
        if (act == LK_ACT_EXIT) { sm.cmd = kCmdExit; break; }
        const uint32_t slot = e.st.slot;
        if (slot >= a.num_slots) { report_error(a, wid, e, LK_WERR_BAD_SLOT, slot + LK_WORK_BASE); sm.cmd = kCmdExit; break; }
        if (e.hint & LK_HINT_EMPTY) {
          // the host staged an EMPTY descriptor in this slot and said so in the
          // word's hint bits: complete without the descriptor round trip to L2
          const uint64_t c_begin_e = clock64();
          const bool tl = (a.flags & LK_CF_TIMELINE) != 0;
          const uint64_t t_b = tl ? globaltimer() : 0;
          const lk_step_out o = lk_complete_work(e.st);
          publish(a, wid, e, o.publish, (a.flags & LK_CF_FENCE_ALWAYS) != 0);
          write_timeline(a, wid, e, t_b, t_b, c_begin_e, clock64(), tl);
          continue;
        }
        // descriptor and the slot's trigger mask: reused from this worker's
        // cache when the host says it is current (LK_HINT_CACHED; the slot is
        // checked too), else one L2 round trip, which refills the cache
        lk_desc d;
        unsigned long long mk[4] = {0ull, 0ull, 0ull, 0ull};
        if ((e.hint & LK_HINT_CACHED) && e.cslot == slot) {
          d = sm.cdesc;
#pragma unroll
          for (int k = 0; k < 4; ++k) mk[k] = sm.cmask[k];
        } else {
          const uint4* src = reinterpret_cast<const uint4*>(a.desc + slot);
          uint4* dst = reinterpret_cast<uint4*>(&d);
          const unsigned long long* m = a.slot_mask + uint64_t(slot) * a.nwords;
          if (a.flags & LK_CF_HOST_DESC) {   // host-mapped table: sys scope, never a stale L2 line
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = ld_sys4(src + k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (uint32_t(k) < a.nwords) mk[k] = ld_cell(m + k, false);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = ld_cg4(src + k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (uint32_t(k) < a.nwords) mk[k] = ld_cg64(m + k);
          }
          sm.cdesc = d;
#pragma unroll
          for (int k = 0; k < 4; ++k) sm.cmask[k] = mk[k];
          e.cslot = slot;
          e.ckind = d.kind;
          e.citer = d.iterations;
        }
        if (d.kind >= LK_KIND_COUNT) { report_error(a, wid, e, LK_WERR_BAD_KIND, slot + LK_WORK_BASE); sm.cmd = kCmdExit; break; }
        if (single_thread_kind(d.kind)) {
          const bool tl = (a.flags & LK_CF_TIMELINE) != 0;
          c_begin = clock64();
          t_begin = tl ? globaltimer() : 0;
          if (d.kind == LK_KIND_BUSY_LOOP) *a.sink = busy_loop(d.iterations);   // global store: the loop must run
          const uint64_t t_end = tl ? globaltimer() : 0;
          const lk_step_out o = lk_complete_work(e.st);
          publish(a, wid, e, o.publish, (a.flags & LK_CF_FENCE_ALWAYS) != 0);
          write_timeline(a, wid, e, t_begin, t_end, c_begin, clock64(), tl);
          continue;
        }
        // payload item: rank/count from the slot's trigger mask
        uint32_t count = 0, rank = 0;
        const uint32_t mw = wid >> 6;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          const unsigned long long bits = mk[k];
          count += __popcll(bits);
          if (k < mw) rank += __popcll(bits);
          else if (k == mw) rank += __popcll(bits & ((1ull << (wid & 63)) - 1ull));
        }
        sm.desc = d;
        sm.rank = rank;
        sm.count = count ? count : 1;
        sm.slot = slot;
        sm.cmd = kCmdWork;
        c_begin = clock64();
        t_begin = globaltimer();
        break;
      }
    }
    wsync(T);
    if (sm.cmd == kCmdExit) break;
    const lk_desc d = sm.desc;
    // a narrow dispatch streams through 128-bit LSU loads: a lone SM moves
    // ~110 GB/s that way against ~85 GB/s through the ring, which wins only
    // once enough SMs share the dispatch to load HBM (tools/tma_vs_lsu_count.py)
    run_multi(d, sm.rank, sm.count, a.reduce_ctr + 4ull * sm.slot, sm.red, T, ring,
              ring_ok && sm.count >= a.tma_min_workers, g, a.red_share8, a.red_claim, (a.flags & LK_CF_TIMELINE) ? a.spans + uint64_t(LK_TIMELINE_WORDS) * wid : nullptr);
    wsync(T);
    if (threadIdx.x == 0) {
      const uint64_t t_end = globaltimer();
      const lk_step_out o = lk_complete_work(e.st);
      // Payload stores of every worker thread (ordered before this thread by the
      // barrier) reach L2, the coherence point the host's copy engine reads,
      // before FINISHED is posted: a gpu-scope fence (~L2 round trip).  A
      // sys-scope release would also wait for this thread's earlier posted
      // host writes (WORKING) to cross PCIe (~1.5 us, tools/probe_costs.cu);
      // Host-mapped buffers (LK_DF_HOSTMEM) and LK_CF_FENCE_ALWAYS take it: the
      // st.release.sys is cumulative over the barrier, so every thread's
      // output stores are visible to the host before it can see FINISHED.
      const bool sys = (a.flags & LK_CF_FENCE_ALWAYS) != 0 || (d.flags & LK_DF_HOSTMEM) != 0;
      if (!sys) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      publish(a, wid, e, o.publish, sys);
      write_timeline(a, wid, e, t_begin, t_end, c_begin, clock64(), true);
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(a.exited, 1u);                      // lets the gateway retire
    *reinterpret_cast<volatile uint32_t*>(&sm.stop) = 1u;   // and this CTA's channel pollers
  }
}

// ---------------------------------------------------------------- baseline
__global__ void __launch_bounds__(kMaxThreads) lk_work_kernel(const lk_desc d, uint32_t* ctr, int use_tma) {
  __shared__ ReduceSmem rs;
  __shared__ uint64_t full[2 * kMaxStages], empty[2 * kMaxStages];
  __shared__ uint32_t tile[kMaxStages], gred;
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  if (single_thread_kind(d.kind)) {
    // the result goes to global memory (the counter line's spare word), which
    // ptxas cannot treat as dead; a dead shared store would let it drop the loop
    if (threadIdx.x == 0 && d.kind == LK_KIND_BUSY_LOOP) ctr[3] = busy_loop(d.iterations);
    return;
  }
  Ring ring{dyn_smem, full, empty, kDefaultStages, tile, &gred};
  uint32_t g = 0;
  if (use_tma) ring_init(ring, blockDim.x);
  run_multi(d, blockIdx.x, gridDim.x, ctr, rs, blockDim.x, ring, use_tma != 0, g);
}

// The fastest conventional task: an empty kernel, one warp, no shared memory
// (the launch+sync floor lk_launch_floor_bench measures LK against).
__global__ void lk_empty_kernel() {}

// ---------------------------------------------------------------- ping-pong
__global__ void lk_pingpong_kernel(volatile uint32_t* flag, volatile uint32_t* echo, uint64_t rounds) {
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    while (ld_relaxed_sys(const_cast<const uint32_t*>(flag)) < want) {   // >=: the host's release value passes all
    }
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(echo), "r"(want) : "memory");
  }
}

// Host/device clock correlation: echo %globaltimer for each host flag value.
__global__ void lk_clocksync_kernel(const uint32_t* flag, unsigned long long* echo, uint32_t rounds) {
  for (uint32_t r = 1; r <= rounds; ++r) {
    while (ld_relaxed_sys(flag) != r) {
    }
    st_relaxed_sys(echo, globaltimer());
    // same 128-B line, posted in order: no release fence (MEMBAR.SYS would skew the echo)
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(echo + 1), "r"(r) : "memory");
  }
}

// SM topology probe: every CTA of a cluster runs on the same GPC, so the SM
// ids of one cluster's CTAs belong to one GPC (lk_sm_topology unions them).
__global__ void lk_topo_kernel(uint32_t* smids) {
  if (threadIdx.x == 0) smids[blockIdx.x] = smid();
}

}  // namespace

// One clustered launch of the topology probe: grid blocks in clusters of
// `cluster` CTAs, one CTA per SM (large dynamic shared memory).
cudaError_t lk_launch_topo(uint32_t* smids, uint32_t grid, uint32_t cluster, size_t smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaFuncSetAttribute(lk_topo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess && cluster > 8)
    e = cudaFuncSetAttribute(lk_topo_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, lk_topo_kernel, smids);
}

cudaError_t lk_launch_clocksync(const uint32_t* flag, unsigned long long* echo, uint32_t rounds,
                                cudaStream_t st) {
  lk_clocksync_kernel<<<1, 1, 0, st>>>(flag, echo, rounds);
  return cudaGetLastError();
}

// CUDA 12 loads kernels lazily on first launch, and loading a module while a
// spinning kernel is resident can wait on it forever.  Load every kernel of
// this library before the persistent kernel launches.
cudaError_t lk_preload_kernels() {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, lk_work_kernel);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lk_work_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kDefaultStages * kStageBytes));
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, lk_pingpong_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, lk_empty_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, lk_clocksync_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, lk_persistent_kernel);
  return e;
}

cudaError_t lk_persistent_configure(size_t smem) {
  return cudaFuncSetAttribute(lk_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

cudaError_t lk_persistent_occupancy(uint32_t threads, size_t smem, int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, lk_persistent_kernel, int(threads), smem);
}

cudaError_t lk_launch_persistent(const lk_dev_args& a, uint32_t grid, uint32_t threads, size_t smem,
                                 cudaStream_t st) {
  void* args[] = {const_cast<lk_dev_args*>(&a)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lk_persistent_kernel), dim3(grid),
                                     dim3(threads), args, smem, st);
}

cudaError_t lk_launch_work(const lk_desc& d, uint32_t grid, uint32_t threads, uint32_t* reduce_ctr,
                           cudaStream_t st, int use_tma) {
  lk_work_kernel<<<grid, threads, use_tma ? kDefaultStages * kStageBytes : 0, st>>>(d, reduce_ctr, use_tma);
  return cudaGetLastError();
}

cudaError_t lk_launch_empty(cudaStream_t st) {
  lk_empty_kernel<<<1, 32, 0, st>>>();
  return cudaGetLastError();
}

size_t lk_ring_bytes(uint32_t stages) { return size_t(stages ? stages : kDefaultStages) * kStageBytes; }
uint32_t lk_ring_max_stages() { return kMaxStages; }

cudaError_t lk_launch_pingpong(volatile uint32_t* flag, volatile uint32_t* echo, uint64_t rounds,
                               cudaStream_t st) {
  lk_pingpong_kernel<<<1, 1, 0, st>>>(flag, echo, rounds);
  return cudaGetLastError();
}
