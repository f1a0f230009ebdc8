// probe_cluster.cu -- does a thread-block-cluster fan-out through distributed
// shared memory beat L2 mailboxes (LK's gateway) or per-SM host polling (LK's
// DIRECT) for a full-mask dispatch?  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_cluster.cu -o tools/probe_cluster
//
// One CTA per SM (large dynamic shared memory).  A round: the host writes
// value r, every CTA echoes r into its own host line, the host sees all G
// echoes.  Modes:
//   direct   every CTA polls its own host line (ld.relaxed.sys)
//   gateway  CTA 0 polls one host doorbell, writes G L2 mailboxes; CTAs poll L2
//   cluster  clusters of C CTAs: rank 0 polls the host doorbell and writes r
//            into each peer's shared memory (st.shared::cluster); peers spin
//            on their own shared memory
//   cl_gw    CTA 0 polls the host doorbell, writes one L2 mailbox per cluster
//            leader; leaders fan out through DSMEM
// Value 0xFFFFFFFF stops every kernel.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <vector>

namespace cg = cooperative_groups;

static inline uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return uint64_t(ts.tv_sec) * 1000000000ull + ts.tv_nsec;
}
__device__ __forceinline__ uint32_t ld_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr uint32_t kStop = 0xFFFFFFFFu;

__global__ void k_direct(const uint32_t* flags, uint32_t* echo) {
  if (threadIdx.x) return;
  const uint32_t* f = flags + 32 * blockIdx.x;
  uint32_t seen = 0;
  for (;;) {
    const uint32_t v = ld_sys(f);
    if (v != seen) {
      seen = v;
      if (v == kStop) return;
      st_sys(echo + 32 * blockIdx.x, v);
    }
  }
}

__global__ void k_gateway(const uint32_t* bell, uint32_t* mb, uint32_t* echo) {
  const uint32_t lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 64) {   // gateway warp
    uint32_t seen = 0;
    for (;;) {
      const uint32_t v = __shfl_sync(0xffffffffu, lane == 0 ? ld_sys(bell) : 0u, 0);
      if (v != seen) {
        seen = v;
        for (uint32_t b = lane; b < gridDim.x; b += 32) st_gpu(mb + 32 * b, v);
        if (v == kStop) return;
      }
    }
  }
  if (threadIdx.x) return;
  uint32_t seen = 0;
  for (;;) {
    const uint32_t v = ld_gpu(mb + 32 * blockIdx.x);
    if (v != seen) {
      seen = v;
      if (v == kStop) return;
      st_sys(echo + 32 * blockIdx.x, v);
    }
  }
}

// cluster fan-out: warp 1 of cluster rank 0 (the leader) polls `src` (the
// host doorbell, or its L2 mailbox when `from_l2`) and its lane k stores the
// value into cluster rank k's shared word; thread 0 of every CTA spins on its
// own shared word and echoes.  With `from_l2`, warp 2 of CTA 0 is a gateway
// that forwards the doorbell to one L2 mailbox per cluster leader.
__global__ void k_cluster(const uint32_t* bell, uint32_t* mb, uint32_t* echo, int from_l2) {
  __shared__ uint32_t word;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) word = 0;
  cl.sync();
  const uint32_t rank = cl.block_rank(), csize = cl.num_blocks();
  if (from_l2 && blockIdx.x == 0 && warp == 2) {
    uint32_t seen = 0;
    for (;;) {
      const uint32_t v = __shfl_sync(0xffffffffu, lane == 0 ? ld_sys(bell) : 0u, 0);
      if (v != seen) {
        seen = v;
        for (uint32_t b = lane * csize; b < gridDim.x; b += 32 * csize) st_gpu(mb + 32 * b, v);
        if (v == kStop) break;
      }
    }
  } else if (rank == 0 && warp == 1) {
    uint32_t seen = 0;
    const uint32_t* src = from_l2 ? mb + 32 * blockIdx.x : bell;
    uint32_t* peer = lane < csize ? cl.map_shared_rank(&word, lane) : nullptr;
    for (;;) {
      const uint32_t v = __shfl_sync(0xffffffffu, lane == 0 ? (from_l2 ? ld_gpu(src) : ld_sys(src)) : 0u, 0);
      if (v != seen) {
        seen = v;
        if (peer) *reinterpret_cast<volatile uint32_t*>(peer) = v;   // a DSMEM store (generic address)
        if (v == kStop) break;
      }
    }
  } else if (threadIdx.x == 0) {
    uint32_t seen = 0;
    volatile uint32_t* w = &word;
    for (;;) {
      const uint32_t v = *w;
      if (v != seen) {
        seen = v;
        if (v == kStop) break;
        st_sys(echo + 32 * blockIdx.x, v);
      }
    }
  }
  cl.sync();   // peers' shared memory outlives the leader's remote stores
}

static void summary(const char* label, std::vector<uint64_t>& v) {
  std::vector<uint64_t> s(v.begin() + v.size() / 10, v.end());
  std::sort(s.begin(), s.end());
  auto q = [&](double p) { return s[size_t(p * (s.size() - 1))] / 1e3; };
  printf("%-28s p50 %6.3f  p90 %6.3f  p99 %6.3f  p99.9 %6.3f us\n", label, q(0.5), q(0.9), q(0.99), q(0.999));
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 20000;
  cudaSetDevice(0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 150 * 1024;   // one CTA per SM
  cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gateway, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  uint32_t* host = nullptr;   // flags (nsm lines) | echo (nsm lines) | bell
  const size_t hbytes = size_t(2 * nsm + 2) * 128;
  cudaHostAlloc(reinterpret_cast<void**>(&host), hbytes, cudaHostAllocMapped | cudaHostAllocPortable);
  uint32_t* mb = nullptr;
  cudaMalloc(&mb, size_t(nsm) * 128);
  uint32_t* flags = host;
  uint32_t* echo = host + 32 * nsm;
  uint32_t* bell = host + 64 * nsm;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);

  auto run = [&](const char* label, int G, auto launch, bool per_cta_flags) {
    memset(host, 0, hbytes);
    cudaMemsetAsync(mb, 0, size_t(nsm) * 128, st);
    cudaStreamSynchronize(st);
    cudaError_t e = launch();
    if (e != cudaSuccess) {
      printf("%-28s launch failed: %s\n", label, cudaGetErrorString(e));
      cudaGetLastError();
      return;
    }
    std::vector<uint64_t> t;
    t.reserve(rounds);
    bool hung = false;
    for (int r = 1; r <= rounds && !hung; ++r) {
      const uint32_t v = uint32_t(r);
      const uint64_t t0 = now_ns();
      if (per_cta_flags) {
        for (int b = 0; b < G; ++b) __atomic_store_n(flags + 32 * b, v, __ATOMIC_RELEASE);
      } else {
        __atomic_store_n(bell, v, __ATOMIC_RELEASE);
      }
      for (int b = 0; b < G; ++b) {
        while (__atomic_load_n(echo + 32 * b, __ATOMIC_ACQUIRE) != v) {
          _mm_pause();
          if (now_ns() - t0 > 1000000000ull) { hung = true; break; }
        }
        if (hung) break;
      }
      t.push_back(now_ns() - t0);
    }
    for (int b = 0; b < G; ++b) __atomic_store_n(flags + 32 * b, kStop, __ATOMIC_RELEASE);
    __atomic_store_n(bell, kStop, __ATOMIC_RELEASE);
    const uint64_t until = now_ns() + 2000000000ull;
    while (cudaStreamQuery(st) == cudaErrorNotReady && now_ns() < until) usleep(100);
    if (hung || cudaStreamQuery(st) != cudaSuccess) {
      printf("%-28s HUNG (G=%d)\n", label, G);
      fflush(stdout);
      exit(1);
    }
    char l2[96];
    snprintf(l2, sizeof l2, "%s G=%d", label, G);
    summary(l2, t);
  };

  // co-residency of each cluster size at one CTA per SM
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm / C * C);
    cfg.blockDim = dim3(96);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_cluster, &cfg);
    printf("cluster %2d: max co-resident clusters %d (%d CTAs)%s\n", C, ncl, ncl * C,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  fflush(stdout);

  for (int rep = 0; rep < 2; ++rep) {
    run("direct (all SMs poll host)", nsm, [&] {
      k_direct<<<nsm, 64, smem, st>>>(flags, echo);
      return cudaGetLastError();
    }, true);
    run("gateway (L2 mailboxes)", nsm, [&] {
      k_gateway<<<nsm, 64, smem, st>>>(bell, mb, echo);
      return cudaGetLastError();
    }, false);
    for (int C : {2, 4, 8, 16}) {
      for (int from_l2 = 0; from_l2 < 2; ++from_l2) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.blockDim = dim3(96);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        int ncl = 0;
        cfg.gridDim = dim3(nsm / C * C);
        if (cudaOccupancyMaxActiveClusters(&ncl, k_cluster, &cfg) != cudaSuccess || ncl < 1) continue;
        const int G = std::min(nsm / C, ncl) * C;   // only co-resident clusters (spinning kernels)
        cfg.gridDim = dim3(G);
        char label[64];
        snprintf(label, sizeof label, "%s C=%d", from_l2 ? "cl_gw (L2 -> DSMEM)" : "cluster (DSMEM)", C);
        const int fl = from_l2;
        run(label, G, [&] { return cudaLaunchKernelEx(&cfg, k_cluster, (const uint32_t*)bell, mb, echo, fl); },
            false);
      }
    }
  }
  return 0;
}
