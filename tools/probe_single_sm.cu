// probe_single_sm.cu -- how fast can ONE SM stream an int32 vector add
// (out = a + b, 12 B/element)?  Variants: 128-bit LSU loads with U vectors
// in flight per thread, and cp.async (LDGSTS) 16-B copies into a shared-
// memory ring with D stages in flight.  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_single_sm.cu -o tools/probe_single_sm
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int U>
__global__ void __launch_bounds__(512, 1) lsu(const uint4* a, const uint4* b, uint4* o, uint64_t nv) {
  const uint32_t t = threadIdx.x, T = blockDim.x;
  uint64_t v = t;
  for (; v + uint64_t(U - 1) * T < nv; v += uint64_t(U) * T) {
    uint4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w) : "l"(a + v + u * T));
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(y[u].x), "=r"(y[u].y), "=r"(y[u].z), "=r"(y[u].w) : "l"(b + v + u * T));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      o[v + u * T] = make_uint4(x[u].x + y[u].x, x[u].y + y[u].y, x[u].z + y[u].z, x[u].w + y[u].w);
  }
  for (; v < nv; v += T) {
    const uint4 x = a[v], y = b[v];
    o[v] = make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
  }
}

// cp.async ring: each thread copies its own 16 B of a and b per stage into
// smem (so it only ever reads what it copied: no CTA barrier), D stages in
// flight (commit groups), then consumes the oldest.
template <int D>
__global__ void __launch_bounds__(512, 1) ldgsts(const uint4* a, const uint4* b, uint4* o, uint64_t nv) {
  extern __shared__ uint4 ring[];   // [D][2][T]
  const uint32_t t = threadIdx.x, T = blockDim.x;
  const uint64_t steps = (nv + T - 1) / T;
  auto issue = [&](uint64_t s) {
    const uint64_t v = s * T + t;
    uint4* sa = ring + (s % D) * 2 * T + t;
    uint4* sb = sa + T;
    if (v < nv) {
      const uint32_t da = uint32_t(__cvta_generic_to_shared(sa)), db = uint32_t(__cvta_generic_to_shared(sb));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(da), "l"(a + v));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(db), "l"(b + v));
    }
    asm volatile("cp.async.commit_group;");
  };
  for (uint64_t s = 0; s < D - 1 && s < steps; ++s) issue(s);
  for (uint64_t s = 0; s < steps; ++s) {
    if (s + D - 1 < steps) issue(s + D - 1);
    else asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1));
    const uint64_t v = s * T + t;
    if (v < nv) {
      const uint4 x = ring[(s % D) * 2 * T + t], y = ring[(s % D) * 2 * T + T + t];
      o[v] = make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    }
  }
}

int main() {
  const uint64_t n = 1 << 22;   // 4 Mi int32 = 16 MiB per vector, 48 MiB moved
  const uint64_t nv = n / 4;
  uint4 *a, *b, *o;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMalloc(&o, n * 4);
  cudaMemset(a, 1, n * 4);
  cudaMemset(b, 2, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    float best = 1e9f;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-28s %7.1f GB/s (1 SM, 512 threads)\n", name, 12.0 * n / (best * 1e6));
    fflush(stdout);
  };
  timeit("LSU U=2", [&] { lsu<2><<<1, 512>>>(a, b, o, nv); });
  timeit("LSU U=4 (LK today)", [&] { lsu<4><<<1, 512>>>(a, b, o, nv); });
  timeit("LSU U=8", [&] { lsu<8><<<1, 512>>>(a, b, o, nv); });
  for (int D : {4, 8, 12}) {
    const size_t sm = size_t(D) * 2 * 512 * 16;
    char name[64];
    snprintf(name, sizeof name, "cp.async ring D=%d (%zu KB)", D, sm / 1024);
    if (D == 4) { cudaFuncSetAttribute(ldgsts<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
                  timeit(name, [&] { ldgsts<4><<<1, 512, sm>>>(a, b, o, nv); }); }
    if (D == 8) { cudaFuncSetAttribute(ldgsts<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
                  timeit(name, [&] { ldgsts<8><<<1, 512, sm>>>(a, b, o, nv); }); }
    if (D == 12) { cudaFuncSetAttribute(ldgsts<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
                   timeit(name, [&] { ldgsts<12><<<1, 512, sm>>>(a, b, o, nv); }); }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
