// probe_green.cu -- can a persistent spinning kernel own a green-context SM
// partition while ordinary kernels run on the rest? (design probe)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_green.cu -o tools/probe_green -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>
#include <stdlib.h>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* m; cuGetErrorString(r_, &m); \
  printf("%s -> %d %s (line %d)\n", #x, int(r_), m, __LINE__); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { \
  printf("%s -> %s (line %d)\n", #x, cudaGetErrorString(r_), __LINE__); return 1; } } while (0)

static inline double now_s() { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + t.tv_nsec * 1e-9; }

__global__ void spinner(volatile uint32_t* stop, uint32_t* smids) {
  if (threadIdx.x == 0) {
    uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smids[blockIdx.x] = s;
    while (*stop == 0) {}
  }
  __syncthreads();
}
__global__ void worker(float* x, size_t n, uint32_t* smids) {
  if (threadIdx.x == 0 && blockIdx.x < 1024) { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); smids[blockIdx.x] = s; }
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = x[i] * 1.0001f + 1.f;
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  RK(cudaSetDevice(0)); RK(cudaFree(0));
  CUcontext primary; CK(cuCtxGetCurrent(&primary));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  CUdevResource part[1], rest; unsigned ng = 1;
  CK(cuDevSmResourceSplitByCount(part, &ng, &all, &rest, 0, 16));
  printf("partition: %u groups, %u SMs; rest %u SMs\n", ng, part[0].sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dA, dB;
  CK(cuDevResourceGenerateDesc(&dA, part, 1));
  CK(cuDevResourceGenerateDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUcontext cA, cB; CK(cuCtxFromGreenCtx(&cA, gA)); CK(cuCtxFromGreenCtx(&cB, gB));
  uint32_t *stop, *smA, *smB;
  RK(cudaHostAlloc(&stop, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(stop, 0, 4096);
  // plain device memory: managed memory would make the driver serialise B behind A
  RK(cudaMalloc(&smA, 4096 * 4)); RK(cudaMalloc(&smB, 4096 * 4));
  static uint32_t hA[4096], hB[4096];
  float* x; RK(cudaMalloc(&x, size_t(64) << 20));
  // load every kernel in every context first: a lazy module load while the
  // spinner is resident would wait for it (the same trap as liblk's preload)
  cudaFuncAttributes fa;
  for (CUcontext c : {primary, cA, cB}) {
    CK(cuCtxSetCurrent(c));
    RK(cudaFuncGetAttributes(&fa, spinner));
    RK(cudaFuncGetAttributes(&fa, worker));
  }
  // A: spinner in partition A, one block per partition SM, cooperative
  CK(cuCtxSetCurrent(cA));
  cudaStream_t sA; RK(cudaStreamCreateWithFlags(&sA, cudaStreamNonBlocking));
  RK(cudaFuncSetAttribute(spinner, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
  unsigned nA = part[0].sm.smCount;
  void* args[] = {&stop, &smA};
  const bool coop = getenv("NOCOOP") == nullptr;
  cudaError_t le = coop ? cudaLaunchCooperativeKernel((void*)spinner, dim3(nA), dim3(512), args, 120 * 1024, sA)
                        : cudaLaunchKernel((void*)spinner, dim3(nA), dim3(512), args, 120 * 1024, sA);
  printf("%s launch of %u blocks in partition A: %s\n", coop ? "cooperative" : "plain", nA, cudaGetErrorString(le));
  usleep(100000);
  // B: ordinary kernel in partition B while A spins
  const bool inPrimary = getenv("BPRIMARY") != nullptr;
  CK(cuCtxSetCurrent(inPrimary ? primary : cB));
  printf("B runs in the %s context\n", inPrimary ? "primary" : "green B");
  cudaStream_t sB; RK(cudaStreamCreateWithFlags(&sB, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1));
  RK(cudaEventRecord(e0, sB));
  for (int k = 0; k < 10; ++k) worker<<<1024, 256, 0, sB>>>(x, (size_t(64) << 20) / 4, smB);
  RK(cudaEventRecord(e1, sB));
  double t0 = now_s();
  bool done = false;
  while (now_s() - t0 < 3.0) { if (cudaEventQuery(e1) == cudaSuccess) { done = true; break; } usleep(100); }
  printf("partition B kernels %s while A spins (%.3f s)\n", done ? "COMPLETED" : "did NOT complete", now_s() - t0);
  float ms = 0; if (done) { cudaEventElapsedTime(&ms, e0, e1); printf("B: 10 x 64 MiB read+write in %.3f ms -> %.0f GB/s\n", ms, 10 * 2 * 64.0 * 1048576 / (ms * 1e6)); }
  *(volatile uint32_t*)stop = 1;
  CK(cuCtxSetCurrent(cA)); RK(cudaStreamSynchronize(sA));
  CK(cuCtxSetCurrent(inPrimary ? primary : cB)); RK(cudaStreamSynchronize(sB));
  // SM sets
  CK(cuCtxSetCurrent(primary));
  RK(cudaMemcpy(hA, smA, sizeof hA, cudaMemcpyDeviceToHost)); RK(cudaMemcpy(hB, smB, sizeof hB, cudaMemcpyDeviceToHost));
  smA = hA; smB = hB;
  unsigned overlap = 0; bool inA[256] = {false};
  for (unsigned i = 0; i < nA; ++i) inA[smA[i] & 255] = true;
  for (int i = 0; i < 1024; ++i) if (inA[smB[i] & 255]) ++overlap;
  printf("A blocks on SMs:"); for (unsigned i = 0; i < nA; ++i) printf(" %u", smA[i]); printf("\n");
  printf("B blocks landing on A's SMs: %u of 1024\n", overlap);
  // primary-context kernel while A spins again?  (skipped: primary may use any SM)
  CK(cuCtxSetCurrent(primary));
  printf("ok\n");
  return 0;
}
