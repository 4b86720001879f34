// Micro-benchmark: cost of one grid-wide barrier for a co-resident cooperative
// grid shaped like the fused reach (512 CTAs x 512 threads, 4 per SM):
// cooperative_groups grid.sync() vs a counter barrier (tuning aid only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_gridsync tools/ubench_gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int ITERS = 200;

__global__ void __launch_bounds__(512, 4) k_cg(int* sink) {
  cg::grid_group g = cg::this_grid();
  int x = 0;
  for (int i = 0; i < ITERS; ++i) {
    x += threadIdx.x ^ i;
    g.sync();
  }
  if (x == 12345678) *sink = x;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(512, 4) k_ctr(unsigned* bar, int* sink) {
  const unsigned n = gridDim.x * gridDim.y;
  int x = 0;
  for (int i = 0; i < ITERS; ++i) {
    x += threadIdx.x ^ i;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned target = unsigned(i + 1) * n;
      while (ld_acquire(bar) < target) {
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && atomicAdd(bar + 1, 1u) == n - 1) {
    bar[0] = 0;
    bar[1] = 0;
  }
  if (x == 12345678) *sink = x;
}

int main() {
  int* sink;
  unsigned* bar;
  cudaMalloc(&sink, 4);
  cudaMalloc(&bar, 8);
  cudaMemset(bar, 0, 8);
  dim3 grid(16, 32), block(512);
  void* args_cg[] = {&sink};
  void* args_ctr[] = {&bar, &sink};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, grid, block, args_cg, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("cg grid.sync:   %.3f us per barrier (%s)\n", ms * 1e3 / ITERS,
           cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_ctr, grid, block, args_ctr, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("counter barrier: %.3f us per barrier (%s)\n", ms * 1e3 / ITERS,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
