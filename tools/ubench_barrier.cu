// Micro-benchmark (tuning aid): cost of one grid-wide barrier vs the number of
// participating CTAs, and a cluster-hierarchical barrier (barrier.cluster, then
// one atomic per cluster).  Informs the reach chain's barrier (ccl.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_barrier tools/ubench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int ITERS = 400;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_cg(int* sink) {
  cg::grid_group g = cg::this_grid();
  int x = 0;
  for (int i = 0; i < ITERS; ++i) {
    x += threadIdx.x ^ i;
    g.sync();
  }
  if (x == 12345678) *sink = x;
}

__global__ void k_ctr(unsigned* bar, int* sink) {
  const unsigned n = gridDim.x;
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
  if (x == 12345678) *sink = x;
}

// cluster-level barrier first, then one arrival per cluster
__global__ void k_cluster(unsigned* bar, int* sink) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned nclusters = gridDim.x / cl.num_blocks();
  int x = 0;
  for (int i = 0; i < ITERS; ++i) {
    x += threadIdx.x ^ i;
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned target = unsigned(i + 1) * nclusters;
      while (ld_acquire(bar) < target) {
      }
    }
    cl.sync();
  }
  if (x == 12345678) *sink = x;
}

int main() {
  int* sink;
  unsigned* bar;
  cudaMalloc(&sink, 4);
  cudaMalloc(&bar, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int block = 256;
  for (int per_sm : {1, 2, 4}) {
    const int grid = 148 * per_sm;
    for (int rep = 0; rep < 2; ++rep) {
      float ms;
      void* args_cg[] = {&sink};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, dim3(grid), dim3(block), args_cg, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%4d CTAs  cg grid.sync      %.3f us (%s)\n", grid, ms * 1e3 / ITERS,
                      cudaGetErrorString(cudaGetLastError()));
      cudaMemset(bar, 0, 8);
      void* args_ctr[] = {&bar, &sink};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_ctr, dim3(grid), dim3(block), args_ctr, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%4d CTAs  counter barrier   %.3f us (%s)\n", grid, ms * 1e3 / ITERS,
                      cudaGetErrorString(cudaGetLastError()));
      for (int cs : {2, 4}) {
        if (grid % cs) continue;
        cudaMemset(bar, 0, 8);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster, bar, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("%4d CTAs  cluster(%d)+ctr    %.3f us (%s / %s)\n", grid, cs,
                        ms * 1e3 / ITERS, cudaGetErrorString(e),
                        cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
