// Micro-benchmark (tuning aid): popcount of a 32 MiB bit image (16384^2), the
// volume primitive's shape, under several grid / unroll / epilogue choices.
// Each variant: 8 launches on 8 distinct images between CUDA events, L2 flushed
// before each group; time per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_volume tools/ubench_volume.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

// U unconditional loads per pass, tail one at a time; EPI 0: per-CTA partial
// stored to an array (no atomics), 1: atomicAdd + fence + done counter (last-CTA
// pattern), 2: one returning atomic on a packed (count << 20 | CTAs) word
template <int U, int EPI>
__global__ void k_pop(const uint4* __restrict__ a, size_t n4, unsigned long long* acc,
                      unsigned* done, unsigned long long* part_out, unsigned long long* out) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long local = 0;
  for (; q + (U - 1) * stride < n4; q += U * stride) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldg(a + q + u * stride);
    unsigned c = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) c += __popc(x[u].x) + __popc(x[u].y) + __popc(x[u].z) + __popc(x[u].w);
    local += c;
  }
  for (; q < n4; q += stride) {
    const uint4 x = __ldg(a + q);
    local += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) part[wid] = local;
  __syncthreads();
  if (wid == 0) {
    local = lane < int(blockDim.x >> 5) ? part[lane] : 0ull;
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if (lane == 0) {
      if (EPI == 0) {
        part_out[blockIdx.x] = local;
      } else if (EPI == 2) {
        const unsigned long long old = atomicAdd(acc, (local << 20) | 1ull);
        if ((old & 0xfffffull) == gridDim.x - 1) {
          *out = (old >> 20) + local;
          *acc = 0ull;
        }
      } else {
        if (local) atomicAdd(acc, local);
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
          __threadfence();
          *out = atomicExch(acc, 0ull);
          *done = 0u;
        }
      }
    }
  }
}

__global__ void k_flush(uint4* p, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_uint4(i, 0, 0, 0);
}

template <int U, int EPI>
void run(const char* name, const uint4* a, size_t n4, int grid, int block, unsigned long long* acc,
         unsigned* done, unsigned long long* part, unsigned long long* out, uint4* fl, size_t fln) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int rep = 0; rep < 25; ++rep) {
    k_flush<<<148 * 8, 256>>>(fl, fln);
    cudaEventRecord(e0);
    for (int c = 0; c < 8; ++c)  // 8 distinct images (256 MiB > L2), like bench.py's table
      k_pop<U, EPI><<<grid, block>>>(a + c * n4, n4, acc, done, part, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep >= 5) ts.push_back(ms * 1e3f / 8);
  }
  std::sort(ts.begin(), ts.end());
  const double gbs = double(n4) * 16 / (ts[ts.size() / 2] * 1e-6) / 1e9;
  printf("%-34s grid %5d x %4d  median %6.2f us  min %6.2f us  %7.1f GB/s (%s)\n", name, grid,
         block, ts[ts.size() / 2], ts[0], gbs, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t bytes = size_t(16384) * 16384 / 8;
  const size_t n4 = bytes / 16;
  uint4 *a, *fl;
  unsigned long long *acc, *part, *out;
  unsigned* done;
  const size_t fln = (size_t(512) << 20) / 16;
  cudaMalloc(&a, 8 * bytes);
  cudaMalloc(&fl, fln * 16);
  cudaMalloc(&acc, 8);
  cudaMalloc(&done, 4);
  cudaMalloc(&part, 8 * 65536);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0x5a, 8 * bytes);
  cudaMemset(acc, 0, 8);
  cudaMemset(done, 0, 4);
  run<8, 1>("U8 atomics (old grid)", a, n4, 1024, 256, acc, done, part, out, fl, fln);
  run<8, 2>("U8 packed atomic (old grid)", a, n4, 1024, 256, acc, done, part, out, fl, fln);
  run<8, 2>("U8 packed atomic 592x256", a, n4, 592, 256, acc, done, part, out, fl, fln);
  run<4, 2>("U4 packed atomic 2048x256", a, n4, 2048, 256, acc, done, part, out, fl, fln);
  run<1, 2>("empty, packed atomic", a, 0, 592, 256, acc, done, part, out, fl, fln);
  run<8, 0>("U8 partials (old grid)", a, n4, 1024, 256, acc, done, part, out, fl, fln);
  run<8, 1>("U8 atomics 592x256", a, n4, 592, 256, acc, done, part, out, fl, fln);
  run<16, 1>("U16 atomics 592x256", a, n4, 592, 256, acc, done, part, out, fl, fln);
  run<8, 1>("U8 atomics 1184x256", a, n4, 1184, 256, acc, done, part, out, fl, fln);
  run<4, 1>("U4 atomics 2048x256", a, n4, 2048, 256, acc, done, part, out, fl, fln);
  run<4, 1>("U4 atomics 1184x512", a, n4, 1184, 512, acc, done, part, out, fl, fln);
  run<2, 1>("U2 atomics 4096x256", a, n4, 4096, 256, acc, done, part, out, fl, fln);
  run<1, 1>("U1 atomics 8192x256", a, n4, 8192, 256, acc, done, part, out, fl, fln);
  run<1, 0>("U1 partials 8192x256", a, n4, 8192, 256, acc, done, part, out, fl, fln);
  run<16, 1>("U16 atomics 296x512", a, n4, 296, 512, acc, done, part, out, fl, fln);
  run<8, 1>("U8 atomics 296x1024", a, n4, 296, 1024, acc, done, part, out, fl, fln);
  // empty-kernel floor: n4 = 0
  run<1, 1>("empty (launch + epilogue)", a, 0, 592, 256, acc, done, part, out, fl, fln);
  return 0;
}
