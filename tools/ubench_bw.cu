// Micro-benchmark of near / volume kernel variants at 16384^2 (tuning aid,
// not product code).  Back-to-back launches over 8 rotating inputs (> L2),
// CUDA events around 64 launches; prints GB/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bw tools/ubench_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t vmask(int j, int wpr, uint32_t last) {
  return j < wpr - 1 ? 0xffffffffu : (j == wpr - 1 ? last : 0u);
}

template <int S, int BLOCK>
__global__ void __launch_bounds__(BLOCK) near1(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                               int h, int wpr, uint32_t last, int pitch4, int nstrips) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = t / pitch4, q = t - s * pitch4;
  if (s >= nstrips) return;
  uint4* dst = reinterpret_cast<uint4*>(out);
  const int r0 = s * S, j0 = 4 * q;
  const int rows = min(S, h - r0);
  const size_t pitch = size_t(pitch4) * 4;
  const bool has_l = j0 > 0, has_r = j0 + 4 < wpr;
  uint32_t hr[S + 2][4];
#pragma unroll
  for (int i = 0; i < S + 2; ++i) {
    const int r = r0 - 1 + i;
    uint32_t w[6];
    if (r < 0 || r >= h) {
#pragma unroll
      for (int e = 0; e < 6; ++e) w[e] = 0;
    } else {
      const uint32_t* row = in + size_t(r) * pitch;
      const uint4 c = __ldg(reinterpret_cast<const uint4*>(row + j0));
      w[0] = has_l ? __ldg(row + j0 - 1) : 0;
      w[1] = c.x; w[2] = c.y; w[3] = c.z; w[4] = c.w;
      w[5] = has_r ? __ldg(row + j0 + 4) : 0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      hr[i][e] = w[e + 1] | __funnelshift_l(w[e], w[e + 1], 1) | __funnelshift_r(w[e + 1], w[e + 2], 1);
  }
#pragma unroll
  for (int i = 0; i < S; ++i)
    if (i < rows) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = (hr[i][e] | hr[i + 1][e] | hr[i + 2][e]) & vmask(j0 + e, wpr, last);
      dst[size_t(r0 + i) * pitch4 + q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// shuffle variant: neighbours from adjacent lanes (rows wider than a warp)
template <int S, int BLOCK>
__global__ void __launch_bounds__(BLOCK) near1_shfl(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                    int h, int wpr, uint32_t last, int pitch4, int nstrips) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = t / pitch4, q = t - s * pitch4;
  const int lane = threadIdx.x & 31;
  uint4* dst = reinterpret_cast<uint4*>(out);
  const int r0 = s * S, j0 = 4 * q;
  const int rows = min(S, h - r0);
  const size_t pitch = size_t(pitch4) * 4;
  uint32_t hr[S + 2][4];
#pragma unroll
  for (int i = 0; i < S + 2; ++i) {
    const int r = r0 - 1 + i;
    uint4 c = make_uint4(0, 0, 0, 0);
    const bool ok = r >= 0 && r < h && s < nstrips;
    const uint32_t* row = in + size_t(r) * pitch;
    if (ok) c = __ldg(reinterpret_cast<const uint4*>(row + j0));
    uint32_t L = __shfl_up_sync(0xffffffffu, c.w, 1);
    uint32_t R = __shfl_down_sync(0xffffffffu, c.x, 1);
    if (lane == 0) L = (ok && j0 > 0) ? __ldg(row + j0 - 1) : 0;
    if (lane == 31) R = (ok && j0 + 4 < wpr) ? __ldg(row + j0 + 4) : 0;
    const uint32_t w[6] = {L, c.x, c.y, c.z, c.w, R};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      hr[i][e] = w[e + 1] | __funnelshift_l(w[e], w[e + 1], 1) | __funnelshift_r(w[e + 1], w[e + 2], 1);
  }
  if (s >= nstrips) return;
#pragma unroll
  for (int i = 0; i < S; ++i)
    if (i < rows) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) o[e] = (hr[i][e] | hr[i + 1][e] | hr[i + 2][e]) & vmask(j0 + e, wpr, last);
      dst[size_t(r0 + i) * pitch4 + q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

template <int UNR>
__global__ void vol(const uint4* __restrict__ a, size_t n4, unsigned long long* acc) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long local = 0;
  for (; q + (UNR - 1) * stride < n4; q += UNR * stride) {
    uint4 x[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) x[u] = __ldg(a + q + u * stride);
    unsigned c = 0;
#pragma unroll
    for (int u = 0; u < UNR; ++u) c += __popc(x[u].x) + __popc(x[u].y) + __popc(x[u].z) + __popc(x[u].w);
    local += c;
  }
  for (; q < n4; q += stride) {
    const uint4 x = __ldg(a + q);
    local += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(acc, local);
}

__global__ void copy4(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n4) {
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += size_t(gridDim.x) * blockDim.x)
    b[q] = a[q];
}

int main() {
  const int n = 16384, wpr = n / 32, pitch4 = wpr / 4;
  const size_t words = size_t(wpr) * n, bytes = words * 4;
  const int R = 8, REPS = 64;
  uint32_t *in[R], *out[R];
  for (int i = 0; i < R; ++i) {
    cudaMalloc(&in[i], bytes);
    cudaMalloc(&out[i], bytes);
    cudaMemset(in[i], 0x5a + i, bytes);
  }
  unsigned long long* acc;
  cudaMalloc(&acc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double bytes_per_launch, auto launch) {
    for (int i = 0; i < 8; ++i) launch(i % R);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < REPS; ++i) launch(i % R);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / REPS;
    printf("%-28s %8.2f us  %7.1f GB/s  (%s)\n", name, us, bytes_per_launch / us / 1e3,
           cudaGetErrorString(cudaGetLastError()));
  };
  const double nb = 2.0 * bytes;
#define NEAR(S, B)                                                                        \
  run("near S=" #S " B=" #B, nb, [&](int i) {                                           \
    int ns = (n + S - 1) / S;                                                             \
    size_t th = size_t(pitch4) * ns;                                                      \
    near1<S, B><<<unsigned((th + B - 1) / B), B>>>(in[i], out[i], n, wpr, ~0u, pitch4, ns); \
  });
  NEAR(4, 128) NEAR(8, 128) NEAR(16, 128) NEAR(8, 256) NEAR(16, 256) NEAR(32, 128)
#define NEARS(S, B)                                                                            \
  run("near_shfl S=" #S " B=" #B, nb, [&](int i) {                                           \
    int ns = (n + S - 1) / S;                                                                  \
    size_t th = size_t(pitch4) * ns;                                                           \
    near1_shfl<S, B><<<unsigned((th + B - 1) / B), B>>>(in[i], out[i], n, wpr, ~0u, pitch4, ns); \
  });
  NEARS(8, 128) NEARS(16, 128) NEARS(16, 256)
#define VOL(U, G)                                                                         \
  run("volume U=" #U " G=148x" #G, double(bytes), [&](int i) {                           \
    vol<U><<<148 * G, 256>>>(reinterpret_cast<const uint4*>(in[i]), words / 4, acc);     \
  });
  VOL(4, 4) VOL(4, 8) VOL(8, 8) VOL(8, 16) VOL(4, 16) VOL(2, 32) VOL(1, 64)
  run("copy (uint4, 148x16x256)", nb, [&](int i) {
    copy4<<<148 * 16, 256>>>(reinterpret_cast<const uint4*>(in[i]), reinterpret_cast<uint4*>(out[i]), words / 4);
  });
  run("cudaMemcpyAsync d2d", nb, [&](int i) { cudaMemcpyAsync(out[i], in[i], bytes, cudaMemcpyDeviceToDevice); });
  return 0;
}
