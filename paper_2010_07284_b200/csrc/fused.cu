// fused.cu -- one launch for a whole chain of thresholds and ! & | over
// bit-packed words (the north star's "chains of elementwise ops and
// thresholds are fused into single launches").
//
// The program (FusedProgram, slcs_internal.h) is a short register-machine
// listing passed by value as a kernel parameter, so every thread decodes the
// same op at the same time: the switch below is a uniform branch.  Bool-only
// listings run on 4-word (128-px) groups per thread; listings with u16
// thresholds (kernels.cpp:75-97, as an integer interval lo <= p <= hi) run one
// word per thread and never materialise a Bool image.
#include "slcs_internal.h"

namespace slcs {
namespace {

// The listing's registers hold 4-word groups (uint4) and live in shared
// memory, one 16 B lane-contiguous slot per thread and register (conflict-free
// 128-bit accesses): a runtime register index costs one LDS/STS instead of a
// chain of selects over a register array.
constexpr int kFusedBlock = 128;
struct Regs {
  uint4* base;  // &fregs[0][threadIdx.x]
  __device__ __forceinline__ uint4 get(int i) const { return base[i * kFusedBlock]; }
  __device__ __forceinline__ void set(int i, uint4 v) const { base[i * kFusedBlock] = v; }
};

// 8 threshold bits of the 8 u16 pixels in x (pixel e -> bit e)
__device__ __forceinline__ uint32_t thresh_byte(uint4 x, unsigned lo, unsigned span) {
  const uint32_t comp[4] = {x.x, x.y, x.z, x.w};
  uint32_t b = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    b |= ((comp[e] & 0xffffu) - lo <= span ? 1u : 0u) << (2 * e);
    b |= ((comp[e] >> 16) - lo <= span ? 1u : 0u) << (2 * e + 1);
  }
  return b;
}

// one word of `lo <= p <= hi` from its 64 B of u16 pixels (4 x 16 B loads)
__device__ __forceinline__ uint32_t thresh_word(const uint16_t* __restrict__ src, unsigned lo,
                                                unsigned span) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
  uint4 x[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) x[v] = __ldg(p + v);
  uint32_t w = 0;
#pragma unroll
  for (int v = 0; v < 4; ++v) w |= thresh_byte(x[v], lo, span) << (8 * v);
  return w;
}

// Listings with u16 thresholds: thread = one 32-px word per grid-stride step
// (the u16 operand dominates the traffic: 64 B per word, so a warp's 4 loads
// cover 2 KB contiguous), registers as u32 slots in shared memory.
template <int NB>
__global__ void __launch_bounds__(256) k_fused_words(const FusedProgram prog, int wpr,
                                                     uint32_t lastmask, size_t bpitch,
                                                     size_t upitch, size_t nwords) {
  slcs_pdl_wait();
  __shared__ uint32_t wregs[kFusedRegs][256];
  uint32_t* R = &wregs[0][threadIdx.x];
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords;
       q += size_t(gridDim.x) * blockDim.x) {
    const size_t row = q / bpitch;
    const int j = int(q - row * bpitch);
    const uint32_t vm = valid_mask(j, wpr, lastmask);
    uint32_t bin[NB > 0 ? NB : 1];
#pragma unroll
    for (int k = 0; k < NB; ++k) bin[k] = k < prog.n_bin ? __ldg(prog.bin[k] + q) : 0u;
    for (int i = 0; i < prog.n_ops; ++i) {
      const FusedOp op = prog.ops[i];
      switch (op.op) {
        case FOP_LOADB: {
          uint32_t v = bin[0];
#pragma unroll
          for (int k = 1; k < NB; ++k) v = (op.a == k) ? bin[k] : v;
          R[op.dst * 256] = v;
          break;
        }
        case FOP_THRESH:
          R[op.dst * 256] = (j < wpr && op.lo <= op.hi)
                                ? thresh_word(prog.uin[op.a] + row * upitch + size_t(j) * 32,
                                              unsigned(op.lo), unsigned(op.hi - op.lo)) & vm
                                : 0u;
          break;
        case FOP_NOT: R[op.dst * 256] = ~R[op.a * 256] & vm; break;
        case FOP_AND: R[op.dst * 256] = R[op.a * 256] & R[op.b * 256]; break;
        case FOP_OR: R[op.dst * 256] = R[op.a * 256] | R[op.b * 256]; break;
        case FOP_ANDNOT: R[op.dst * 256] = R[op.a * 256] & ~R[op.b * 256]; break;
        case FOP_STORE: prog.out[op.a][q] = R[op.dst * 256]; break;
        default: break;
      }
    }
  }
}

__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
  return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}

// Bool-only listings: thread = U 4-word groups (q, q + stride, ...) per
// grid-stride step.  The NB bool inputs of all U groups are loaded before the
// listing runs (U x NB independent 16 B loads in flight).  Padding bits/words
// are re-masked on NOT (zero-padding invariant).
template <int NB, int U>
__global__ void __launch_bounds__(kFusedBlock) k_fused(const FusedProgram prog, int wpr,
                                                       uint32_t lastmask, size_t bpitch,
                                                       size_t upitch, size_t ngroups) {
  slcs_pdl_wait();
  __shared__ uint4 fregs[kFusedRegs][kFusedBlock];
  const Regs R{&fregs[0][threadIdx.x]};
  const size_t pitch4 = bpitch / 4;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t q0 = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q0 < ngroups;
       q0 += U * stride) {
    uint4 bin[U][NB > 0 ? NB : 1];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const size_t q = q0 + u * stride;
        bin[u][k] = (k < prog.n_bin && q < ngroups)
                        ? __ldg(reinterpret_cast<const uint4*>(prog.bin[k]) + q)
                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t q = q0 + u * stride;
      if (q >= ngroups) break;
      const size_t row = q / pitch4;
      const int j0 = int(q - row * pitch4) * 4;
      const uint4 vm = make_uint4(valid_mask(j0, wpr, lastmask), valid_mask(j0 + 1, wpr, lastmask),
                                  valid_mask(j0 + 2, wpr, lastmask),
                                  valid_mask(j0 + 3, wpr, lastmask));
      for (int i = 0; i < prog.n_ops; ++i) {
        const FusedOp op = prog.ops[i];
        switch (op.op) {
          case FOP_LOADB: {
            uint4 v = bin[u][0];
#pragma unroll
            for (int k = 1; k < NB; ++k) v = (op.a == k) ? bin[u][k] : v;
            R.set(op.dst, v);
            break;
          }
          case FOP_NOT: {
            const uint4 v = R.get(op.a);
            R.set(op.dst, make_uint4(~v.x & vm.x, ~v.y & vm.y, ~v.z & vm.z, ~v.w & vm.w));
            break;
          }
          case FOP_AND: R.set(op.dst, and4(R.get(op.a), R.get(op.b))); break;
          case FOP_OR: {
            const uint4 x = R.get(op.a), y = R.get(op.b);
            R.set(op.dst, make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w));
            break;
          }
          case FOP_ANDNOT: {
            const uint4 x = R.get(op.a), y = R.get(op.b);
            R.set(op.dst, make_uint4(x.x & ~y.x, x.y & ~y.y, x.z & ~y.z, x.w & ~y.w));
            break;
          }
          case FOP_STORE:
            reinterpret_cast<uint4*>(prog.out[op.a])[q] = R.get(op.dst);
            break;
          default: break;
        }
      }
    }
  }
}

template <int NB, int U>
void fused_launch(const FusedProgram& p, const Geo& gb, const Geo& gu, cudaStream_t st) {
  const size_t groups = gb.slice * size_t(gb.batch) / 4;
  size_t blocks = (groups + kFusedBlock * U - 1) / (kFusedBlock * U);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  pdl(k_fused<NB, U>, unsigned(blocks), kFusedBlock, 0, st, p, gb.wpr, gb.lastmask,
      gb.pitch, gu.pitch, groups);
}

template <int NB>
void fused_words_launch(const FusedProgram& p, const Geo& gb, const Geo& gu, cudaStream_t st) {
  const size_t n = gb.slice * size_t(gb.batch);
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  pdl(k_fused_words<NB>, unsigned(blocks), 256, 0, st, p, gb.wpr, gb.lastmask, gb.pitch, gu.pitch,
      n);
}

}  // namespace

int launch_fused(const FusedProgram& p, const Geo& gb, const Geo& gu, cudaStream_t st) {
  bool has_t = false;
  for (int i = 0; i < p.n_ops; ++i) has_t |= p.ops[i].op == FOP_THRESH;
  if (has_t) {
    switch (p.n_bin) {
      case 0: fused_words_launch<0>(p, gb, gu, st); break;
      case 1: fused_words_launch<1>(p, gb, gu, st); break;
      case 2: fused_words_launch<2>(p, gb, gu, st); break;
      case 3:
      case 4: fused_words_launch<4>(p, gb, gu, st); break;
      default: fused_words_launch<kFusedMaxIn>(p, gb, gu, st); break;
    }
  } else {
    switch (p.n_bin) {
      case 0:
      case 1: fused_launch<1, 8>(p, gb, gu, st); break;
      case 2: fused_launch<2, 4>(p, gb, gu, st); break;
      case 3:
      case 4: fused_launch<4, 2>(p, gb, gu, st); break;
      default: fused_launch<kFusedMaxIn, 1>(p, gb, gu, st); break;
    }
  }
  return 1;
}

}  // namespace slcs
