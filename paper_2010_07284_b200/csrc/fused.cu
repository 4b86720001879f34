// fused.cu -- one launch for a whole chain of thresholds and ! & | over
// bit-packed words (the north star's "chains of elementwise ops and
// thresholds are fused into single launches").
//
// The program (FusedProgram, slcs_internal.h) is a short register-machine
// listing passed by value as a kernel parameter, so every thread decodes the
// same op at the same time: the switch below is a uniform branch, and the 8
// registers stay in registers (the accessors are fully unrolled selects).
// Each thread produces one 32-px word per output; u16 thresholds read their
// 64 B of pixels with 4 x 16 B loads and never materialise a Bool image.
#include "slcs_internal.h"

namespace slcs {
namespace {

struct Regs {
  uint32_t r[kFusedRegs];
  __device__ __forceinline__ uint32_t get(int i) const {
    uint32_t v = r[0];
#pragma unroll
    for (int k = 1; k < kFusedRegs; ++k) v = (i == k) ? r[k] : v;
    return v;
  }
  __device__ __forceinline__ void set(int i, uint32_t v) {
#pragma unroll
    for (int k = 0; k < kFusedRegs; ++k) r[k] = (i == k) ? v : r[k];
  }
};

__device__ __forceinline__ uint32_t thresh_word(const uint16_t* __restrict__ src, int lo, int hi) {
  if (lo > hi) return 0u;
  const unsigned span = unsigned(hi - lo);
  const uint4* p = reinterpret_cast<const uint4*>(src);
  uint32_t word = 0;
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    uint4 x = __ldg(p + v);
    uint32_t comp[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      unsigned p0 = comp[e] & 0xffffu, p1 = comp[e] >> 16;
      word |= (unsigned(p0 - unsigned(lo)) <= span ? 1u : 0u) << (v * 8 + e * 2);
      word |= (unsigned(p1 - unsigned(lo)) <= span ? 1u : 0u) << (v * 8 + e * 2 + 1);
    }
  }
  return word;
}

__global__ void k_fused(const FusedProgram prog, int wpr, uint32_t lastmask, size_t bpitch,
                        size_t upitch, size_t nwords_total) {
  slcs_pdl_wait();
  for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords_total;
       q += size_t(gridDim.x) * blockDim.x) {
    size_t row = q / bpitch;
    int j = int(q - row * bpitch);
    const bool valid = j < wpr;
    const uint32_t vmask = j < wpr - 1 ? 0xffffffffu : (j == wpr - 1 ? lastmask : 0u);
    Regs R;
#pragma unroll
    for (int k = 0; k < kFusedRegs; ++k) R.r[k] = 0;
    for (int i = 0; i < prog.n_ops; ++i) {
      const FusedOp op = prog.ops[i];
      switch (op.op) {
        case FOP_LOADB: R.set(op.dst, prog.bin[op.a][q]); break;
        case FOP_THRESH:
          R.set(op.dst, valid ? thresh_word(prog.uin[op.a] + row * upitch + size_t(j) * 32,
                                            op.lo, op.hi) & vmask
                              : 0u);
          break;
        case FOP_NOT: R.set(op.dst, ~R.get(op.a) & vmask); break;
        case FOP_AND: R.set(op.dst, R.get(op.a) & R.get(op.b)); break;
        case FOP_OR: R.set(op.dst, R.get(op.a) | R.get(op.b)); break;
        case FOP_ANDNOT: R.set(op.dst, R.get(op.a) & ~R.get(op.b)); break;
        case FOP_STORE: prog.out[op.a][q] = R.get(op.dst); break;
        default: break;
      }
    }
  }
}

}  // namespace

int launch_fused(const FusedProgram& p, const Geo& gb, const Geo& gu, cudaStream_t st) {
  size_t n = gb.slice * size_t(gb.batch);
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  pdl(k_fused, unsigned(blocks), 256, 0, st, p, gb.wpr, gb.lastmask, gb.pitch, gu.pitch, n);
  return 1;
}

}  // namespace slcs
