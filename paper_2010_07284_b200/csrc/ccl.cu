// ccl.cu -- union-find connected components, reach and maxvol for sm_100a.
//
// Replaces the reference's pointer-jumping labelling (ccl::label,
// proj/src/ccl.cpp:127-165, paper Alg. 1) and the CCL-based reach
// (proj/src/reach.cpp:10-50) with block-based union-find:
//
//  * Union-find nodes are 2x2 pixel blocks: under 8-connectivity every
//    foreground pixel of a block is adjacent to every other one, so a block
//    is always inside one component (4x fewer nodes than pixels).
//  * A block's key is its row-first max foreground pixel, packed (r<<s)|c
//    (slcs_internal.h KeyGeo).  Linking always hangs the smaller root under
//    the larger (atomicMax), so every root is the block holding its
//    component's lexicographic-max pixel and the final label is exactly the
//    reference's canonical `max index + 1` (ccl.hpp:52-60) -- no relabel pass.
//  * Tiles of 64x64 px are resolved in shared memory; only tile-border links
//    touch global memory.  Images up to 256x256 (C1, the C3 slices) run as
//    one CTA per image with everything -- labelling, seeds, selection and the
//    closing near -- in shared memory, one launch per batch of slices.
//  * reach never materialises labels: seeds (through & near(target)) flag
//    local roots, flags propagate to global roots, and the selected
//    components are written as bits.
#include "slcs_internal.h"

namespace slcs {

KeyGeo key_geo(int w, int h) {
  KeyGeo k;
  int s = 1;
  while ((1ll << s) < (long long)w) ++s;
  k.s = s;
  k.cmask = (1u << s) - 1u;
  k.bw = (w + 1) / 2;
  k.bh = (h + 1) / 2;
  k.slice_blocks = size_t(k.bw) * size_t(k.bh);
  return k;
}

namespace {

// pattern bits of a 2x2 block: (r0,c0)=1 (r0,c0+1)=2 (r1,c0)=4 (r1,c0+1)=8
constexpr uint32_t P00 = 1, P01 = 2, P10 = 4, P11 = 8;

struct G {
  int W, H, wpr;
  size_t pitch, slice;  // bool layout (words)
  int BW, BH;
  int s;
  uint32_t cmask;
  size_t sb;  // blocks per slice
};

G make_g(const Geo& gb) {
  KeyGeo k = key_geo(gb.w, gb.h);
  G g;
  g.W = gb.w;
  g.H = gb.h;
  g.wpr = gb.wpr;
  g.pitch = gb.pitch;
  g.slice = gb.slice;
  g.BW = k.bw;
  g.BH = k.bh;
  g.s = k.s;
  g.cmask = k.cmask;
  g.sb = k.slice_blocks;
  return g;
}

__device__ __forceinline__ uint32_t load_pattern(const uint32_t* __restrict__ bits, const G& g,
                                                 int br, int bc) {
  if (br >= g.BH || bc >= g.BW || br < 0 || bc < 0) return 0;
  int r = 2 * br, c = 2 * bc;
  const uint32_t* row = bits + size_t(r) * g.pitch + (c >> 5);
  int sh = c & 31;
  uint32_t p = (__ldg(row) >> sh) & 3u;
  if (r + 1 < g.H) p |= ((__ldg(row + g.pitch) >> sh) & 3u) << 2;
  return p;
}

// 4 bits of row r at columns c-1..c+2 (bit 0 = column c-1); out of image = 0
__device__ __forceinline__ uint32_t window4(const uint32_t* __restrict__ bits, const G& g, int r,
                                            int c) {
  if (r < 0 || r >= g.H) return 0;
  const uint32_t* row = bits + size_t(r) * g.pitch;
  int j = c >> 5, sh = c & 31;
  uint32_t w0 = __ldg(row + j);
  if (sh == 0) {
    uint32_t wm = j > 0 ? __ldg(row + j - 1) : 0u;
    return (wm >> 31) | ((w0 << 1) & 14u);
  }
  uint32_t wp = (sh > 29 && j + 1 < g.wpr) ? __ldg(row + j + 1) : 0u;
  uint64_t x = (uint64_t(wp) << 32) | w0;
  return uint32_t(x >> (sh - 1)) & 15u;
}

// 2x2 pattern of near(t) at block (br, bc)
__device__ __forceinline__ uint32_t near_pattern(const uint32_t* __restrict__ t, const G& g,
                                                 int br, int bc) {
  int r = 2 * br, c = 2 * bc;
  uint32_t n[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t v = window4(t, g, r - 1 + i, c);
    n[i] = ((v | (v >> 1) | (v << 1)) >> 1) & 3u;
  }
  return (n[0] | n[1] | n[2]) | ((n[1] | n[2] | n[3]) << 2);
}

// ---------------------------------------------------------------------------
// shared-memory union-find over a tile of (1<<TBW_LOG) x tbh blocks
template <int TBW_LOG>
struct Tile {
  static constexpr int TBW = 1 << TBW_LOG;
  static constexpr int KW = TBW_LOG + 1;  // log2 tile width in pixels
  uint8_t* pat;
  uint32_t* par;
  int nb;

  __device__ __forceinline__ static int blk(uint32_t lk) {
    return int((lk >> (KW + 1)) << TBW_LOG) | int((lk & ((1u << KW) - 1u)) >> 1);
  }
  __device__ __forceinline__ static uint32_t key(int lb, uint32_t p) {
    int lbr = lb >> TBW_LOG, lbc = lb & (TBW - 1);
    int dr = (p & (P10 | P11)) ? 1 : 0;
    int dc = dr ? int((p >> 3) & 1u) : int((p >> 1) & 1u);
    return (uint32_t(2 * lbr + dr) << KW) | uint32_t(2 * lbc + dc);
  }
  // find with path halving (plain stores are safe: parents only ever move to
  // ancestors, and a racing atomicMax link is completed by the union loop)
  __device__ __forceinline__ uint32_t find(uint32_t k) const {
    volatile uint32_t* vp = par;
    for (;;) {
      uint32_t p = vp[blk(k)];
      if (p == k) return k;
      uint32_t gp = vp[blk(p)];
      if (gp == p) return p;
      vp[blk(k)] = gp;
      k = gp;
    }
  }
  __device__ __forceinline__ uint32_t find_ro(uint32_t k) const {
    volatile uint32_t* vp = par;
    uint32_t q = vp[blk(k)];
    while (q != k) {
      k = q;
      q = vp[blk(k)];
    }
    return k;
  }
  __device__ __forceinline__ void unite(uint32_t a, uint32_t b) const {
    for (;;) {
      a = find(a);
      b = find(b);
      if (a == b) return;
      if (a < b) {
        uint32_t t = a;
        a = b;
        b = t;
      }
      uint32_t old = atomicMax(par + blk(b), a);
      if (old == b) return;
      b = old;
    }
  }
  // True iff upper lanes lo..hi (any order) lie in one upper-row segment.
  __device__ __forceinline__ static bool same_seg(int a, int b, uint32_t hcu) {
    int lo = a < b ? a : b, hi = a < b ? b : a;
    if (lo < 0 || hi > 31) return false;
    if (lo == hi) return true;
    uint32_t m = (hi == 31 ? 0xffffffffu : ((2u << hi) - 1u)) & ~((2u << lo) - 1u);
    return (hcu & m) == m;
  }
  // Patterns must be in pat[].  Builds par[] and flattens it (par[lb] = root
  // key).  Warp-per-32-block row span:
  //  1. horizontal runs of connected blocks ("segments") are found with two
  //     ballots and every block points straight at its segment's max key --
  //     no atomics for horizontal adjacency;
  //  2. only links to the row above (and across span boundaries) need
  //     unions, and a link is skipped when the left neighbour in the same
  //     segment already links into the same upper segment, so a solid region
  //     costs one union per segment instead of three per block;
  //  3. flatten.
  __device__ void solve() const {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SPANS = TBW / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int items = (nb >> TBW_LOG) * SPANS;
    for (int it = warp; it < items; it += nw) {
      const int lbr = it / SPANS, lbc = (it % SPANS) * 32 + lane;
      const int lb = (lbr << TBW_LOG) | lbc;
      const uint32_t p = pat[lb];
      const uint32_t pl = __shfl_up_sync(FULL, p, 1);
      const uint32_t hc = __ballot_sync(FULL, lane > 0 && (p & (P00 | P10)) && (pl & (P01 | P11)));
      const uint32_t le = lane == 31 ? FULL : ((2u << lane) - 1u);
      const int s = 31 - __clz(~hc & le);
      const int e = lane == 31 ? 31 : lane + __ffs(~(hc >> (lane + 1))) - 1;
      const uint32_t segmask = (e == 31 ? FULL : ((2u << e) - 1u)) & ~((1u << s) - 1u);
      const uint32_t bot = __ballot_sync(FULL, (p & (P10 | P11)) != 0);
      const uint32_t cb = bot & segmask;
      const int ml = cb ? 31 - __clz(cb) : e;
      const uint32_t k = p ? key(lb, p) : 0u;
      const uint32_t rk = __shfl_sync(FULL, k, ml);
      par[lb] = p ? rk : 0xffffffffu;
    }
    __syncthreads();
    for (int it = warp; it < items; it += nw) {
      const int lbr = it / SPANS, lbc = (it % SPANS) * 32 + lane;
      const int lb = (lbr << TBW_LOG) | lbc;
      const uint32_t p = pat[lb];
      const bool up = lbr > 0;
      const uint32_t qu = up ? pat[lb - TBW] : 0u;
      const uint32_t qul = (up && lbc > 0) ? pat[lb - TBW - 1] : 0u;
      const uint32_t qur = (up && lbc < TBW - 1) ? pat[lb - TBW + 1] : 0u;
      uint32_t tset = ((p & P00) && (qul & P11) ? 1u : 0u) |
                      ((p & (P00 | P01)) && (qu & (P10 | P11)) ? 2u : 0u) |
                      ((p & P01) && (qur & P10) ? 4u : 0u);
      const uint32_t qleft = __shfl_up_sync(FULL, qu, 1);
      const uint32_t hcu =
          __ballot_sync(FULL, lane > 0 && (qu & (P00 | P10)) && (qleft & (P01 | P11)));
      const uint32_t pl = __shfl_up_sync(FULL, p, 1);
      const bool joined_left = lane > 0 && (p & (P00 | P10)) && (pl & (P01 | P11));
      const uint32_t prev = __shfl_up_sync(FULL, tset, 1);
      if (p) {
        const uint32_t mine = par[lb];
        if (lane == 0 && lbc > 0 && (p & (P00 | P10)) && (pat[lb - 1] & (P01 | P11)))
          unite(mine, par[lb - 1]);
        for (int t = 0; t < 3; ++t) {
          if (!(tset & (1u << t))) continue;
          const int j = lane - 1 + t;
          bool covered = false;
          if (joined_left)
            for (int t2 = 0; t2 < 3; ++t2)
              if ((prev & (1u << t2)) && same_seg(lane - 2 + t2, j, hcu)) covered = true;
          if (!covered) unite(mine, par[lb - TBW - 1 + t]);
        }
      }
      // reconverge: lanes leave their union loops at different times, and
      // the block barrier below must not release a partially-arrived warp
      __syncwarp();
    }
    __syncwarp();
    __syncthreads();
    // flatten: roots are found (with halving) into registers first and
    // written only after a barrier -- a halving write by another thread must
    // never overwrite a slot its owner already set to the final root
    constexpr int MAXPER = 16;  // nb <= 16 * blockDim.x on both paths
    uint32_t rr[MAXPER];
#pragma unroll
    for (int i = 0; i < MAXPER; ++i) {
      const int lb = threadIdx.x + i * int(blockDim.x);
      rr[i] = (lb < nb && pat[lb]) ? find(par[lb]) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MAXPER; ++i) {
      const int lb = threadIdx.x + i * int(blockDim.x);
      if (lb < nb && pat[lb]) par[lb] = rr[i];
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------
// global union-find over per-block values v = packed key + 1 (0 = empty)
__device__ __forceinline__ size_t gblk(const G& g, uint32_t v) {
  uint32_t k = v - 1u;
  return size_t((k >> g.s) >> 1) * size_t(g.BW) + size_t((k & g.cmask) >> 1);
}

// find during concurrent unions: L2-coherent loads, path halving
__device__ __forceinline__ uint32_t gfind_cg(uint32_t* P, const G& g, uint32_t v) {
  for (;;) {
    uint32_t p = __ldcg(P + gblk(g, v));
    if (p == v) return v;
    uint32_t gp = __ldcg(P + gblk(g, p));
    if (gp == p) return p;
    __stcg(P + gblk(g, v), gp);
    v = gp;
  }
}

__device__ void gunite(uint32_t* P, const G& g, uint32_t a, uint32_t b) {
  for (;;) {
    a = gfind_cg(P, g, a);
    b = gfind_cg(P, g, b);
    if (a == b) return;
    if (a < b) {
      uint32_t t = a;
      a = b;
      b = t;
    }
    uint32_t old = atomicMax(P + gblk(g, b), a);
    if (old == b) return;
    b = old;
  }
}

__device__ __forceinline__ uint32_t linear_label(const G& g, uint32_t v) {
  uint32_t k = v - 1u;
  return (k >> g.s) * uint32_t(g.W) + (k & g.cmask) + 1u;
}

// interleave: bit 2i <- x bit i, bit 2i+1 <- y bit i (16-bit inputs)
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// A warp holds 2x2 patterns of 32 consecutive blocks of one block row
// (bc0 = 32*k); writes the 2 words of each of the two pixel rows.
__device__ __forceinline__ void warp_store_patterns(uint32_t* __restrict__ out, const G& g,
                                                    int br, int bc0, uint32_t pat,
                                                    const uint32_t* __restrict__ orsrc) {
  const int lane = threadIdx.x & 31;
  uint32_t m0 = __ballot_sync(0xffffffffu, pat & P00);
  uint32_t m1 = __ballot_sync(0xffffffffu, pat & P01);
  uint32_t m2 = __ballot_sync(0xffffffffu, pat & P10);
  uint32_t m3 = __ballot_sync(0xffffffffu, pat & P11);
  if (lane < 4) {
    int rsel = lane >> 1, half = lane & 1;
    int r = 2 * br + rsel;
    int word = (bc0 >> 4) + half;  // 16 blocks = 32 px per word
    if (r < g.H && word < int(g.pitch)) {
      uint32_t x = rsel ? m2 : m0, y = rsel ? m3 : m1;
      if (half) {
        x >>= 16;
        y >>= 16;
      }
      uint32_t w = spread16(x) | (spread16(y) << 1);
      size_t idx = size_t(r) * g.pitch + size_t(word);
      if (orsrc) w |= orsrc[idx];
      out[idx] = w;
    }
  }
}

// ===========================================================================
// Large-image path: 64x64-px tiles, 3-5 launches.
constexpr int LT_LOG = 5;  // 32 blocks = 64 px wide
constexpr int LT_H = 64;   // 64 block rows = 128 px high
constexpr int LT_N = (1 << LT_LOG) * LT_H;
constexpr int LT_THREADS = 256;

enum { MODE_CCL = 0, MODE_REACH = 1 };

constexpr int LT_ROWS = 2 * LT_H;          // pixel rows per tile
constexpr int LT_WORDS = LT_ROWS * 2;       // 2 words (64 px) per row
constexpr int LT_LIST = 192;                // per-tile list: count + <= 188 ring roots

// near(t) word (r, j) from global bits: 3x3 OR, out of image = 0
__device__ __forceinline__ uint32_t near_word(const uint32_t* __restrict__ t, const G& g, int r,
                                              int j) {
  uint32_t acc = 0;
#pragma unroll
  for (int d = -1; d <= 1; ++d) {
    int rr = r + d;
    if (rr < 0 || rr >= g.H) continue;
    const uint32_t* row = t + size_t(rr) * g.pitch;
    uint32_t C = __ldg(row + j);
    uint32_t L = j > 0 ? __ldg(row + j - 1) : 0u;
    uint32_t R = j + 1 < g.wpr ? __ldg(row + j + 1) : 0u;
    acc |= C | __funnelshift_l(L, C, 1) | __funnelshift_r(C, R, 1);
  }
  return acc;
}

// 2x2 pattern of block (lbr, lbc) from a staged 2-word-wide tile of rows
__device__ __forceinline__ uint32_t staged_pattern(const uint32_t* w, int lbr, int lbc) {
  const int jj = lbc >> 4, sh = (2 * lbc) & 31;
  return ((w[(2 * lbr) * 2 + jj] >> sh) & 3u) | (((w[(2 * lbr + 1) * 2 + jj] >> sh) & 3u) << 2);
}

// Tile-local pass.  Writes, per block, P = local root key + 1 (0 = empty);
// per local root, F = "holds a seed" (reach); and a per-tile list of the
// local roots that touch the tile ring -- the only ones a border union can
// link, so the only ones the root-flatten pass must visit.
template <int MODE>
__global__ void __launch_bounds__(LT_THREADS) k_tile_local(const uint32_t* __restrict__ ubits,
                                                           const uint32_t* __restrict__ tbits,
                                                           uint32_t* __restrict__ P,
                                                           uint8_t* __restrict__ F,
                                                           uint32_t* __restrict__ lists, G g) {
  __shared__ uint8_t pat[LT_N];
  __shared__ uint32_t par[LT_N];
  __shared__ uint8_t touch[LT_N];
  __shared__ uint8_t fl[MODE == MODE_REACH ? LT_N : 1];
  __shared__ uint32_t su[LT_WORDS];
  __shared__ uint32_t snt[MODE == MODE_REACH ? LT_WORDS : 1];
  __shared__ int s_cnt;
  using T = Tile<LT_LOG>;
  const int slice = blockIdx.z;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const int tbr0 = blockIdx.y * LT_H, tbc0 = blockIdx.x * T::TBW;
  const int r0 = 2 * tbr0, c0 = 2 * tbc0, j0 = c0 >> 5;
  // stage the tile's bit rows (and near(target) rows) in shared memory
  for (int q = threadIdx.x; q < LT_WORDS; q += blockDim.x) {
    const int r = r0 + (q >> 1), j = j0 + (q & 1);
    const bool in = r < g.H && j < g.wpr;
    su[q] = in ? __ldg(u + size_t(r) * g.pitch + j) : 0u;
    if (MODE == MODE_REACH)
      snt[q] = in ? near_word(tbits + size_t(slice) * g.slice, g, r, j) : 0u;
  }
  for (int lb = threadIdx.x; lb < LT_N; lb += blockDim.x) {
    touch[lb] = 0;
    if (MODE == MODE_REACH) fl[lb] = 0;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  for (int lb = threadIdx.x; lb < LT_N; lb += blockDim.x)
    pat[lb] = uint8_t(staged_pattern(su, lb >> LT_LOG, lb & (T::TBW - 1)));
  __syncthreads();
  T tile{pat, par, LT_N};
  tile.solve();

  uint32_t* Ps = P + size_t(slice) * g.sb;
  for (int lb = threadIdx.x; lb < LT_N; lb += blockDim.x) {
    const uint32_t p = pat[lb];
    const int lbr = lb >> LT_LOG, lbc = lb & (T::TBW - 1);
    const int br = tbr0 + lbr, bc = tbc0 + lbc;
    uint32_t v = 0;
    if (p) {
      const uint32_t lk = par[lb];
      const uint32_t gr = uint32_t(r0) + (lk >> T::KW);
      const uint32_t gc = uint32_t(c0) + (lk & ((1u << T::KW) - 1u));
      v = ((gr << g.s) | gc) + 1u;
      if (lbr == 0 || lbr == LT_H - 1 || lbc == 0 || lbc == T::TBW - 1) touch[T::blk(lk)] = 1;
      if (MODE == MODE_REACH && (p & staged_pattern(snt, lbr, lbc))) fl[T::blk(lk)] = 1;
    }
    if (br < g.BH && bc < g.BW) Ps[size_t(br) * g.BW + bc] = v;
  }
  __syncthreads();
  const size_t tile_id = (size_t(slice) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  uint32_t* L = lists + tile_id * LT_LIST;
  for (int lb = threadIdx.x; lb < LT_N; lb += blockDim.x) {
    const uint32_t p = pat[lb];
    if (!p || par[lb] != T::key(lb, p)) continue;  // local roots only
    const int br = tbr0 + (lb >> LT_LOG), bc = tbc0 + (lb & (T::TBW - 1));
    const size_t gbi = size_t(br) * g.BW + bc;
    if (MODE == MODE_REACH) F[size_t(slice) * g.sb + gbi] = fl[lb];
    if (touch[lb]) L[1 + atomicAdd(&s_cnt, 1)] = Ps[gbi];
  }
  __syncthreads();
  if (threadIdx.x == 0) L[0] = uint32_t(s_cnt);
}

// read-only find (concurrent writers only ever store final roots)
__device__ __forceinline__ uint32_t gfind_ro(const uint32_t* P, const G& g, uint32_t v) {
  uint32_t q = __ldcg(P + gblk(g, v));
  while (q != v) {
    v = q;
    q = __ldcg(P + gblk(g, v));
  }
  return v;
}

// After the border merge: every ring-touching local root points straight at
// its global root (and hands its seed flag over, for reach).  Afterwards any
// block's global root is exactly two loads away: P[b] -> P[local root].
__global__ void k_root_flatten(uint32_t* P, uint8_t* F, const uint32_t* __restrict__ lists, G g,
                               int ntiles, int reach) {
  const int slice = blockIdx.y;
  const int tile = int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (tile >= ntiles) return;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  uint8_t* Fs = reach ? F + size_t(slice) * g.sb : nullptr;
  const uint32_t* L = lists + (size_t(slice) * ntiles + tile) * LT_LIST;
  const int n = int(L[0]);
  for (int i = lane; i < n; i += 32) {
    const uint32_t r = L[1 + i];
    const uint32_t R = gfind_ro(Ps, g, r);
    if (R != r) {
      Ps[gblk(g, r)] = R;
      if (reach && Fs[gblk(g, r)]) Fs[gblk(g, R)] = 1;
    }
  }
}

// global root of a block after k_root_flatten (v = P[b] != 0)
__device__ __forceinline__ uint32_t groot(const uint32_t* P, const G& g, uint32_t v) {
  return P[gblk(g, v)];
}

// unions across tile borders (see DESIGN.md for the link enumeration)
__global__ void k_tile_merge(const uint32_t* __restrict__ ubits, uint32_t* P, G g, int nhb,
                             int nvb) {
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const long long nA = (long long)nhb * g.BW, nB = (long long)nvb * g.BH;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nA + nB;
       i += (long long)gridDim.x * blockDim.x) {
    if (i < nA) {
      int t = int(i / g.BW), bc = int(i - (long long)t * g.BW);
      int br = (t + 1) * LT_H;
      uint32_t p = load_pattern(u, g, br, bc);
      if (!(p & (P00 | P01))) continue;
      uint32_t vx = Ps[size_t(br) * g.BW + bc];
      uint32_t q = load_pattern(u, g, br - 1, bc);
      if (q & (P10 | P11)) gunite(Ps, g, vx, Ps[size_t(br - 1) * g.BW + bc]);
      if (bc > 0 && (p & P00)) {
        q = load_pattern(u, g, br - 1, bc - 1);
        if (q & P11) gunite(Ps, g, vx, Ps[size_t(br - 1) * g.BW + bc - 1]);
      }
      if (bc + 1 < g.BW && (p & P01)) {
        q = load_pattern(u, g, br - 1, bc + 1);
        if (q & P10) gunite(Ps, g, vx, Ps[size_t(br - 1) * g.BW + bc + 1]);
      }
    } else {
      long long j = i - nA;
      int t = int(j / g.BH), br = int(j - (long long)t * g.BH);
      int bc = (t + 1) * (1 << LT_LOG);
      uint32_t px = load_pattern(u, g, br, bc);
      uint32_t py = load_pattern(u, g, br, bc - 1);
      uint32_t vx = px ? Ps[size_t(br) * g.BW + bc] : 0u;
      uint32_t vy = py ? Ps[size_t(br) * g.BW + bc - 1] : 0u;
      if ((px & (P00 | P10)) && (py & (P01 | P11))) gunite(Ps, g, vx, vy);
      if (br % LT_H != 0) {
        if (px & P00) {
          uint32_t q = load_pattern(u, g, br - 1, bc - 1);
          if (q & P11) gunite(Ps, g, vx, Ps[size_t(br - 1) * g.BW + bc - 1]);
        }
        if (py & P01) {
          uint32_t q = load_pattern(u, g, br - 1, bc);
          if (q & P10) gunite(Ps, g, vy, Ps[size_t(br - 1) * g.BW + bc]);
        }
      }
    }
  }
}

// labels: one thread per block, 2 rows x 2 px each
__global__ void k_tile_labels(const uint32_t* __restrict__ ubits, uint32_t* P,
                              uint32_t* __restrict__ L, G g) {
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  uint32_t* Ls = L + size_t(slice) * size_t(g.W) * size_t(g.H);
  const bool even = (g.W & 1) == 0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < g.sb;
       i += size_t(gridDim.x) * blockDim.x) {
    int br = int(i / g.BW), bc = int(i - size_t(br) * g.BW);
    uint32_t v = Ps[i];
    uint32_t lab = 0, p = 0;
    if (v) {
      lab = linear_label(g, groot(Ps, g, v));
      p = load_pattern(u, g, br, bc);
    }
    int r = 2 * br, c = 2 * bc;
    size_t o = size_t(r) * g.W + c;
    uint32_t a0 = (p & P00) ? lab : 0u, a1 = (p & P01) ? lab : 0u;
    uint32_t b0 = (p & P10) ? lab : 0u, b1 = (p & P11) ? lab : 0u;
    if (even) {
      *reinterpret_cast<uint2*>(Ls + o) = make_uint2(a0, a1);
      if (r + 1 < g.H) *reinterpret_cast<uint2*>(Ls + o + g.W) = make_uint2(b0, b1);
    } else {
      Ls[o] = a0;
      if (c + 1 < g.W) Ls[o + 1] = a1;
      if (r + 1 < g.H) {
        Ls[o + g.W] = b0;
        if (c + 1 < g.W) Ls[o + g.W + 1] = b1;
      }
    }
  }
}

// reach: out bits = target | (through components with a flagged root).
// Warp = 32 consecutive blocks of one block row; covers the full row pitch.
__global__ void k_reach_select(const uint32_t* __restrict__ ubits,
                               const uint32_t* __restrict__ tbits,
                               uint32_t* P, const uint8_t* __restrict__ F,
                               uint32_t* __restrict__ out, G g) {
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint8_t* Fs = F + size_t(slice) * g.sb;
  const int wpb = int(g.pitch / 2);  // warps per block row (2 words per warp)
  const long long nw = (long long)g.BH * wpb;
  const int lane = threadIdx.x & 31;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    int br = int(w / wpb), bc0 = int(w - (long long)br * wpb) * 32;
    int bc = bc0 + lane;
    uint32_t p = 0;
    if (bc < g.BW) {
      uint32_t v = Ps[size_t(br) * g.BW + bc];
      if (v && Fs[gblk(g, groot(Ps, g, v))]) p = load_pattern(u, g, br, bc);
    }
    warp_store_patterns(out + size_t(slice) * g.slice, g, br, bc0, p,
                        tbits + size_t(slice) * g.slice);
  }
}

// maxvol: component sizes accumulated at the root block
__global__ void k_maxvol_size(const uint32_t* __restrict__ ubits, uint32_t* P,
                              uint32_t* SZ, G g) {
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  uint32_t* Ss = SZ + size_t(slice) * g.sb;
  // grid-stride with whole warps alive for __match_any_sync
  const size_t n = g.sb;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t base = size_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    size_t i = base + threadIdx.x;
    uint32_t v = 0, cnt = 0;
    size_t rb = ~size_t(0);
    if (i < n) {
      v = Ps[i];
      if (v) {
        int br = int(i / g.BW), bc = int(i - size_t(br) * g.BW);
        cnt = __popc(load_pattern(u, g, br, bc));
        rb = gblk(g, groot(Ps, g, v));
      }
    }
    unsigned peers = __match_any_sync(0xffffffffu, (unsigned long long)rb);
    int leader = __ffs(peers) - 1;
    uint32_t sum = __reduce_add_sync(peers, cnt);
    if ((threadIdx.x & 31) == leader && v) atomicAdd(Ss + rb, sum);
  }
}

__global__ void k_maxvol_max(uint32_t* P, const uint32_t* __restrict__ SZ,
                             unsigned int* maxv, G g) {
  const int slice = blockIdx.y;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* Ss = SZ + size_t(slice) * g.sb;
  uint32_t best = 0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < g.sb;
       i += size_t(gridDim.x) * blockDim.x) {
    uint32_t v = Ps[i];
    if (v && gblk(g, v) == i) best = max(best, Ss[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(maxv + slice, best);
}

__global__ void k_maxvol_select(const uint32_t* __restrict__ ubits,
                                uint32_t* P, const uint32_t* __restrict__ SZ,
                                const unsigned int* __restrict__ maxv, uint32_t* __restrict__ out,
                                G g) {
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* Ss = SZ + size_t(slice) * g.sb;
  const uint32_t mx = maxv[slice];
  const int wpb = int(g.pitch / 2);
  const long long nw = (long long)g.BH * wpb;
  const int lane = threadIdx.x & 31;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    int br = int(w / wpb), bc0 = int(w - (long long)br * wpb) * 32;
    int bc = bc0 + lane;
    uint32_t p = 0;
    if (bc < g.BW) {
      uint32_t v = Ps[size_t(br) * g.BW + bc];
      if (v && Ss[gblk(g, groot(Ps, g, v))] == mx) p = load_pattern(u, g, br, bc);
    }
    warp_store_patterns(out + size_t(slice) * g.slice, g, br, bc0, p, nullptr);
  }
}

// ===========================================================================
// Small-image path: one CTA per image (W, H <= 256), everything in smem.
constexpr int ST_LOG = 7;  // 128 blocks = 256 px
constexpr int ST_THREADS = 1024;

struct SmallLayout {
  int nb;  // 128 * BH
  size_t off_par, off_pat, off_aux, off_bits, total;
};

SmallLayout small_layout(int bh, int pitch_words, int h, int mode) {
  SmallLayout s;
  s.nb = (1 << ST_LOG) * bh;
  s.off_par = 0;
  s.off_pat = s.off_par + size_t(s.nb) * 4;
  s.off_aux = s.off_pat + round_up(size_t(s.nb), 16);
  size_t aux = mode == 2 ? size_t(s.nb) * 4 : (mode == 1 ? round_up(size_t(s.nb), 16) : 0);
  s.off_bits = s.off_aux + aux;
  size_t bits = mode == 1 ? size_t(pitch_words) * size_t(h) * 4 : 0;
  s.total = s.off_bits + bits + 64;
  return s;
}

// mode 0 = labels, 1 = reach, 2 = maxvol
template <int MODE>
__global__ void __launch_bounds__(ST_THREADS) k_small(const uint32_t* __restrict__ ubits,
                                                      const uint32_t* __restrict__ tbits,
                                                      uint32_t* __restrict__ out, G g,
                                                      SmallLayout lay) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* par = reinterpret_cast<uint32_t*>(smem + lay.off_par);
  uint8_t* pat = smem + lay.off_pat;
  using T = Tile<ST_LOG>;
  const int slice = blockIdx.x;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const int nb = lay.nb;
  for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) {
    int br = lb >> ST_LOG, bc = lb & (T::TBW - 1);
    pat[lb] = uint8_t(load_pattern(u, g, br, bc));
  }
  if (MODE == 1) {
    uint8_t* fl = smem + lay.off_aux;
    for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) fl[lb] = 0;
  }
  if (MODE == 2) {
    uint32_t* sz = reinterpret_cast<uint32_t*>(smem + lay.off_aux);
    for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) sz[lb] = 0;
  }
  __syncthreads();
  T tile{pat, par, nb};
  tile.solve();

  if (MODE == 0) {
    uint32_t* Ls = out + size_t(slice) * size_t(g.W) * size_t(g.H);
    // row-major over pixels for coalesced stores
    const size_t npx = size_t(g.W) * g.H;
    for (size_t i = threadIdx.x; i < npx; i += blockDim.x) {
      int r = int(i / g.W), c = int(i - size_t(r) * g.W);
      int lb = ((r >> 1) << ST_LOG) | (c >> 1);
      uint32_t p = pat[lb];
      uint32_t bit = 1u << (((r & 1) << 1) | (c & 1));
      uint32_t lab = 0;
      if (p & bit) {
        uint32_t lk = par[lb];
        lab = (lk >> T::KW) * uint32_t(g.W) + (lk & ((1u << T::KW) - 1u)) + 1u;
      }
      Ls[i] = lab;
    }
    return;
  }
  if (MODE == 1) {
    uint8_t* fl = smem + lay.off_aux;
    uint32_t* sb = reinterpret_cast<uint32_t*>(smem + lay.off_bits);
    const uint32_t* t = tbits + size_t(slice) * g.slice;
    for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) {
      uint32_t p = pat[lb];
      if (!p) continue;
      int br = lb >> ST_LOG, bc = lb & (T::TBW - 1);
      if (p & near_pattern(t, g, br, bc)) fl[T::blk(par[lb])] = 1;
    }
    __syncthreads();
    // S | t into smem bit rows (one thread per word)
    const int nwords = int(g.pitch) * g.H;
    for (int q = threadIdx.x; q < nwords; q += blockDim.x) {
      int r = q / int(g.pitch), j = q - r * int(g.pitch);
      uint32_t w = t[q];
      if (j < g.wpr) {
        int br = r >> 1, sh = (r & 1) << 1;
        for (int k = 0; k < 16; ++k) {
          int bc = j * 16 + k;
          if (bc >= g.BW) break;
          int lb = (br << ST_LOG) | bc;
          uint32_t p = pat[lb];
          if (p && fl[T::blk(par[lb])]) w |= ((p >> sh) & 3u) << (2 * k);
        }
      }
      sb[q] = w;
    }
    __syncthreads();
    // closing near over the smem rows
    uint32_t* o = out + size_t(slice) * g.slice;
    for (int q = threadIdx.x; q < nwords; q += blockDim.x) {
      int r = q / int(g.pitch), j = q - r * int(g.pitch);
      uint32_t acc = 0;
      if (j < g.wpr) {
        for (int rr = max(0, r - 1); rr <= min(g.H - 1, r + 1); ++rr) {
          const uint32_t* row = sb + rr * int(g.pitch);
          uint32_t C = row[j];
          uint32_t L = j > 0 ? row[j - 1] : 0u;
          uint32_t R = j + 1 < g.wpr ? row[j + 1] : 0u;
          acc |= C | __funnelshift_l(L, C, 1) | __funnelshift_r(C, R, 1);
        }
        acc &= j == g.wpr - 1 ? ((g.W & 31) ? ((1u << (g.W & 31)) - 1u) : 0xffffffffu)
                              : 0xffffffffu;
      }
      o[q] = acc;
    }
    return;
  }
  if (MODE == 2) {
    uint32_t* sz = reinterpret_cast<uint32_t*>(smem + lay.off_aux);
    __shared__ unsigned int s_max;
    if (threadIdx.x == 0) s_max = 0;
    // nb is a multiple of 32, so every warp runs whole iterations
    for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) {
      uint32_t p = pat[lb];
      int rb = p ? T::blk(par[lb]) : -1;
      unsigned peers = __match_any_sync(0xffffffffu, rb);
      uint32_t sum = __reduce_add_sync(peers, uint32_t(__popc(p)));
      if (p && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(sz + rb, sum);
    }
    __syncthreads();
    uint32_t best = 0;
    for (int lb = threadIdx.x; lb < nb; lb += blockDim.x) best = max(best, sz[lb]);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o2));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(&s_max, best);
    __syncthreads();
    const uint32_t mx = s_max;
    uint32_t* o = out + size_t(slice) * g.slice;
    const int nwords = int(g.pitch) * g.H;
    for (int q = threadIdx.x; q < nwords; q += blockDim.x) {
      int r = q / int(g.pitch), j = q - r * int(g.pitch);
      uint32_t w = 0;
      if (j < g.wpr && mx) {
        int br = r >> 1, sh = (r & 1) << 1;
        for (int k = 0; k < 16; ++k) {
          int bc = j * 16 + k;
          if (bc >= g.BW) break;
          int lb = (br << ST_LOG) | bc;
          uint32_t p = pat[lb];
          if (p && sz[T::blk(par[lb])] == mx) w |= ((p >> sh) & 3u) << (2 * k);
        }
      }
      o[q] = w;
    }
  }
}

template <int MODE>
int small_launch(const uint32_t* u, const uint32_t* t, uint32_t* out, const G& g, int batch,
                 int pitch, cudaStream_t st) {
  SmallLayout lay = small_layout(g.BH, pitch, g.H, MODE);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_small<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_small<MODE><<<batch, ST_THREADS, lay.total, st>>>(u, t, out, g, lay);
  return 1;
}

int grid_blocks(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return int(b);
}

void check_label_range(const Geo& gb) {
  KeyGeo k = key_geo(gb.w, gb.h);
  unsigned long long maxkey = ((unsigned long long)(gb.h - 1) << k.s) | (unsigned long long)(gb.w - 1);
  if ((unsigned long long)gb.w * (unsigned long long)gb.h >= 0xfffffffeull || maxkey + 1 >= 0xffffffffull)
    fail(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
}

}  // namespace

bool ccl_small_path(int w, int h) { return w <= 256 && h <= 256; }

static size_t n_tiles(const KeyGeo& k) {
  return size_t((k.bw + 31) / 32) * size_t((k.bh + LT_H - 1) / LT_H);
}

size_t ccl_scratch_bytes(int w, int h, int batch, bool flags, bool sizes) {
  if (ccl_small_path(w, h)) return 0;
  KeyGeo k = key_geo(w, h);
  size_t n = k.slice_blocks * size_t(batch);
  size_t b = round_up(n * 4, 256) + round_up(n_tiles(k) * size_t(batch) * LT_LIST * 4, 256);
  if (flags) b += round_up(n, 256);
  if (sizes) b += round_up(n * 4, 256) + round_up(size_t(batch) * 4, 256);
  return b;
}

void ccl_scratch_carve(void* base, int w, int h, int batch, bool flags, bool sizes,
                       CclScratch* s) {
  *s = CclScratch{};
  if (ccl_small_path(w, h)) return;
  KeyGeo k = key_geo(w, h);
  size_t n = k.slice_blocks * size_t(batch);
  unsigned char* p = static_cast<unsigned char*>(base);
  s->parent = reinterpret_cast<uint32_t*>(p);
  p += round_up(n * 4, 256);
  s->lists = reinterpret_cast<uint32_t*>(p);
  p += round_up(n_tiles(k) * size_t(batch) * LT_LIST * 4, 256);
  if (flags) {
    s->flag = p;
    p += round_up(n, 256);
  }
  if (sizes) {
    s->size = reinterpret_cast<uint32_t*>(p);
    p += round_up(n * 4, 256);
    s->maxv = reinterpret_cast<unsigned int*>(p);
  }
}

static void large_local_and_merge(const uint32_t* u, const uint32_t* t, const G& g, int batch,
                                  CclScratch& s, bool reach, cudaStream_t st, int& launches) {
  dim3 grid(unsigned((g.BW + 31) / 32), unsigned((g.BH + LT_H - 1) / LT_H), unsigned(batch));
  if (reach)
    k_tile_local<MODE_REACH><<<grid, LT_THREADS, 0, st>>>(u, t, s.parent, s.flag, s.lists, g);
  else
    k_tile_local<MODE_CCL><<<grid, LT_THREADS, 0, st>>>(u, t, s.parent, s.flag, s.lists, g);
  ++launches;
  int nhb = int(grid.y) - 1, nvb = int(grid.x) - 1;
  size_t links = size_t(nhb) * g.BW + size_t(nvb) * g.BH;
  if (links) {
    dim3 mg(unsigned(grid_blocks(links, 256)), unsigned(batch));
    k_tile_merge<<<mg, 256, 0, st>>>(u, s.parent, g, nhb, nvb);
    int ntiles = int(grid.x * grid.y);
    dim3 fg(unsigned((ntiles * 32 + 255) / 256), unsigned(batch));
    k_root_flatten<<<fg, 256, 0, st>>>(s.parent, s.flag, s.lists, g, ntiles, reach ? 1 : 0);
    launches += 2;
  }
}

int launch_ccl(const uint32_t* bits, uint32_t* labels, const Geo& gb, CclScratch& s,
               cudaStream_t st) {
  check_label_range(gb);
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h))
    return small_launch<0>(bits, nullptr, labels, g, gb.batch, int(gb.pitch), st);
  int launches = 0;
  large_local_and_merge(bits, nullptr, g, gb.batch, s, false, st, launches);
  dim3 lg(unsigned(grid_blocks(g.sb, 256)), unsigned(gb.batch));
  k_tile_labels<<<lg, 256, 0, st>>>(bits, s.parent, labels, g);
  return launches + 1;
}

int launch_reach(const uint32_t* target, const uint32_t* through, uint32_t* out,
                 uint32_t* tmp_bits, const Geo& gb, CclScratch& s, cudaStream_t st) {
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h))
    return small_launch<1>(through, target, out, g, gb.batch, int(gb.pitch), st);
  // keys are internal here (no label output), but must still fit 32 bits
  KeyGeo k = key_geo(gb.w, gb.h);
  if ((((unsigned long long)(gb.h - 1) << k.s) | (unsigned long long)(gb.w - 1)) + 1 >=
      0xffffffffull)
    fail(SLCS_ERR_TOO_LARGE, "reach: image too large for 32-bit block keys");
  int launches = 0;
  large_local_and_merge(through, target, g, gb.batch, s, true, st, launches);
  size_t warps = size_t(g.BH) * (gb.pitch / 2);
  dim3 sg(unsigned(grid_blocks(warps * 32, 256)), unsigned(gb.batch));
  k_reach_select<<<sg, 256, 0, st>>>(through, target, s.parent, s.flag, tmp_bits, g);
  launches += 1;
  launches += launch_near(tmp_bits, out, gb, 1, false, st);
  return launches;
}

int launch_maxvol(const uint32_t* bits, uint32_t* out, const Geo& gb, CclScratch& s,
                  cudaStream_t st) {
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h))
    return small_launch<2>(bits, nullptr, out, g, gb.batch, int(gb.pitch), st);
  KeyGeo k = key_geo(gb.w, gb.h);
  if ((((unsigned long long)(gb.h - 1) << k.s) | (unsigned long long)(gb.w - 1)) + 1 >=
      0xffffffffull)
    fail(SLCS_ERR_TOO_LARGE, "maxvol: image too large for 32-bit block keys");
  int launches = 0;
  large_local_and_merge(bits, nullptr, g, gb.batch, s, false, st, launches);
  cudaMemsetAsync(s.size, 0, g.sb * size_t(gb.batch) * 4, st);
  cudaMemsetAsync(s.maxv, 0, size_t(gb.batch) * 4, st);
  dim3 pg(unsigned(grid_blocks(g.sb, 256)), unsigned(gb.batch));
  k_maxvol_size<<<pg, 256, 0, st>>>(bits, s.parent, s.size, g);
  k_maxvol_max<<<pg, 256, 0, st>>>(s.parent, s.size, s.maxv, g);
  size_t warps = size_t(g.BH) * (gb.pitch / 2);
  dim3 sg(unsigned(grid_blocks(warps * 32, 256)), unsigned(gb.batch));
  k_maxvol_select<<<sg, 256, 0, st>>>(bits, s.parent, s.size, s.maxv, out, g);
  return launches + 3;
}

}  // namespace slcs
