// ccl.cu -- run-based union-find connected components, reach and maxvol for
// sm_100a.
//
// Replaces the reference's pointer-jumping labelling (ccl::label,
// proj/src/ccl.cpp:127-165, paper Alg. 1) and the CCL-based reach
// (proj/src/reach.cpp:10-50).
//
// Nodes.  The image is cut into 2-row bands.  One thread owns one 32-px word
// of a band -- the two bit-packed words T (row 2k) and B (row 2k+1) -- and
// its union-find nodes are the runs of the column occupancy c = T | B: under
// 8-connectivity every pixel of such a run touches the next column's pixels,
// so a run is connected, and runs split by an empty column are not.  Runs are
// found with a handful of bit operations per word, never per pixel.
//
// Keys.  A run's key is its row-first max pixel, packed (r << s) | c
// (KeyGeo).  Two runs of one band never share a 2x2 block column pair for
// their key pixels, so the key's 2x2 block indexes the node's parent slot.
// Unions hang the smaller root under the larger (atomicMax), so every root is
// the max pixel of its component and the final label is exactly the
// reference's canonical max index + 1 (ccl.hpp:52-60): no relabel pass.
//
// Passes (large images; images <= 256x256 run everything in one CTA):
//   tile_local  128x256-px tile in shared memory: runs, unions with the band
//               above / the word to the right, flatten; writes per run
//               P = local root, per tile the list of ring-touching roots
//   tile_merge  unions across tile borders on the global P (bit-parallel)
//   root_flatten  listed local roots -> their global root
//   select / labels / maxvol  per word: every run's global root is P[P[key]]
#include "slcs_internal.h"

#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

#ifndef SLCS_COOP_PDL
#define SLCS_COOP_PDL 2
#endif
#ifndef SLCS_MERGE_QUEUE
#define SLCS_MERGE_QUEUE 1
#endif
#ifndef SLCS_FUSED_QUEUE
#define SLCS_FUSED_QUEUE 0
#endif
#ifndef SLCS_TL_QUEUE
#define SLCS_TL_QUEUE 1
#endif
#ifndef SLCS_TL_PHASES
#define SLCS_TL_PHASES 0  // diagnostics: per-phase clock64 of k_tile_local (stderr)
#endif
#ifndef SLCS_TL_FUSED_ROOTS
#define SLCS_TL_FUSED_ROOTS 1
#endif
#ifndef SLCS_CH_SLEEP
#define SLCS_CH_SLEEP 32  // reach chain: back-off (ns) between halo-record polls
#endif
#ifndef SLCS_TL_HINTS
#define SLCS_TL_HINTS 1
#endif

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

constexpr uint32_t FULL = 0xffffffffu;

struct G {
  int W, H, wpr;
  uint32_t pitch;   // words per row
  size_t slice;     // words per slice
  int BW, BH;       // 2x2 block grid (BH = number of bands)
  int s;
  uint32_t cmask;
  uint32_t sb;      // blocks per slice
  uint32_t lastmask;  // valid bits of word wpr - 1
};

G make_g(const Geo& gb) {
  KeyGeo k = key_geo(gb.w, gb.h);
  G g;
  g.W = gb.w;
  g.H = gb.h;
  g.wpr = gb.wpr;
  g.pitch = uint32_t(gb.pitch);
  g.slice = gb.slice;
  g.BW = k.bw;
  g.BH = k.bh;
  g.s = k.s;
  g.cmask = k.cmask;
  g.sb = uint32_t(k.slice_blocks);
  g.lastmask = gb.lastmask;
  return g;
}

// ---- run helpers ------------------------------------------------------------
// the run of x that starts at its lowest set bit
__device__ __forceinline__ uint32_t first_run(uint32_t x) {
  // adding the lowest set bit carries through exactly that run (a run ending
  // at bit 31 carries out): the bits it clears are the run -- ALU ops only
  // (no FLO/BREV: 3 % faster CCL and reach than an __ffs-based mask)
  return x & ~(x + (x & (0u - x)));
}

// the run of c containing bit p (bit p must be set)
__device__ __forceinline__ uint32_t run_at(uint32_t c, int p) {
  const uint32_t z = ~c;
  const uint32_t above = z & (0xfffffffeu << p);
  const uint32_t below = z & ((1u << p) - 1u);
  const uint32_t hi = above ? ((above & (0u - above)) - 1u) : FULL;
  const uint32_t lo = below ? (FULL << (32 - __clz(below))) : FULL;
  return hi & lo;
}

// row offset (0/1) and column (0..31) of the run's max pixel
__device__ __forceinline__ void run_max(uint32_t T, uint32_t B, uint32_t m, int& dr, int& col) {
  const uint32_t bm = B & m;
  dr = bm ? 1 : 0;
  col = 31 - __clz(bm ? bm : (T & m));
}

__device__ __forceinline__ uint32_t dil1(uint32_t x) { return x | (x << 1) | (x >> 1); }

// ---- global union-find over P ------------------------------------------------
// Global nodes are identified by an invertible hash of their key, and unions
// hang the smaller id under the larger: random priorities keep the trees
// O(log n) deep.  (Max-key linking over a regular grid of tiles builds
// linear chains -- tile after tile along a row, row after row -- and every
// find then walks ~20 dependent L2 hops.)  The canonical max key of a
// component is carried separately where labels need it (MK).
constexpr uint32_t HMUL = 0x9E3779B1u, HINV = 0x0E8B2F51u;
__device__ __forceinline__ uint32_t hnode(uint32_t key) {
  return (key ^ (key >> 16)) * HMUL;
}
__device__ __forceinline__ uint32_t hkey(uint32_t node) {
  const uint32_t x = node * HINV;
  return x ^ (x >> 16);
}
__device__ __forceinline__ uint32_t kblk(const G& g, uint32_t k) {
  return ((k >> g.s) >> 1) * uint32_t(g.BW) + ((k & g.cmask) >> 1);
}
// parent slot of a node: the 2x2 block of its key
__device__ __forceinline__ uint32_t gblk(const G& g, uint32_t n) { return kblk(g, hkey(n)); }

__device__ __forceinline__ uint32_t gkey(const G& g, int row, int col) {
  return (uint32_t(row) << g.s) | uint32_t(col);
}
__device__ __forceinline__ uint32_t gnode(const G& g, int row, int col) {
  return hnode(gkey(g, row, col));
}

// global node of the run m of word j in band k
__device__ __forceinline__ uint32_t grun(const G& g, int k, int j, uint32_t T, uint32_t B,
                                         uint32_t m) {
  int dr, col;
  run_max(T, B, m, dr, col);
  return gnode(g, 2 * k + dr, 32 * j + col);
}

// find during concurrent unions: L2-coherent loads, path halving
__device__ __forceinline__ uint32_t gfind_cg(uint32_t* P, const G& g, uint32_t v) {
  for (;;) {
    const uint32_t p = __ldcg(P + gblk(g, v));
    if (p == v) return v;
    const uint32_t gp = __ldcg(P + gblk(g, p));
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
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMax(P + gblk(g, b), a);
    if (old == b) return;
    b = old;
  }
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

__device__ __forceinline__ uint32_t linear_label(const G& g, uint32_t k) {
  return (k >> g.s) * uint32_t(g.W) + (k & g.cmask) + 1u;
}

// near(t) word (r, j): 3x3 OR, out of image = 0
__device__ __forceinline__ uint32_t near_word(const uint32_t* __restrict__ t, const G& g, int r,
                                              int j) {
  uint32_t acc = 0;
#pragma unroll
  for (int d = -1; d <= 1; ++d) {
    const int rr = r + d;
    if (rr < 0 || rr >= g.H) continue;
    const uint32_t* row = t + size_t(rr) * g.pitch;
    const uint32_t C = __ldg(row + j);
    const uint32_t L = j > 0 ? __ldg(row + j - 1) : 0u;
    const uint32_t R = j + 1 < g.wpr ? __ldg(row + j + 1) : 0u;
    acc |= C | __funnelshift_l(L, C, 1) | __funnelshift_r(C, R, 1);
  }
  return acc;
}

// ---- shared-memory tile of runs ---------------------------------------------
// Tile = bands x (1 << KW) px; unit u = band * TWW + word, one per thread.
// Local keys (lrow << KW) | lcol; parent slot = the key's 2x2 block.
template <int KW>
struct RunTile {
  static constexpr int TWW = (1 << KW) / 32;
  static constexpr int BL = KW - 1;
  uint32_t* par;
  const uint32_t* sT;
  const uint32_t* sB;

  __device__ __forceinline__ static int slot(uint32_t lk) {
    return int(((lk >> (KW + 1)) << BL) | ((lk & ((1u << KW) - 1u)) >> 1));
  }
  __device__ __forceinline__ static uint32_t key(int band, int w, uint32_t T, uint32_t B,
                                                 uint32_t m) {
    int dr, col;
    run_max(T, B, m, dr, col);
    return (uint32_t(2 * band + dr) << KW) | uint32_t(32 * w + col);
  }
  // Union-find nodes are (priority << 16) | slot: the high half is a hash of
  // the local key (a random linking order), the low half the parent slot, so
  // a find step needs no key arithmetic.  Linking by key order (root = max
  // pixel) builds long chains along rows/bands; random linking keeps trees
  // O(log n) deep, and atomicMax linking lets concurrent unions on one root
  // all make progress.  Roots are therefore arbitrary representatives; the
  // canonical max key is recovered separately where labels need it.
  // priority = the slot's bits reversed (a van der Corput order: along any run
  // of consecutive slots the maxima are spread like a ruler sequence, so chains
  // link into O(log n)-deep trees) -- two instructions instead of a hash
  __device__ __forceinline__ static uint32_t snode(uint32_t sl) { return __brev(sl) | sl; }
  __device__ __forceinline__ static uint32_t node(uint32_t k) { return snode(uint32_t(slot(k))); }
  // node of run m of word w in `band` without composing the key
  __device__ __forceinline__ static uint32_t rnode(int band, int w, uint32_t T, uint32_t B,
                                                  uint32_t m) {
    const uint32_t bm = B & m;
    const int col = 31 - __clz(bm ? bm : (T & m));
    return snode((uint32_t(band) << BL) | (uint32_t(32 * w + col) >> 1));
  }
  __device__ __forceinline__ static int nslot(uint32_t v) { return int(v & 0xffffu); }
  // a representative key of a slot's 2x2 block (top-left pixel)
  __device__ __forceinline__ static uint32_t bkey(int sl) {
    return (uint32_t(sl >> BL) << (KW + 1)) | (uint32_t(sl & ((1 << BL) - 1)) << 1);
  }
  __device__ __forceinline__ uint32_t find(uint32_t v) const {
    volatile uint32_t* vp = par;
    for (;;) {
      const uint32_t p = vp[nslot(v)];
      if (p == v) return v;
      const uint32_t gp = vp[nslot(p)];
      if (gp == p) return p;
      vp[nslot(v)] = gp;
      v = gp;
    }
  }
  // returns a node of the merged set (the winning root at link time)
  __device__ __forceinline__ uint32_t unite(uint32_t a, uint32_t b) const {
    for (;;) {
      a = find(a);
      b = find(b);
      if (a == b) return a;
      if (a < b) {
        const uint32_t t = a;
        a = b;
        b = t;
      }
      const uint32_t old = atomicMax(par + nslot(b), a);
      if (old == b) return a;
      b = old;
    }
  }
  // After roots(): the max key of each run's component into the root's slot
  // (par is free again).  Afterwards par[nslot(r[i])] is run i's component max
  // key (read it there: a per-run register copy spills at 32 registers).
  __device__ void max_keys_only(int u, uint32_t T, uint32_t B, const uint32_t (&r)[16]) const {
    const int band = u / TWW, w = u % TWW;
    uint32_t x = T | B;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      const uint32_t m = first_run(x);
      x &= ~m;
      if (r[i] == node(key(band, w, T, B, m))) par[nslot(r[i])] = 0;
    }
    __syncthreads();
    // consecutive runs of a word mostly share a root: one atomic per stretch
    // of equal roots (inside a dense tile every run hits the same slot)
    x = T | B;
    uint32_t cr = 0, ck = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t k = key(band, w, T, B, m);
      if (i > 0 && r[i] != cr) atomicMax(par + nslot(cr), ck);
      ck = (i > 0 && r[i] == cr) ? max(ck, k) : k;
      cr = r[i];
    }
    if (T | B) atomicMax(par + nslot(cr), ck);
    __syncthreads();
  }
  // max_keys_only, then this thread's per-run component max keys in registers
  __device__ void max_keys(int u, uint32_t T, uint32_t B, const uint32_t (&r)[16],
                           uint32_t (&mk)[16]) const {
    max_keys_only(u, T, B, r);
#pragma unroll
    for (int i = 0; i < 16; ++i) mk[i] = par[nslot(r[i])];
  }
  // Roots of all runs, then unions with the band above (pixel adjacency
  // between B of band-1 and T of this band, incl. the diagonals into the
  // neighbouring words) and with the next word of the same band.  Links
  // leaving the tile are left to the global merge.
  // q (optional): a per-warp queue in shared memory (256 node-slot pairs per warp,
  // counters qn[warp]); the band-above pairs are queued and then united 32 per warp
  // step instead of inside each lane's divergent run/overlap loops
  __device__ void link(int u, uint32_t T, uint32_t B, uint32_t* q = nullptr,
                       int* qn = nullptr, int qcap = 256) const {
    const int band = u / TWW, w = u % TWW;
    for (uint32_t x = T | B; x;) {
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t v = rnode(band, w, T, B, m);
      par[nslot(v)] = v;
    }
    // Row links without union-find: a run crossing word boundaries is one chain
    // of pieces along the band, and the band's TWW words are TWW consecutive
    // lanes.  A segmented scan over those lanes hands every continuing piece the
    // node of the chain's leftmost piece, which it points at directly.
    {
      static_assert(32 % TWW == 0, "a band's words must share a warp");
      const uint32_t c = T | B;
      const uint32_t prev_c = __shfl_up_sync(0xffffffffu, c, 1, TWW);
      const bool cont = w > 0 && (c & 1u) && (prev_c >> 31);
      const uint32_t first = c ? rnode(band, w, T, B, first_run(c)) : 0u;
      const uint32_t last = c ? rnode(band, w, T, B, run_at(c, 31 - __clz(c))) : 0u;
      const bool single = c && first == last;
      uint32_t rep_first = first, rep_last = last;
#pragma unroll
      for (int step = 1; step < TWW; ++step) {
        const uint32_t left = __shfl_up_sync(0xffffffffu, rep_last, 1, TWW);
        if (cont) rep_first = left;
        rep_last = single ? rep_first : last;
      }
      if (cont) par[nslot(first)] = rep_first;
    }
    __syncthreads();
    // Links to the band above.  Each lane's first (run, upper run) pair is held
    // back and deduplicated across the warp: inside a blob all 8 words of a band
    // link the same two row chains, and one union suffices.
    bool have = false;
    uint32_t fa = 0, fb = 0;
    if (band > 0 && T) {
      const int uu = u - TWW;
      const uint32_t Tu = sT[uu], Bu = sB[uu], cu = Tu | Bu;
      for (uint32_t x = T | B; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        const uint32_t td = T & m;
        if (!td) continue;
        // a: the last known root of this run (saves re-finding from the run)
        uint32_t a = rnode(band, w, T, B, m);
        auto link_to = [&](uint32_t b) {
          if (!have) {
            have = true;
            fa = a;
            fb = b;
          } else {
            // queued pairs are filtered when the warp unites them
            if (q) {
              const int wq = threadIdx.x >> 5;
              const int at = atomicAdd(qn + wq, 1);
              if (at < qcap) {
                q[wq * qcap + at] = (uint32_t(nslot(a)) << 16) | uint32_t(nslot(b));
                return;
              }
            }
            if (par[nslot(b)] == a) return;  // b hangs under a already: same set
            a = unite(a, b);
          }
        };
        for (uint32_t ov = dil1(td) & Bu; ov;) {
          const uint32_t mu = run_at(cu, __ffs(ov) - 1);
          ov &= ~mu;
          link_to(rnode(band - 1, w, Tu, Bu, mu));
        }
        // a diagonal link is redundant when the pixel straight above is set:
        // that pixel's run is linked both ways already (vertical + row link)
        if ((td & 1u) && w > 0 && !(Bu & 1u)) {
          const uint32_t Tl = sT[uu - 1], Bl = sB[uu - 1];
          if (Bl >> 31) link_to(rnode(band - 1, w - 1, Tl, Bl, run_at(Tl | Bl, 31)));
        }
        if ((td >> 31) && w + 1 < TWW && !(Bu >> 31)) {
          const uint32_t Tr = sT[uu + 1], Br = sB[uu + 1];
          if (Br & 1u) link_to(rnode(band - 1, w + 1, Tr, Br, run_at(Tr | Br, 0)));
        }
      }
    }
    {
      // compare the pair's current parents (row-chain representatives or later
      // ancestors -- either way the same sets) with the previous lane's; an equal
      // pair is united by that lane (or, transitively, by an earlier one)
      const uint32_t pa = have ? par[nslot(fa)] : 0u, pb = have ? par[nslot(fb)] : 0u;
      const uint32_t lo = pa < pb ? pa : pb, hi = pa < pb ? pb : pa;
      const int lane = threadIdx.x & 31;
      const uint32_t plo = __shfl_up_sync(0xffffffffu, lo, 1);
      const uint32_t phi = __shfl_up_sync(0xffffffffu, hi, 1);
      const bool phave = __shfl_up_sync(0xffffffffu, have ? 1u : 0u, 1) != 0u;
#if SLCS_TL_HINTS
      if (have && lo != hi && !(lane > 0 && phave && plo == lo && phi == hi)) unite(fa, fb);
      if (q) {
        __syncwarp();
        const int wq = threadIdx.x >> 5;
        const int n = min(qn[wq], qcap);
        for (int i = lane; i < n; i += 32) {
          const uint32_t e = q[wq * qcap + i];
          const uint32_t a = snode(e >> 16), b = snode(e & 0xffffu);
          if (par[nslot(b)] != a) unite(a, b);
        }
      }
#else
      if (have && !(lane > 0 && phave && plo == lo && phi == hi)) unite(fa, fb);
#endif
    }
    __syncwarp();
    __syncthreads();
  }
  // The root of each of this word's runs (<= 16), in run order.  Finds halve
  // paths, so results go to registers and the caller must __syncthreads()
  // before reusing par.
  __device__ void roots(int u, uint32_t T, uint32_t B, uint32_t (&r)[16]) const {
    const int band = u / TWW, w = u % TWW;
    uint32_t x = T | B;
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = 0;
#if SLCS_TL_HINTS
    // no unions are in flight: a run whose parent is the previous run's root
    // (or itself) needs no find
    uint32_t last = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t v = rnode(band, w, T, B, m);
      const uint32_t p = static_cast<volatile uint32_t*>(par)[nslot(v)];
      last = (p == v || p == last) ? p : find(p);
      r[i] = last;
    }
#else
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      const uint32_t m = first_run(x);
      x &= ~m;
      r[i] = find(rnode(band, w, T, B, m));
    }
#endif
  }
};

// ===========================================================================
// Large-image path: 128x256-px tiles (64 bands x 8 words = 512 threads, 4 CTAs per SM).
constexpr int LKW = 8;
constexpr int LTWW = 8;
#ifndef SLCS_LTNB
#define SLCS_LTNB 64
#endif
constexpr int LTNB = SLCS_LTNB;
constexpr int LUNITS = LTNB * LTWW;              // 512
constexpr int LSLOTS = LTNB * (1 << (LKW - 1));  // 8192 blocks per tile
constexpr int LT_LIST = 520;                     // count + <= 512 ring roots
constexpr int LT_THREADS = LUNITS;

// MODE_BOTH: reach's seed flags (F) and the labels' max keys (SZ as MK) from one
// labelling -- a band's reach and ccl::label of the same image share it
enum { MODE_CCL = 0, MODE_REACH = 1, MODE_SIZE = 2, MODE_BOTH = 3 };
#if SLCS_TL_PHASES
__device__ unsigned long long tl_phase_acc[8];
#define TL_MARK(i)                                                   \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      const long long t_ = clock64();                                \
      atomicAdd(&tl_phase_acc[i], (unsigned long long)(t_ - tl_t0)); \
      tl_t0 = t_;                                                    \
    }                                                                \
  } while (0)
#else
#define TL_MARK(i) \
  do {             \
  } while (0)
#endif

// Tile-local pass.  Per run: P[key block] = local root + 1.  Per local root:
// F = "holds a seed" (reach) or SZ = local pixel count (maxvol).  Per tile:
// the local roots touching the tile ring -- the only ones a border union can
// link, hence the only ones root_flatten visits.
#ifndef SLCS_TL_MINB
#define SLCS_TL_MINB (2048 / LT_THREADS)
#endif
template <int MODE>
__global__ void __launch_bounds__(LT_THREADS, SLCS_TL_MINB) k_tile_local(const uint32_t* __restrict__ ubits,
                                                           const uint32_t* __restrict__ tbits,
                                                           uint32_t* __restrict__ P,
                                                           uint8_t* __restrict__ F,
                                                           uint32_t* __restrict__ SZ,
                                                           uint32_t* __restrict__ lists, G g) {
  slcs_pdl_wait();
  extern __shared__ __align__(16) unsigned char lsm[];
  uint32_t* par = reinterpret_cast<uint32_t*>(lsm);           // LSLOTS
  uint32_t* sT = par + LSLOTS;                                 // LUNITS
  uint32_t* sB = sT + LUNITS;                                  // LUNITS
  // MODE_SIZE: per-root pixel counts reuse the union-find slots once every
  // run's root is in registers (keeps the tile at four CTAs per SM)
  uint32_t* lsz = par;
  uint8_t* touch = reinterpret_cast<uint8_t*>(sB + LUNITS);
  uint8_t* fl = touch + LSLOTS;                                // LSLOTS (MODE_REACH)
  __shared__ int s_cnt;
  using T = RunTile<LKW>;
  const int slice = blockIdx.z;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const int u0 = threadIdx.x;
  const int band = u0 / LTWW, w = u0 % LTWW;
  const int kb = blockIdx.y * LTNB + band;  // global band
  const int j = blockIdx.x * LTWW + w;      // global word
  const int r = 2 * kb;
  const bool in = kb < g.BH && j < g.wpr;
  const uint32_t Tw = in ? __ldg(u + size_t(r) * g.pitch + j) : 0u;
  const uint32_t Bw = (in && r + 1 < g.H) ? __ldg(u + size_t(r + 1) * g.pitch + j) : 0u;
  // the word's seed pixels: through & near(target), both rows folded into one
  // column mask (a run is seeded iff it meets it; one live register across link)
  uint32_t sdw = 0;
  constexpr bool SEEDS = MODE == MODE_REACH || MODE == MODE_BOTH;
  constexpr bool MAXK = MODE == MODE_CCL || MODE == MODE_BOTH;
  if (SEEDS && (Tw | Bw)) {
    const uint32_t* t = tbits + size_t(slice) * g.slice;
    sdw = (Tw & near_word(t, g, r, j)) | (r + 1 < g.H ? Bw & near_word(t, g, r + 1, j) : 0u);
  }
  sT[u0] = Tw;
  sB[u0] = Bw;
#if SLCS_TL_PHASES
  long long tl_t0 = clock64();
#endif
#if SLCS_TL_QUEUE
  // touch + fl (16 KB) are free until the roots are known: the link queue
  __shared__ int s_qn[LT_THREADS / 32];
  if (threadIdx.x < LT_THREADS / 32) s_qn[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  TL_MARK(0);
  T tile{par, sT, sB};
  tile.link(u0, Tw, Bw, reinterpret_cast<uint32_t*>(touch), s_qn);
  TL_MARK(1);
  uint32_t rt[16];
  // FUSED: the roots are found inside the per-run output loop below (one pass
  // over the runs instead of two); maxvol's sizes alias par, so it keeps the
  // separate roots() pass
  constexpr bool FUSED = SLCS_TL_FUSED_ROOTS && MODE != MODE_SIZE;
  if (!FUSED) tile.roots(u0, Tw, Bw, rt);
  for (int q = threadIdx.x; q < LSLOTS / 4; q += blockDim.x) {
    reinterpret_cast<uint32_t*>(touch)[q] = 0;
    if (SEEDS) reinterpret_cast<uint32_t*>(fl)[q] = 0;
  }
  __syncthreads();
#else
  constexpr bool FUSED = false;
  for (int q = threadIdx.x; q < LSLOTS / 4; q += blockDim.x) {
    reinterpret_cast<uint32_t*>(touch)[q] = 0;
    if (SEEDS) reinterpret_cast<uint32_t*>(fl)[q] = 0;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  T tile{par, sT, sB};
  tile.link(u0, Tw, Bw);
  uint32_t rt[16];
  tile.roots(u0, Tw, Bw, rt);
  __syncthreads();
#endif
  if (MODE == MODE_SIZE) {
    for (int q = threadIdx.x; q < LSLOTS / 4; q += blockDim.x)
      reinterpret_cast<uint4*>(lsz)[q] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
  }

  const int R0 = blockIdx.y * LTNB * 2, C0 = blockIdx.x * LTWW * 32;
  const uint32_t lmask = (1u << LKW) - 1u;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  {
    uint32_t x = Tw | Bw;
    int cs = -1;       // MODE_SIZE: the stretch of runs sharing root slot cs
    uint32_t cn = 0;   // and its pixel count (one shared atomic per stretch)
    uint32_t last = 0xffffffffu;  // FUSED: the previous run's root (a find hint)
    if (FUSED) {
#pragma unroll
      for (int i = 0; i < 16; ++i) rt[i] = 0;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      {
        const uint32_t m = first_run(x);
        x &= ~m;
        const uint32_t k = T::key(band, w, Tw, Bw, m);
        if (FUSED) {  // as roots(): no unions are in flight any more
          const uint32_t v = T::node(k);
          const uint32_t p = static_cast<volatile uint32_t*>(par)[T::nslot(v)];
          last = (p == v || p == last) ? p : tile.find(p);
          rt[i] = last;
        }
        const int rs = T::nslot(rt[i]);
        if (band == 0 || band == LTNB - 1 || (w == 0 && (m & 1u)) || (w == LTWW - 1 && (m >> 31)))
          touch[rs] = 1;
        if (SEEDS && (sdw & m)) fl[rs] = 1;
        if (MODE == MODE_SIZE) {
          const uint32_t n = uint32_t(__popc(Tw & m) + __popc(Bw & m));
          if (rs != cs && cs >= 0) atomicAdd(lsz + cs, cn);
          cn = rs == cs ? cn + n : n;
          cs = rs;
        }
      }
    }
    if (MODE == MODE_SIZE && cs >= 0) atomicAdd(lsz + cs, cn);
  }
  __syncthreads();
  TL_MARK(2);
  // MODE_CCL: component max keys (roots are hash-ordered) land in par at the
  // roots' slots
  if (MAXK && SZ) tile.max_keys_only(u0, Tw, Bw, rt);
  TL_MARK(3);
  const size_t tile_id = (size_t(slice) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  uint32_t* L = lists + tile_id * LT_LIST;
  {
    uint32_t x = Tw | Bw;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      {
        const uint32_t m = first_run(x);
        x &= ~m;
        const uint32_t k = T::key(band, w, Tw, Bw, m);
        const int ks = T::slot(k);
        // P (run key block -> local root node) is staged in par, whose LSLOTS
        // slots are exactly the tile's 2x2 blocks, and leaves below as whole
        // 512 B band rows (scattered 4 B stores left partial sectors that L2
        // refilled from DRAM: ~1 B/px of reads).  A slot is the key block of one
        // run only, so this thread is its only reader (a root's size / max key)
        // and writer from here on; slots without a run key keep stale values,
        // which nothing reads.
        const uint32_t rk = T::bkey(T::nslot(rt[i]));  // the root's block stands for it globally
        const uint32_t pv = gnode(g, R0 + int(rk >> LKW), C0 + int(rk & lmask));
        if (rt[i] == T::node(k)) {  // local root
          const uint32_t bk = T::bkey(ks);
          const uint32_t gk = gkey(g, R0 + int(bk >> LKW), C0 + int(bk & lmask));
          const uint32_t b = kblk(g, gk);
          if (SEEDS) F[size_t(slice) * g.sb + b] = fl[ks];
          if (MODE == MODE_SIZE) SZ[size_t(slice) * g.sb + b] = lsz[ks];
          if (MAXK && SZ) {  // component max key (MK)
            const uint32_t mk = par[ks];
            SZ[size_t(slice) * g.sb + b] = gkey(g, R0 + int(mk >> LKW), C0 + int(mk & lmask));
          }
          if (touch[ks]) L[1 + atomicAdd(&s_cnt, 1)] = hnode(gk);
        }
        par[ks] = pv;
      }
    }
  }
  __syncthreads();
  TL_MARK(4);
  if (threadIdx.x == 0) L[0] = uint32_t(s_cnt);
  {
    constexpr int BPR = 1 << (LKW - 1);  // blocks per tile band row (128)
    const int bx0 = blockIdx.x * BPR, nbx = min(BPR, g.BW - bx0);
    const int kb0 = blockIdx.y * LTNB, nkb = min(LTNB, g.BH - kb0);
    if ((g.BW & 3) == 0) {
      for (int e = threadIdx.x; e < nkb * (BPR / 4); e += blockDim.x) {
        const int bi = e / (BPR / 4), q = e % (BPR / 4);
        if (4 * q < nbx)
          *reinterpret_cast<uint4*>(Ps + size_t(kb0 + bi) * size_t(g.BW) + bx0 + 4 * q) =
              *reinterpret_cast<const uint4*>(par + bi * BPR + 4 * q);
      }
    } else {
      for (int e = threadIdx.x; e < nkb * BPR; e += blockDim.x) {
        const int bi = e / BPR, c = e % BPR;
        if (c < nbx) Ps[size_t(kb0 + bi) * size_t(g.BW) + bx0 + c] = par[e];
      }
    }
  }
}

__device__ __forceinline__ void load_unit(const uint32_t* u, const G& g, int k, int j,
                                          uint32_t& T, uint32_t& B) {
  if (k < 0 || k >= g.BH || j < 0 || j >= g.wpr) {
    T = B = 0;
    return;
  }
  const uint32_t* row = u + size_t(2 * k) * g.pitch + j;
  T = __ldg(row);
  B = 2 * k + 1 < g.H ? __ldg(row + g.pitch) : 0u;
}

// Unions across tile borders.  Part A: the first band of every tile row
// against the band above (all three column offsets).  Part B: the word pair
// straddling every vertical tile border (the horizontal link, and the two
// diagonals into the band above when that band is in the same tile row).
__global__ void k_tile_merge(const uint32_t* __restrict__ ubits, uint32_t* P, G g, int nhb,
                             int nvb) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t nA = uint32_t(nhb) * uint32_t(g.wpr), nB = uint32_t(nvb) * uint32_t(g.BH);
#if SLCS_MERGE_QUEUE
  // a horizontal-border word's further pairs are queued per warp and united by
  // all lanes together at the end: divergent lanes would run their L2 find
  // chains one after another, the compacted warp runs 32 of them in parallel
  constexpr int MQ = 64;
  __shared__ uint32_t s_qa[8][MQ], s_qb[8][MQ];
  __shared__ int s_qn[8];
  const int mw = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) s_qn[mw] = 0;
  __syncwarp();
#endif
  // units [0, nA): horizontal tile borders; [nA, nA + nB): vertical ones.  The
  // loop is warp-uniform so the vertical-border lanes of a warp can dedupe their
  // unions together.
  const int lane = threadIdx.x & 31;
  for (uint32_t base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < nA + nB;
       base += gridDim.x * blockDim.x) {
    const uint32_t i = base + uint32_t(lane);
    const unsigned maskA = __ballot_sync(FULL, i < nA);
    const unsigned maskB = __ballot_sync(FULL, i < nA + nB && i >= nA);
    if (i >= nA + nB) continue;
    if (i < nA) {
      const int t = int(i / uint32_t(g.wpr)), j = int(i - uint32_t(t) * uint32_t(g.wpr));
      const int k = (t + 1) * LTNB;
      uint32_t T, B, Tu, Bu;
      load_unit(u, g, k, j, T, B);
      load_unit(u, g, k - 1, j, Tu, Bu);
      uint32_t Tl = 0, Bl = 0, Tr = 0, Br = 0;
      // diagonals are redundant when the pixel straight above is set
      if ((T & 1u) && !(Bu & 1u)) load_unit(u, g, k - 1, j - 1, Tl, Bl);
      if ((T >> 31) && !(Bu >> 31)) load_unit(u, g, k - 1, j + 1, Tr, Br);
      const uint32_t cu = Tu | Bu;
      // Links are made between the endpoints' current ancestors (their local
      // roots after tile_local, or anything above them): along a tile border
      // most links join the same two pieces (the giant component of the tiles
      // above and below), so a lane skips a pair equal to the pair it linked
      // last, and the first pair of every word goes through the warp dedupe.
      bool first = true;
      uint32_t fa = 0, fb = 0, clo = 0, chi = 0;
      for (uint32_t x = T | B; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        const uint32_t td = T & m;
        if (!td) continue;
        const uint32_t la = __ldcg(Ps + gblk(g, grun(g, k, j, T, B, m)));
        auto link = [&](uint32_t wnode) {
          const uint32_t lb = __ldcg(Ps + gblk(g, wnode));
          const uint32_t lo = la < lb ? la : lb, hi = la < lb ? lb : la;
          if (lo == hi || (lo == clo && hi == chi)) return;
          clo = lo;
          chi = hi;
          if (first) {
            fa = la;
            fb = lb;
            first = false;
          } else {
#if SLCS_MERGE_QUEUE
            const int at = atomicAdd(&s_qn[mw], 1);
            if (at < MQ) {
              s_qa[mw][at] = la;
              s_qb[mw][at] = lb;
              return;
            }
#endif
            gunite(Ps, g, la, lb);
          }
        };
        for (uint32_t a = dil1(td) & Bu; a;) {
          const uint32_t mu = run_at(cu, __ffs(a) - 1);
          a &= ~mu;
          link(grun(g, k - 1, j, Tu, Bu, mu));
        }
        if ((td & 1u) && (Bl >> 31)) link(grun(g, k - 1, j - 1, Tl, Bl, run_at(Tl | Bl, 31)));
        if ((td >> 31) && (Br & 1u)) link(grun(g, k - 1, j + 1, Tr, Br, run_at(Tr | Br, 0)));
      }
      {
        // each lane's first pair: one union per distinct pair of the warp
        const uint32_t lo = min(fa, fb), hi = max(fa, fb);
        const bool need = !first && lo != hi;
        const unsigned long long key = (static_cast<unsigned long long>(hi) << 32) | lo;
        const unsigned grp = __match_any_sync(maskA, need ? key : 0ull);
        if (need && lane == __ffs(grp) - 1) gunite(Ps, g, fa, fb);
      }
    } else {
      const uint32_t i2 = i - nA;
      const int t = int(i2 / uint32_t(g.BH)), k = int(i2 - uint32_t(t) * uint32_t(g.BH));
      const int jr = (t + 1) * LTWW, jl = jr - 1;
      uint32_t Tl, Bl, Tr, Br;
      load_unit(u, g, k, jl, Tl, Bl);
      load_unit(u, g, k, jr, Tr, Br);
      const uint32_t cl = Tl | Bl, cr = Tr | Br;
      // Up to three links per band: the horizontal one and the two diagonals into
      // the band above (when that band is in the same tile row and the pixel
      // straight above is clear).  Each is taken between the endpoints' current
      // ancestors (local roots or above).  Down one border the links mostly join
      // the same two pieces, so the warp's lanes match their pairs and one lane
      // per distinct pair unites: a dense border costs a union per warp, not per
      // band.
      uint32_t pa[3] = {0u, 0u, 0u}, pb[3] = {0u, 0u, 0u};
      if ((cl >> 31) && (cr & 1u)) {
        pa[0] = __ldcg(Ps + gblk(g, grun(g, k, jl, Tl, Bl, run_at(cl, 31))));
        pb[0] = __ldcg(Ps + gblk(g, grun(g, k, jr, Tr, Br, run_at(cr, 0))));
      }
      if (k % LTNB != 0 && ((Tr & 1u) || (Tl >> 31))) {
        uint32_t Tul, Bul, Tur, Bur;
        load_unit(u, g, k - 1, jl, Tul, Bul);
        load_unit(u, g, k - 1, jr, Tur, Bur);
        if ((Tr & 1u) && (Bul >> 31) && !(Bur & 1u)) {
          pa[1] = __ldcg(Ps + gblk(g, grun(g, k, jr, Tr, Br, run_at(cr, 0))));
          pb[1] = __ldcg(Ps + gblk(g, grun(g, k - 1, jl, Tul, Bul, run_at(Tul | Bul, 31))));
        }
        if ((Tl >> 31) && (Bur & 1u) && !(Bul >> 31)) {
          pa[2] = __ldcg(Ps + gblk(g, grun(g, k, jl, Tl, Bl, run_at(cl, 31))));
          pb[2] = __ldcg(Ps + gblk(g, grun(g, k - 1, jr, Tur, Bur, run_at(Tur | Bur, 0))));
        }
      }
      unsigned long long prev[2] = {0ull, 0ull};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint32_t lo = min(pa[q], pb[q]), hi = max(pa[q], pb[q]);
        const unsigned long long key = (static_cast<unsigned long long>(hi) << 32) | lo;
        // absent or already-joined pairs (lo == hi) and a lane's repeats drop out
        const bool need = lo != hi && (q < 1 || key != prev[0]) && (q < 2 || key != prev[1]);
        if (q < 2) prev[q] = key;
        const unsigned grp = __match_any_sync(maskB, need ? key : 0ull);
        if (need && lane == __ffs(grp) - 1) gunite(Ps, g, pa[q], pb[q]);
      }
    }
  }
#if SLCS_MERGE_QUEUE
  __syncwarp();
  const int n = min(s_qn[mw], MQ);
  for (int q = threadIdx.x & 31; q < n; q += 32) gunite(Ps, g, s_qa[mw][q], s_qb[mw][q]);
#endif
}

// After the merge: every listed local root points straight at its global
// root and hands over its seed flag (reach) or pixel count (maxvol).  Then a
// run's global root is exactly P[P[key block]].  One thread per list entry
// (two 256-entry chunks per tile), so each SM keeps hundreds of independent
// find chains in flight; the flag / size / max-key updates are aggregated per
// warp over the lanes that found the same global root (inside a dense tile
// most ring roots belong to one giant component, and one L2 atomic per warp
// replaces up to 32 on the same address).
__global__ void __launch_bounds__(256) k_root_flatten(uint32_t* P, uint8_t* F, uint32_t* SZ,
                                                      const uint32_t* __restrict__ lists, G g,
                                                      int ntiles, int mode) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const int tile = int(blockIdx.x >> 1);
  if (tile >= ntiles) return;
  const int i = int((blockIdx.x & 1u) * 256u + threadIdx.x);
  uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* L = lists + (size_t(slice) * ntiles + tile) * LT_LIST;
  const int n = int(__ldg(L));
  if ((blockIdx.x & 1u) * 256u >= uint32_t(n)) return;  // whole-CTA exit
  const bool act = i < n;
  const uint32_t rv = act ? __ldg(L + 1 + i) : 0u;
  const uint32_t R = act ? gfind_ro(Ps, g, rv) : 0u;
  const bool moved = act && R != rv;
  if (moved) Ps[gblk(g, rv)] = R;
  if (mode == MODE_CCL && !SZ) return;
  const unsigned part = __ballot_sync(FULL, moved);
  if (!moved) return;
  const unsigned grp = __match_any_sync(part, R);
  const bool leader = (threadIdx.x & 31) == __ffs(grp) - 1;
  if (mode == MODE_REACH || mode == MODE_BOTH) {
    uint8_t* Fs = F + size_t(slice) * g.sb;
    const unsigned any = __ballot_sync(part, Fs[gblk(g, rv)] != 0) & grp;
    if (leader && any) Fs[gblk(g, R)] = 1;
  }
  if (mode != MODE_REACH && SZ) {
    uint32_t* Ss = SZ + size_t(slice) * g.sb;
    const uint32_t v = Ss[gblk(g, rv)];
    if (mode == MODE_SIZE) {
      const uint32_t sum = __reduce_add_sync(grp, v);
      if (leader) atomicAdd(Ss + gblk(g, R), sum);
    } else {  // MODE_CCL: SZ holds the max key of each root (MK)
      const uint32_t mx = __reduce_max_sync(grp, v);
      if (leader) atomicMax(Ss + gblk(g, R), mx);
    }
  }
}

__device__ __forceinline__ uint32_t groot(const uint32_t* P, const G& g, uint32_t v) {
  return P[gblk(g, P[gblk(g, v)])];
}

// The global root block of each run of word (k, j), in run order, as two
// rounds of independent loads instead of a dependent chain per run.  Runs of a
// word mostly share their local root (one piece of a large component), so a
// repeat of the previous run's local root skips its second load.
__device__ __forceinline__ int run_root_blocks(const uint32_t* Ps, const G& g, int k, int j,
                                               uint32_t T, uint32_t B, uint32_t (&v)[16]) {
  uint32_t x = T | B;
  int nr = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    v[q] = 0;
    if (x) {
      const uint32_t m = first_run(x);
      x &= ~m;
      v[q] = Ps[gblk(g, grun(g, k, j, T, B, m))];
      nr = q + 1;
    }
  }
  uint32_t w[16];
#pragma unroll
  for (int q = 0; q < 16; ++q)
    w[q] = (q < nr && (q == 0 || v[q] != v[q - 1])) ? Ps[gblk(g, v[q])] : 0u;
#pragma unroll
  for (int q = 1; q < 16; ++q)
    if (q < nr && v[q] == v[q - 1]) w[q] = w[q - 1];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = gblk(g, w[q]);
  return nr;
}

// reach: out = target | through-runs whose global root holds a seed.
// Thread = word (band k, word j), j fastest: each warp stores 128 B per row.
__global__ void k_reach_select(const uint32_t* __restrict__ ubits,
                               const uint32_t* __restrict__ tbits, const uint32_t* __restrict__ P,
                               const uint8_t* __restrict__ F, uint32_t* __restrict__ out, G g) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* t = tbits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint8_t* Fs = F + size_t(slice) * g.sb;
  uint32_t* o = out + size_t(slice) * g.slice;
  const uint32_t n = uint32_t(g.BH) * g.pitch;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = int(i / g.pitch), j = int(i - uint32_t(k) * g.pitch);
    const size_t row = size_t(2 * k) * g.pitch + j;
    const bool two = 2 * k + 1 < g.H;
    uint32_t ST = 0, SB = 0;
    if (j < g.wpr) {
      const uint32_t T = __ldg(u + row), B = two ? __ldg(u + row + g.pitch) : 0u;
      for (uint32_t x = T | B; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        if (Fs[gblk(g, groot(Ps, g, grun(g, k, j, T, B, m)))]) {
          ST |= T & m;
          SB |= B & m;
        }
      }
      ST |= __ldg(t + row);
      if (two) SB |= __ldg(t + row + g.pitch);
    }
    o[row] = ST;
    if (two) o[row + g.pitch] = SB;
  }
}

// ---- reach against a precomputed labelling (label CSE) ------------------------
// Flags are stamps: the labelling step zeroes the per-block flag array once per
// program run, and the reaches sharing that labelling stamp gen = idx + 1
// (idx < 4096 distinct per labelling), so a stamp is never 0 and never reused
// within a run.

__global__ void k_reach_seed(const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ tbits,
                             const uint32_t* __restrict__ P, uint32_t* __restrict__ F32,
                             uint32_t gen, G g) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* t = tbits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  uint32_t* Fs = F32 + size_t(slice) * g.sb;
  const uint32_t n = uint32_t(g.BH) * uint32_t(g.wpr);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = int(i / uint32_t(g.wpr)), j = int(i - uint32_t(k) * uint32_t(g.wpr));
    const size_t row = size_t(2 * k) * g.pitch + j;
    const bool two = 2 * k + 1 < g.H;
    const uint32_t T = __ldg(u + row), B = two ? __ldg(u + row + g.pitch) : 0u;
    if (!(T | B)) continue;
    const uint32_t sd = (T & near_word(t, g, 2 * k, j)) | (two ? (B & near_word(t, g, 2 * k + 1, j)) : 0u);
    for (uint32_t x = T | B; x;) {
      const uint32_t m = first_run(x);
      x &= ~m;
      if (sd & m) Fs[gblk(g, groot(Ps, g, grun(g, k, j, T, B, m)))] = gen;
    }
  }
}

__global__ void k_reach_select_gen(const uint32_t* __restrict__ ubits,
                                   const uint32_t* __restrict__ tbits,
                                   const uint32_t* __restrict__ P,
                                   const uint32_t* __restrict__ F32,
                                   uint32_t gen, uint32_t* __restrict__ out, G g) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* t = tbits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* Fs = F32 + size_t(slice) * g.sb;
  uint32_t* o = out + size_t(slice) * g.slice;
  const uint32_t n = uint32_t(g.BH) * g.pitch;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = int(i / g.pitch), j = int(i - uint32_t(k) * g.pitch);
    const size_t row = size_t(2 * k) * g.pitch + j;
    const bool two = 2 * k + 1 < g.H;
    uint32_t ST = 0, SB = 0;
    if (j < g.wpr) {
      const uint32_t T = __ldg(u + row), B = two ? __ldg(u + row + g.pitch) : 0u;
      for (uint32_t x = T | B; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        if (Fs[gblk(g, groot(Ps, g, grun(g, k, j, T, B, m)))] == gen) {
          ST |= T & m;
          SB |= B & m;
        }
      }
      ST |= __ldg(t + row);
      if (two) SB |= __ldg(t + row + g.pitch);
    }
    o[row] = ST;
    if (two) o[row + g.pitch] = SB;
  }
}

// ---- row-band support (multi-GPU) ------------------------------------
// Per pixel of row r: the global root node of its through-component and a
// class byte (0 background, 1 unseeded, 2 seeded).  Used to stitch bands.
__global__ void k_band_row(const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ P,
                           const uint8_t* __restrict__ F, int r, uint32_t* __restrict__ roots,
                           uint8_t* __restrict__ cls, G g) {
  slcs_pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.wpr) return;
  const int k = r >> 1;
  uint32_t T, B;
  {
    const uint32_t* row = ubits + size_t(2 * k) * g.pitch + j;
    T = __ldg(row);
    B = 2 * k + 1 < g.H ? __ldg(row + g.pitch) : 0u;
  }
  const uint32_t mine = (r & 1) ? B : T;
  const int c0 = 32 * j, ncol = min(32, g.W - c0);
  for (int b = 0; b < ncol; ++b) {
    roots[c0 + b] = 0;
    cls[c0 + b] = 0;
  }
  for (uint32_t x = T | B; x;) {
    const uint32_t m = first_run(x);
    x &= ~m;
    const uint32_t px = mine & m;
    if (!px) continue;
    const uint32_t R = groot(P, g, grun(g, k, j, T, B, m));
    const uint8_t c = F[gblk(g, R)] ? 2 : 1;
    for (uint32_t y = px; y;) {
      const int b = __ffs(y) - 1;
      y &= y - 1;
      roots[c0 + b] = R;
      cls[c0 + b] = c;
    }
  }
}

__global__ void k_band_set_flags(const uint32_t* __restrict__ roots, int n, uint8_t* F, G g) {
  slcs_pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) F[gblk(g, roots[i])] = 1;
}

// the same with the list and its length in device memory (cross-band merge
// output, bands.cu); the grid covers the list's capacity
__global__ void k_band_set_flags_dev(const uint32_t* __restrict__ roots, const int* n, uint8_t* F,
                                     G g) {
  slcs_pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *n) F[gblk(g, roots[i])] = 1;
}

__device__ __forceinline__ uint32_t pick16(const uint32_t (&labs)[16], int ri) {
  uint32_t lab = 0;
#pragma unroll
  for (int z = 0; z < 16; ++z) lab = (ri == z) ? labs[z] : lab;
  return lab;
}

// labels: each run's pixels get linear(component max key) + 1.  A warp owns 32
// consecutive words of one band: lanes resolve their runs' labels into a
// per-warp shared table (stride 17, conflict-free), then the warp writes each
// output row cooperatively -- lane l stores pixels 4l..4l+3 of every 128-px
// stretch, so each warp store is 512 contiguous bytes (the label image is the
// 4 B/px bulk of the CCL traffic).
#ifndef SLCS_TL_WARPS
#define SLCS_TL_WARPS 8
#endif
// OUT = uint32_t: the labels; OUT = u64: a band's global 64-bit labels, each
// run's label mapped once through `map` (the cross-band merge), so the band
// CCL writes its 8 B/px output directly instead of a u32 image plus a relabel
constexpr int TL_WARPS = SLCS_TL_WARPS;
template <class OUT>
__global__ void __launch_bounds__(TL_WARPS * 32) k_tile_labels(const uint32_t* __restrict__ ubits,
                                                             const uint32_t* __restrict__ P,
                                                             const uint32_t* __restrict__ MKall,
                                                             OUT* __restrict__ L, G g,
                                                             LabelMap64 map, int vec_ok) {
  slcs_pdl_wait();
  __shared__ OUT tab[TL_WARPS][32 * 17];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* MK = MKall + size_t(slice) * g.sb;
  OUT* Ls = L + size_t(slice) * size_t(g.W) * size_t(g.H);
  OUT* tb = tab[wib];
  const int groups = (g.wpr + 31) / 32;
  const size_t nw = size_t(g.BH) * size_t(groups);
  const bool vec = (g.W & 3) == 0 && vec_ok;
  for (size_t wg = size_t(blockIdx.x) * TL_WARPS + wib; wg < nw; wg += size_t(gridDim.x) * TL_WARPS) {
    const int k = int(wg / size_t(groups)), gi = int(wg - size_t(k) * groups);
    const int j = gi * 32 + lane;
    const bool two = 2 * k + 1 < g.H;
    uint32_t T = 0, B = 0;
    if (j < g.wpr) {
      const size_t row = size_t(2 * k) * g.pitch + j;
      T = __ldg(u + row);
      B = two ? __ldg(u + row + g.pitch) : 0u;
    }
    uint32_t starts = 0;
    {
      // run -> global root block -> max key, one load round each (see
      // run_root_blocks); runs sharing a root share its label
      uint32_t rb[16], lab[16];
      const int nr = run_root_blocks(Ps, g, k, j, T, B, rb);
      starts = (T | B) & ~((T | B) << 1);
#pragma unroll
      for (int q = 0; q < 16; ++q)
        lab[q] = (q < nr && (q == 0 || rb[q] != rb[q - 1])) ? MK[rb[q]] : 0u;
      OUT prev = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q >= nr) break;
        OUT v;
        if (q > 0 && rb[q] == rb[q - 1]) {
          v = prev;
        } else if (sizeof(OUT) == 8) {
          v = OUT(map_label64(linear_label(g, lab[q]), map));
        } else {
          v = OUT(linear_label(g, lab[q]));
        }
        prev = v;
        tb[lane * 17 + q] = v;
      }
    }
    __syncwarp();
    const size_t c0 = size_t(gi) * 1024;
    for (int rr = 0; rr < (two ? 2 : 1); ++rr) {
      const uint32_t bits = rr ? B : T;
      OUT* dst = Ls + size_t(2 * k + rr) * g.W + c0;
      if (vec) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int wi = it * 4 + (lane >> 3), x0 = (lane & 7) * 4;
          const uint32_t wb = __shfl_sync(0xffffffffu, bits, wi);
          const uint32_t ws = __shfl_sync(0xffffffffu, starts, wi);
          const size_t p = size_t(it) * 128 + size_t(lane) * 4;
          if (c0 + p < size_t(g.W)) {
            OUT v[4];
            // run index of pixel x0 (runs starting at or before it, minus one), then
            // advanced by the run starts at x0+1 .. x0+3
            const uint32_t sb = ws >> x0, pb = wb >> x0;
            const OUT* trow = tb + wi * 17 + __popc(ws & ((2u << x0) - 1u)) - 1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (e > 0) trow += (sb >> e) & 1u;
              v[e] = ((pb >> e) & 1u) ? *trow : OUT(0);
            }
            if (sizeof(OUT) == 8) {
              ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst + p);
              d2[0] = make_ulonglong2(v[0], v[1]);
              d2[1] = make_ulonglong2(v[2], v[3]);
            } else {
              *reinterpret_cast<uint4*>(dst + p) =
                  make_uint4(uint32_t(v[0]), uint32_t(v[1]), uint32_t(v[2]), uint32_t(v[3]));
            }
          }
        }
      } else {
        for (int it = 0; it < 32; ++it) {
          const uint32_t wb = __shfl_sync(0xffffffffu, bits, it);
          const uint32_t ws = __shfl_sync(0xffffffffu, starts, it);
          const size_t p = size_t(it) * 32 + lane;
          if (c0 + p < size_t(g.W))
            dst[p] = ((wb >> lane) & 1u) ? tb[it * 17 + __popc(ws & ((2u << lane) - 1u)) - 1]
                                         : OUT(0);
        }
      }
    }
    __syncwarp();
  }
}

// maxvol: max size over global roots (a run is a global root iff its block
// slot points at a node of its own block)
__global__ void k_maxvol_max(const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ P,
                             const uint32_t* __restrict__ SZ, unsigned int* maxv, G g) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* Ss = SZ + size_t(slice) * g.sb;
  const uint32_t n = uint32_t(g.BH) * uint32_t(g.wpr);
  uint32_t best = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = int(i / uint32_t(g.wpr)), j = int(i - uint32_t(k) * uint32_t(g.wpr));
    const size_t row = size_t(2 * k) * g.pitch + j;
    const uint32_t T = __ldg(u + row), B = 2 * k + 1 < g.H ? __ldg(u + row + g.pitch) : 0u;
    for (uint32_t x = T | B; x;) {
      const uint32_t m = first_run(x);
      x &= ~m;
      // a global root's block holds a node of that same block (roots are
      // represented by their block, not by the run's own key)
      const uint32_t b = gblk(g, grun(g, k, j, T, B, m));
      if (gblk(g, Ps[b]) == b) best = max(best, Ss[b]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(FULL, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(maxv + slice, best);
}

__global__ void k_maxvol_select(const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ P,
                                const uint32_t* __restrict__ SZ,
                                const unsigned int* __restrict__ maxv, uint32_t* __restrict__ out,
                                G g) {
  slcs_pdl_wait();
  const int slice = blockIdx.y;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* Ps = P + size_t(slice) * g.sb;
  const uint32_t* Ss = SZ + size_t(slice) * g.sb;
  uint32_t* o = out + size_t(slice) * g.slice;
  const uint32_t mx = maxv[slice];
  const uint32_t n = uint32_t(g.BH) * g.pitch;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = int(i / g.pitch), j = int(i - uint32_t(k) * g.pitch);
    const size_t row = size_t(2 * k) * g.pitch + j;
    const bool two = 2 * k + 1 < g.H;
    uint32_t ST = 0, SB = 0;
    if (j < g.wpr && mx) {
      const uint32_t T = __ldg(u + row), B = two ? __ldg(u + row + g.pitch) : 0u;
      for (uint32_t x = T | B; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        if (Ss[gblk(g, groot(Ps, g, grun(g, k, j, T, B, m)))] == mx) {
          ST |= T & m;
          SB |= B & m;
        }
      }
    }
    o[row] = ST;
    if (two) o[row + g.pitch] = SB;
  }
}

// ===========================================================================
// Small-image path: one CTA per image (W, H <= 256); 1024 threads = 128 bands
// x 8 words; everything in shared memory, one launch per batch of slices.
constexpr int SKW = 8;
constexpr int STWW = 8;
constexpr int ST_THREADS = 1024;
constexpr int SSLOTS = 128 * 128;

size_t small_smem_bytes() { return size_t(SSLOTS) * 4 + 2 * ST_THREADS * 4 + 256 * STWW * 4 + 64; }

// up to kSmallJobs independent same-shape problems in one launch (the program
// batches independent reaches): CTA x = job * batch + slice
constexpr int kSmallJobs = 4;
struct SmallJobs {
  const uint32_t* u[kSmallJobs];
  const uint32_t* t[kSmallJobs];
  uint32_t* out[kSmallJobs];
  int batch;
};

// optional bool-only listings around a small-image kernel: the operand words
// computed by `pro`, the result words passed through `epi` (FOP_PRESET = result)
struct SmallListings {
  FusedProgram pro, epi;
  int has_pro = 0, has_epi = 0;
};

__device__ uint32_t eval_listing(const FusedProgram& p, size_t q, uint32_t vm, uint32_t preset) {
  uint32_t R[kFusedRegs];
  uint32_t res = 0;
  for (int i = 0; i < p.n_ops; ++i) {
    const FusedOp op = p.ops[i];
    switch (op.op) {
      case FOP_LOADB: R[op.dst] = __ldg(p.bin[op.a] + q); break;
      case FOP_PRESET: R[op.dst] = preset; break;
      case FOP_NOT: R[op.dst] = ~R[op.a] & vm; break;
      case FOP_AND: R[op.dst] = R[op.a] & R[op.b]; break;
      case FOP_OR: R[op.dst] = R[op.a] | R[op.b]; break;
      case FOP_ANDNOT: R[op.dst] = R[op.a] & ~R[op.b]; break;
      case FOP_STORE: res = R[op.dst]; break;
      default: break;
    }
  }
  return res;
}

// mode 0 = labels, 1 = reach, 2 = maxvol
template <int MODE>
__global__ void __launch_bounds__(ST_THREADS, 2) k_small(const SmallJobs jobs, G g,
                                                      const SmallListings lst) {
  slcs_pdl_wait();
  const int job = int(blockIdx.x) / jobs.batch;
  // constant indices keep the job table in parameter space (no local copy)
  const uint32_t* __restrict__ ubits = jobs.u[0];
  const uint32_t* __restrict__ tbits = jobs.t[0];
  uint32_t* __restrict__ out = jobs.out[0];
#pragma unroll
  for (int i = 1; i < kSmallJobs; ++i)
    if (job == i) {
      ubits = jobs.u[i];
      tbits = jobs.t[i];
      out = jobs.out[i];
    }
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* par = reinterpret_cast<uint32_t*>(smem);  // SSLOTS
  uint32_t* sT = par + SSLOTS;                         // 1024
  uint32_t* sB = sT + ST_THREADS;                      // 1024
  uint32_t* rows = sB + ST_THREADS;                    // 256 rows x 8 words
  __shared__ unsigned int s_max;
  using T = RunTile<SKW>;
  const int slice = int(blockIdx.x) - job * jobs.batch;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const int u0 = threadIdx.x;
  const int band = u0 / STWW, w = u0 % STWW;
  const int r = 2 * band;
  const bool in = band < g.BH && w < g.wpr;
  const uint32_t vm = w + 1 < g.wpr ? FULL : (w + 1 == g.wpr && (g.W & 31)) ? (1u << (g.W & 31)) - 1u
                                                                           : (w < g.wpr ? FULL : 0u);
  const size_t q0 = size_t(slice) * g.slice + size_t(r) * g.pitch + w;
  uint32_t Tw = 0, Bw = 0;
  bool loaded = false;
  if constexpr (MODE == 2) {
    if (lst.has_pro) {
      Tw = in ? eval_listing(lst.pro, q0, vm, 0u) : 0u;
      Bw = (in && r + 1 < g.H) ? eval_listing(lst.pro, q0 + g.pitch, vm, 0u) : 0u;
      loaded = true;
    }
  }
  if (!loaded) {
    Tw = in ? __ldg(u + size_t(r) * g.pitch + w) : 0u;
    Bw = (in && r + 1 < g.H) ? __ldg(u + size_t(r + 1) * g.pitch + w) : 0u;
  }
  sT[u0] = Tw;
  sB[u0] = Bw;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  T tile{par, sT, sB};
  tile.link(u0, Tw, Bw);
  uint32_t rt[16];
  tile.roots(u0, Tw, Bw, rt);
  __syncthreads();

  if constexpr (MODE == 0) {
    uint32_t mk[16];  // labels are the component max index + 1 (ccl.hpp:52-60)
    tile.max_keys(u0, Tw, Bw, rt, mk);
    if (!in) return;
    uint32_t* Ls = out + size_t(slice) * size_t(g.W) * size_t(g.H);
    uint32_t labs[16];
    uint32_t starts = 0;
    {
      uint32_t x = Tw | Bw;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        labs[q] = 0;
        if (x) {
          const uint32_t m = first_run(x);
          x &= ~m;
          starts |= m & (0u - m);
          labs[q] = (mk[q] >> SKW) * uint32_t(g.W) + (mk[q] & ((1u << SKW) - 1u)) + 1u;
        }
      }
    }
    const int c0 = 32 * w, ncol = min(32, g.W - c0);
    for (int rr = 0; rr < (r + 1 < g.H ? 2 : 1); ++rr) {
      const uint32_t bits = rr ? Bw : Tw;
      uint32_t* dst = Ls + size_t(r + rr) * g.W + c0;
      for (int x = 0; x < ncol; ++x)
        dst[x] = ((bits >> x) & 1u) ? pick16(labs, __popc(starts & ((2u << x) - 1u)) - 1) : 0u;
    }
    return;
  }
  // modes 1 and 2 reuse par (free after roots()) as a per-root value array
  else {
  for (int q = threadIdx.x; q < SSLOTS; q += blockDim.x) par[q] = 0;
  __syncthreads();
  uint32_t ST = 0, SB = 0;
  if (MODE == 1) {
    const uint32_t* t = tbits + size_t(slice) * g.slice;
    uint32_t ntT = 0, ntB = 0;
    if (Tw | Bw) {
      ntT = near_word(t, g, r, w);
      ntB = r + 1 < g.H ? near_word(t, g, r + 1, w) : 0u;
    }
    {
      uint32_t x = Tw | Bw;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (x) {
          const uint32_t m = first_run(x);
          x &= ~m;
          if (((Tw & ntT) | (Bw & ntB)) & m) par[T::nslot(rt[q])] = 1;
        }
    }
    __syncthreads();
    {
      uint32_t x = Tw | Bw;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (x) {
          const uint32_t m = first_run(x);
          x &= ~m;
          if (par[T::nslot(rt[q])]) {
            ST |= Tw & m;
            SB |= Bw & m;
          }
        }
    }
    // S | target into smem rows, then the closing near from smem
    if (in) {
      rows[r * STWW + w] = ST | __ldg(t + size_t(r) * g.pitch + w);
      if (r + 1 < g.H) rows[(r + 1) * STWW + w] = SB | __ldg(t + size_t(r + 1) * g.pitch + w);
    }
    __syncthreads();
    uint32_t* o = out + size_t(slice) * g.slice;
    const int nwords = int(g.pitch) * g.H;
    for (int q = threadIdx.x; q < nwords; q += blockDim.x) {
      const int rr = q / int(g.pitch), j = q - rr * int(g.pitch);
      uint32_t acc = 0;
      if (j < g.wpr) {
        for (int y = max(0, rr - 1); y <= min(g.H - 1, rr + 1); ++y) {
          const uint32_t* row = rows + y * STWW;
          const uint32_t C = row[j];
          const uint32_t L = j > 0 ? row[j - 1] : 0u;
          const uint32_t R = j + 1 < g.wpr ? row[j + 1] : 0u;
          acc |= C | __funnelshift_l(L, C, 1) | __funnelshift_r(C, R, 1);
        }
        if (j == g.wpr - 1 && (g.W & 31)) acc &= (1u << (g.W & 31)) - 1u;
      }
      o[q] = acc;
    }
    return;
  }
  if (MODE == 2) {
    {
      uint32_t x = Tw | Bw;
      uint32_t cr = 0, cn = 0;  // one shared atomic per stretch of runs sharing a root
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (x) {
          const uint32_t m = first_run(x);
          x &= ~m;
          const uint32_t n = uint32_t(__popc(Tw & m) + __popc(Bw & m));
          if (q > 0 && rt[q] != cr) atomicAdd(par + T::nslot(cr), cn);
          cn = (q > 0 && rt[q] == cr) ? cn + n : n;
          cr = rt[q];
        }
      if (Tw | Bw) atomicAdd(par + T::nslot(cr), cn);
    }
    __syncthreads();
    uint32_t best = 0;
    for (int q = threadIdx.x; q < SSLOTS; q += blockDim.x) best = max(best, par[q]);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) best = max(best, __shfl_xor_sync(FULL, best, o2));
    if ((threadIdx.x & 31) == 0 && best) atomicMax(&s_max, best);
    __syncthreads();
    const uint32_t mx = s_max;
    {
      uint32_t x = Tw | Bw;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (x) {
          const uint32_t m = first_run(x);
          x &= ~m;
          if (par[T::nslot(rt[q])] == mx) {
            ST |= Tw & m;
            SB |= Bw & m;
          }
        }
    }
    uint32_t* o = out + size_t(slice) * g.slice;
    if (band < g.BH && w < int(g.pitch)) {
      // unit (band, w) owns both words; words >= wpr (padding) are zero
      if (lst.has_epi) {
        ST = eval_listing(lst.epi, q0, vm, ST);
        if (r + 1 < g.H) SB = eval_listing(lst.epi, q0 + g.pitch, vm, SB);
      }
      o[size_t(r) * g.pitch + w] = ST;
      if (r + 1 < g.H) o[size_t(r + 1) * g.pitch + w] = SB;
    }
  }
  }
}

template <int MODE>
int small_launch_jobs(const SmallJobs& jobs, int n, const G& g, cudaStream_t st,
                      const SmallListings& lst = SmallListings{}) {
  static PerDevice<int> attr;
  smem_opt_in(attr, k_small<MODE>, small_smem_bytes());
  pdl(k_small<MODE>, n * jobs.batch, ST_THREADS, small_smem_bytes(), st, jobs, g, lst);
  return 1;
}

template <int MODE>
int small_launch(const uint32_t* u, const uint32_t* t, uint32_t* out, const G& g, int batch,
                 cudaStream_t st) {
  SmallJobs jobs{};
  jobs.u[0] = u;
  jobs.t[0] = t;
  jobs.out[0] = out;
  jobs.batch = batch;
  return small_launch_jobs<MODE>(jobs, 1, g, st);
}

// ===========================================================================
// Fused single-launch reach for images whose tiles are all co-resident
// (NB bands x 256 px per CTA, e.g. 4096^2 = 512 tiles of 128x256 px on 148
// SMs): one cooperative launch with three grid barriers instead of five
// kernels.
//   A  the tile's target words (+ a 1-word/1-row halo) are staged in shared
//      memory and near(t) is taken from there; tile-local run union-find; per
//      local root a record {seeded, touches the ring, compact index}.  Ring
//      roots get compact ids c = tile * 512 + idx (<= 508 per tile) and a
//      node in a small global union-find GP; a seeded ring root starts out
//      under the virtual root SEED (the largest node value), so "seeded" is
//      simply "its root is SEED".  Runs that touch the ring publish
//      P[key block] = c.
//   B  each tile unites its own left and top borders on GP (atomicMax links).
//   C  (no barrier) each tile resolves its ring roots (root == SEED?) into
//      the records, then selects S | t per word from shared memory; the words
//      go to `sel` (global, for the neighbours' halos) and to shared memory.
//   D  the closing near^KOUT of the tile from shared memory, halo words of
//      the neighbouring tiles read from `sel`.
// Data written during the launch by other CTAs is read with ld.global.cg.
constexpr uint32_t REC_SEED = 1u << 31, REC_RING = 1u << 30, REC_ROOT = 1u << 29, REC_IDX = 511u;
constexpr uint32_t SEED = 0xffffffffu;  // no compact id hashes to it (ids < 2^31)
constexpr int FT_LIST = 512;
// per-tile words of the `lists` scratch region: LT_LIST for the multi-kernel
// path, or GP (512 u32) per fused tile (fused tiles may be half as tall: two per
// multi-kernel tile)
constexpr int FT_WORDS = 1280;
static_assert(FT_WORDS >= LT_LIST && FT_WORDS >= 2 * FT_LIST, "lists region too small");

__device__ __forceinline__ uint32_t cfind(uint32_t* GP, uint32_t v) {
  for (;;) {
    if (v == SEED) return v;
    const uint32_t p = __ldcg(GP + hkey(v));
    if (p == v || p == SEED) return p;
    const uint32_t gp = __ldcg(GP + hkey(p));
    if (gp == p) return p;
    __stcg(GP + hkey(v), gp);
    v = gp;
  }
}

__device__ void cunite(uint32_t* GP, uint32_t a, uint32_t b) {
  for (;;) {
    a = cfind(GP, a);
    b = cfind(GP, b);
    if (a == b) return;
    if (a < b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMax(GP + hkey(b), a);  // b != SEED: SEED is the largest
    if (old == b) return;
    b = old;
  }
}

// compact node of the ring run m of word j in band k (published in phase A)
__device__ __forceinline__ uint32_t cnode(const uint32_t* P, const G& g, int k, int j, uint32_t T,
                                          uint32_t B, uint32_t m) {
  int dr, col;
  run_max(T, B, m, dr, col);
  return hnode(__ldcg(P + kblk(g, gkey(g, 2 * k + dr, 32 * j + col))));
}

__device__ __forceinline__ void cunite_dedup(uint32_t* GP, uint32_t a, uint32_t b, bool active) {
  const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
  const uint32_t plo = __shfl_up_sync(mask, lo, 1), phi = __shfl_up_sync(mask, hi, 1);
  const bool prev_active = lane > 0 && ((mask >> (lane - 1)) & 1u);
  if (!active || a == b) return;
  if (prev_active && plo == lo && phi == hi) return;
  cunite(GP, a, b);
}

// word (r, j) of a bit image or 0 outside the image (halo staging)
__device__ __forceinline__ uint32_t word_or0(const uint32_t* img, const G& g, int r, int j,
                                             bool coherent) {
  if (r < 0 || r >= g.H || j < 0 || j >= g.wpr) return 0u;
  const uint32_t* p = img + size_t(r) * g.pitch + j;
  return coherent ? __ldcg(p) : __ldg(p);
}

// near^K of the word at (row sr, column sc) of a shared-memory window of
// 10-word rows (columns j0-1 .. j0+8), rows r0 .. r1 of the window valid
template <int K>
__device__ __forceinline__ uint32_t near_smem(const uint32_t* win, int sr, int sc, int r0, int r1) {
  uint32_t acc = 0;
#pragma unroll
  for (int d = -K; d <= K; ++d) {
    const int rr = sr + d;
    if (rr < r0 || rr > r1) continue;
    const uint32_t* row = win + rr * 10;
    const uint32_t C = row[sc], L = row[sc - 1], R = row[sc + 1];
    acc |= C;
#pragma unroll
    for (int e = 1; e <= K; ++e) acc |= __funnelshift_l(L, C, e) | __funnelshift_r(C, R, e);
  }
  return acc;
}

// TK: the target operand is near^TK(tbits) (nears folded into the reach by the
// program planner; the window then carries a TK+1 halo).  KOUT = 0 emits the
// selection S | t itself (no closing near: the consumer folds it as its TK).
template <int KOUT, int NB, int TK>
__global__ void __launch_bounds__(NB * LTWW, 2048 / (NB * LTWW)) k_reach_fused(const uint32_t* __restrict__ ubits,
                                                               const uint32_t* __restrict__ tbits,
                                                               uint32_t* P, uint32_t* GP,
                                                               uint32_t* sel,
                                                               uint32_t* __restrict__ out, G g,
                                                               long long* tstamp, int early) {
  cg::grid_group grid = cg::this_grid();
  // diagnostics (SLCS_PHASE_TIMING=1): per-CTA %globaltimer (ns) at phase boundaries
  int tsn = 0;
  auto stamp = [&]() {
    if (tstamp) {
      __syncthreads();
      if (threadIdx.x == 0) {
        long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        tstamp[(size_t((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x)) * 16 + tsn] =
            ns;
      }
      ++tsn;
    }
  };
  stamp();
  extern __shared__ __align__(16) unsigned char lsm[];
  constexpr int UNITS = NB * LTWW, SLOTS = NB * (1 << (LKW - 1));
  constexpr int TH = TK + 1;  // target window halo rows
  constexpr int TROWS = 2 * NB + 2 * TH, SROWS = KOUT > 0 ? 2 * NB + 2 * KOUT : 1;
  uint32_t* par = reinterpret_cast<uint32_t*>(lsm);  // SLOTS: union-find, then records
  uint32_t* sT = par + SLOTS;                         // UNITS
  uint32_t* sB = sT + UNITS;                          // UNITS
  uint32_t* tw = sB + UNITS;                          // TROWS x 10: target + halo
  uint32_t* sw = tw + TROWS * 10;                     // SROWS x 10: selection + halo
  uint16_t* ring = reinterpret_cast<uint16_t*>(sw + SROWS * 10);  // FT_LIST: idx -> root slot
  // the neighbour tiles' border words, prefetched in phase A for phase B: per
  // band the left tile's last word (T, B), then the upper tile's last band at
  // words j0-1 .. j0+8 (T, B)
  uint32_t* nbw = reinterpret_cast<uint32_t*>(ring + FT_LIST);  // 2 * NB + 20
  __shared__ int s_cnt;
  using T = RunTile<LKW>;
  const int slice = blockIdx.z;
  const uint32_t* u = ubits + size_t(slice) * g.slice;
  const uint32_t* t = tbits + size_t(slice) * g.slice;
  uint32_t* Ps = P + size_t(slice) * g.sb;
  uint32_t* ss = sel + size_t(slice) * g.slice;
  const int u0 = threadIdx.x;
  const int band = u0 / LTWW, w = u0 % LTWW;
  const int kb = blockIdx.y * NB + band;
  const int j0 = blockIdx.x * LTWW, j = j0 + w;
  const int R0 = blockIdx.y * NB * 2;  // first row of the tile
  const int r = 2 * kb;
  const bool in = kb < g.BH && j < g.wpr;
  const bool two = r + 1 < g.H;
#if !SLCS_COOP_PDL
  (void)early;
#else
  // Programmatic dependent launch: when `through` was not written by the
  // previous launch (early), everything up to the flattened tile union-find
  // reads only `through` and shared memory, so it runs while the previous
  // kernel drains; the target window and all scratch writes wait for it.
  // Otherwise even `through` is read only after the wait: the previous grid's
  // writes are guaranteed visible only once griddepcontrol.wait returns.
  if (!early) slcs_pdl_wait();
#endif
  const uint32_t Tw = in ? __ldcg(u + size_t(r) * g.pitch + j) : 0u;
  const uint32_t Bw = (in && two) ? __ldcg(u + size_t(r + 1) * g.pitch + j) : 0u;
  uint32_t tT, tB, seedT, seedB;
  auto stage_target = [&]() {
    // target window: rows R0-TH .. R0+2NB+TH-1, columns j0-1 .. j0+8 (halo words by
    // threads < 20TH + 4NB).  With TK > 0 the window holds the operand before its
    // folded nears and tbits may be written by the previous kernel of a chain.
    tw[(r - R0 + TH) * 10 + w + 1] = word_or0(t, g, r, j, false);
    tw[(r - R0 + TH + 1) * 10 + w + 1] = word_or0(t, g, r + 1, j, false);
    if (u0 < 20 * TH) {
      const int q = u0 % (10 * TH);
      const int hr = u0 < 10 * TH ? R0 - TH + q / 10 : R0 + 2 * NB + q / 10;
      tw[(hr - R0 + TH) * 10 + q % 10] = word_or0(t, g, hr, j0 - 1 + q % 10, false);
    } else if (u0 < 20 * TH + 4 * NB) {
      const int q = u0 - 20 * TH, side = q / (2 * NB), hr = R0 + q % (2 * NB);
      tw[(hr - R0 + TH) * 10 + (side ? 9 : 0)] = word_or0(t, g, hr, side ? j0 + 8 : j0 - 1, false);
    }
  };
  auto seeds = [&]() {
    // the target operand t = near^TK(window) at this unit's two words, and the
    // seeds through & near(t) = through & near^(TK+1)(window).  The box stencil is
    // separable: vertical ORs of the (L, C, R) column words first (shared by the
    // two rows and by both radii), then one horizontal pass per result.
    {
      const int base = r - R0;  // window row of r - TH
      uint3 rows[2 * TH + 2];
#pragma unroll
      for (int i = 0; i < 2 * TH + 2; ++i) {
        const uint32_t* wr = tw + (base + i) * 10 + w;
        rows[i] = make_uint3(wr[0], wr[1], wr[2]);
      }
      auto orv = [](uint3 a, uint3 b) { return make_uint3(a.x | b.x, a.y | b.y, a.z | b.z); };
      auto hdil = [](uint3 v, int k) {
        uint32_t acc = v.y;
#pragma unroll
        for (int e = 1; e <= TH; ++e)
          if (e <= k) acc |= __funnelshift_l(v.x, v.y, e) | __funnelshift_r(v.y, v.z, e);
        return acc;
      };
      // rows[TH] is row r, rows[TH + 1] is row r + 1
      uint3 inner = rows[TH];  // rows r - TK + 1 .. r + TK (shared core of both rows)
#pragma unroll
      for (int d = 1; d < TK; ++d) inner = orv(inner, orv(rows[TH - d], rows[TH + d]));
      if (TK > 0) inner = orv(inner, rows[TH + TK]);
      // row r: rows r-TK .. r+TK; row r+1: rows r-TK+1 .. r+TK+1
      const uint3 vT = TK > 0 ? orv(inner, rows[TH - TK]) : rows[TH];
      const uint3 vB = TK > 0 ? orv(inner, rows[TH + TK + 1]) : rows[TH + 1];
      tT = TK > 0 ? hdil(vT, TK) : rows[TH].y;
      tB = TK > 0 ? hdil(vB, TK) : rows[TH + 1].y;
      const uint3 sTv = orv(orv(vT, rows[TH - TK - 1]), rows[TH + TK + 1]);
      const uint3 sBv = orv(orv(vB, rows[TH - TK]), rows[2 * TH + 1]);  // rows r-TK .. r+TK+2
      seedT = Tw & hdil(sTv, TK + 1);
      seedB = Bw & hdil(sBv, TK + 1);
    }
  };
#if !SLCS_COOP_PDL
  stage_target();
#endif
  if (u0 < NB) {  // inputs only: safe to read before any barrier
    uint32_t a = 0, b = 0;
    if (blockIdx.x > 0) load_unit(u, g, blockIdx.y * NB + u0, j0 - 1, a, b);
    nbw[2 * u0] = a;
    nbw[2 * u0 + 1] = b;
  } else if (u0 < NB + 10) {
    uint32_t a = 0, b = 0;
    if (blockIdx.y > 0) load_unit(u, g, blockIdx.y * NB - 1, j0 - 1 + (u0 - NB), a, b);
    nbw[2 * NB + 2 * (u0 - NB)] = a;
    nbw[2 * NB + 2 * (u0 - NB) + 1] = b;
  }
  sT[u0] = Tw;
  sB[u0] = Bw;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
#if !SLCS_COOP_PDL
  seeds();
#endif
  stamp();  // 1: loads
  T tile{par, sT, sB};
#if SLCS_COOP_PDL && SLCS_FUSED_QUEUE
  {
    // the target/selection windows and the ring list are staged after the
    // union-find: their shared memory holds the link queue meanwhile
    constexpr int QWORDS = (TROWS * 10 + SROWS * 10 + FT_LIST / 2) / (UNITS / 32);
    __shared__ int s_qn[UNITS / 32];
    if (threadIdx.x < UNITS / 32) s_qn[threadIdx.x] = 0;
    __syncthreads();
    tile.link(u0, Tw, Bw, tw, s_qn, QWORDS);
  }
#else
  tile.link(u0, Tw, Bw);
#endif
  stamp();  // 2: link
  // flatten in place: a run's slot holds its root's slot, a root's slot holds
  // its record (REC_ROOT set) -- no per-run root registers stay live afterwards
  {
    uint32_t rt[16];
    tile.roots(u0, Tw, Bw, rt);
    __syncthreads();
    uint32_t x = Tw | Bw;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (!x) break;
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t k = T::key(band, w, Tw, Bw, m);
      par[T::slot(k)] = rt[i] == T::node(k) ? REC_ROOT : uint32_t(T::nslot(rt[i]));
    }
  }
#if SLCS_COOP_PDL
  if (early) slcs_pdl_wait();
  stage_target();
  __syncthreads();
  seeds();
#endif
  __syncthreads();
  stamp();  // 3: roots
  auto root_of = [&](uint32_t k) {  // the root's slot
    const uint32_t v = par[T::slot(k)];
    return (v & REC_ROOT) ? uint32_t(T::slot(k)) : v;
  };

  // ---- A: per-root records, compact ids of ring roots, ring runs -> P
  const uint32_t tile_id = (uint32_t(slice) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  const int C0 = j0 * 32;
  const uint32_t lmask = (1u << LKW) - 1u;
  auto ring_run = [&](uint32_t m) {
    return band == 0 || band == NB - 1 || (w == 0 && (m & 1u)) || (w == LTWW - 1 && (m >> 31));
  };
  for (uint32_t x = Tw | Bw; x;) {
    const uint32_t m = first_run(x);
    x &= ~m;
    const uint32_t marks = (ring_run(m) ? REC_RING : 0u) | (((seedT | seedB) & m) ? REC_SEED : 0u);
    if (marks) atomicOr(par + root_of(T::key(band, w, Tw, Bw, m)), marks);
  }
  __syncthreads();
  for (uint32_t x = Tw | Bw; x;) {
    const uint32_t m = first_run(x);
    x &= ~m;
    const uint32_t k = T::key(band, w, Tw, Bw, m);
    const uint32_t rec = par[T::slot(k)];
    if ((rec & REC_ROOT) && (rec & REC_RING)) {
      const uint32_t idx = uint32_t(atomicAdd(&s_cnt, 1));
      par[T::slot(k)] = rec | idx;
      ring[idx] = uint16_t(T::slot(k));
      const uint32_t c = tile_id * FT_LIST + idx;
      __stcg(GP + c, (rec & REC_SEED) ? SEED : hnode(c));
    }
  }
  __syncthreads();
  // publish only what the right and lower neighbours read in phase B: runs of
  // the last band and word-7 runs reaching bit 31 (this tile's own border side
  // comes from its records)
  for (uint32_t x = (band == NB - 1 || w == LTWW - 1) ? (Tw | Bw) : 0u; x;) {
    const uint32_t m = first_run(x);
    x &= ~m;
    if (band == NB - 1 || (m >> 31)) {
      const uint32_t k = T::key(band, w, Tw, Bw, m);
      const uint32_t c = tile_id * FT_LIST + (par[root_of(k)] & REC_IDX);
      __stcg(Ps + kblk(g, gkey(g, R0 + int(k >> LKW), C0 + int(k & lmask))), c);
    }
  }
  stamp();  // 4: records + publish
  grid.sync();
  stamp();  // 5: barrier

  // ---- B: unions across this tile's left border (threads 0..NB-1) and top
  // border (threads NB..NB+7).  This tile's side comes from shared memory (words
  // and root records), the neighbour's words were prefetched in phase A; only
  // the neighbour's published compact ids (P) are read from L2 here.
  auto own_cnode = [&](int bnd, int ww, uint32_t T, uint32_t B, uint32_t m) {
    return hnode(tile_id * FT_LIST + (par[root_of(T::key(bnd, ww, T, B, m))] & REC_IDX));
  };
  if (u0 < NB) {
    const int k = blockIdx.y * NB + u0;
    const int jr = j0, jl = jr - 1;
    if (blockIdx.x > 0 && k < g.BH) {
      const uint32_t Tl = nbw[2 * u0], Bl = nbw[2 * u0 + 1];
      const uint32_t Tr = sT[u0 * LTWW], Br = sB[u0 * LTWW];
      const uint32_t cl = Tl | Bl, cr = Tr | Br;
      const bool hlink = (cl >> 31) && (cr & 1u);
      const uint32_t va = hlink ? cnode(Ps, g, k, jl, Tl, Bl, run_at(cl, 31)) : 0u;
      const uint32_t vb = hlink ? own_cnode(u0, 0, Tr, Br, run_at(cr, 0)) : 0u;
      cunite_dedup(GP, va, vb, hlink);
      if (u0 != 0 && ((Tr & 1u) || (Tl >> 31))) {
        const uint32_t Tul = nbw[2 * u0 - 2], Bul = nbw[2 * u0 - 1];
        const uint32_t Tur = sT[(u0 - 1) * LTWW], Bur = sB[(u0 - 1) * LTWW];
        if ((Tr & 1u) && (Bul >> 31) && !(Bur & 1u))
          cunite(GP, own_cnode(u0, 0, Tr, Br, run_at(cr, 0)),
                 cnode(Ps, g, k - 1, jl, Tul, Bul, run_at(Tul | Bul, 31)));
        if ((Tl >> 31) && (Bur & 1u) && !(Bul >> 31))
          cunite(GP, cnode(Ps, g, k, jl, Tl, Bl, run_at(cl, 31)),
                 own_cnode(u0 - 1, 0, Tur, Bur, run_at(Tur | Bur, 0)));
      }
    }
  } else if (u0 < NB + LTWW) {
    const int k = blockIdx.y * NB;
    const int wo = u0 - NB, jj = j0 + wo;
    if (blockIdx.y > 0 && jj < g.wpr) {
      const uint32_t T0 = sT[wo], B0 = sB[wo];
      const uint32_t* up = nbw + 2 * NB + 2 * (wo + 1);  // upper band, word jj
      const uint32_t Tu = up[0], Bu = up[1];
      uint32_t Tl = 0, Bl = 0, Tr = 0, Br = 0;
      if ((T0 & 1u) && !(Bu & 1u)) {
        Tl = up[-2];
        Bl = up[-1];
      }
      if ((T0 >> 31) && !(Bu >> 31)) {
        Tr = up[2];
        Br = up[3];
      }
      const uint32_t cu = Tu | Bu;
      for (uint32_t x = T0 | B0; x;) {
        const uint32_t m = first_run(x);
        x &= ~m;
        const uint32_t td = T0 & m;
        if (!td) continue;
        const uint32_t v = own_cnode(0, wo, T0, B0, m);
        for (uint32_t a = dil1(td) & Bu; a;) {
          const uint32_t mu = run_at(cu, __ffs(a) - 1);
          a &= ~mu;
          cunite(GP, v, cnode(Ps, g, k - 1, jj, Tu, Bu, mu));
        }
        if ((td & 1u) && (Bl >> 31)) cunite(GP, v, cnode(Ps, g, k - 1, jj - 1, Tl, Bl, run_at(Tl | Bl, 31)));
        if ((td >> 31) && (Br & 1u)) cunite(GP, v, cnode(Ps, g, k - 1, jj + 1, Tr, Br, run_at(Tr | Br, 0)));
      }
    }
  }
  stamp();  // 6: merge
  grid.sync();
  stamp();  // 7: barrier
#if SLCS_COOP_PDL == 2
  // the next launch may start its through-only prologue on free SM slots.  Only
  // after this grid's last grid.sync: a cooperative launch re-arms the grid
  // barrier, so an earlier trigger breaks this grid's remaining barriers
  // (measured: triggering after the first barrier corrupts chained reaches)
  if (KOUT == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif

  // ---- C: resolve this tile's ring roots (read-only finds), then select
  if (u0 < s_cnt) {
    uint32_t v = hnode(tile_id * FT_LIST + uint32_t(u0));
    while (v != SEED) {
      const uint32_t q = __ldcg(GP + hkey(v));
      if (q == v) break;
      v = q;
    }
    if (v == SEED) par[ring[u0]] |= REC_SEED;
  }
  __syncthreads();
  stamp();  // 8: resolve
  {
    uint32_t ST = 0, SB = 0;
    for (uint32_t x = Tw | Bw; x;) {
      const uint32_t m = first_run(x);
      x &= ~m;
      if (par[root_of(T::key(band, w, Tw, Bw, m))] & REC_SEED) {
        ST |= Tw & m;
        SB |= Bw & m;
      }
    }
    ST |= tT;
    SB |= tB;
    if constexpr (KOUT == 0) {
      // the selection is the result (its consumer applies the closing near)
      if (kb < g.BH && j < int(g.pitch)) {
        uint32_t* o = out + size_t(slice) * g.slice;
        o[size_t(r) * g.pitch + j] = in ? ST : 0u;
        if (two) o[size_t(r + 1) * g.pitch + j] = in ? SB : 0u;
      }
      stamp();  // 9: select
      return;
    }
    sw[(r - R0 + KOUT) * 10 + w + 1] = ST;
    sw[(r - R0 + KOUT + 1) * 10 + w + 1] = SB;
    if (in) {
      __stcg(ss + size_t(r) * g.pitch + j, ST);
      if (two) __stcg(ss + size_t(r + 1) * g.pitch + j, SB);
    }
  }
  stamp();  // 9: select
  grid.sync();
  stamp();  // 10: barrier
#if SLCS_COOP_PDL == 2
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // after the last grid.sync
#endif

  // ---- D: closing near^KOUT; halo from the neighbours' selections
  constexpr int KO = KOUT > 0 ? KOUT : 1;  // (KOUT == 0 returned above)
  if (u0 < 20 * KOUT) {
    const int q = u0 % (10 * KOUT), hr = u0 < 10 * KOUT ? R0 - KOUT + q / 10 : R0 + 2 * NB + q / 10;
    sw[(hr - R0 + KOUT) * 10 + q % 10] = word_or0(ss, g, hr, j0 - 1 + q % 10, true);
  } else if (u0 < 20 * KOUT + 4 * NB) {
    const int q = u0 - 20 * KOUT, side = q / (2 * NB), hr = R0 + q % (2 * NB);
    sw[(hr - R0 + KOUT) * 10 + (side ? 9 : 0)] = word_or0(ss, g, hr, side ? j0 + 8 : j0 - 1, true);
  }
  __syncthreads();
  if (kb < g.BH && j < int(g.pitch)) {
    uint32_t* o = out + size_t(slice) * g.slice;
    const uint32_t vm = valid_mask(j, g.wpr, g.lastmask);
    o[size_t(r) * g.pitch + j] =
        j < g.wpr ? near_smem<KO>(sw, r - R0 + KOUT, w + 1, 0, SROWS - 1) & vm : 0u;
    if (two)
      o[size_t(r + 1) * g.pitch + j] =
          j < g.wpr ? near_smem<KO>(sw, r - R0 + KOUT + 1, w + 1, 0, SROWS - 1) & vm : 0u;
  }
  stamp();  // 11: near
}


// ---- chains of reaches against ONE labelling: one persistent launch ----------------
// The config-2 chain  x -> near -> reach(., u) -> near -> reach(., u) ...  runs
// 500 reaches of ONE `through` image u.  With label CSE the program labels u
// once (launch_labels); what is left of every reach is flag propagation:
//   seeds   S_s = components of u touching near(T_s)
//   select  U_s = T_s | S_s,     reach_s = near^k(U_s),  T_{s+1} = reach_s.
// k_reach_chain keeps a grid of co-resident tiles alive for the whole chain
// (cooperative launch, two grid barriers per reach):
//   setup   each tile finds the global root of every run of u it owns (two
//           loads per run, once) and gives the tile's distinct roots compact
//           local ids (shared-memory hash); runs keep their local id.
//   seed    the tile stages its slice of the previous U (+3-row / 1-word halo,
//           L2) in shared memory, applies near^(a+1) (a = the previous closing
//           radius), marks the local ids of runs touching it, then publishes
//           one flag stamp per seeded distinct root (F[root] = gen).
//   --- grid barrier ---
//   select  one flag load per distinct root of the tile, U = near^a(prev) | S
//           (same staged window), stored for the next step.
//   --- grid barrier ---
// No per-reach labelling, no per-run root lookups, and per step only the
// staged window, the tile's roots' flags and the U words touch L2.  Runs of
// tiles with more than CH_MAXL distinct roots fall back to a direct root
// lookup (correct, slower).  Flags are the label-CSE stamps (gen = reach
// index + 1; the labelling step zeroes them once per run).
constexpr int CH_TW = 8;     // words per tile row (256 px)
// Tile = 32 bands (64 rows) x 8 words (256 px), 128 threads: 4096^2 -> 16 x 64 =
// 1024 tiles, 7 co-resident per SM.  Smaller tiles hide the per-step latency better
// (measured C2: 56 bands / 4 per SM 2.50 ms, 32 / 7 2.30 ms, 16 / 14 2.43 ms,
// 28 / 8 with a partial warp 2.53 ms).
#ifndef SLCS_CH_TB
#define SLCS_CH_TB 32
#endif
#ifndef SLCS_CH_MAXL
#define SLCS_CH_MAXL 1024
#endif
#ifndef SLCS_CH_MINB
#define SLCS_CH_MINB 7
#endif
constexpr int CH_TB = SLCS_CH_TB;  // bands per tile
constexpr int CH_THREADS = CH_TW * CH_TB / 2;  // a thread owns two stacked bands of one word
constexpr int CH_R = 3;                       // max stencil radius
constexpr int CH_ROWS = 2 * CH_TB + 2 * CH_R;  // staged rows
constexpr int CH_SW = 16;     // staged row stride: halo word, 8 words (16 B aligned), halo word
constexpr int CH_C0 = 4;      // column of the tile's first word in a staged row
constexpr int CH_MAXL = SLCS_CH_MAXL;  // distinct roots with a local id
constexpr int CH_HASH = 2 * CH_MAXL;
constexpr int CH_HASH_BITS = CH_HASH == 4096 ? 12 : (CH_HASH == 2048 ? 11 : (CH_HASH == 1024 ? 10 : 13));
static_assert((1 << CH_HASH_BITS) == CH_HASH, "CH_HASH must be 1024 .. 8192");
constexpr uint16_t CH_NOL = 0xffffu;
constexpr size_t CH_SMEM_LIDS = size_t(CH_TW) * CH_TB * 16 * 2;
constexpr size_t CH_SMEM_ROOTS = size_t(CH_MAXL) * 4;
constexpr size_t CH_SMEM_FLAGS = 2 * size_t(CH_MAXL);  // flags + neighbour masks
constexpr size_t CH_SMEM_STAGE = size_t(CH_ROWS) * CH_SW * 4;
constexpr size_t CH_SMEM_HROWS = 2 * size_t(CH_ROWS) * CH_TW * 4;  // H_a, H_(a+1)
constexpr size_t CH_SMEM_REGION = size_t(CH_HASH) * 6 > CH_SMEM_STAGE + CH_SMEM_HROWS
                                      ? size_t(CH_HASH) * 6
                                      : CH_SMEM_STAGE + CH_SMEM_HROWS;
constexpr size_t CH_SMEM = CH_SMEM_LIDS + CH_SMEM_ROOTS + CH_SMEM_FLAGS + CH_SMEM_REGION;
// a tile's halo record (u64 = step tag << 32 | word): its top 3 rows and bottom 3
// rows (8 words each), its first and last word of every row
constexpr int CH_H_TOP = 0, CH_H_BOT = 3 * CH_TW, CH_H_LEFT = 6 * CH_TW,
              CH_H_RIGHT = 6 * CH_TW + 2 * CH_TB, CH_HALO = 6 * CH_TW + 4 * CH_TB;

struct ChainArgs {
  const uint32_t* x;  // target of the first reach
  const uint32_t* u;  // through
  const uint32_t* P;  // labelling of u (launch_labels)
  uint32_t* F;        // per root block: the first step that seeded it (min stamp; 0xff..)
  unsigned long long* halo;  // per tile: its boundary words of every step, tagged (ch_halo)
  unsigned int* arrive;      // per step: tiles that published that step's seeds (zeroed)
  unsigned int* tilecnt;     // per root block: tiles holding the root (zeroed)
  unsigned int* tile_arrive;  // per tile: 1 + the last step it published seeds for (zeroed)
  unsigned int* tile_roots;   // per tile: count + its distinct roots (CH_MAXL + 1 words)
  uint32_t* out;      // near^klast(U of the last reach)
  int steps;
  int kmid;           // closing radius of every reach but the last (0..2)
  int klast;          // closing radius of the last reach (1..3)
  uint32_t gen0;      // flag stamp of the first reach
  unsigned long long* ts;  // diagnostics (SLCS_PHASE_TIMING=1): per CTA phase ns sums, or null
};

__device__ __forceinline__ unsigned long long ch_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// horizontal dilations of staged word (row r, column c) by R and R + 1 bits
template <int R>
__device__ __forceinline__ void ch_hdil2(const uint32_t* st, int r, int c, uint32_t& da,
                                         uint32_t& db) {
  const uint32_t* p = st + r * CH_SW + c;
  const uint32_t m = p[0], l = p[-1], rr = p[1];
  uint32_t d = m;
#pragma unroll
  for (int k = 1; k <= R; ++k) d |= __funnelshift_l(l, m, k) | __funnelshift_r(m, rr, k);
  da = d;
  db = d | __funnelshift_l(l, m, R + 1) | __funnelshift_r(m, rr, R + 1);
}

// rows r0 .. r0+3 of a vertical R-window OR over the per-row dilations H
template <int R>
__device__ __forceinline__ void ch_vwin4(const uint32_t* H, int r0, int c, uint32_t (&o)[4]) {
  uint32_t v[4 + 2 * R];
#pragma unroll
  for (int i = 0; i < 4 + 2 * R; ++i) v[i] = H[(r0 - R + i) * CH_TW + c];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t acc = v[q];
#pragma unroll
    for (int i = 1; i <= 2 * R; ++i) acc |= v[q + i];
    o[q] = acc;
  }
}

__device__ __forceinline__ void ch_vwin4_dyn(const uint32_t* H, int r0, int c, int R,
                                             uint32_t (&o)[4]) {
  switch (R) {
    case 0: ch_vwin4<0>(H, r0, c, o); break;
    case 1: ch_vwin4<1>(H, r0, c, o); break;
    case 2: ch_vwin4<2>(H, r0, c, o); break;
    default: ch_vwin4<3>(H, r0, c, o); break;
  }
}

// halo records: one 64-bit word carries (step tag, data), so each is written and
// read with a single-copy-atomic relaxed gpu-scope access and validates itself
__device__ __forceinline__ void ch_rec_store(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ch_rec_load(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ch_hash(uint32_t key) {
  return (key * 0x9E3779B1u) >> (32 - CH_HASH_BITS);
}

__global__ void __launch_bounds__(CH_THREADS, SLCS_CH_MINB) k_reach_chain(ChainArgs a, G g) {
  slcs_pdl_wait();
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* lids = reinterpret_cast<uint16_t*>(smem);
  uint32_t* lroot = reinterpret_cast<uint32_t*>(smem + CH_SMEM_LIDS);
  uint8_t* lflag = smem + CH_SMEM_LIDS + CH_SMEM_ROOTS;
  uint8_t* lnbr = lflag + CH_MAXL;  // per root: which of the 8 neighbour tiles hold it
  unsigned char* region = smem + CH_SMEM_LIDS + CH_SMEM_ROOTS + CH_SMEM_FLAGS;
  uint32_t* hkeys = reinterpret_cast<uint32_t*>(region);
  uint16_t* hlid = reinterpret_cast<uint16_t*>(region + size_t(CH_HASH) * 4);
  uint32_t* stage = reinterpret_cast<uint32_t*>(region);
  uint32_t* Ha = reinterpret_cast<uint32_t*>(region + CH_SMEM_STAGE);  // [row][word]
  uint32_t* Hb = Ha + CH_ROWS * CH_TW;
  __shared__ int nl_sh, has_nol, pend_global, pend_mask, pub_any;

  const int tid = threadIdx.x;
  const int tiles_x = (int(g.pitch) + CH_TW - 1) / CH_TW;
  const int j0 = (int(blockIdx.x) % tiles_x) * CH_TW;
  const int k0 = (int(blockIdx.x) / tiles_x) * CH_TB;
  const int jw = tid % CH_TW, kb0 = 2 * (tid / CH_TW);  // bands kb0, kb0 + 1 of word jw
  const int j = j0 + jw;
  const uint32_t EMPTYK = 0xffffffffu;
  const unsigned long long t_start = (a.ts != nullptr && tid == 0) ? ch_now() : 0ull;

  // ---- setup: runs of u, their roots, compact local ids ----
  for (int i = tid; i < CH_HASH; i += CH_THREADS) hkeys[i] = EMPTYK;
  if (tid == 0) {
    nl_sh = 0;
    has_nol = 0;
    pub_any = 0;
  }
  uint32_t T[2], B[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = k0 + kb0 + q;
    T[q] = B[q] = 0u;
    if (k < g.BH && j < g.wpr) {
      const uint32_t* row = a.u + size_t(2 * k) * g.pitch + j;
      T[q] = __ldg(row);
      B[q] = 2 * k + 1 < g.H ? __ldg(row + g.pitch) : 0u;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = k0 + kb0 + q;
    for (uint32_t x = T[q] | B[q]; x;) {
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t rb = gblk(g, groot(a.P, g, grun(g, k, j, T[q], B[q], m)));
      uint32_t h = ch_hash(rb);
      bool stored = false;
      for (int probe = 0; probe < CH_HASH; ++probe, h = (h + 1) & (CH_HASH - 1)) {
        const uint32_t old = atomicCAS(hkeys + h, EMPTYK, rb);
        if (old == EMPTYK || old == rb) {
          stored = true;
          break;
        }
      }
      // a full table: the root goes without a local id, but still counts as held
      // here (possibly more than once -- an over-count only makes the other
      // holders treat it as shared, i.e. wait for it)
      if (!stored) atomicAdd(a.tilecnt + rb, 1u);
    }
  }
  __syncthreads();
  for (int i = tid; i < CH_HASH; i += CH_THREADS) {
    if (hkeys[i] == EMPTYK) continue;
    const int l = atomicAdd(&nl_sh, 1);
    hlid[i] = l < CH_MAXL ? uint16_t(l) : CH_NOL;
    // a root beyond the local ids is seeded here through F (global stamps): the
    // other tiles that hold it must count this tile as a holder too
    if (l >= CH_MAXL) atomicAdd(a.tilecnt + hkeys[i], 1u);
    if (l < CH_MAXL) lroot[l] = hkeys[i];
  }
  __syncthreads();
  const int nl = min(nl_sh, CH_MAXL);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = k0 + kb0 + q, unit = (kb0 + q) * CH_TW + jw;
    int ri = 0;
    for (uint32_t x = T[q] | B[q]; x; ++ri) {
      const uint32_t m = first_run(x);
      x &= ~m;
      const uint32_t rb = gblk(g, groot(a.P, g, grun(g, k, j, T[q], B[q], m)));
      uint16_t l = CH_NOL;
      uint32_t h = ch_hash(rb);
      for (int probe = 0; probe < CH_HASH; ++probe, h = (h + 1) & (CH_HASH - 1)) {
        const uint32_t kk = hkeys[h];
        if (kk == rb) {
          l = hlid[h];
          break;
        }
        if (kk == EMPTYK) break;
      }
      lids[unit * 16 + ri] = l;
      if (l == CH_NOL) has_nol = 1;
    }
  }
  // roots held by more than one tile ("shared") can be seeded elsewhere; the
  // others only here.  A shared root whose holders are all among the 8
  // neighbouring tiles only ever needs those neighbours' progress.  lflag bits:
  // 1 seeded (sticky), 2 shared, 4 seeded this step, 8 held beyond the neighbours
  const int tiles_y = (g.BH + CH_TB - 1) / CH_TB;
  const int tx = int(blockIdx.x) % tiles_x, ty = int(blockIdx.x) / tiles_x;
  {
    unsigned int* mine = a.tile_roots + size_t(blockIdx.x) * (CH_MAXL + 1);
    for (int i = tid; i < nl; i += CH_THREADS) {
      atomicAdd(a.tilecnt + lroot[i], 1u);
      mine[1 + i] = lroot[i];
      lnbr[i] = 0;
    }
    if (tid == 0) mine[0] = unsigned(nl);
  }
  grid.sync();
  for (int n = 0; n < 8; ++n) {
    const int dx = n < 3 ? n - 1 : (n == 3 ? -1 : (n == 4 ? 1 : n - 6));
    const int dy = n < 3 ? -1 : (n < 5 ? 0 : 1);
    const int ntx = tx + dx, nty = ty + dy;
    if (ntx < 0 || ntx >= tiles_x || nty < 0 || nty >= tiles_y) continue;
    const unsigned int* list = a.tile_roots + (size_t(nty) * tiles_x + ntx) * (CH_MAXL + 1);
    const int cnt = int(__ldcg(list));
    for (int e = tid; e < cnt; e += CH_THREADS) {
      const uint32_t rb = __ldcg(list + 1 + e);
      uint32_t h = ch_hash(rb);
      for (int probe = 0; probe < CH_HASH; ++probe, h = (h + 1) & (CH_HASH - 1)) {
        const uint32_t kk = hkeys[h];
        if (kk == rb) {
          const uint16_t l = hlid[h];
          if (l != CH_NOL)
            atomicOr(reinterpret_cast<unsigned*>(lnbr + (l & ~3)), (1u << n) << (8 * (l & 3)));
          break;
        }
        if (kk == EMPTYK) break;
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < nl; i += CH_THREADS) {
    const unsigned cnt = __ldcg(a.tilecnt + lroot[i]);
    uint8_t f = cnt > 1u ? 2 : 0;
    if (cnt > 1u && unsigned(__popc(lnbr[i])) + 1u < cnt) f |= 8;
    lflag[i] = f;
  }
  __syncthreads();  // the hash region becomes the staging window
  unsigned long long tacc[7] = {0, 0, 0, 0, 0, 0, 0}, tprev = 0, nbr_waits = 0;
  const bool timing = a.ts != nullptr && tid == 0;
  auto mark = [&](int ph) {
    if (a.ts != nullptr && timing) {
      const unsigned long long t = ch_now();
      tacc[ph] += t - tprev;
      tprev = t;
    }
  };
  if (timing) {
    tprev = ch_now();
    tacc[0] = tprev - t_start;
  }

  // stage rows [2 k0 - 3, 2 k0 + 2 CH_TB + 3) of the first target: two 16 B loads
  // per row for the tile's 8 words, one word of halo on each side; zeros outside
  auto stage_rows = [&](const uint32_t* src) {
    for (int i = tid; i < CH_ROWS * 4; i += CH_THREADS) {
      const int r = i >> 2, part = i & 3;
      const int gr = 2 * k0 - CH_R + r;
      const bool in_row = gr >= 0 && gr < g.H;
      const uint32_t* row = src + size_t(gr) * g.pitch;
      uint32_t* dst = stage + r * CH_SW;
      if (part < 2) {
        const int w = j0 + 4 * part;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (in_row && w < int(g.pitch)) v = __ldcg(reinterpret_cast<const uint4*>(row + w));
        *reinterpret_cast<uint4*>(dst + CH_C0 + 4 * part) = v;
      } else if (part == 2) {
        dst[CH_C0 - 1] = in_row && j0 > 0 ? __ldcg(row + j0 - 1) : 0u;
      } else {
        dst[CH_C0 + CH_TW] = in_row && j0 + CH_TW < g.wpr ? __ldcg(row + j0 + CH_TW) : 0u;
      }
    }
  };
  // later steps: the tile's own rows are already in the window (its select wrote
  // them); the neighbours' boundary words come from their halo records, each
  // word tagged with its step, so waiting for the data IS the synchronisation
  // (no grid barrier between a step's select and the next step's seed).
  // Each thread owns at most two halo words of the window; where they come from
  // is fixed for the whole chain, so it is resolved once.  Words outside the
  // image stay the zeros the first full staging wrote.
  constexpr int CH_NHALO = 6 * (CH_TW + 2) + 2 * 2 * CH_TB;
  static_assert(CH_NHALO <= 2 * CH_THREADS, "each thread stages at most two halo words");
  const unsigned long long* hsrc[2] = {nullptr, nullptr};
  int hdst[2] = {0, 0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = tid + q * CH_THREADS;
    if (i >= CH_NHALO) continue;
    int ntx, nty, idx, dst;
    if (i < 6 * (CH_TW + 2)) {
      const int rr = i / (CH_TW + 2), c = i - rr * (CH_TW + 2);  // c: staged col - (C0-1)
      const bool above = rr < 3;
      const int r = above ? rr : CH_R + 2 * CH_TB + (rr - 3);
      nty = above ? ty - 1 : ty + 1;
      const int base = above ? CH_H_BOT + rr * CH_TW : CH_H_TOP + (rr - 3) * CH_TW;
      if (c == 0) {
        ntx = tx - 1;
        idx = base + CH_TW - 1;
      } else if (c == CH_TW + 1) {
        ntx = tx + 1;
        idx = base;
      } else {
        ntx = tx;
        idx = base + c - 1;
      }
      dst = r * CH_SW + CH_C0 - 1 + c;
    } else {
      const int qq = i - 6 * (CH_TW + 2);
      const int row = qq >> 1, right = qq & 1;
      nty = ty;
      ntx = right ? tx + 1 : tx - 1;
      idx = right ? CH_H_LEFT + row : CH_H_RIGHT + row;
      dst = (CH_R + row) * CH_SW + (right ? CH_C0 + CH_TW : CH_C0 - 1);
    }
    if (ntx < 0 || ntx >= tiles_x || nty < 0 || nty >= tiles_y) continue;
    hsrc[q] = a.halo + (size_t(nty) * tiles_x + ntx) * CH_HALO + size_t(idx);
    hdst[q] = dst;
  }
  // records are double-buffered by tag parity: a tile that does not wait for the
  // others can run one step ahead of a neighbour, never two (it needs that
  // neighbour's previous step to stage its own)
  const size_t halo_bank = size_t(gridDim.x) * CH_HALO;
  auto stage_halo = [&](unsigned long long tag) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!hsrc[q]) continue;
      const unsigned long long* p = hsrc[q] + (tag & 1) * halo_bank;
      unsigned long long v = ch_rec_load(p);
      for (int spin = 0; (v >> 32) != tag; ++spin) {
        if (spin > (1 << 22)) __trap();  // a producer never arrived: fail, never hang
        __nanosleep(SLCS_CH_SLEEP);
        v = ch_rec_load(p);
      }
      stage[hdst[q]] = uint32_t(v);
    }
  };
  // per staged row, the tile's words dilated horizontally by ra and ra + 1
  auto hrows = [&](int ra) {
    for (int i = tid; i < CH_ROWS * CH_TW; i += CH_THREADS) {
      const int r = i / CH_TW, c = i - r * CH_TW;
      switch (ra) {
        case 0: ch_hdil2<0>(stage, r, CH_C0 + c, Ha[i], Hb[i]); break;
        case 1: ch_hdil2<1>(stage, r, CH_C0 + c, Ha[i], Hb[i]); break;
        case 2: ch_hdil2<2>(stage, r, CH_C0 + c, Ha[i], Hb[i]); break;
        default: ch_hdil2<3>(stage, r, CH_C0 + c, Ha[i], Hb[i]); break;
      }
    }
  };

  const int lr0 = CH_R + 2 * kb0;  // staged row of this thread's first row
  const unsigned ntiles = gridDim.x;
  bool unseeded = (T[0] | B[0] | T[1] | B[1]) != 0u;  // this thread has unseeded runs
  // The chain is monotone: T(s+1) = near^kmid(U(s)) contains U(s), which contains
  // T(s), so a component seeded once stays seeded.  Seeds are therefore sticky:
  // a tile publishes a root only the step it becomes seeded (F = min stamp), and
  // waits for the other tiles only while it still holds SHARED roots that are
  // unseeded -- a tile whose roots are all seeded or all its own never waits.
  for (int s = 0; s < a.steps; ++s) {
    const int ra = s == 0 ? 0 : a.kmid;  // prev -> target radius
    const uint32_t gen = a.gen0 + uint32_t(s);
    if (s == 0) stage_rows(a.x);
    else stage_halo((unsigned long long)s);
    __syncthreads();
    mark(6);
    hrows(ra);
    __syncthreads();
    mark(1);
    // seed: runs of u touching near(target) = near^(ra+1)(prev), not yet seeded
    // (a thread whose runs were all seeded at its last select has nothing to do)
    // Stamping F sets pub_any; thread 0 then makes its arrival a release (fence +
    // relaxed write) only in steps where this tile stamped something.  A release
    // on every arrival made thread 0 pay a full fence every step; stamps are rare.
    bool pub = false;
    if (unseeded) {
      uint32_t n[4];
      ch_vwin4_dyn(Hb, lr0, jw, ra + 1, n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t sd = (T[q] & n[2 * q]) | (B[q] & n[2 * q + 1]);
        if (!sd) continue;
        const int unit = (kb0 + q) * CH_TW + jw;
        int ri = 0;
        for (uint32_t x = T[q] | B[q]; x; ++ri) {
          const uint32_t m = first_run(x);
          x &= ~m;
          if (!(sd & m)) continue;
          const uint16_t l = lids[unit * 16 + ri];
          if (l != CH_NOL) {
            if (!(lflag[l] & 1)) lflag[l] |= 4;
          } else {
            atomicMin(a.F + gblk(g, groot(a.P, g, grun(g, k0 + kb0 + q, j, T[q], B[q], m))), gen);
            pub = true;
          }
        }
      }
    }
    if (tid == 0) {
      pend_global = has_nol;
      pend_mask = 0;
    }
    __syncthreads();
    for (int i = tid; i < nl; i += CH_THREADS) {
      uint8_t f = lflag[i];
      if (f & 4) {
        f = uint8_t((f & ~4) | 1);
        lflag[i] = f;
        if (f & 2) {
          atomicMin(a.F + lroot[i], gen);
          pub = true;
        }
      }
      if ((f & 3) == 2) {  // shared and still unseeded: another tile may seed it
        if (f & 8) pend_global = 1;
        else atomicOr(&pend_mask, int(lnbr[i]));
      }
    }
    if (pub) pub_any = 1;
    __syncthreads();
    mark(2);
    // arrive (this tile's seeds of step s are published); then wait for the
    // tiles that can still seed one of this tile's unseeded shared roots: all
    // of them, only some neighbours, or none
    const bool wait = pend_global || pend_mask;
    if (a.ts != nullptr && tid == 0) {  // diagnostics: steps with a global / neighbour wait
      if (pend_global) tacc[5] += 1000;
      else if (pend_mask) ++nbr_waits;
    }
    if (tid == 0) {
      // release pattern when stamps were made (fence.acq_rel.gpu, cumulative
      // over the block barrier, then the relaxed writes): a reader that observes
      // these arrivals with ld.acquire sees this step's stamps
      if (pub_any) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        pub_any = 0;
      }
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.arrive + s) : "memory");
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a.tile_arrive + blockIdx.x),
                   "r"(unsigned(s + 1))
                   : "memory");
      auto spin_until = [&](const unsigned* p, unsigned target) {
        for (int spin = 0;; ++spin) {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
          if (v >= target) return;
          if (spin > (1 << 24)) __trap();  // never hang
          __nanosleep(32);
        }
      };
      if (pend_global) {
        spin_until(a.arrive + s, ntiles);
      } else {
        for (int n = 0; n < 8; ++n) {
          if (!((pend_mask >> n) & 1)) continue;
          const int dx = n < 3 ? n - 1 : (n == 3 ? -1 : (n == 4 ? 1 : n - 6));
          const int dy = n < 3 ? -1 : (n < 5 ? 0 : 1);
          spin_until(a.tile_arrive + (size_t(ty + dy) * tiles_x + (tx + dx)), unsigned(s + 1));
        }
      }
    }
    mark(3);
    if (wait) {  // shared roots seeded elsewhere this step
      __syncthreads();
      for (int i = tid; i < nl; i += CH_THREADS) {
        const uint8_t f = lflag[i];
        if ((f & 3) == 2 && __ldcg(a.F + lroot[i]) <= gen) lflag[i] = uint8_t(f | 1);
      }
      __syncthreads();
    }
    // select: U = near^ra(prev) | seeded components
    uint32_t uo_keep[4] = {0u, 0u, 0u, 0u};
    bool still_unseeded = false;
    if (j < int(g.pitch)) {
      uint32_t (&uo)[4] = uo_keep;
      if (j < g.wpr) {
        ch_vwin4_dyn(Ha, lr0, jw, ra, uo);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int unit = (kb0 + q) * CH_TW + jw;
          int ri = 0;
          for (uint32_t x = T[q] | B[q]; x; ++ri) {
            const uint32_t m = first_run(x);
            x &= ~m;
            const uint16_t l = lids[unit * 16 + ri];
            const bool sel =
                l != CH_NOL ? (lflag[l] & 1) != 0
                            : __ldcg(a.F + gblk(g, groot(a.P, g, grun(g, k0 + kb0 + q, j, T[q],
                                                                      B[q], m)))) <= gen;
            if (sel) {
              uo[2 * q] |= T[q] & m;
              uo[2 * q + 1] |= B[q] & m;
            } else {
              still_unseeded = true;
            }
          }
        }
        const uint32_t vm = valid_mask(j, g.wpr, g.lastmask);
#pragma unroll
        for (int i = 0; i < 4; ++i) uo[i] &= vm;
      }
    }
    // the next window's own rows (stage is free: this step read it through Ha/Hb),
    // and this tile's boundary words for its neighbours, tagged with the step
    unseeded = still_unseeded;
#pragma unroll
    for (int i = 0; i < 4; ++i) stage[(lr0 + i) * CH_SW + CH_C0 + jw] = uo_keep[i];
    {
      const unsigned long long tag = (unsigned long long)(s + 1) << 32;
      unsigned long long* my_halo = a.halo + ((s + 1) & 1) * halo_bank +
                                    size_t(blockIdx.x) * CH_HALO;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 2 * kb0 + i;  // tile-relative
        const unsigned long long v = tag | uo_keep[i];
        if (row < 3) ch_rec_store(my_halo + CH_H_TOP + row * CH_TW + jw, v);
        if (row >= 2 * CH_TB - 3)
          ch_rec_store(my_halo + CH_H_BOT + (row - (2 * CH_TB - 3)) * CH_TW + jw, v);
        if (jw == 0) ch_rec_store(my_halo + CH_H_LEFT + row, v);
        if (jw == CH_TW - 1) ch_rec_store(my_halo + CH_H_RIGHT + row, v);
      }
    }
    __syncthreads();
    mark(4);
  }
  if (timing)
  {
    for (int i = 0; i < 7; ++i) a.ts[size_t(blockIdx.x) * 8 + i] = tacc[i];
    a.ts[size_t(blockIdx.x) * 8 + 7] = nbr_waits * 1000;
  }

  // closing near of the last reach
  stage_halo((unsigned long long)a.steps);
  __syncthreads();
  hrows(a.klast);
  __syncthreads();
  if (j < int(g.pitch)) {
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    if (j < g.wpr) {
      ch_vwin4_dyn(Ha, lr0, jw, a.klast, o);
      const uint32_t vm = valid_mask(j, g.wpr, g.lastmask);
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] &= vm;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = 2 * (k0 + kb0) + i;
      if (r < g.H) a.out[size_t(r) * g.pitch + j] = o[i];
    }
  }
}

int grid_blocks(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return int(b);
}

void check_key_range(const Geo& gb, const char* what) {
  KeyGeo k = key_geo(gb.w, gb.h);
  unsigned long long maxkey =
      ((unsigned long long)(gb.h - 1) << k.s) | (unsigned long long)(gb.w - 1);
  if (maxkey > 0xffffffffull)
    fail(SLCS_ERR_TOO_LARGE, std::string(what) + ": image too large for 32-bit run keys");
}

}  // namespace

bool ccl_small_path(int w, int h) { return w <= 256 && h <= 256; }

static size_t n_tiles(int w, int h) {
  return size_t((((w + 31) / 32) + LTWW - 1) / LTWW) * size_t(((h + 1) / 2 + LTNB - 1) / LTNB);
}

size_t ccl_scratch_bytes(int w, int h, int batch, bool flags, bool sizes) {
  if (ccl_small_path(w, h)) return 0;
  return ccl_scratch_bytes_large(w, h, batch, flags, sizes);
}

size_t ccl_scratch_bytes_large(int w, int h, int batch, bool flags, bool sizes) {
  KeyGeo k = key_geo(w, h);
  size_t n = k.slice_blocks * size_t(batch);
  size_t b = round_up(n * 4, 256) + round_up(n_tiles(w, h) * size_t(batch) * FT_WORDS * 4, 256);
  if (flags) b += round_up(n, 256);
  if (sizes) b += round_up(n * 4, 256) + round_up(size_t(batch) * 4, 256);
  return b;
}

void ccl_scratch_carve(void* base, int w, int h, int batch, bool flags, bool sizes,
                       CclScratch* s) {
  *s = CclScratch{};
  if (ccl_small_path(w, h)) return;
  ccl_scratch_carve_large(base, w, h, batch, flags, sizes, s);
}

void ccl_scratch_carve_large(void* base, int w, int h, int batch, bool flags, bool sizes,
                             CclScratch* s) {
  *s = CclScratch{};
  KeyGeo k = key_geo(w, h);
  size_t n = k.slice_blocks * size_t(batch);
  unsigned char* p = static_cast<unsigned char*>(base);
  s->parent = reinterpret_cast<uint32_t*>(p);
  p += round_up(n * 4, 256);
  s->lists = reinterpret_cast<uint32_t*>(p);
  p += round_up(n_tiles(w, h) * size_t(batch) * FT_WORDS * 4, 256);
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

template <int MODE>
size_t tile_smem() {
  return size_t(LSLOTS) * 4 + 2 * size_t(LUNITS) * 4 + 2 * size_t(LSLOTS) + 16;
}

template <int MODE>
void tile_launch(dim3 grid, const uint32_t* u, const uint32_t* t, CclScratch& s, const G& g,
                 cudaStream_t st) {
  static PerDevice<int> attr;
  smem_opt_in(attr, k_tile_local<MODE>, tile_smem<MODE>());
#if SLCS_TL_PHASES
  {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbolAsync(tl_phase_acc, z, sizeof z, 0, cudaMemcpyHostToDevice, st);
  }
#endif
  pdl(k_tile_local<MODE>, grid, LT_THREADS, tile_smem<MODE>(), st, u, t, s.parent, s.flag, s.size,
                                                                 s.lists, g);
#if SLCS_TL_PHASES
  {
    unsigned long long z[8];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(z, tl_phase_acc, sizeof z);
    const double n = double(grid.x) * grid.y * grid.z;
    std::fprintf(stderr, "[tile_local<%d> %0.f tiles, cycles per tile] init %.0f link %.0f "
                 "roots+out %.0f maxkeys %.0f lists %.0f\n", MODE, n, z[0] / n, z[1] / n,
                 z[2] / n, z[3] / n, z[4] / n);
  }
#endif
}

static void large_local_and_merge(const uint32_t* u, const uint32_t* t, const G& g, int batch,
                                  CclScratch& s, int mode, cudaStream_t st, int& launches) {
  dim3 grid(unsigned((g.wpr + LTWW - 1) / LTWW), unsigned((g.BH + LTNB - 1) / LTNB),
            unsigned(batch));
  if (mode == MODE_REACH)
    tile_launch<MODE_REACH>(grid, u, t, s, g, st);
  else if (mode == MODE_BOTH)
    tile_launch<MODE_BOTH>(grid, u, t, s, g, st);
  else if (mode == MODE_SIZE)
    tile_launch<MODE_SIZE>(grid, u, t, s, g, st);
  else
    tile_launch<MODE_CCL>(grid, u, t, s, g, st);
  ++launches;
  const int nhb = int(grid.y) - 1, nvb = int(grid.x) - 1;
  const size_t links = size_t(nhb) * g.wpr + size_t(nvb) * g.BH;
  if (links) {
    dim3 mg(unsigned(grid_blocks(links, 256)), unsigned(batch));
    pdl(k_tile_merge, mg, 256, 0, st, u, s.parent, g, nhb, nvb);
    ++launches;
    const int ntiles = int(grid.x * grid.y);
    dim3 fg(unsigned(ntiles) * 2u, unsigned(batch));
    pdl(k_root_flatten, fg, 256, 0, st, s.parent, s.flag, s.size, s.lists, g, ntiles, mode);
    launches += 1;
  }
}

size_t ccl_labels_bytes(int w, int h, int batch) {
  return ccl_scratch_bytes(w, h, batch, false, false);
}

int launch_labels(const uint32_t* through, void* labels, const Geo& gb, cudaStream_t st) {
  check_key_range(gb, "reach");
  G g = make_g(gb);
  CclScratch s;
  ccl_scratch_carve(labels, gb.w, gb.h, gb.batch, false, false, &s);
  int launches = 0;
  large_local_and_merge(through, nullptr, g, gb.batch, s, MODE_CCL, st, launches);
  return launches;
}

bool reach_chain_fits(const Geo& gb, int steps, int kmid, int klast) {
  if (gb.batch != 1 || steps < 1 || kmid < 0 || kmid > 2 || klast < 1 || klast > CH_R) return false;
  static PerDevice<int> cap;
  const int capacity = cap.get([](int dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaFuncSetAttribute(k_reach_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(CH_SMEM)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_reach_chain, CH_THREADS, CH_SMEM) !=
            cudaSuccess)
      per = 0;
    cudaGetLastError();
    return per * sms;
  });
  const size_t tiles = size_t((gb.pitch + CH_TW - 1) / CH_TW) *
                       size_t((size_t(gb.h) + 2 * CH_TB - 1) / (2 * CH_TB));
  return tiles <= size_t(capacity);
}

size_t reach_chain_scratch_bytes(const Geo& gb, int steps) {
  const size_t tiles = size_t((gb.pitch + CH_TW - 1) / CH_TW) *
                       size_t((size_t(gb.h) + 2 * CH_TB - 1) / (2 * CH_TB));
  return 2 * tiles * CH_HALO * 8 + (size_t(steps) + tiles + tiles * (CH_MAXL + 1)) * 4;
}

int launch_reach_chain(const uint32_t* x, const uint32_t* through, const void* labels,
                       uint32_t* flags32, uint32_t idx0, int steps, int kmid, int klast,
                       uint32_t* out, uint32_t* tmp2, const Geo& gb, cudaStream_t st) {
  if (!reach_chain_fits(gb, steps, kmid, klast))
    fail(SLCS_ERR_ARG, "reach chain does not fit one cooperative launch");
  if (idx0 + uint32_t(steps) > 4096u) fail(SLCS_ERR_ARG, "too many reaches share one labelling");
  G g = make_g(gb);
  ChainArgs a;
  a.x = x;
  a.u = through;
  a.P = static_cast<const uint32_t*>(labels);
  a.F = flags32;
  const unsigned tiles = unsigned(((gb.pitch + CH_TW - 1) / CH_TW) *
                                  ((size_t(gb.h) + 2 * CH_TB - 1) / (2 * CH_TB)));
  // scratch: halo records, per-step arrival counters; the labelling's two flag
  // copies: min seed stamps (0xff..) and per-root tile counts (0)
  a.halo = reinterpret_cast<unsigned long long*>(tmp2);
  a.arrive = reinterpret_cast<unsigned int*>(a.halo + 2 * size_t(tiles) * CH_HALO);
  a.tile_arrive = a.arrive + steps;
  a.tile_roots = a.tile_arrive + tiles;
  a.tilecnt = flags32 + g.sb;
  a.out = out;
  a.steps = steps;
  a.kmid = kmid;
  a.klast = klast;
  a.gen0 = idx0 + 1u;
  a.ts = nullptr;
  static const bool timing = [] {
    const char* e = std::getenv("SLCS_PHASE_TIMING");
    return e && *e == '1';
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles);
  cfg.blockDim = dim3(CH_THREADS);
  cfg.dynamicSmemBytes = CH_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaMemsetAsync(a.halo, 0,
                             2 * size_t(tiles) * CH_HALO * 8 + (size_t(steps) + tiles) * 4, st),
             "chain halo");
  cuda_check(cudaMemsetAsync(a.F, 0xff, size_t(g.sb) * 4, st), "chain flags");
  cuda_check(cudaMemsetAsync(a.tilecnt, 0, size_t(g.sb) * 4, st), "chain tile counts");
  if (timing) cuda_check(cudaMalloc(&a.ts, size_t(tiles) * 8 * 8), "timing buffer");
  cuda_check(cudaLaunchKernelEx(&cfg, k_reach_chain, a, g), "reach chain launch");
  if (timing) {  // diagnostics only: per-step phase times, mean and max over CTAs (us)
    std::vector<unsigned long long> h(size_t(tiles) * 8);
    cuda_check(cudaStreamSynchronize(st), "timing sync");
    cuda_check(cudaMemcpy(h.data(), a.ts, h.size() * 8, cudaMemcpyDeviceToHost), "timing copy");
    cudaFree(a.ts);
    const char* names[] = {"setup", "hdil", "seed+publish", "arrive/wait", "select+store",
                           "global-wait share", "stage/halo wait", "neighbour-wait share"};
    std::fprintf(stderr, "[reach chain: %u tiles, %d steps; us per step (setup: total), mean/max]",
                 tiles, steps);
    for (int ph = 0; ph < 8; ++ph) {
      double sum = 0, mx = 0;
      for (unsigned t = 0; t < tiles; ++t) {
        const double v = double(h[size_t(t) * 8 + ph]) / 1e3 / (ph ? steps : 1);
        sum += v;
        mx = v > mx ? v : mx;
      }
      std::fprintf(stderr, " %s %.2f/%.2f", names[ph], sum / tiles, mx);
    }
    std::fprintf(stderr, "\n");
  }
  return 1;
}

int launch_reach_labeled(const uint32_t* target, const uint32_t* through, const void* labels,
                         uint32_t* flags32, uint32_t idx, uint32_t* out,
                         uint32_t* tmp_bits, const Geo& gb, cudaStream_t st, int k_out) {
  if (idx >= 4096u) fail(SLCS_ERR_ARG, "too many reaches share one labelling");
  const uint32_t gen = idx + 1u;
  G g = make_g(gb);
  const uint32_t* P = static_cast<const uint32_t*>(labels);
  dim3 ug(unsigned(grid_blocks(size_t(g.BH) * g.wpr, 256)), unsigned(gb.batch));
  pdl(k_reach_seed, ug, 256, 0, st, through, target, P, flags32, gen, g);
  dim3 sg(unsigned(grid_blocks(size_t(g.BH) * g.pitch, 256)), unsigned(gb.batch));
  pdl(k_reach_select_gen, sg, 256, 0, st, through, target, P, flags32, gen, tmp_bits, g);
  return 2 + launch_near(tmp_bits, out, gb, k_out, false, st);
}

// reach split in phases for row bands: prepare (labels + seed flags), export a
// row's roots/classes, import resolved flags, finish (select [+ closing near])
int launch_reach_prepare(const uint32_t* target, const uint32_t* through, const Geo& gb,
                         CclScratch& s, cudaStream_t st, bool max_keys) {
  check_key_range(gb, "reach");
  if (max_keys && (unsigned long long)gb.w * (unsigned long long)gb.h >= 0xfffffffeull)
    fail(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
  G g = make_g(gb);
  int launches = 0;
  large_local_and_merge(through, target, g, gb.batch, s, max_keys ? MODE_BOTH : MODE_REACH, st,
                        launches);
  return launches;
}

int launch_reach_row(const uint32_t* through, const CclScratch& s, const Geo& gb, int row,
                     uint32_t* roots, uint8_t* cls, cudaStream_t st) {
  G g = make_g(gb);
  pdl(k_band_row, (g.wpr + 127) / 128, 128, 0, st, through, s.parent, s.flag, row, roots, cls, g);
  return 1;
}

int launch_reach_set_flags(const CclScratch& s, const Geo& gb, const uint32_t* roots, int n,
                           cudaStream_t st) {
  if (n <= 0) return 0;
  G g = make_g(gb);
  pdl(k_band_set_flags, (n + 255) / 256, 256, 0, st, roots, n, s.flag, g);
  return 1;
}

int launch_reach_set_flags_dev(const CclScratch& s, const Geo& gb, const uint32_t* roots,
                               const int* n_dev, int max_n, cudaStream_t st) {
  if (max_n <= 0) return 0;
  G g = make_g(gb);
  pdl(k_band_set_flags_dev, (max_n + 255) / 256, 256, 0, st, roots, n_dev, s.flag, g);
  return 1;
}

int launch_reach_finish(const uint32_t* target, const uint32_t* through, const CclScratch& s,
                        uint32_t* out, uint32_t* tmp_bits, const Geo& gb, int k_out,
                        cudaStream_t st) {
  G g = make_g(gb);
  dim3 sg(unsigned(grid_blocks(size_t(g.BH) * g.pitch, 256)), unsigned(gb.batch));
  uint32_t* dst = k_out > 0 ? tmp_bits : out;
  pdl(k_reach_select, sg, 256, 0, st, through, target, s.parent, s.flag, dst, g);
  return 1 + (k_out > 0 ? launch_near(tmp_bits, out, gb, k_out, false, st) : 0);
}

int launch_ccl(const uint32_t* bits, uint32_t* labels, const Geo& gb, CclScratch& s,
               cudaStream_t st) {
  if ((unsigned long long)gb.w * (unsigned long long)gb.h >= 0xfffffffeull)
    fail(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
  check_key_range(gb, "ccl");
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h)) return small_launch<0>(bits, nullptr, labels, g, gb.batch, st);
  int launches = 0;
  large_local_and_merge(bits, nullptr, g, gb.batch, s, MODE_CCL, st, launches);
  const size_t warps = size_t(g.BH) * size_t((g.wpr + 31) / 32);
  dim3 lg(unsigned(std::min<size_t>((warps + TL_WARPS - 1) / TL_WARPS, 148 * 16)),
          unsigned(gb.batch));
  pdl(k_tile_labels<uint32_t>, lg, TL_WARPS * 32, 0, st, bits, s.parent, s.size, labels, g,
      LabelMap64{}, 1);
  return launches + 1;
}

int launch_ccl_prepare(const uint32_t* bits, const Geo& gb, CclScratch& s, cudaStream_t st) {
  if ((unsigned long long)gb.w * (unsigned long long)gb.h >= 0xfffffffeull)
    fail(SLCS_ERR_TOO_LARGE, "image too large for packed coordinate labels");
  if (ccl_small_path(gb.w, gb.h) || gb.batch != 1)
    fail(SLCS_ERR_ARG, "ccl_prepare: a single image larger than 256x256");
  check_key_range(gb, "ccl");
  G g = make_g(gb);
  int launches = 0;
  large_local_and_merge(bits, nullptr, g, 1, s, MODE_CCL, st, launches);
  return launches;
}

// the u32 labels of one row (a band's border record), from the union-find
__global__ void k_row_labels(const uint32_t* __restrict__ ubits, const uint32_t* __restrict__ P,
                             const uint32_t* __restrict__ MK, G g, int row,
                             uint32_t* __restrict__ out) {
  slcs_pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= g.wpr) return;
  const int k = row >> 1;
  const uint32_t T = __ldg(ubits + size_t(2 * k) * g.pitch + j);
  const uint32_t B = 2 * k + 1 < g.H ? __ldg(ubits + size_t(2 * k + 1) * g.pitch + j) : 0u;
  uint32_t rb[16];
  run_root_blocks(P, g, k, j, T, B, rb);
  const uint32_t starts = (T | B) & ~((T | B) << 1), bits = (row & 1) ? B : T;
  for (int x = 0; x < 32 && 32 * j + x < g.W; ++x)
    out[32 * j + x] = ((bits >> x) & 1u)
                          ? linear_label(g, MK[pick16(rb, __popc(starts & ((2u << x) - 1u)) - 1)])
                          : 0u;
}

int launch_ccl_row_labels(const uint32_t* bits, const Geo& gb, const CclScratch& s, int row,
                          uint32_t* out, cudaStream_t st) {
  G g = make_g(gb);
  pdl(k_row_labels, unsigned((g.wpr + 127) / 128), 128, 0, st, bits, s.parent, s.size, g, row,
      out);
  return 1;
}

int launch_ccl_labels64(const uint32_t* bits, const Geo& gb, const CclScratch& s,
                        const LabelMap64& map, unsigned long long* out, cudaStream_t st) {
  G g = make_g(gb);
  const size_t warps = size_t(g.BH) * size_t((g.wpr + 31) / 32);
  dim3 lg(unsigned(std::min<size_t>((warps + TL_WARPS - 1) / TL_WARPS, 148 * 16)), 1u);
  const int vec_ok = reinterpret_cast<uintptr_t>(out) % 16 == 0;
  pdl(k_tile_labels<unsigned long long>, lg, TL_WARPS * 32, 0, st, bits, s.parent, s.size, out, g,
      map, vec_ok);
  return 1;
}

template <int KOUT, int NB, int TK>
bool reach_fused_try(const uint32_t* target, const uint32_t* through, uint32_t* out,
                     uint32_t* tmp_bits, const G& g, int batch, CclScratch& s, cudaStream_t st,
                     bool early) {
  constexpr int THREADS = NB * LTWW;
  constexpr size_t smem = size_t(NB) * (1 << (LKW - 1)) * 4 + 2 * size_t(THREADS) * 4 +
                          size_t(2 * NB + 2 * (TK + 1)) * 40 +
                          size_t(KOUT > 0 ? 2 * NB + 2 * KOUT : 1) * 40 + FT_LIST * 2 +
                          size_t(2 * NB + 20) * 4;
  // co-resident CTAs on this device (thread-safe one-time initialisation)
  static PerDevice<int> cap;
  const int capacity = cap.get([](int dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaFuncSetAttribute(k_reach_fused<KOUT, NB, TK>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_reach_fused<KOUT, NB, TK>, THREADS,
                                                      smem) != cudaSuccess)
      per = 0;
    cudaGetLastError();  // a failed opt-in only disables the fused path
    return per * sms;
  });
  dim3 grid(unsigned((g.wpr + LTWW - 1) / LTWW), unsigned((g.BH + NB - 1) / NB),
            unsigned(batch));
  const size_t tiles = size_t(grid.x) * grid.y * grid.z;
  if (tiles > size_t(capacity)) return false;
  uint32_t* GP = s.lists;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (SLCS_COOP_PDL && pdl_enabled()) ? 2 : 1;
  static const bool timing = [] {
    const char* e = std::getenv("SLCS_PHASE_TIMING");
    return e && *e == '1';
  }();
  long long* ts = nullptr;
  if (timing) cuda_check(cudaMalloc(&ts, tiles * 16 * sizeof(long long)), "timing buffer");
  cuda_check(cudaLaunchKernelEx(&cfg, k_reach_fused<KOUT, NB, TK>, through, target, s.parent, GP,
                                tmp_bits, out, g, ts, early ? 1 : 0),
             "fused reach launch");
  if (timing) {  // diagnostics only: timeline of phase ends, min/max over CTAs (us)
    std::vector<long long> h(tiles * 16);
    cuda_check(cudaStreamSynchronize(st), "timing sync");
    cuda_check(cudaMemcpy(h.data(), ts, h.size() * sizeof(long long), cudaMemcpyDeviceToHost),
               "timing copy");
    cudaFree(ts);
    const char* names[] = {"start", "load", "link", "roots", "records", "bar1", "merge", "bar2",
                           "resolve", "select", "bar3", "near"};
    long long t0 = h[0];
    for (size_t t = 0; t < tiles; ++t) t0 = h[t * 16] < t0 ? h[t * 16] : t0;
    std::fprintf(stderr, "[fused reach %zu tiles, us since first CTA: min/max]", tiles);
    for (int ph = 0; ph <= 11; ++ph) {
      long long mn = h[ph], mx = h[ph];
      for (size_t t = 0; t < tiles; ++t) {
        mn = h[t * 16 + ph] < mn ? h[t * 16 + ph] : mn;
        mx = h[t * 16 + ph] > mx ? h[t * 16 + ph] : mx;
      }
      std::fprintf(stderr, " %s %.1f/%.1f", names[ph], (mn - t0) / 1e3, (mx - t0) / 1e3);
    }
    std::fprintf(stderr, "\n");
    std::vector<std::pair<long long, size_t>> ld;
    for (size_t t = 0; t < tiles; ++t) ld.push_back({h[t * 16 + 2] - h[t * 16 + 1], t});
    std::sort(ld.begin(), ld.end());
    std::fprintf(stderr, "  link us: median %.1f, slowest tiles (x,y):", ld[tiles / 2].first / 1e3);
    for (size_t q = tiles > 6 ? tiles - 6 : 0; q < tiles; ++q)
      std::fprintf(stderr, " %.1f@(%zu,%zu)", ld[q].first / 1e3, ld[q].second % grid.x,
                   (ld[q].second / grid.x) % grid.y);
    std::fprintf(stderr, "\n");
  }
  return true;
}

bool fused_reach_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SLCS_NO_FUSED_REACH");
    return !(e && *e && *e != '0');
  }();
  return on;
}

int launch_maxvol_small_listing(const FusedProgram* pro, const FusedProgram* epi,
                                const uint32_t* bits, uint32_t* out, const Geo& gb,
                                cudaStream_t st) {
  if (!ccl_small_path(gb.w, gb.h)) fail(SLCS_ERR_ARG, "maxvol listings need a small image");
  SmallListings lst;
  if (pro) {
    lst.pro = *pro;
    lst.has_pro = 1;
  }
  if (epi) {
    lst.epi = *epi;
    lst.has_epi = 1;
  }
  SmallJobs jobs{};
  jobs.u[0] = bits;
  jobs.out[0] = out;
  jobs.batch = gb.batch;
  return small_launch_jobs<2>(jobs, 1, make_g(gb), st, lst);
}

// n (<= 4) independent small-image reaches of one shape in one k_small launch
int launch_reach_small_multi(const uint32_t* const* target, const uint32_t* const* through,
                             uint32_t* const* out, int n, const Geo& gb, cudaStream_t st) {
  if (!ccl_small_path(gb.w, gb.h) || n < 1 || n > kSmallJobs)
    fail(SLCS_ERR_ARG, "reach: batched launch needs 1-4 small images");
  G g = make_g(gb);
  SmallJobs jobs{};
  for (int i = 0; i < n; ++i) {
    jobs.u[i] = through[i];
    jobs.t[i] = target[i];
    jobs.out[i] = out[i];
  }
  jobs.batch = gb.batch;
  return small_launch_jobs<1>(jobs, n, g, st);
}

int launch_reach(const uint32_t* target, const uint32_t* through, uint32_t* out,
                 uint32_t* tmp_bits, const Geo& gb, CclScratch& s, cudaStream_t st, int k_out,
                 int tk, bool early_through) {
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h)) {
    if (k_out != 1 || tk != 0)
      fail(SLCS_ERR_ARG, "reach: folded nears need the tiled path");
    return small_launch<1>(through, target, out, g, gb.batch, st);
  }
  if (k_out < 0 || k_out > 8 || tk < 0 || tk > 8) fail(SLCS_ERR_ARG, "reach: near radius out of range");
  check_key_range(gb, "reach");
  if (fused_reach_enabled()) {
    static const int nb = [] {
      const char* e = std::getenv("SLCS_FUSED_NB");
      // A/B switch; 32-band tiles measured equal (10.72 vs 10.62 ms on the chain)
      return (e && std::atoi(e) == 128) ? 128 : 64;
    }();
    bool done = false;
#define SLCS_FUSED(KO, NBV, TKV)                                                                \
  case (KO) * 10000 + (NBV) * 10 + (TKV):                                                      \
    done = reach_fused_try<KO, NBV, TKV>(target, through, out, tmp_bits, g, gb.batch, s, st,  \
                                         early_through);                                       \
    break;
    switch (k_out * 10000 + nb * 10 + tk) {
      SLCS_FUSED(0, 64, 0) SLCS_FUSED(0, 64, 1) SLCS_FUSED(0, 64, 2)
      SLCS_FUSED(1, 64, 0) SLCS_FUSED(1, 64, 1) SLCS_FUSED(1, 64, 2)
      SLCS_FUSED(2, 64, 0) SLCS_FUSED(2, 64, 1) SLCS_FUSED(2, 64, 2)
      SLCS_FUSED(3, 64, 0) SLCS_FUSED(3, 64, 1) SLCS_FUSED(3, 64, 2)
      SLCS_FUSED(4, 64, 0) SLCS_FUSED(4, 64, 1) SLCS_FUSED(4, 64, 2)
      SLCS_FUSED(1, 128, 0) SLCS_FUSED(2, 128, 0)
      default: break;
    }
#undef SLCS_FUSED
    if (done) return 1;
  }
  // tiled multi-kernel path.  Folded target nears are applied first (into `out`,
  // which is free until the end: the select reads and writes each word in place)
  int launches = 0;
  const uint32_t* tgt = target;
  if (tk > 0) {
    launches += launch_near(target, out, gb, tk, false, st);
    tgt = out;
  }
  large_local_and_merge(through, tgt, g, gb.batch, s, MODE_REACH, st, launches);
  dim3 sg(unsigned(grid_blocks(size_t(g.BH) * g.pitch, 256)), unsigned(gb.batch));
  uint32_t* dst = k_out > 0 ? tmp_bits : out;
  pdl(k_reach_select, sg, 256, 0, st, through, tgt, s.parent, s.flag, dst, g);
  launches += 1;
  if (k_out > 0) launches += launch_near(tmp_bits, out, gb, k_out, false, st);
  return launches;
}

int launch_maxvol(const uint32_t* bits, uint32_t* out, const Geo& gb, CclScratch& s,
                  cudaStream_t st) {
  G g = make_g(gb);
  if (ccl_small_path(gb.w, gb.h)) return small_launch<2>(bits, nullptr, out, g, gb.batch, st);
  check_key_range(gb, "maxvol");
  int launches = 0;
  cudaMemsetAsync(s.maxv, 0, size_t(gb.batch) * 4, st);
  large_local_and_merge(bits, nullptr, g, gb.batch, s, MODE_SIZE, st, launches);
  dim3 pg(unsigned(grid_blocks(size_t(g.BH) * g.wpr, 256)), unsigned(gb.batch));
  pdl(k_maxvol_max, pg, 256, 0, st, bits, s.parent, s.size, s.maxv, g);
  dim3 sg(unsigned(grid_blocks(size_t(g.BH) * g.pitch, 256)), unsigned(gb.batch));
  pdl(k_maxvol_select, sg, 256, 0, st, bits, s.parent, s.size, s.maxv, out, g);
  return launches + 2;
}


}  // namespace slcs
