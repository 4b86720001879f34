// bands.cu -- cross-band merges for row-band decomposition.
//
// A very large image is split into row bands, one per GPU.  Each band runs the
// single-image kernels on its own rows; what crosses a band border is resolved
// here, on the device, from a small per-band BORDER RECORD that the caller
// all-gathers (NCCL all_gather_into_tensor over NVLink): every rank then runs
// the same tiny union-find over all records and keeps its own part.  Nothing
// goes through the host.
//
// Nodes are border pixels: slot s = (band b, side, column c), side 0 = the
// band's first row, 1 = its last row.  Slots of one band that belong to the
// same band-local component (same root node / same local label) are joined
// through a hash table keyed (band, component); slots touching across a band
// border (8-connectivity: columns c-1, c, c+1) are united with a lock-free
// union-find (link the larger slot under the smaller, atomicCAS).
//
//  reach   record = roots + classes of the first/last row (k_band_row) and the
//          first/last TARGET row.  A component is seeded if any of its border
//          pixels is seeded locally or touches a target pixel across the border
//          (near(t) reaching into the neighbour band, reach.cpp:20-37).  Each
//          rank flags its own newly seeded roots (then select + closing near).
//  ccl     record = band-local labels (local max index + 1) of the first/last
//          row.  Global label = row0 * W + local; a component crossing borders
//          takes the max over its parts -- the canonical label of the whole
//          image, ccl.hpp:52-60.  Each rank relabels its band to 64 bits.
#include "slcs_internal.h"

namespace slcs {
namespace {

constexpr uint32_t NONE = 0xffffffffu;
constexpr unsigned long long EMPTY = ~0ull;

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__device__ __forceinline__ uint32_t hash_slot(unsigned long long key, uint32_t mask) {
  return band_hash_slot(key, mask);  // the same slots the label writers probe
}

// insert `key` (absent: EMPTY) and keep the smallest slot id as its representative
__device__ void hash_insert_min(unsigned long long* keys, uint32_t* rep, uint32_t mask,
                                unsigned long long key, uint32_t s) {
  uint32_t h = hash_slot(key, mask);
  for (;;) {
    const unsigned long long old = atomicCAS(keys + h, EMPTY, key);
    if (old == EMPTY || old == key) {
      atomicMin(rep + h, s);
      return;
    }
    h = (h + 1) & mask;
  }
}

__device__ uint32_t hash_find(const unsigned long long* keys, uint32_t mask,
                              unsigned long long key) {
  uint32_t h = hash_slot(key, mask);
  for (;;) {
    const unsigned long long k = __ldcg(keys + h);
    if (k == key) return h;
    if (k == EMPTY) return NONE;
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* P, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(P + x);
    if (p == x) return x;
    const uint32_t gp = __ldcg(P + p);
    if (gp != p) __stcg(P + x, gp);  // path halving (benign race: gp is an ancestor)
    x = p;
  }
}

__device__ void uf_unite(uint32_t* P, uint32_t a, uint32_t b) {
  for (;;) {
    a = uf_find(P, a);
    b = uf_find(P, b);
    if (a == b) return;
    const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
    if (atomicCAS(P + hi, hi, lo) == hi) return;
  }
}

// ---- border record accessors -------------------------------------------------------
struct ReachRec {  // byte offsets inside one band's record
  size_t roots[2], cls[2], tgt[2], bytes;
};
ReachRec reach_rec(int w, size_t pitch_words) {
  ReachRec r;
  const size_t w4 = align16(size_t(w) * 4), w1 = align16(size_t(w)), p4 = pitch_words * 4;
  r.roots[0] = 0;
  r.roots[1] = w4;
  r.cls[0] = 2 * w4;
  r.cls[1] = 2 * w4 + w1;
  r.tgt[0] = 2 * w4 + 2 * w1;
  r.tgt[1] = r.tgt[0] + p4;
  r.bytes = r.tgt[1] + p4;
  return r;
}
struct LabelRec {
  size_t lab[2], bytes;
};
LabelRec label_rec(int w) {
  LabelRec r;
  const size_t w4 = align16(size_t(w) * 4);
  r.lab[0] = 0;
  r.lab[1] = w4;
  r.bytes = 2 * w4;
  return r;
}

struct MergeGeo {
  int nb, w;
  uint32_t nslots;  // nb * 2 * w
  uint32_t hmask;   // hash capacity - 1
  size_t rec_bytes;
};

__device__ __forceinline__ void slot_parts(const MergeGeo& m, uint32_t s, int& b, int& side,
                                           int& c) {
  b = int(s / (2u * uint32_t(m.w)));
  const uint32_t r = s - uint32_t(b) * 2u * uint32_t(m.w);
  side = int(r / uint32_t(m.w));
  c = int(r - uint32_t(side) * uint32_t(m.w));
}
__device__ __forceinline__ uint32_t slot_of(const MergeGeo& m, int b, int side, int c) {
  return (uint32_t(b) * 2u + uint32_t(side)) * uint32_t(m.w) + uint32_t(c);
}

// component id of a slot (0 = background) and its hash key
struct ReachView {
  const unsigned char* rec;
  ReachRec off;
  __device__ bool fg(const MergeGeo& m, int b, int side, int c) const {
    return cls(m, b, side, c) != 0;
  }
  // root node of the pixel's band-local component (any value, 0 included)
  __device__ uint32_t comp(const MergeGeo& m, int b, int side, int c) const {
    return reinterpret_cast<const uint32_t*>(rec + size_t(b) * m.rec_bytes + off.roots[side])[c];
  }
  __device__ uint8_t cls(const MergeGeo& m, int b, int side, int c) const {
    return reinterpret_cast<const uint8_t*>(rec + size_t(b) * m.rec_bytes + off.cls[side])[c];
  }
  __device__ bool tgt(const MergeGeo& m, int b, int side, int c) const {
    if (c < 0 || c >= m.w) return false;
    const uint32_t* t =
        reinterpret_cast<const uint32_t*>(rec + size_t(b) * m.rec_bytes + off.tgt[side]);
    return (t[c >> 5] >> (c & 31)) & 1u;
  }
};
struct LabelView {
  const unsigned char* rec;
  LabelRec off;
  __device__ bool fg(const MergeGeo& m, int b, int side, int c) const {
    return comp(m, b, side, c) != 0;
  }
  __device__ uint32_t comp(const MergeGeo& m, int b, int side, int c) const {
    return reinterpret_cast<const uint32_t*>(rec + size_t(b) * m.rec_bytes + off.lab[side])[c];
  }
};

__device__ __forceinline__ unsigned long long comp_key(int b, uint32_t comp) {
  return (static_cast<unsigned long long>(b) << 32) | comp;
}

template <class V>
__global__ void k_merge_insert(V v, MergeGeo m, unsigned long long* keys, uint32_t* rep) {
  slcs_pdl_wait();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.nslots;
       s += gridDim.x * blockDim.x) {
    int b, side, c;
    slot_parts(m, s, b, side, c);
    if (v.fg(m, b, side, c)) hash_insert_min(keys, rep, m.hmask, comp_key(b, v.comp(m, b, side, c)), s);
  }
}

// parent of a foreground slot = the representative slot of its band component
template <class V>
__global__ void k_merge_init(V v, MergeGeo m, const unsigned long long* keys, const uint32_t* rep,
                             uint32_t* P, uint32_t* Rp) {
  slcs_pdl_wait();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.nslots;
       s += gridDim.x * blockDim.x) {
    int b, side, c;
    slot_parts(m, s, b, side, c);
    const uint32_t r =
        v.fg(m, b, side, c) ? rep[hash_find(keys, m.hmask, comp_key(b, v.comp(m, b, side, c)))] : s;
    P[s] = r;
    Rp[s] = r;
  }
}

// unions across each band border: last row of band b with first row of b + 1
template <class V>
__global__ void k_merge_unite(V v, MergeGeo m, uint32_t* P) {
  slcs_pdl_wait();
  const uint32_t n = uint32_t(m.nb - 1) * uint32_t(m.w);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int b = int(i / uint32_t(m.w)), c = int(i - uint32_t(b) * uint32_t(m.w));
    if (!v.fg(m, b, 1, c)) continue;
    const uint32_t s1 = slot_of(m, b, 1, c);
    for (int d = -1; d <= 1; ++d) {
      const int c2 = c + d;
      if (c2 < 0 || c2 >= m.w || !v.fg(m, b + 1, 0, c2)) continue;
      uf_unite(P, s1, slot_of(m, b + 1, 0, c2));
    }
  }
}

// reach: a set is seeded if a member is seeded in its band or touches a target
// pixel of the neighbouring band across the border
__global__ void k_merge_seed(ReachView v, MergeGeo m, uint32_t* P, uint8_t* seeded) {
  slcs_pdl_wait();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.nslots;
       s += gridDim.x * blockDim.x) {
    int b, side, c;
    slot_parts(m, s, b, side, c);
    const uint8_t k = v.cls(m, b, side, c);
    if (!k) continue;
    bool seed = k == 2;
    if (!seed && side == 0 && b > 0)
      seed = v.tgt(m, b - 1, 1, c - 1) || v.tgt(m, b - 1, 1, c) || v.tgt(m, b - 1, 1, c + 1);
    if (!seed && side == 1 && b + 1 < m.nb)
      seed = v.tgt(m, b + 1, 0, c - 1) || v.tgt(m, b + 1, 0, c) || v.tgt(m, b + 1, 0, c + 1);
    if (seed) seeded[uf_find(P, s)] = 1;
  }
}

// this band's roots whose merged set is seeded: one entry per band component,
// reported by its representative slot
__global__ void k_merge_collect_reach(ReachView v, MergeGeo m, int me, uint32_t* P,
                                      const uint32_t* Rp, const uint8_t* seeded, uint32_t* out,
                                      int* count) {
  slcs_pdl_wait();
  const uint32_t n = 2u * uint32_t(m.w);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = uint32_t(me) * n + i;
    const int side = int(i / uint32_t(m.w)), c = int(i - uint32_t(side) * uint32_t(m.w));
    if (v.cls(m, me, side, c) != 1) continue;  // background, or already seeded locally
    if (Rp[s] != s || !seeded[uf_find(P, s)]) continue;
    out[atomicAdd(count, 1)] = v.comp(m, me, side, c);
  }
}

// ccl: global label of a slot and the max over its merged set
__global__ void k_merge_max_label(LabelView v, MergeGeo m, const unsigned long long* row0w,
                                  uint32_t* P, unsigned long long* gmax) {
  slcs_pdl_wait();
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m.nslots;
       s += gridDim.x * blockDim.x) {
    int b, side, c;
    slot_parts(m, s, b, side, c);
    const uint32_t l = v.comp(m, b, side, c);
    if (l) atomicMax(gmax + uf_find(P, s), row0w[b] + l);
  }
}

// this band's labels whose global value changes -> relabel hash (key = local label)
__global__ void k_merge_collect_labels(LabelView v, MergeGeo m, int me,
                                       const unsigned long long* row0w, uint32_t* P,
                                       const unsigned long long* gmax, unsigned long long* rkeys,
                                       unsigned long long* rvals, uint32_t rmask) {
  slcs_pdl_wait();
  const uint32_t n = 2u * uint32_t(m.w);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = uint32_t(me) * n + i;
    const int side = int(i / uint32_t(m.w)), c = int(i - uint32_t(side) * uint32_t(m.w));
    const uint32_t l = v.comp(m, me, side, c);
    if (!l) continue;
    const unsigned long long g = gmax[uf_find(P, s)];
    if (g == row0w[me] + l) continue;
    uint32_t h = hash_slot(l, rmask);
    for (;;) {
      const unsigned long long old = atomicCAS(rkeys + h, EMPTY, (unsigned long long)l);
      if (old == EMPTY || old == l) {
        rvals[h] = g;  // every slot of the component writes the same value
        break;
      }
      h = (h + 1) & rmask;
    }
  }
}

// band labels -> global 64-bit labels: offset + local, or the merged value.
// Four labels per thread (one 16 B load, two 16 B stores); neighbouring pixels
// mostly share a label, so a label equal to the previous one reuses its value
// instead of probing the hash again.
__global__ void k_relabel_hash(const uint32_t* __restrict__ lab, size_t n, LabelMap64 map,
                               int vec, unsigned long long* __restrict__ out) {
  slcs_pdl_wait();
  const size_t n4 = vec ? n / 4 : 0;  // vec: both buffers 16 B aligned
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  uint32_t pl = 0;
  unsigned long long pv = 0;
  auto one = [&](uint32_t l) {
    if (l != pl) {
      pv = map_label64(l, map);
      pl = l;
    }
    return pv;
  };
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint4 l = __ldcs(reinterpret_cast<const uint4*>(lab) + i);
    ulonglong2 a, b;
    a.x = one(l.x);
    a.y = one(l.y);
    b.x = one(l.z);
    b.y = one(l.w);
    __stcs(reinterpret_cast<ulonglong2*>(out) + 2 * i, a);
    __stcs(reinterpret_cast<ulonglong2*>(out) + 2 * i + 1, b);
  }
  for (size_t i = 4 * n4 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = map_label64(__ldg(lab + i), map);
}

uint32_t pow2_at_least(size_t n) {
  uint32_t c = 16;
  while (c < n) c <<= 1;
  return c;
}

unsigned grid_of(size_t n) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8)));
}

}  // namespace

size_t band_record_bytes(int kind, int w, size_t pitch_words) {
  return kind == 0 ? reach_rec(w, pitch_words).bytes : label_rec(w).bytes;
}

// offsets of the reach record pieces (written by api.cu)
void band_reach_record_offsets(int w, size_t pitch_words, size_t* roots, size_t* cls,
                               size_t* tgt) {
  const ReachRec r = reach_rec(w, pitch_words);
  for (int i = 0; i < 2; ++i) {
    roots[i] = r.roots[i];
    cls[i] = r.cls[i];
    tgt[i] = r.tgt[i];
  }
}
void band_label_record_offsets(int w, size_t* lab) {
  const LabelRec r = label_rec(w);
  lab[0] = r.lab[0];
  lab[1] = r.lab[1];
}

size_t band_merge_scratch_bytes(int nb, int w) {
  const size_t nslots = size_t(nb) * 2 * size_t(w);
  const size_t hc = pow2_at_least(2 * nslots);
  const size_t rc = pow2_at_least(4 * size_t(w));
  return align16(hc * 8) + align16(hc * 4) + 2 * align16(nslots * 4) + align16(nslots * 8) +
         align16(rc * 16) + align16(2 * size_t(w) * 4) + 16 + align16(size_t(nb) * 8);
}

namespace {
struct MergeScratch {
  unsigned long long* keys;
  uint32_t* rep;
  uint32_t* P;
  uint32_t* Rp;  // representative slot of each slot's band component
  unsigned long long* gmax;  // ccl: per slot max label / reach: seeded bytes
  unsigned long long* rkeys;
  unsigned long long* rvals;
  uint32_t* out;
  int* count;
  unsigned long long* row0w;
  uint32_t hc, rc;
};
MergeScratch carve(void* base, int nb, int w) {
  MergeScratch s;
  const size_t nslots = size_t(nb) * 2 * size_t(w);
  s.hc = pow2_at_least(2 * nslots);
  s.rc = pow2_at_least(4 * size_t(w));
  char* p = static_cast<char*>(base);
  s.keys = reinterpret_cast<unsigned long long*>(p);
  p += align16(size_t(s.hc) * 8);
  s.rep = reinterpret_cast<uint32_t*>(p);
  p += align16(size_t(s.hc) * 4);
  s.P = reinterpret_cast<uint32_t*>(p);
  p += align16(nslots * 4);
  s.Rp = reinterpret_cast<uint32_t*>(p);
  p += align16(nslots * 4);
  s.gmax = reinterpret_cast<unsigned long long*>(p);
  p += align16(nslots * 8);
  s.rkeys = reinterpret_cast<unsigned long long*>(p);
  s.rvals = s.rkeys + s.rc;
  p += align16(size_t(s.rc) * 16);
  s.out = reinterpret_cast<uint32_t*>(p);
  p += align16(2 * size_t(w) * 4);
  s.count = reinterpret_cast<int*>(p);
  p += 16;
  s.row0w = reinterpret_cast<unsigned long long*>(p);
  return s;
}

MergeGeo merge_geo(int nb, int w, size_t rec_bytes, const MergeScratch& s) {
  MergeGeo m;
  m.nb = nb;
  m.w = w;
  m.nslots = uint32_t(size_t(nb) * 2 * size_t(w));
  m.hmask = s.hc - 1;
  m.rec_bytes = rec_bytes;
  return m;
}

void clear_tables(const MergeScratch& s, size_t nslots, cudaStream_t st) {
  cuda_check(cudaMemsetAsync(s.keys, 0xff, size_t(s.hc) * 8, st), "merge tables");
  cuda_check(cudaMemsetAsync(s.rep, 0xff, size_t(s.hc) * 4, st), "merge tables");
  cuda_check(cudaMemsetAsync(s.gmax, 0, nslots * 8, st), "merge tables");
  cuda_check(cudaMemsetAsync(s.rkeys, 0xff, size_t(s.rc) * 8, st), "merge tables");
  cuda_check(cudaMemsetAsync(s.count, 0, sizeof(int), st), "merge tables");
}
}  // namespace

int launch_band_reach_merge(int nb, int w, size_t pitch_words, int me, const void* records,
                            void* scratch, uint32_t** roots_out, int** count_out,
                            cudaStream_t st) {
  MergeScratch s = carve(scratch, nb, w);
  const ReachRec off = reach_rec(w, pitch_words);
  MergeGeo m = merge_geo(nb, w, off.bytes, s);
  ReachView v{static_cast<const unsigned char*>(records), off};
  clear_tables(s, m.nslots, st);
  uint8_t* seeded = reinterpret_cast<uint8_t*>(s.gmax);
  pdl(k_merge_insert<ReachView>, grid_of(m.nslots), 256, 0, st, v, m, s.keys, s.rep);
  pdl(k_merge_init<ReachView>, grid_of(m.nslots), 256, 0, st, v, m, s.keys, s.rep, s.P, s.Rp);
  pdl(k_merge_unite<ReachView>, grid_of(size_t(nb) * w), 256, 0, st, v, m, s.P);
  pdl(k_merge_seed, grid_of(m.nslots), 256, 0, st, v, m, s.P, seeded);
  pdl(k_merge_collect_reach, grid_of(2 * size_t(w)), 256, 0, st, v, m, me, s.P,
      static_cast<const uint32_t*>(s.Rp), static_cast<const uint8_t*>(seeded), s.out, s.count);
  *roots_out = s.out;
  *count_out = s.count;
  return 5;
}

int launch_band_ccl_merge(int nb, int w, int me, const void* records,
                          const unsigned long long* row0w_host, void* scratch, LabelMap64* map,
                          cudaStream_t st) {
  MergeScratch s = carve(scratch, nb, w);
  const LabelRec off = label_rec(w);
  MergeGeo m = merge_geo(nb, w, off.bytes, s);
  LabelView v{static_cast<const unsigned char*>(records), off};
  clear_tables(s, m.nslots, st);
  cuda_check(cudaMemcpyAsync(s.row0w, row0w_host, size_t(nb) * 8, cudaMemcpyHostToDevice, st),
             "band offsets");
  int launches = 0;
  if (nb > 1) {
    pdl(k_merge_insert<LabelView>, grid_of(m.nslots), 256, 0, st, v, m, s.keys, s.rep);
    pdl(k_merge_init<LabelView>, grid_of(m.nslots), 256, 0, st, v, m, s.keys, s.rep, s.P, s.Rp);
    pdl(k_merge_unite<LabelView>, grid_of(size_t(nb) * w), 256, 0, st, v, m, s.P);
    pdl(k_merge_max_label, grid_of(m.nslots), 256, 0, st, v, m,
        static_cast<const unsigned long long*>(s.row0w), s.P, s.gmax);
    pdl(k_merge_collect_labels, grid_of(2 * size_t(w)), 256, 0, st, v, m, me,
        static_cast<const unsigned long long*>(s.row0w), s.P,
        static_cast<const unsigned long long*>(s.gmax), s.rkeys, s.rvals, s.rc - 1);
    launches = 5;
  }
  map->offset = row0w_host[me];
  map->rkeys = s.rkeys;
  map->rvals = s.rvals;
  map->rmask = s.rc - 1;
  map->any = nb > 1 ? 1 : 0;
  return launches;
}

int launch_band_ccl_merge_relabel(int nb, int w, int me, const void* records,
                                  const unsigned long long* row0w_host, void* scratch,
                                  const uint32_t* labels, size_t npx, unsigned long long* out,
                                  cudaStream_t st) {
  LabelMap64 map;
  const int launches = launch_band_ccl_merge(nb, w, me, records, row0w_host, scratch, &map, st);
  const int vec = (reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(out)) % 16 == 0;
  pdl(k_relabel_hash, unsigned(std::min<size_t>((npx + 1023) / 1024, 148 * 32)), 256, 0, st, labels,
      npx, map, vec, out);
  return launches + 1;
}

}  // namespace slcs
