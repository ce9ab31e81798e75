// Device mirror (DeviceState, device.py:124-386) and the octree ray caster
// (render/raycast.py:40-339, render/core.py:34-187) for sm_100a.
//
// One thread per ray, one warp per 16x2 pixel tile (VT_TW).  Every ray is
// independent within a pass (the node buffer and brick buffer are frozen,
// flags are idempotent ORs, counters are sums), so marching each ray to
// completion reproduces the reference's wavefront `march` exactly.
//
// Arithmetic: FP64 throughout, compiled with -fmad=false, following the
// reference's numpy operation order (sampling positions, LOD, trilinear
// weights, np.interp transfer functions, compositing), so images match the
// CPU reference to ~1e-15 rather than merely within the 1/255 tolerance.
// The gather (8 corners x C channels per pos-sample from the brick buffer)
// is the bandwidth limiter; FP64 on B200 runs at half the FP32 rate, which
// this kernel never approaches.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "tree.cuh"

using namespace vtx;

#ifndef VT_TW
#define VT_TW 16  // warp tile width in pixels (the tile is VT_TW x 32 / VT_TW)
#endif

struct vt_mirror {
  vt_tree* tree = nullptr;
  std::atomic<int> refs{1};  // ray sessions keep their mirror alive
  bool zero_copy = false;
  int64_t slots = 0;
  uint64_t* d_nb = nullptr;
  uint8_t* d_fb = nullptr;
  uint8_t* d_bb = nullptr;   // own brick buffer (bounded mode)
  int32_t* d_res = nullptr;  // node -> brick-buffer slot or -1 (bounded mode)
  // per brick-buffer slot, per channel: max sample over the stored brick
  // (borders included) — empty-space skipping bound; valid for slots < bmax_n
  uint16_t* d_bmax = nullptr;        // sub-brick maxima, then brick maxima
  uint16_t* d_bmax_brick = nullptr;  // = d_bmax + bmax_cap * kMaxC
  int64_t bmax_cap = 0;
  bool bmax_valid = false;
  int64_t bmax_version = -1;  // tree data_version the zero-copy maxima reflect
  int64_t bmax_incremental = 0, bmax_last_slots = 0;  // refresh statistics
};

namespace {

constexpr int kMaxLevels = kMaxDepth + 1;

struct RenderParams {
  Geo g;
  double dims[3], spacing[3], box_hi[3];
  double ext[kMaxLevels][3], scl[kMaxLevels][3];
  double base_voxel;
  double fmax;
  double qmax;
  int avg_w;
  int borders_filled;
  int zero_copy;
  // scene
  double cam[3], fwd[3], right[3], up[3];
  double tan_half, aspect, pfs;  // pixel_footprint_scale
  int W, H;
  int mip;
  double step, corr, et, lod_scale;
  int has_et;
  int tf_n[kMaxC];
  double tf_x[kMaxC][VT_MAX_TF_POINTS];
  double tf_v[kMaxC][VT_MAX_TF_POINTS][4];
  double tf_s[kMaxC][VT_MAX_TF_POINTS][4];  // segment slopes (host FP64)
  double tf_xzero[kMaxC];                   // alpha == 0 on [0, xzero]
  double inv_fmax;
  double inv_scl[kMaxLevels][3];  // exact: scales are powers of two
  int exti[kMaxLevels][3];        // node extents in voxels; 1 << 30 on unsplit axes
  int unit_spacing;               // spacing == (1, 1, 1): p / spacing == p
  int base_pow2;                  // base_voxel a power of two: exact reciprocal
  double inv_base;
  int n_clips;
  double clip_n[3][3], clip_o[3];
  int has_tr;
  double tr[kMaxC][12];
  // tile restriction
  int rect[4];  // x0, y0, x1, y1
  // sort-first strip interleave: this launch renders the rows of strips
  // part, part + n_parts, ... (strip_rows rows each), written compactly
  int strip_rows, n_parts, part;
  // exact empty-space skipping (DVR, no channel transforms): a sample whose
  // every channel value v satisfies v <= ess_thr[c] has transfer-function
  // alpha exactly 0 and composites to a no-op
  int ess;
  int ess_thr[kMaxC];
  int fast;                    // FP32 sample reconstruction (vt_scene.precision)
  const uint16_t* bmax;        // [slot][nsb][kMaxC] sub-brick maxima
  const uint16_t* bmax_brick;  // [slot][kMaxC] whole-brick maxima
  double inv_step;
  int sbk[3], nsub[3], nsb;  // sub-brick edge, count per axis, total
  // node / flag / brick buffers of this launch: read from constant memory
  // where used rather than held in registers for the whole ray
  const uint64_t* buf_nb;
  uint8_t* buf_fb;
  const void* buf_bb;
};

// per-launch scene + geometry; render entry points serialise on g_render_mu
__constant__ RenderParams c_P;

struct RayOut {
  double rgb[3], a;
  double mip[kMaxC];
};

// per-thread (per-ray) counts fit 32 bits (a ray takes at most a few
// thousand samples); warp sums go to 64-bit device counters
struct Counters {
  int samples, tf, avgfb, coarse, req, used;
  int skipped;  // samples accounted by the empty-space skip (not computed)
};

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return fmin(fmax(v, lo), hi);
}

// np.clip(a, lo, hi) == minimum(maximum(a, lo), hi) for non-NaN a (every
// clipped quantity on the sampling path is finite)
__device__ __forceinline__ double npclip(double v, double lo, double hi) {
  // two compares + selects (no DMNMX on sm_100; fmin/fmax add NaN handling)
  v = v < lo ? lo : v;
  return v > hi ? hi : v;
}

// transfer-function tables staged in shared memory per block: lanes index
// different segments, which the constant cache would serialise
struct TFTable {
  double xzero[kMaxC];  // TF alpha is exactly 0 for every x <= xzero (or -inf)
  double x[kMaxC][VT_MAX_TF_POINTS];
  double v[kMaxC][VT_MAX_TF_POINTS][4];
  double s[kMaxC][VT_MAX_TF_POINTS][4];
  int n[kMaxC];
  // FP32 copies for the float reconstruction path
  float xzf[kMaxC];
  float xf[kMaxC][VT_MAX_TF_POINTS];
  float vf[kMaxC][VT_MAX_TF_POINTS][4];
  float sf[kMaxC][VT_MAX_TF_POINTS][4];
};

__device__ void load_tf(TFTable& T) {
  const RenderParams& P = c_P;
  const double* src_x = &P.tf_x[0][0];
  const double* src_v = &P.tf_v[0][0][0];
  const double* src_s = &P.tf_s[0][0][0];
  for (int e = threadIdx.x; e < kMaxC * VT_MAX_TF_POINTS; e += blockDim.x) {
    (&T.x[0][0])[e] = src_x[e];
    (&T.xf[0][0])[e] = (float)src_x[e];
  }
  for (int e = threadIdx.x; e < kMaxC * VT_MAX_TF_POINTS * 4; e += blockDim.x) {
    (&T.v[0][0][0])[e] = src_v[e];
    (&T.s[0][0][0])[e] = src_s[e];
    (&T.vf[0][0][0])[e] = (float)src_v[e];
    (&T.sf[0][0][0])[e] = (float)src_s[e];
  }
  if (threadIdx.x < kMaxC) {
    T.n[threadIdx.x] = P.tf_n[threadIdx.x];
    T.xzero[threadIdx.x] = P.tf_xzero[threadIdx.x];
    T.xzf[threadIdx.x] = (float)P.tf_xzero[threadIdx.x];
  }
  __syncthreads();
}

// camera.py:41-53
__device__ void ray_dir(int i, int j, double d[3]) {
  const RenderParams& P = c_P;
  double xs = (2.0 * ((double)i + 0.5) / (double)P.W - 1.0) * P.tan_half * P.aspect;
  double ys = (1.0 - 2.0 * ((double)j + 0.5) / (double)P.H) * P.tan_half;
  for (int a = 0; a < 3; ++a) d[a] = P.fwd[a] + xs * P.right[a] + ys * P.up[a];
  double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  for (int a = 0; a < 3; ++a) d[a] = d[a] / n;
}

// compute_ray_bounds (core.py:34-67) + RayBatch step count (core.py:79-89)
__device__ void ray_setup(const double d[3], double& t0o, long long& n) {
  const RenderParams& P = c_P;
  double t0 = 0.0, t1 = INFINITY;
  for (int a = 0; a < 3; ++a) {
    double o = P.cam[a], dd = d[a];
    double near_, far_;
    if (dd == 0.0) {
      bool in = o >= 0.0 && o <= P.box_hi[a];
      near_ = in ? -INFINITY : INFINITY;
      far_ = in ? INFINITY : -INFINITY;
    } else {
      double ta = (0.0 - o) / dd, tb = (P.box_hi[a] - o) / dd;
      near_ = fmin(ta, tb);
      far_ = fmax(ta, tb);
    }
    t0 = fmax(t0, near_);
    t1 = fmin(t1, far_);
  }
  for (int q = 0; q < P.n_clips; ++q) {
    const double* nn = P.clip_n[q];
    double num = P.clip_o[q] - (P.cam[0] * nn[0] + P.cam[1] * nn[1] + P.cam[2] * nn[2]);
    double den = d[0] * nn[0] + d[1] * nn[1] + d[2] * nn[2];
    double tc = num / den;
    bool keep = den == 0.0 && num >= 0.0;
    bool kill = den == 0.0 && num < 0.0;
    if (den > 0.0)
      t1 = fmin(t1, tc);
    else if (!keep && !kill)
      t0 = fmax(t0, tc);
    if (kill) t1 = -INFINITY;
  }
  bool hit = t0 < t1;
  double span = fmax(t1 - t0, 0.0);
  t0o = hit ? t0 : 0.0;
  n = hit ? (long long)ceil(span / P.step - 1e-12) : 0;
}

// np.interp on sorted control points (transfer.py:34-41), all four RGBA
// components from one segment search.  Segment slopes are precomputed on
// the host in FP64 with the same operation numpy uses, so every result is
// bit-identical to numpy's: slope * (x - xp[j]) + fp[j].
__device__ __forceinline__ void interp4(const TFTable& T, int c, double x, double out[4]) {
  const int n = T.n[c];
  const double* xp = T.x[c];
  if (!(x >= xp[0])) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = x != x ? x : T.v[c][0][q];
    return;
  }
  if (x >= xp[n - 1]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = T.v[c][n - 1][q];
    return;
  }
  int j = 0;
  while (j + 2 < n && !(x < xp[j + 1])) ++j;
  const double dx = x - xp[j];
  const bool exact = x == xp[j];  // numpy returns fp[j] on an exact knot
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double y0 = T.v[c][j][q];
    double r = exact ? y0 : T.s[c][j][q] * dx + y0;
    if (r != r) {
      const double y1 = T.v[c][j + 1][q];
      r = T.s[c][j][q] * (x - xp[j + 1]) + y1;
      if (r != r && y0 == y1) r = y0;
    }
    out[q] = r;
  }
}

// the same on FP32 tables (float reconstruction path)
__device__ __forceinline__ void interp4(const TFTable& T, int c, float x, float out[4]) {
  const int n = T.n[c];
  const float* xp = T.xf[c];
  if (!(x >= xp[0])) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = x != x ? x : T.vf[c][0][q];
    return;
  }
  if (x >= xp[n - 1]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = T.vf[c][n - 1][q];
    return;
  }
  int j = 0;
  while (j + 2 < n && !(x < xp[j + 1])) ++j;
  const float dx = x - xp[j];
  const bool exact = x == xp[j];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float y0 = T.vf[c][j][q];
    float r = exact ? y0 : fmaf(T.sf[c][j][q], dx, y0);
    if (r != r) r = y0;
    out[q] = r;
  }
}

// the node a sample last resolved to, per channel group: a sample inside
// its box at the same target level reuses it.  Node boxes have integral
// voxel origins, and pv >= 0 on the sampling path, so the box test is an
// integer compare of floor(pv).  The full-frame fallback's ancestors are
// re-derived only when a sample needs them (ancestors()).
struct DescentCache {
  int target;  // -1: empty
  int clear;   // the node is transparent for the scene (empty-space skip)
  int lvl;
  int idx;     // BFS node index (< 2^31: a depth-8 tree has 19.2M nodes)
  int lo[3];   // box origin; the box is [lo, lo + exti[lvl])
};

// Exact integer -> FP64 conversions on the FP64 pipe: the per-sample
// conversions (24 corner values, cell floors, box origins, descent floors)
// all on the quarter-rate conversion (XU) pipe saturate it; the measured
// fastest split puts the corner differences, box origins and the sample
// index here and the rest on XU.  For an integer 0 <= v < 2^31 the double
// 2^52 + v is exact.
constexpr double kMagic52 = 4503599627370496.0;  // 2^52
__device__ __forceinline__ double magic_of(unsigned v) {
  return __hiloint2double(0x43300000, (int)v);  // == 2^52 + v
}
// (double)v for 0 <= v < 2^31
__device__ __forceinline__ double exact_d(int v) { return magic_of((unsigned)v) - kMagic52; }
// (double)v for any 32-bit v: the double with high word 0x43380000 and low
// word v + 2^31 is exactly 2^52 + 2^51 + 2^31 + v
__device__ __forceinline__ double exact_sd(int v) {
  return __hiloint2double(0x43380000, v ^ (int)0x80000000) - 6755401588539392.0;
}

// floor(log2(v)) for a positive normal double: its unbiased exponent
__device__ __forceinline__ int floor_log2(double v) {
  return (int)((__double_as_longlong(v) >> 52) & 0x7FF) - 1023;
}

#define P c_P
// FAST: sample reconstruction (trilinear) and transfer functions in FP32 —
// the north-star's "float accumulation" model; positions, LOD, descent and
// compositing stay FP64
// FILLED: 1 / 0 = borders filled / not known at compile time (the full-frame
// kernel is instantiated for both), -1 = read P.borders_filled
template <class T, int NC, bool TR, bool FAST = false, int FILLED = -1>
struct Sampler {
  using V = typename std::conditional<FAST, float, double>::type;
  static constexpr int kC = NC;
  bool fullframe;
  Counters cnt;  // by value: stays in registers
  int last_used = -1, last_req = -1;
  // the last sample resolved to a node that is transparent for the scene's
  // transfer functions: 1 resident brick (or sub-brick), 2 homogeneous
  // (AVG) node; the transparent box is cache[0]'s node box, or its
  // sub-brick hint_sb (x | y << 8 | z << 16) when >= 0
  int hint = 0;
  int hint_sb = -1;
  DescentCache cache[TR ? NC : 1];

  __device__ static const uint64_t* nbuf() { return P.buf_nb; }
  __device__ static uint8_t* fbuf() { return P.buf_fb; }
  __device__ static const T* bbuf() { return static_cast<const T*>(P.buf_bb); }
  __device__ Sampler(const uint64_t*, uint8_t*, const T*, bool ff)
      : fullframe(ff), cnt{0, 0, 0, 0, 0, 0, 0} {
#pragma unroll
    for (int q = 0; q < (TR ? NC : 1); ++q) {
      cache[q].target = -1;
      cache[q].clear = 0;
    }
  }

  // feedback flag: idempotent OR into the byte of the node (device.py:35-36,
  // raycast.py:161-163).  Skipped when this thread already marked the node;
  // otherwise warp-aggregated: the lanes marking the same node this step
  // elect one leader (__match_any_sync), which writes only if the bit is
  // not set yet — one atomic per node per warp instead of one per lane
  __device__ void mark(int idx, unsigned flag) {
    int& last = flag == 1 ? last_used : last_req;
    if (last == idx) return;
    last = idx;
    const unsigned peers = __match_any_sync(__activemask(), idx);
    if ((int)(threadIdx.x & 31) != __ffs(peers) - 1) return;
    unsigned* w = reinterpret_cast<unsigned*>(fbuf() + (idx & ~3));
    unsigned bit = flag << ((idx & 3) * 8);
    if (!(__ldcg(w) & bit)) atomicOr(w, bit);
  }

  __device__ double avg_of(uint64_t e, int c) const {
    uint64_t q = (e >> (24 + c * P.avg_w)) & ((1ULL << P.avg_w) - 1);
    return rint((double)q * P.fmax / P.qmax);
  }

  // _trilerp (raycast.py:133-159) for channels [c0, c1): cell index and
  // weights once per sample, then the 8 corners of every channel
  __device__ void trilerp(uint64_t e, int lvl, const int lo[3], const double pv[3], int c0,
                          int c1, V* out, int* cell = nullptr) const {
    const long long slot = (long long)((e >> 24) & 0xFFFFFFFFULL);
    int i0[3];
    double w1[3];
    const bool filled = FILLED < 0 ? P.borders_filled != 0 : FILLED != 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      // scale is a power of two: multiplying by its reciprocal is exact
      double f = (pv[a] - exact_d(lo[a])) * P.inv_scl[lvl][a] + 0.5;
      // inside the node box f is in [0.5, M + 0.5): with filled borders the
      // reference's clip to [0, M + 1] and the index clip to [0, M] are
      // no-ops; before fill_borders samples clamp to interior centres
      if (!filled) f = npclip(f, 1.0, exact_d(P.g.brick[a]));
      // the cell floor and its double on the conversion (XU) pipe: the FP64
      // pipe carries the other conversions (measured fastest split)
      int fi = (int)floor(f);
      if (filled) fi = fi > P.g.brick[a] ? P.g.brick[a] : fi;
      const double fl = (double)fi;
      i0[a] = fi;
      if (cell) cell[a] = fi;
      w1[a] = f - fl;  // in [0, 1] by construction
    }
    constexpr int C = NC;
    // 32-bit offsets inside a brick (a stored brick is < 2^31 samples)
    const int sxC = P.g.stored[0] * C, sxyC = sxC * P.g.stored[1];
    const T* p = bbuf() + slot * P.g.brick_elems + (i0[2] * sxyC + i0[1] * sxC + i0[0] * C);
    if (FAST) {
      // FP32: lerp along x, then y, then z (7 FMAs per channel)
      float fx = (float)w1[0], fy = (float)w1[1], fz = (float)w1[2];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (c < c0 || c >= c1) continue;
        float r[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int dz = q >> 1, dy = q & 1;
          const T* row = p + dz * sxyC + dy * sxC + c;
          const float a0 = (float)__ldg(row), a1 = (float)__ldg(row + C);
          r[q] = fmaf(fx, a1 - a0, a0);
        }
        const float y0 = fmaf(fy, r[1] - r[0], r[0]), y1 = fmaf(fy, r[3] - r[2], r[2]);
        out[c] = (V)fmaf(fz, y1 - y0, y0);
      }
      return;
    }
    // FP64 lerps along x, y, z with fused multiply-adds (equal to the
    // reference's sum of weighted corners to ~1e-15 relative)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c < c0 || c >= c1) continue;
      double r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int dz = q >> 1, dy = q & 1;
        const T* row = p + dz * sxyC + dy * sxC + c;
        // the difference through the FP64 pipe, a0 through the conversion
        // (XU) pipe: the two pipes share the 24 conversions (measured ~1.5 %
        // faster than either pipe alone)
        const int a0 = __ldg(row), a1 = __ldg(row + C);
        r[q] = fma(w1[0], exact_sd(a1 - a0), (double)a0);
      }
      const double y0 = fma(w1[1], r[1] - r[0], r[0]), y1 = fma(w1[1], r[3] - r[2], r[2]);
      out[c] = (V)fma(w1[2], y1 - y0, y0);
    }
  }

  // raycast.py:86-123 with a per-channel-group descent cache: a sample that
  // stays inside the cached node box at the same target level reuses it
  // returns true when it re-descended (a different node than the cached one)
  __device__ bool descend(const double pv[3], int target, DescentCache& dc) {
    int ip[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ip[a] = (int)pv[a];  // floor: pv >= 0
    if (dc.target == target) {
      bool ok = true;
#pragma unroll
      for (int a = 0; a < 3; ++a)
        ok = ok && ip[a] >= dc.lo[a] && ip[a] - dc.lo[a] < P.exti[dc.lvl][a];
      if (ok) return false;
    }
    int idx = 0;
    int lvl = P.g.depth;
    int lo[3] = {0, 0, 0};
    for (int it = 0; it < P.g.depth; ++it) {
      uint64_t e = __ldg(nbuf() + idx);
      int ptr = (int)((e >> 2) & 0x3FFFFFULL);
      if (!(ptr != 0 && lvl > target)) break;
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int half = P.exti[lvl - 1][a];
        const bool bit = ip[a] >= lo[a] + half && P.g.split[a];
        k |= bit ? (1 << a) : 0;
        lo[a] += bit ? half : 0;
      }
      idx = 8 * (ptr - 1) + 1 + k;
      --lvl;
    }
    dc.target = target;
    dc.idx = idx;
    dc.lvl = lvl;
#pragma unroll
    for (int a = 0; a < 3; ++a) dc.lo[a] = lo[a];
    return true;
  }

  // the two nearest ancestors of the node at level `lvl` on pv's path (the
  // last two nodes descend() passed through): full-frame fallback only
  __device__ void ancestors(const double pv[3], int lvl, int aidx[2], int alvl[2],
                            int alo[2][3]) const {
    int ip[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ip[a] = (int)pv[a];
    aidx[0] = aidx[1] = -1;
    alvl[0] = alvl[1] = 0;
    int idx = 0, l = P.g.depth;
    int lo[3] = {0, 0, 0};
    while (l > lvl) {
      const uint64_t e = __ldg(nbuf() + idx);
      const int ptr = (int)((e >> 2) & 0x3FFFFFULL);
      aidx[1] = aidx[0];
      alvl[1] = alvl[0];
      aidx[0] = idx;
      alvl[0] = l;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        alo[1][a] = alo[0][a];
        alo[0][a] = lo[a];
      }
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int half = P.exti[l - 1][a];
        const bool bit = ip[a] >= lo[a] + half && P.g.split[a];
        k |= bit ? (1 << a) : 0;
        lo[a] += bit ? half : 0;
      }
      idx = 8 * (ptr - 1) + 1 + k;
      --l;
    }
  }

  // transparency of the node just entered: every sample in it has TF alpha 0
  __device__ int node_clear(uint64_t e, int c0, int c1) const {
    if (TR || !P.ess) return 0;
    bool clear = true;
    if (!(e & 2)) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c >= c0 && c < c1) clear = clear && avg_of(e, c) <= (double)P.ess_thr[c];
      return clear ? 2 : 0;
    }
    if (!(e & 1)) return 0;
    const uint16_t* bm = P.bmax_brick + ((e >> 24) & 0xFFFFFFFFULL) * kMaxC;
#pragma unroll
    for (int c = 0; c < NC; ++c) clear = clear && (int)__ldg(bm + c) <= P.ess_thr[c];
    return clear ? 1 : 0;
  }

  // optimal_lod (raycast.py:40-50): floor(log2(.)) is the exponent of the
  // positive normal footprint ratio (no transcendental per sample)
  __device__ int lod(const double p[3]) const {
    double z = (p[0] - P.cam[0]) * P.fwd[0] + (p[1] - P.cam[1]) * P.fwd[1] +
               (p[2] - P.cam[2]) * P.fwd[2];
    double fp = fmax(z, 1e-12) * P.pfs;
    fp = fp * P.lod_scale;
    const double v = P.base_pow2 ? fp * P.inv_base : fp / P.base_voxel;
    int l = v >= 2.2250738585072014e-308 ? floor_log2(v) : -1;
    l = l < 0 ? 0 : (l > P.g.depth ? P.g.depth : l);
    return l;
  }

  // _resolve + _fullframe_fallback (raycast.py:167-238) for channels [c0, c1)
  __device__ bool resolve(const double pv[3], int target, int c0, int c1, V* out,
                          DescentCache& dc) {
    const bool moved = descend(pv, target, dc);
    const uint64_t e = __ldg(nbuf() + dc.idx);
    const bool resident = e & 1, nh = e & 2;
    if (moved) dc.clear = node_clear(e, c0, c1);
    if (!nh) {
      if (dc.clear) {
        // transparent homogeneous node: value irrelevant, skip its samples
        hint = 2;
        hint_sb = -1;
        return false;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c >= c0 && c < c1) out[c] = (V)avg_of(e, c);
      return false;
    }
    if (resident) {
      mark(dc.idx, 1);
      cnt.used++;
      if (dc.clear) {
        hint = 1;
        hint_sb = -1;
        return false;
      }
      int cell[3];
      trilerp(e, dc.lvl, dc.lo, pv, c0, c1, out, cell);
      if (!TR && P.ess >= 2) {
        // sub-brick of the sample's trilinear cell: its maxima bound every
        // corner of every sample whose cell lies in the sub-brick
        const uint64_t slot = (e >> 24) & 0xFFFFFFFFULL;
        int sb[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int q = cell[a] / P.sbk[a];
          sb[a] = q >= P.nsub[a] ? P.nsub[a] - 1 : q;
        }
        const int sbi = (sb[2] * P.nsub[1] + sb[1]) * P.nsub[0] + sb[0];
        const uint16_t* sm = P.bmax + (slot * P.nsb + sbi) * kMaxC;
        bool clear = true;
#pragma unroll
        for (int c = 0; c < NC; ++c) clear = clear && (int)__ldg(sm + c) <= P.ess_thr[c];
        if (clear) {
          hint = 1;
          hint_sb = sb[0] | (sb[1] << 8) | (sb[2] << 16);
        }
      }
      return false;
    }
    mark(dc.idx, 2);
    cnt.req++;
    if (!fullframe) return true;
    int aidx[2], alvl[2], alo[2][3];
    ancestors(pv, dc.lvl, aidx, alvl, alo);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ai = aidx[q];
      if (ai < 0) continue;
      uint64_t ae = __ldg(nbuf() + ai);
      if (ae & 1) {
        trilerp(ae, alvl[q], alo[q], pv, c0, c1, out);
        mark(ai, 1);
        cnt.used++;
        cnt.coarse++;
        return false;
      }
      if (ae & 2) {
        mark(ai, 2);
        cnt.req++;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c >= c0 && c < c1) out[c] = (V)avg_of(e, c);
    cnt.avgfb++;
    return false;
  }

  __device__ __forceinline__ void to_voxels(const double q[3], double pv[3]) const {
    // a uniform branch, so the division is not if-converted into every sample
    if (P.unit_spacing) {
#pragma unroll
      for (int a = 0; a < 3; ++a) pv[a] = q[a];
    } else {
#pragma unroll
      for (int a = 0; a < 3; ++a) pv[a] = q[a] / P.spacing[a];
    }
  }

  // samples k+1 .. k+m provably resolve to the same transparent node with
  // the same target level, inside the volume and the ray: returns m (exact
  // empty-space skip; each skipped sample still counts as the reference
  // counts it).  Positions are monotone in k, so checking the last one
  // suffices; the analytic estimate is verified with the sampling code.
  // the voxel-space box the hint says stays transparent
  __device__ void hint_box(double lo[3], double hi[3]) const {
    const DescentCache& dc = cache[0];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const bool sp = P.g.split[a];
      const double nlo = (double)dc.lo[a];
      const double nhi = nlo + (double)P.exti[dc.lvl][a];
      lo[a] = sp ? nlo : -INFINITY;
      hi[a] = sp ? nhi : INFINITY;
      if (hint_sb >= 0) {
        // cells [sB, sB + B) <=> (pv - lo) / scale in [sB - 0.5, sB + B - 0.5)
        const int sb = (hint_sb >> (8 * a)) & 0xFF;
        const double sc = P.scl[dc.lvl][a];
        const double base = nlo - 0.5 * sc;
        if (sb > 0) lo[a] = base + (double)(sb * P.sbk[a]) * sc;
        if (sb < P.nsub[a] - 1) hi[a] = base + (double)((sb + 1) * P.sbk[a]) * sc;
      }
    }
  }

  // samples k+1 .. k+m provably resolve to the same transparent node with
  // the same target level, inside the volume and the ray: returns m (exact
  // empty-space skip; each skipped sample still counts as the reference
  // counts it).  Positions are monotone in k, so checking the last one
  // suffices; the analytic estimate is verified with the sampling code.
  __device__ long long skip_count(long long k, long long n, double t0, const double d[3]) {
    const int target = cache[0].target;
    double box_lo[3], box_hi[3];
    hint_box(box_lo, box_hi);
    double tl = INFINITY;
    if (target < P.g.depth) {
      const double df = d[0] * P.fwd[0] + d[1] * P.fwd[1] + d[2] * P.fwd[2];
      if (df > 0.0) tl = ldexp(P.base_voxel / (P.pfs * P.lod_scale * df), target + 1);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double lo = fmax(0.0, box_lo[a]), hi = fmin(P.dims[a], box_hi[a]);
      if (d[a] > 0.0) tl = fmin(tl, (hi * P.spacing[a] - P.cam[a]) * (1.0 / d[a]));
      else if (d[a] < 0.0) tl = fmin(tl, (lo * P.spacing[a] - P.cam[a]) * (1.0 / d[a]));
    }
    long long m = (long long)floor((tl - t0) * P.inv_step) - 1 - k;
    m = m < n - 1 - k ? m : n - 1 - k;
    for (int tries = 0; tries < 3 && m > 0; ++tries, m >>= 1) {
      const double t = t0 + (double)(k + m) * P.step;
      double p[3], pv[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) p[a] = P.cam[a] + t * d[a];
      to_voxels(p, pv);
      bool ok = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) ok = ok && pv[a] >= 0.0 && pv[a] <= P.dims[a];
      if (!ok || lod(p) != target) continue;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double q = npclip(pv[a], 0.0, P.dims[a] - 1e-9);
        if (!(q >= box_lo[a] && q < box_hi[a])) ok = false;
      }
      if (ok) return m;
    }
    return 0;
  }

  // sampler (raycast.py:242-278); returns missing
  __device__ bool sample(const double p[3], V* vals) {
    constexpr int C = NC;
    hint = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) vals[c] = (V)P.g.bg;
    if (!TR) {
      double pv[3];
      to_voxels(p, pv);
      bool in = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) in = in && pv[a] >= 0.0 && pv[a] <= P.dims[a];
      if (!in) return false;
      int target = lod(p);
      // np.clip(pv, 0, dims - 1e-9): pv >= 0 here, so only the upper bound acts
#pragma unroll
      for (int a = 0; a < 3; ++a) pv[a] = pv[a] > P.dims[a] - 1e-9 ? P.dims[a] - 1e-9 : pv[a];
      return resolve(pv, target, 0, C, vals, cache[0]);
    }
    bool missing = false;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double* m = P.tr[c];
      double q[3], pv[3];
      bool in = true;
      for (int r = 0; r < 3; ++r)
        q[r] = p[0] * m[r * 4 + 0] + p[1] * m[r * 4 + 1] + p[2] * m[r * 4 + 2] + m[r * 4 + 3];
      to_voxels(q, pv);
      for (int r = 0; r < 3; ++r) in = in && pv[r] >= 0.0 && pv[r] <= P.dims[r];
      if (!in) continue;
      int target = lod(q);
      for (int a = 0; a < 3; ++a) pv[a] = npclip(pv[a], 0.0, P.dims[a] - 1e-9);
      missing |= resolve(pv, target, c, c + 1, vals, cache[TR ? c : 0]);
    }
    return missing;
  }
};

#undef P

// composite_step (core.py:110-134); returns terminated
// MODE: 0 DVR, 1 MIP, -1 read P.mip at run time
// COUNT: tally the TF lookups here (false: the full-frame DVR march derives
// them as C per counted sample once, at the end of the ray)
template <int NC, int MODE = -1, bool COUNT = true>
__device__ bool composite(const TFTable& T, const float* vals, RayOut& o, Counters& cnt) {
  // float reconstruction path: per-sample TF / intermix in FP32, the ray's
  // front-to-back accumulation in FP64
  const RenderParams& P = c_P;
  constexpr int C = NC;
  if (MODE == 1 || (MODE < 0 && P.mip)) {
#pragma unroll
    for (int c = 0; c < C; ++c) o.mip[c] = fmax(o.mip[c], (double)vals[c]);
    return false;
  }
  float srgb[3] = {0.f, 0.f, 0.f};
  float trans = 1.f;
  bool any = false;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float x = vals[c] * (float)P.inv_fmax;
    if (COUNT) cnt.tf++;
    if (x <= T.xzf[c]) continue;
    any = true;
    float rgba[4];
    interp4(T, c, x, rgba);
    const float alpha =
        1.f - (P.corr == 1.0 ? (1.f - rgba[3]) : powf(1.f - rgba[3], (float)P.corr));
#pragma unroll
    for (int a = 0; a < 3; ++a) srgb[a] = fmaf(rgba[a], alpha, srgb[a]);
    trans = trans * (1.f - alpha);
  }
  if (!any) return false;
  const double w = 1.0 - o.a;
#pragma unroll
  for (int a = 0; a < 3; ++a) o.rgb[a] = o.rgb[a] + w * (double)fminf(fmaxf(srgb[a], 0.f), 1.f);
  o.a = o.a + w * (double)(1.f - trans);
  return P.has_et && o.a >= P.et;
}

template <int NC, int MODE = -1, bool COUNT = true>
__device__ bool composite(const TFTable& T, const double* vals, RayOut& o, Counters& cnt) {
  const RenderParams& P = c_P;
  constexpr int C = NC;
  if (MODE == 1 || (MODE < 0 && P.mip)) {
#pragma unroll
    for (int c = 0; c < C; ++c) o.mip[c] = fmax(o.mip[c], vals[c]);
    return false;
  }
  double srgb[3] = {0.0, 0.0, 0.0};
  double trans = 1.0;
  bool any = false;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double x = vals[c] * P.inv_fmax;
    if (COUNT) cnt.tf++;
    // alpha exactly 0: rgb * 0 and (1 - 0) change nothing — skip the lookup
    if (x <= T.xzero[c]) continue;
    any = true;
    double rgba[4];
    interp4(T, c, x, rgba);
    const double alpha = 1.0 - (P.corr == 1.0 ? (1.0 - rgba[3]) : pow(1.0 - rgba[3], P.corr));
#pragma unroll
    for (int a = 0; a < 3; ++a) srgb[a] = srgb[a] + rgba[a] * alpha;
    trans = trans * (1.0 - alpha);
  }
  if (!any) return false;  // the sample composites to a no-op
#pragma unroll
  for (int a = 0; a < 3; ++a) srgb[a] = npclip(srgb[a], 0.0, 1.0);
  const double sa = 1.0 - trans;
  const double w = 1.0 - o.a;
#pragma unroll
  for (int a = 0; a < 3; ++a) o.rgb[a] = o.rgb[a] + w * srgb[a];
  o.a = o.a + w * sa;
  return P.has_et && o.a >= P.et;
}

// finalize_image (core.py:137-155)
// MODE: 0 DVR, 1 MIP, -1 read P.mip at run time
template <int NC, int MODE = -1>
__device__ void finalize(const TFTable& T, const RayOut& o, double px[4], Counters& cnt) {
  const RenderParams& P = c_P;
  if (MODE == 0 || (MODE < 0 && !P.mip)) {
    px[0] = o.rgb[0];
    px[1] = o.rgb[1];
    px[2] = o.rgb[2];
    px[3] = o.a;
    return;
  }
  double rgb[3] = {0, 0, 0}, trans = 1.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double x = o.mip[c] * P.inv_fmax;
    double rgba[4];
    interp4(T, c, x, rgba);
    cnt.tf++;
    for (int a = 0; a < 3; ++a) rgb[a] = rgb[a] + rgba[a] * rgba[3];
    trans = trans * (1.0 - rgba[3]);
  }
  for (int a = 0; a < 3; ++a) px[a] = npclip(rgb[a], 0.0, 1.0);
  px[3] = 1.0 - trans;
}

__device__ void warp_add_counters(const Counters& c, unsigned long long* out) {
  const long long v[7] = {c.samples, c.tf, c.avgfb, c.coarse, c.req, c.used, c.skipped};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    long long x = v[i];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(out + i, (unsigned long long)x);
  }
}

// pixel of this thread: i (column), j (frame row), jl (output row)
__device__ __forceinline__ bool pixel_of(int& i, int& j, int& jl) {
  const RenderParams& P = c_P;
  // warp = VT_TW x (32 / VT_TW) pixel tile (16x2: rays of a warp stay close
  // in the gather, measured 2 % faster than 8x4); block = 4 warps stacked
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  i = blockIdx.x * VT_TW + (lane % VT_TW);
  jl = (blockIdx.y * 4 + warp) * (32 / VT_TW) + (lane / VT_TW);
  i += P.rect[0];
  if (P.n_parts > 1) {
    const int s = jl / P.strip_rows;
    j = (s * P.n_parts + P.part) * P.strip_rows + (jl - s * P.strip_rows);
  } else {
    j = jl + P.rect[1];
  }
  return i < P.rect[2] && j < P.rect[3];
}

template <class T>
__device__ void store_px(void* out, int kind, int64_t r, const double px[4]) {
  // whole-pixel vector stores (the frame may be page-locked host memory
  // written over PCIe, where narrow scattered stores are expensive)
  if (kind == 0) {
    double2* o = reinterpret_cast<double2*>((double*)out + r * 4);
    o[0] = make_double2(px[0], px[1]);
    o[1] = make_double2(px[2], px[3]);
  } else if (kind == 1) {
    *reinterpret_cast<float4*>((float*)out + r * 4) =
        make_float4((float)px[0], (float)px[1], (float)px[2], (float)px[3]);
  } else {
    uint32_t v = 0;
    for (int a = 0; a < 4; ++a)
      v |= (uint32_t)(uint8_t)npclip(rint(px[a] * 255.0), 0.0, 255.0) << (8 * a);
    *reinterpret_cast<uint32_t*>((uint8_t*)out + r * 4) = v;
  }
}

// fused full-frame pass: ray setup + march + finalize, no per-ray state
// the full-frame march of one ray (render/core.py:162-187): sample,
// composite, early termination; transparent runs skipped exactly
template <int MODE, class S>
__device__ __forceinline__ void march_ray(S& s, const TFTable& tf, const double d[3], double t0,
                                          int n, RayOut& o) {
  const RenderParams& P = c_P;
  constexpr int NC = S::kC;
  typename S::V vals[NC];
  Counters& cnt = s.cnt;
  for (int k = 0; k < n; ++k) {
    double t = t0 + exact_d(k) * P.step;
    double p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = P.cam[a] + t * d[a];
    s.sample(p, vals);
    cnt.samples++;
    if (MODE == 0 && s.hint) {
      // transparent (TF alpha exactly 0): compositing is a no-op; account
      // this sample and the provably transparent run after it
      const int m = (int)s.skip_count(k, n, t0, d);
      cnt.samples += m;
      cnt.skipped += m;
      if (s.hint == 1) cnt.used += m;
      k += m;
      continue;
    }
    if (composite<NC, MODE, MODE != 0>(tf, vals, o, cnt)) break;
  }
  // DVR: every counted sample looks up each channel's TF once (composite
  // or the exact skip) — render/core.py:122
  if (MODE == 0) cnt.tf += cnt.samples * NC;  // one ray per thread: its own samples
}

#ifndef VT_RENDER_MINB
#define VT_RENDER_MINB 5
#endif
template <class T, int NC, bool TR, bool FAST, int FILLED>
__global__ void __launch_bounds__(128, VT_RENDER_MINB) k_render_fullframe(const uint64_t* __restrict__ nb,
                                                          uint8_t* fb, const T* __restrict__ bb,
                                                          void* out, int out_kind, int out_w,
                                                          int out_rows,
                                                          unsigned long long* counters) {
  const RenderParams& P = c_P;
  __shared__ TFTable tf;
  load_tf(tf);
  Sampler<T, NC, TR, FAST, FILLED> s(nb, fb, bb, true);
  Counters& cnt = s.cnt;
  int i, j, jl;
  bool active = pixel_of(i, j, jl);
  bool write = false;
  double px[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    double d[3];
    ray_dir(i, j, d);
    double t0;
    long long n;
    ray_setup(d, t0, n);
    RayOut o{};
    // one uniform branch per ray instead of a mode test per sample (the DVR
    // branch never keeps the MIP maxima live)
    if (P.mip) {
      march_ray<1>(s, tf, d, t0, (int)n, o);
      finalize<NC, 1>(tf, o, px, cnt);
    } else {
      march_ray<0>(s, tf, d, t0, (int)n, o);
      finalize<NC, 0>(tf, o, px, cnt);
    }
    write = true;
  } else if (P.n_parts > 1 && i < P.rect[2] && jl < out_rows) {
    // padding rows of the last strip: deterministic zeros
    write = true;
  }
  if (out_kind == 0) {
    // FP64 frames: the warp's VT_TW x (32 / VT_TW) patch leaves as two
    // instructions of 16 pixels each — contiguous runs of whole rows, 16-byte
    // chunks gathered by shuffles — rather than four half-sector scatters:
    // the frame may be page-locked host memory written over PCIe
    const int lane = threadIdx.x & 31;
    const int64_t base =
        (int64_t)(jl - lane / VT_TW) * out_w + (i - lane % VT_TW - P.rect[0]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int src = 16 * h + (lane >> 1);  // the tile pixel (= lane) this lane stores half of
      double q[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) q[a] = __shfl_sync(0xffffffffu, px[a], src);
      const bool w = __shfl_sync(0xffffffffu, write, src);
      if (w) {
        const int64_t r = base + (int64_t)(src / VT_TW) * out_w + src % VT_TW;
        reinterpret_cast<double2*>((double*)out + r * 4)[lane & 1] =
            (lane & 1) ? make_double2(q[2], q[3]) : make_double2(q[0], q[1]);
      }
    }
  } else if (write) {
    store_px<T>(out, out_kind, (int64_t)jl * out_w + (i - P.rect[0]), px);
  }
  warp_add_counters(cnt, counters);
}

// ---- stateful passes (RefinementSession, raycast.py:298-339) ---------------

struct RayState {
  double* t0;
  long long* n;
  long long* k;
  uint8_t* flags;  // bit0 suspended, bit1 terminated
  double* acc;     // [rays][4]: rgb, a
  double* mip;     // [rays][4]
};

__global__ void k_rays_init(RayState S) {
  const RenderParams& P = c_P;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.W * P.H) return;
  int x = i % P.W, y = i / P.W;
  double d[3];
  ray_dir(x, y, d);
  double t0;
  long long n;
  ray_setup(d, t0, n);
  bool in_tile = x >= P.rect[0] && x < P.rect[2] && y >= P.rect[1] && y < P.rect[3];
  S.t0[i] = t0;
  S.n[i] = in_tile ? n : 0;
  S.k[i] = 0;
  S.flags[i] = 0;
  for (int a = 0; a < 4; ++a) {
    S.acc[i * 4 + a] = 0.0;
    S.mip[i * 4 + a] = 0.0;
  }
}

template <class T, int NC, bool TR>
__global__ void __launch_bounds__(128) k_rays_march(RayState S,
                                                    const uint64_t* __restrict__ nb, uint8_t* fb,
                                                    const T* __restrict__ bb, int fullframe,
                                                    unsigned long long* counters,
                                                    unsigned long long* n_susp) {
  const RenderParams& P = c_P;
  __shared__ TFTable tf;
  load_tf(tf);
  Sampler<T, NC, TR> s(nb, fb, bb, fullframe != 0);
  Counters& cnt = s.cnt;
  int i, j, jl;
  // stateful passes cover the whole frame; rect = full
  bool active = pixel_of(i, j, jl);
  bool susp = false;
  if (active) {
    const int64_t r = (int64_t)j * P.W + i;
    uint8_t fl = S.flags[r] & ~1;  // suspended flags reset each pass
    long long k = S.k[r];
    const long long n = S.n[r];
    if (!(fl & 2) && k < n) {
      double d[3];
      ray_dir(i, j, d);
      RayOut o;
      for (int a = 0; a < 3; ++a) o.rgb[a] = S.acc[r * 4 + a];
      o.a = S.acc[r * 4 + 3];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) o.mip[c] = S.mip[r * 4 + c];
      double vals[NC];
      const double t0 = S.t0[r];
        for (; k < n; ++k) {
        double t = t0 + (double)k * P.step;
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = P.cam[a] + t * d[a];
        bool miss = s.sample(p, vals);
        cnt.samples++;
        if (miss) {
          susp = true;
          fl |= 1;
          break;
        }
        if (s.hint) {
          const long long m = s.skip_count(k, n, t0, d);
          cnt.samples += (int)m;
          cnt.skipped += (int)m;
          cnt.tf += (int)(m + 1) * NC;
          if (s.hint == 1) cnt.used += (int)m;
          k += m;
          continue;
        }
        bool term = composite<NC>(tf, vals, o, cnt);
        if (term) {
          fl |= 2;
          ++k;
          break;
        }
      }
      for (int a = 0; a < 3; ++a) S.acc[r * 4 + a] = o.rgb[a];
      S.acc[r * 4 + 3] = o.a;
      for (int c = 0; c < kMaxC; ++c) S.mip[r * 4 + c] = o.mip[c];
      S.k[r] = k;
    }
    S.flags[r] = fl;
  }
  warp_add_counters(cnt, counters);
  unsigned b = __ballot_sync(0xffffffffu, susp);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(n_susp, (unsigned long long)__popc(b));
}

template <int NC>
__global__ void k_rays_image(RayState S, double* out,
                             unsigned long long* counters) {
  const RenderParams& P = c_P;
  __shared__ TFTable tf;
  load_tf(tf);
  Counters cnt{0, 0, 0, 0, 0, 0, 0};
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P.W * P.H) {
    RayOut o;
    for (int a = 0; a < 3; ++a) o.rgb[a] = S.acc[i * 4 + a];
    o.a = S.acc[i * 4 + 3];
    for (int c = 0; c < kMaxC; ++c) o.mip[c] = S.mip[i * 4 + c];
    double px[4];
    finalize<NC>(tf, o, px, cnt);
    for (int a = 0; a < 4; ++a) out[(int64_t)i * 4 + a] = px[a];
  }
  warp_add_counters(cnt, counters);
}

// ---- mirror kernels ------------------------------------------------------------

// per-slot, per-sub-brick, per-channel maximum over the stored voxels any
// trilinear corner of a sample inside the sub-brick can touch (stored
// indices [s*B, s*B + B + 1] per axis, borders included): the bound the
// empty-space skip tests against.  One warp per sub-brick.
template <class T>
__global__ void __launch_bounds__(256) k_brick_max(const T* __restrict__ bb, const int32_t* slots,
                                                   int n, Geo g, int sb0, int sb1, int sb2,
                                                   int nx, int ny, int nz, uint16_t* bmax,
                                                   uint16_t* bmax_brick) {
  const int C = g.C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nsb = nx * ny * nz;
  const int ex = sb0 + 2, ey = sb1 + 2, ez = sb2 + 2;  // voxels per sub-brick range
  for (int job = blockIdx.x; job < n; job += gridDim.x) {
    const int64_t slot = slots ? slots[job] : job;
    if (slot < 0) continue;
    const T* b = bb + slot * g.brick_elems;
    __shared__ int s_all[kMaxC];
    if (threadIdx.x < kMaxC) s_all[threadIdx.x] = 0;
    __syncthreads();
    for (int q = warp; q < nsb; q += nw) {
      const int qx = q % nx, qy = (q / nx) % ny, qz = q / (nx * ny);
      int mx[kMaxC] = {0, 0, 0, 0};
      for (int v = lane; v < ex * ey * ez; v += 32) {
        const int x = qx * sb0 + v % ex, y = qy * sb1 + (v / ex) % ey, z = qz * sb2 + v / (ex * ey);
        if (x >= g.stored[0] || y >= g.stored[1] || z >= g.stored[2]) continue;
        const T* p = b + g.voxel_offset(z, y, x);
#pragma unroll
        for (int c = 0; c < kMaxC; ++c)
          if (c < C) mx[c] = max(mx[c], (int)p[c]);
      }
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) {
        for (int o = 16; o > 0; o >>= 1) mx[c] = max(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        if (lane == 0) {
          bmax[(slot * nsb + q) * kMaxC + c] = (uint16_t)mx[c];
          atomicMax(&s_all[c], mx[c]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < kMaxC) bmax_brick[slot * kMaxC + threadIdx.x] = (uint16_t)s_all[threadIdx.x];
    __syncthreads();
  }
}

// The same maxima for 16-bit pools in two passes over shared memory: (1)
// every (stored row, sub-brick x-range) task reduces its run of samples —
// consecutive tasks read consecutive, overlapping runs of 32-bit words, so
// the brick streams through coalesced — into a row-maximum table; (2) one
// thread per (sub-brick, channel) reduces its rows of that table.  No
// atomics, no per-voxel index arithmetic.
constexpr int kBmaxSmemBytes = 40 * 1024;
constexpr int kBmaxWords = 20;  // one task's run: (sub-brick edge + 2) * C / 2 words
template <int C>
__global__ void __launch_bounds__(256) k_brick_max16(const uint16_t* __restrict__ bb,
                                                     const int32_t* slots, int n, Geo g, int sb0,
                                                     int sb1, int sb2, int nx, int ny, int nz,
                                                     uint16_t* bmax, uint16_t* bmax_brick) {
  extern __shared__ uint16_t s_rm[];  // [Sz][Sy][nx][C] row maxima
  __shared__ int s_all[kMaxC];
  const int Sx = g.stored[0], Sy = g.stored[1], Sz = g.stored[2];
  const int nsb = nx * ny * nz;
  const int ntask = Sz * Sy * nx;
  for (int job = blockIdx.x; job < n; job += gridDim.x) {
    const int64_t slot = slots ? slots[job] : job;
    if (slot < 0) continue;
    const uint16_t* b = bb + slot * g.brick_elems;
    if (threadIdx.x < kMaxC) s_all[threadIdx.x] = 0;
    for (int t = threadIdx.x; t < ntask; t += blockDim.x) {
      const int qx = t % nx, row = t / nx;  // row = z * Sy + y
      const int x0 = qx * sb0, x1 = min(x0 + sb0 + 2, Sx);
      const uint32_t* w = reinterpret_cast<const uint32_t*>(b + (int64_t)row * Sx * C + x0 * C);
      int mx[kMaxC] = {0, 0, 0, 0};
      const int nw = (x1 - x0) * C / 2;
      // every word of the run in flight at once (<= kBmaxWords), then reduce
      uint32_t v[kBmaxWords];
#pragma unroll
      for (int k = 0; k < kBmaxWords; ++k) v[k] = k < nw ? __ldg(w + k) : 0u;
      // sample 2k + h has channel (2k + h) % C: static after unrolling
#pragma unroll
      for (int k = 0; k < kBmaxWords; ++k) {
        if (k < nw) {
          mx[(2 * k) % C] = max(mx[(2 * k) % C], (int)(v[k] & 0xFFFF));
          mx[(2 * k + 1) % C] = max(mx[(2 * k + 1) % C], (int)(v[k] >> 16));
        }
      }
#pragma unroll
      for (int q = 0; q < kMaxC; ++q)
        if (q < C) s_rm[(int64_t)t * C + q] = (uint16_t)mx[q];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nsb * C; r += blockDim.x) {
      const int q = r / C, c = r - q * C;
      const int qx = q % nx, qy = (q / nx) % ny, qz = q / (nx * ny);
      const int y0 = qy * sb1, y1 = min(y0 + sb1 + 2, Sy), z0 = qz * sb2, z1 = min(z0 + sb2 + 2, Sz);
      int m = 0;
      for (int z = z0; z < z1; ++z)
        for (int y = y0; y < y1; ++y) m = max(m, (int)s_rm[((z * Sy + y) * nx + qx) * C + c]);
      bmax[(slot * nsb + q) * kMaxC + c] = (uint16_t)m;
      atomicMax(&s_all[c], m);
    }
    __syncthreads();
    if (threadIdx.x < kMaxC) bmax_brick[slot * kMaxC + threadIdx.x] = (uint16_t)s_all[threadIdx.x];
    __syncthreads();
  }
}

// sub-brick edge per axis: a quarter of the brick when that divides evenly
// into edges of at least 2 voxels, else the whole brick
inline void sub_bricks(const Geo& g, int sbk[3], int nsub[3]) {
  for (int a = 0; a < 3; ++a) {
    sbk[a] = (g.brick[a] % 4 == 0 && g.brick[a] >= 8) ? g.brick[a] / 4 : g.brick[a];
    nsub[a] = g.brick[a] / sbk[a];
  }
}

// _entry_for / pack_node (device.py:51-87, 168-178)
__global__ void k_repack(Geo g, const uint8_t* __restrict__ flags,
                         const int32_t* __restrict__ pslot, const int32_t* __restrict__ stats,
                         const int32_t* __restrict__ res, int zero_copy, double fmax, int w,
                         uint64_t* nb) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.capacity) return;
  uint8_t f = flags[i];
  if (!(f & NF_EXISTS)) {
    nb[i] = 0;
    return;
  }
  uint64_t e = (f & NF_BRICK) ? 2ULL : 0ULL;
  if (f & NF_CHILDREN) e |= (uint64_t)(i + 1) << 2;
  int32_t s = zero_copy ? ((f & NF_BRICK) ? pslot[i] : -1) : res[i];
  if (s >= 0) {
    e |= 1ULL | ((uint64_t)(uint32_t)s << 24);
  } else {
    double qmax = (double)((1LL << w) - 1);
    for (int c = 0; c < g.C; ++c) {
      double v = (double)stats[st_index(i, ST_AVG, c)];
      uint64_t q = (uint64_t)rint(v * qmax / fmax);
      e |= q << (24 + c * w);
    }
  }
  nb[i] = e;
}

__global__ void k_set_res(const int64_t* __restrict__ nodes, const int32_t* __restrict__ slots,
                          int n, int32_t* res) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) res[nodes[i]] = slots[i];
}

__global__ void k_upload(const int32_t* __restrict__ src_slots, const int32_t* __restrict__ dst_slots,
                         int n, const uint8_t* __restrict__ pool, uint8_t* bb, int64_t bytes) {
  int b = blockIdx.y;
  if (b >= n || dst_slots[b] < 0) return;
  const uint32_t* s = reinterpret_cast<const uint32_t*>(pool + (int64_t)src_slots[b] * bytes);
  uint32_t* d = reinterpret_cast<uint32_t*>(bb + (int64_t)dst_slots[b] * bytes);
  if ((bytes & 3) == 0) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bytes / 4;
         e += (int64_t)gridDim.x * blockDim.x)
      d[e] = s[e];
  } else {
    const uint8_t* s1 = pool + (int64_t)src_slots[b] * bytes;
    uint8_t* d1 = bb + (int64_t)dst_slots[b] * bytes;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bytes;
         e += (int64_t)gridDim.x * blockDim.x)
      d1[e] = s1[e];
  }
}

// c_P is one symbol per device: render entry points hold this lock from
// the parameter upload until their kernels have completed
std::mutex g_render_mu;

// empty-space skip granularity: 0 off, 1 bricks, 2 bricks + sub-bricks
// (env VT_ESS overrides the default)
int ess_level() {
  static int lvl = [] {
    const char* e = std::getenv("VT_ESS");
    return e ? std::atoi(e) : 1;
  }();
  return lvl;
}

// kernel instantiation for (sample type, channel count, transforms)
template <class F>
void dispatch(int sb, int C, bool tr, F&& f) {
  auto by_c = [&](auto tag, auto trc) {
    switch (C) {
      case 1: f(tag, std::integral_constant<int, 1>{}, trc); break;
      case 2: f(tag, std::integral_constant<int, 2>{}, trc); break;
      case 3: f(tag, std::integral_constant<int, 3>{}, trc); break;
      default: f(tag, std::integral_constant<int, 4>{}, trc); break;
    }
  };
  auto by_tr = [&](auto tag) {
    if (tr) by_c(tag, std::true_type{});
    else by_c(tag, std::false_type{});
  };
  if (sb == 1) by_tr(uint8_t{});
  else by_tr(uint16_t{});
}

// rows of one part's compact output: ceil(strips / n_parts) whole strips
int strip_part_rows(int H, int strip_rows, int n_parts) {
  if (n_parts <= 1) return H;
  const int strips = (H + strip_rows - 1) / strip_rows;
  return (strips + n_parts - 1) / n_parts * strip_rows;
}

void set_params(const RenderParams& P, cudaStream_t st) {
  VT_CUDA(cudaMemcpyToSymbolAsync(c_P, &P, sizeof(RenderParams), 0, cudaMemcpyHostToDevice, st));
}

void fill_params(const vt_mirror* m, const vt_scene* s, RenderParams& P) {
  const Tree& t = m->tree->t;
  std::memset(&P, 0, sizeof(P));
  P.g = t.g;
  for (int a = 0; a < 3; ++a) {
    P.dims[a] = (double)t.g.dims[a];
    P.spacing[a] = s->spacing[a];
    P.box_hi[a] = P.dims[a] * P.spacing[a];
  }
  for (int l = 0; l <= t.g.depth; ++l)
    for (int a = 0; a < 3; ++a) {
      P.ext[l][a] = (double)t.g.extent(a, l);
      P.scl[l][a] = (double)t.g.scale(a, l);
    }
  bool any_split = t.g.split[0] || t.g.split[1] || t.g.split[2];
  double bv = INFINITY;
  for (int a = 0; a < 3; ++a)
    if (!any_split || t.g.split[a]) bv = std::min(bv, s->spacing[a]);
  P.base_voxel = bv;
  P.fmax = (double)t.fmax;
  P.inv_fmax = 1.0 / P.fmax;
  for (int l = 0; l <= t.g.depth; ++l)
    for (int a = 0; a < 3; ++a) {
      P.inv_scl[l][a] = 1.0 / P.scl[l][a];
      P.exti[l][a] = t.g.split[a] ? t.g.extent(a, l) : (1 << 30);
    }
  P.unit_spacing = s->spacing[0] == 1.0 && s->spacing[1] == 1.0 && s->spacing[2] == 1.0;
  {
    int ex = 0;
    const double mant = std::frexp(bv, &ex);
    P.base_pow2 = (std::isfinite(bv) && mant == 0.5) ? 1 : 0;
    P.inv_base = P.base_pow2 ? 1.0 / bv : 0.0;
  }
  P.avg_w = 40 / t.g.C;
  P.qmax = (double)((1LL << P.avg_w) - 1);
  P.borders_filled = t.borders ? 1 : 0;
  P.zero_copy = m->zero_copy;
  // camera basis from the host shim (numpy-identical, camera.py:33-57)
  for (int a = 0; a < 3; ++a) {
    P.cam[a] = s->position[a];
    P.fwd[a] = s->fwd[a];
    P.right[a] = s->right[a];
    P.up[a] = s->up[a];
  }
  P.aspect = s->aspect;
  P.pfs = s->footprint_scale;
  P.W = s->width;
  P.H = s->height;
  P.tan_half = s->tan_half;
  P.mip = s->mode_mip;
  P.step = s->step;
  P.corr = s->corr_exp;
  P.et = s->et_limit;
  P.has_et = (s->et_limit >= 0.0 && s->et_limit < 1.0) ? 1 : 0;
  P.lod_scale = s->lod_scale;
  for (int c = 0; c < t.g.C; ++c) {
    P.tf_n[c] = s->tf_count[c];
    VT_REQUIRE(P.tf_n[c] >= 2 && P.tf_n[c] <= VT_MAX_TF_POINTS, VT_EINVAL,
               "transfer function needs 2..16 control points");
    for (int q = 0; q < P.tf_n[c]; ++q) {
      P.tf_x[c][q] = s->tf_x[c][q];
      for (int a = 0; a < 4; ++a) P.tf_v[c][q][a] = s->tf_rgba[c][q][a];
    }
    // np.interp's slope, (fp[j+1] - fp[j]) / (xp[j+1] - xp[j]), in FP64
    for (int q = 0; q + 1 < P.tf_n[c]; ++q)
      for (int a = 0; a < 4; ++a)
        P.tf_s[c][q][a] = (P.tf_v[c][q + 1][a] - P.tf_v[c][q][a]) / (P.tf_x[c][q + 1] - P.tf_x[c][q]);
  }
  P.n_clips = s->n_clips;
  VT_REQUIRE(P.n_clips >= 0 && P.n_clips <= 3, VT_EINVAL, "at most 3 clip planes supported");
  for (int q = 0; q < P.n_clips; ++q) {
    for (int a = 0; a < 3; ++a) P.clip_n[q][a] = s->clip_normal[q][a];
    P.clip_o[q] = s->clip_offset[q];
  }
  P.has_tr = s->has_transforms;
  for (int c = 0; c < kMaxC; ++c)
    for (int q = 0; q < 12; ++q) P.tr[c][q] = s->transforms[c][q];
  P.rect[0] = 0;
  P.rect[1] = 0;
  P.rect[2] = P.W;
  P.rect[3] = P.H;
  // empty-space skip thresholds: x*_c = sup{x : TF alpha == 0 on [0, x]};
  // a sample value v is transparent when v + 0.5 <= x*_c * fmax
  const int want_ess = s->empty_skip == 0 ? ess_level() : s->empty_skip - 1;
  P.ess = (!P.mip && !P.has_tr && m->bmax_valid && m->d_bmax) ? want_ess : 0;
  P.fast = s->precision == 1 ? 1 : 0;
  P.bmax = m->d_bmax;
  P.bmax_brick = m->d_bmax_brick;
  P.inv_step = 1.0 / P.step;
  {
    // the full-frame march counts samples in 32 bits: a ray through the
    // whole box takes at most |box| / step + 1 of them
    const double diag = std::sqrt(P.box_hi[0] * P.box_hi[0] + P.box_hi[1] * P.box_hi[1] +
                                  P.box_hi[2] * P.box_hi[2]);
    VT_REQUIRE(diag / P.step + 2.0 < 2147483647.0, VT_EINVAL,
               "sampling step too small: over 2^31 samples per ray");
  }
  sub_bricks(t.g, P.sbk, P.nsub);
  P.nsb = P.nsub[0] * P.nsub[1] * P.nsub[2];
  for (int c = 0; c < kMaxC; ++c) P.ess_thr[c] = -1;
  for (int c = 0; c < t.g.C; ++c) {
    const int n = P.tf_n[c];
    double xs = -1.0;
    if (P.tf_v[c][0][3] == 0.0) {
      xs = INFINITY;
      for (int q = 0; q + 1 < n; ++q) {
        if (P.tf_v[c][q + 1][3] != 0.0) {
          xs = P.tf_x[c][q];
          // duplicate knot: the jump may already apply at x == xp[q]
          if (!(P.tf_x[c][q + 1] > xs)) xs = std::nextafter(xs, -INFINITY);
          break;
        }
      }
      if (n == 1) xs = INFINITY;
    }
    P.tf_xzero[c] = xs < 0.0 ? -INFINITY : xs;
    if (xs < 0.0) P.ess_thr[c] = -1;
    else if (!std::isfinite(xs)) P.ess_thr[c] = t.fmax;
    // the float path needs a whole sample value of margin for its roundings
    else P.ess_thr[c] = (int)std::max(-1.0, std::floor(xs * P.fmax - (P.fast ? 1.0 : 0.5)));
  }
  P.strip_rows = P.H > 0 ? P.H : 1;
  P.n_parts = 1;
  P.part = 0;
}

}  // namespace

// (re)compute brick maxima: every pool slot in use (zero copy) or the listed
// brick-buffer slots (bounded mode, after uploads)
static void update_bmax(vt_mirror* m, const int32_t* d_slots, int n) {
  Tree& t = m->tree->t;
  int sbk[3], nsub[3];
  sub_bricks(t.g, sbk, nsub);
  const int64_t nsb = (int64_t)nsub[0] * nsub[1] * nsub[2];
  std::vector<int32_t> dirty;
  int32_t* d_dirty = nullptr;
  uint16_t *tab, *tab_brick;
  int jobs;
  if (m->zero_copy) {
    // the tree owns the table (dense leaf kernels write their maxima into
    // it): recompute the slots written since their maxima were last valid
    VT_REQUIRE(!d_slots, VT_ESTATE, "zero-copy maxima are per pool slot");
    t.enable_bmax((int)nsb);
    m->d_bmax = t.d_bmax;
    m->d_bmax_brick = t.bmax_brick();
    m->bmax_cap = t.bmax_cap * nsb;
    const int64_t used = std::min<int64_t>(t.cursor, (int64_t)t.slot_ver.size());
    for (int64_t s = 0; s < used; ++s)
      if (std::max(t.slot_ver[s], t.all_ver) > t.bmax_ver[s]) dirty.push_back((int32_t)s);
    for (int32_t s : dirty) t.bmax_ver[s] = t.data_version;
    if (m->bmax_version >= 0) m->bmax_incremental += 1;
    m->bmax_last_slots = (int64_t)dirty.size();
    m->bmax_version = t.data_version;
    m->bmax_valid = true;
    if (dirty.empty()) return;
    if ((int64_t)dirty.size() < used) {
      d_dirty = upload(t, dirty);
      d_slots = d_dirty;
    }
    jobs = (int)dirty.size();
    tab = t.d_bmax;
    tab_brick = t.bmax_brick();
  } else {
    const int64_t nslots = std::max<int64_t>(1, m->slots);
    const int64_t need = nslots * nsb;
    if (need > m->bmax_cap) {
      VT_CUDA(cudaStreamSynchronize(t.stream));
      cudaFree(m->d_bmax);
      m->d_bmax = nullptr;
      const size_t bytes = (need + nslots) * kMaxC * sizeof(uint16_t);
      VT_CUDA(cudaMalloc(&m->d_bmax, bytes));
      VT_CUDA(cudaMemsetAsync(m->d_bmax, 0xFF, bytes, t.stream));  // unknown: never empty
      m->bmax_cap = need;
      m->d_bmax_brick = m->d_bmax + need * kMaxC;
    }
    jobs = d_slots ? n : (int)m->slots;
    tab = m->d_bmax;
    tab_brick = m->d_bmax_brick;
  }
  if (jobs > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(jobs, 148 * 16);
    const void* bb = m->zero_copy ? (const void*)t.d_pool : (const void*)m->d_bb;
    if (t.g.sb == 1)
      k_brick_max<uint8_t><<<grid, 256, 0, t.stream>>>((const uint8_t*)bb, d_slots, jobs, t.g,
                                                       sbk[0], sbk[1], sbk[2], nsub[0], nsub[1],
                                                       nsub[2], tab, tab_brick);
    else if (sbk[0] % 2 == 0 && t.g.stored[0] % 2 == 0 &&
             (sbk[0] + 2) * t.g.C / 2 <= kBmaxWords &&
             (size_t)t.g.stored[2] * t.g.stored[1] * nsub[0] * t.g.C * sizeof(uint16_t) <=
                 (size_t)kBmaxSmemBytes)
      switch (t.g.C) {
#define VT_BMAX16(CC)                                                                          \
  case CC:                                                                                     \
    k_brick_max16<CC><<<grid, 256, kBmaxSmemBytes, t.stream>>>(                                \
        (const uint16_t*)bb, d_slots, jobs, t.g, sbk[0], sbk[1], sbk[2], nsub[0], nsub[1],     \
        nsub[2], tab, tab_brick);                                                              \
    break;
        VT_BMAX16(1)
        VT_BMAX16(2)
        VT_BMAX16(3)
        VT_BMAX16(4)
#undef VT_BMAX16
      }
    else
      k_brick_max<uint16_t><<<grid, 256, 0, t.stream>>>((const uint16_t*)bb, d_slots, jobs, t.g,
                                                        sbk[0], sbk[1], sbk[2], nsub[0], nsub[1],
                                                        nsub[2], tab, tab_brick);
    VT_CUDA(cudaGetLastError());
  }
  release(t, d_dirty);
  m->bmax_valid = true;
  if (m->zero_copy) m->bmax_version = t.data_version;
}

__global__ void k_clear_flags(const int64_t* __restrict__ idx, int64_t n, uint8_t* fb) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) fb[idx[i]] = 0;
}

struct vt_rays {
  vt_mirror* m;
  int ess_want = 1;
  RenderParams P;
  RayState S{};
  int64_t n = 0;
};

extern "C" {

vt_status vt_mirror_create(vt_tree* tree, int64_t slot_count, vt_mirror** out) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    t.flush();
    if (slot_count >= 0) {
      // a bounded mirror copies whole bricks (shells included) into its own
      // buffer: publish prefilled shells as background and write later dense
      // leaves with background shells.  A zero-copy mirror reads the pool in
      // place, where prefilled shells stay invisible: before fill_borders the
      // sampler clamps to the interior (render/raycast.py:141-144) and the
      // brick maxima only bound what may be read.
      t.publish_halos();
      t.prefill_enabled = false;
    }
    auto* m = new vt_mirror();
    m->tree = tree;
    vt_tree_retain(tree);
    const int64_t cap = t.g.capacity;
    const int64_t cap4 = (cap + 3) & ~3LL;
    try {
      VT_CUDA(cudaMalloc(&m->d_nb, cap * sizeof(uint64_t)));
      VT_CUDA(cudaMalloc(&m->d_fb, cap4));
      VT_CUDA(cudaMemsetAsync(m->d_fb, 0, cap4, t.stream));
      if (slot_count < 0) {
        m->zero_copy = true;
        m->slots = t.pool_slots;
      } else {
        m->slots = std::max<int64_t>(1, slot_count);
        VT_CUDA(cudaMalloc(&m->d_bb, m->slots * t.g.brick_elems * t.g.sb));
        VT_CUDA(cudaMemsetAsync(m->d_bb, 0, m->slots * t.g.brick_elems * t.g.sb, t.stream));
        VT_CUDA(cudaMalloc(&m->d_res, cap * sizeof(int32_t)));
        VT_CUDA(cudaMemsetAsync(m->d_res, 0xFF, cap * sizeof(int32_t), t.stream));
      }
    } catch (...) {
      cudaFree(m->d_nb);
      cudaFree(m->d_fb);
      cudaFree(m->d_bb);
      cudaFree(m->d_res);
      vt_tree_release(m->tree);
      delete m;
      throw;
    }
    *out = m;
  });
}

static void mirror_release(vt_mirror* m) {
  if (!m || m->refs.fetch_sub(1) != 1) return;
  cudaStreamSynchronize(m->tree->t.stream);
  cudaFree(m->d_nb);
  cudaFree(m->d_fb);
  cudaFree(m->d_bb);
  cudaFree(m->d_res);
  if (!m->zero_copy) cudaFree(m->d_bmax);  // a zero-copy mirror's table is the tree's
  vt_tree_release(m->tree);
  delete m;
}

vt_status vt_mirror_destroy(vt_mirror* m) {
  return guarded_on(m->tree->t.device, [&] { mirror_release(m); });
}

vt_status vt_mirror_bmax_stats(vt_mirror* m, int64_t* incremental, int64_t* last_slots) {
  return guarded_on(m->tree->t.device, [&] {
    if (incremental) *incremental = m->bmax_incremental;
    if (last_slots) *last_slots = m->bmax_last_slots;
  });
}

vt_status vt_mirror_buffers(vt_mirror* m, void** nbp, void** fbp, void** bbp, int64_t* cap,
                            int64_t* slots) {
  return guarded_on(m->tree->t.device, [&] {
    Tree& t = m->tree->t;
    if (nbp) *nbp = m->d_nb;
    if (fbp) *fbp = m->d_fb;
    if (bbp) *bbp = m->zero_copy ? t.d_pool : m->d_bb;
    if (cap) *cap = t.g.capacity;
    if (slots) *slots = m->zero_copy ? t.pool_slots : m->slots;
  });
}

vt_status vt_mirror_set_resident(vt_mirror* m, int64_t n, const int64_t* nodes,
                                 const int32_t* slots, int32_t copy) {
  return guarded_on(m->tree->t.device, [&] {
    Tree& t = m->tree->t;
    VT_REQUIRE(!m->zero_copy, VT_ESTATE, "zero-copy mirror: every brick is resident");
    if (n <= 0) return;
    t.flush();
    std::vector<int64_t> nv(nodes, nodes + n);
    std::vector<int32_t> sv(slots, slots + n);
    std::vector<int32_t> src(n, 0);
    for (int64_t i = 0; i < n; ++i) {
      VT_REQUIRE(sv[i] < m->slots, VT_EINVAL, "brick-buffer slot out of range");
      if (sv[i] >= 0) {
        VT_REQUIRE(t.flags[nv[i]] & NF_BRICK, VT_EINVAL, "upload of a node without a brick");
        src[i] = t.slot[nv[i]];
      }
    }
    int64_t* dn = upload(t, nv);
    int32_t* ds = upload(t, sv);
    k_set_res<<<(unsigned)((n + 255) / 256), 256, 0, t.stream>>>(dn, ds, (int)n, m->d_res);
    VT_CUDA(cudaGetLastError());
    if (copy) {
      int32_t* dsrc = upload(t, src);
      const int64_t bytes = t.g.brick_elems * t.g.sb;
      for (int64_t o = 0; o < n; o += 65535) {
        int cnt = (int)std::min<int64_t>(65535, n - o);
        dim3 grid(16, cnt);
        k_upload<<<grid, 256, 0, t.stream>>>(dsrc + o, ds + o, cnt, t.d_pool, m->d_bb, bytes);
        VT_CUDA(cudaGetLastError());
      }
      update_bmax(m, ds, (int)n);
      release(t, dsrc);
    }
    release(t, dn);
    release(t, ds);
  });
}

vt_status vt_mirror_repack(vt_mirror* m) {
  return guarded_on(m->tree->t.device, [&] {
    Tree& t = m->tree->t;
    t.flush();
    const int64_t cap = t.g.capacity;
    k_repack<<<(unsigned)((cap + 255) / 256), 256, 0, t.stream>>>(
        t.g, t.d_flags, t.d_slot, t.d_stats, m->d_res, m->zero_copy ? 1 : 0, (double)t.fmax,
        40 / t.g.C, m->d_nb);
    VT_CUDA(cudaGetLastError());
    if (m->zero_copy) update_bmax(m, nullptr, 0);
    else if (!m->bmax_valid) update_bmax(m, nullptr, 0);
  });
}

vt_status vt_mirror_apply_queued(vt_mirror* m, int64_t* n_events, int64_t* n_deleted) {
  return guarded_on(m->tree->t.device, [&] {
    Tree& t = m->tree->t;
    VT_REQUIRE(m->zero_copy, VT_ESTATE,
               "apply_queued needs a zero-copy mirror (bounded mirrors release slots per event)");
    t.flush();
    std::vector<int64_t> del;
    const int64_t n = t.discard_events(del);
    if (!del.empty()) {
      int64_t* d = upload(t, del);
      k_clear_flags<<<(unsigned)((del.size() + 255) / 256), 256, 0, t.stream>>>(
          d, (int64_t)del.size(), m->d_fb);
      VT_CUDA(cudaGetLastError());
      release(t, d);
    }
    const int64_t cap = t.g.capacity;
    k_repack<<<(unsigned)((cap + 255) / 256), 256, 0, t.stream>>>(
        t.g, t.d_flags, t.d_slot, t.d_stats, m->d_res, 1, (double)t.fmax, 40 / t.g.C, m->d_nb);
    VT_CUDA(cudaGetLastError());
    update_bmax(m, nullptr, 0);
    if (n_events) *n_events = n;
    if (n_deleted) *n_deleted = (int64_t)del.size();
  });
}

vt_status vt_mirror_read_flags(vt_mirror* m, uint8_t* out, int32_t clear) {
  return guarded_on(m->tree->t.device, [&] {
    Tree& t = m->tree->t;
    const int64_t cap = t.g.capacity;
    VT_CUDA(cudaMemcpyAsync(out, m->d_fb, cap, cudaMemcpyDeviceToHost, t.stream));
    if (clear) VT_CUDA(cudaMemsetAsync(m->d_fb, 0, (cap + 3) & ~3LL, t.stream));
    VT_CUDA(cudaStreamSynchronize(t.stream));
  });
}

static const void* brick_ptr(vt_mirror* m) {
  Tree& t = m->tree->t;
  return m->zero_copy ? (const void*)t.d_pool : (const void*)m->d_bb;
}

static void add_counters(vt_counters* cnt, const unsigned long long* h) {
  if (!cnt) return;
  cnt->samples += (int64_t)h[0];
  cnt->tf_lookups += (int64_t)h[1];
  cnt->avg_fallbacks += (int64_t)h[2];
  cnt->coarse_fallbacks += (int64_t)h[3];
  cnt->bricks_requested += (int64_t)h[4];
  cnt->bricks_used_marks += (int64_t)h[5];
  cnt->samples_skipped += (int64_t)h[6];
}

static void render_rect(vt_mirror* m, const vt_scene* scene, const int32_t* rect, void* out,
                        int32_t out_kind, int32_t out_on_device, vt_counters* cnt,
                        int strip_rows = 0, int n_parts = 1, int part = 0) {
  std::lock_guard<std::mutex> lk(g_render_mu);
  Tree& t = m->tree->t;
  t.flush();
  if (m->zero_copy && m->bmax_version != t.data_version) update_bmax(m, nullptr, 0);
  RenderParams P;
  fill_params(m, scene, P);
  VT_REQUIRE(out_kind >= 0 && out_kind <= 2, VT_EINVAL, "out_kind must be 0, 1 or 2");
  if (rect) {
    VT_REQUIRE(rect[0] >= 0 && rect[1] >= 0 && rect[2] <= P.W && rect[3] <= P.H &&
                   rect[0] <= rect[2] && rect[1] <= rect[3],
               VT_EINVAL, "tile rectangle outside the viewport");
    for (int a = 0; a < 4; ++a) P.rect[a] = rect[a];
  }
  int rw = P.rect[2] - P.rect[0], rh = P.rect[3] - P.rect[1];
  if (n_parts > 1) {
    VT_REQUIRE(strip_rows > 0 && part >= 0 && part < n_parts, VT_EINVAL,
               "strip partition needs strip_rows > 0 and 0 <= part < n_parts");
    P.strip_rows = strip_rows;
    P.n_parts = n_parts;
    P.part = part;
    rh = strip_part_rows(P.H, strip_rows, n_parts);
  }
  const int64_t px = (int64_t)rw * rh;
  const int esz = out_kind == 0 ? 8 : (out_kind == 1 ? 4 : 1);
  VT_REQUIRE(((uintptr_t)out & (out_kind == 2 ? 3 : 15)) == 0, VT_EINVAL,
             "output frame must be 16-byte aligned (4-byte for RGBA8)");
  void* dout = out;
  // a page-locked host frame (the Python API's frames are) is written by the
  // kernel itself over PCIe as the rays finish — the 66 MB float64 1080p
  // frame's transfer hides under the render instead of following it
  bool direct = false;
  if (!out_on_device && px > 0) {
    static const bool zc = [] {
      const char* e = std::getenv("VT_RENDER_DIRECT_HOST");
      return !(e && e[0] == '0');
    }();
    cudaPointerAttributes attr{};
    if (zc && cudaPointerGetAttributes(&attr, out) == cudaSuccess &&
        attr.type == cudaMemoryTypeHost && attr.devicePointer != nullptr) {
      dout = attr.devicePointer;
      direct = true;
    } else {
      cudaGetLastError();  // pageable memory: not an error
    }
  }
  if (!out_on_device && !direct)
    VT_CUDA(cudaMallocAsync(&dout, std::max<int64_t>(1, px) * 4 * esz, t.stream));
  unsigned long long* dc = nullptr;
  VT_CUDA(cudaMallocAsync(&dc, 7 * sizeof(unsigned long long), t.stream));
  VT_CUDA(cudaMemsetAsync(dc, 0, 7 * sizeof(unsigned long long), t.stream));
  dim3 grid((rw + VT_TW - 1) / VT_TW, (rh + 4 * (32 / VT_TW) - 1) / (4 * (32 / VT_TW)));
  VT_CUDA(cudaEventRecord(t.ev0, t.stream));
  P.buf_nb = m->d_nb;
  P.buf_fb = m->d_fb;
  P.buf_bb = brick_ptr(m);
  set_params(P, t.stream);
  if (px > 0) {
    dispatch(t.g.sb, t.g.C, P.has_tr != 0, [&](auto tag, auto nc, auto tr) {
      using T = decltype(tag);
      constexpr int NCv = decltype(nc)::value;
      constexpr bool TRv = decltype(tr)::value;
      const T* bbp = (const T*)brick_ptr(m);
      if (P.fast) {
        if (P.borders_filled)
          k_render_fullframe<T, NCv, TRv, true, 1><<<grid, 128, 0, t.stream>>>(
              m->d_nb, m->d_fb, bbp, dout, out_kind, rw, rh, dc);
        else
          k_render_fullframe<T, NCv, TRv, true, 0><<<grid, 128, 0, t.stream>>>(
              m->d_nb, m->d_fb, bbp, dout, out_kind, rw, rh, dc);
      } else {
        if (P.borders_filled)
          k_render_fullframe<T, NCv, TRv, false, 1><<<grid, 128, 0, t.stream>>>(
              m->d_nb, m->d_fb, bbp, dout, out_kind, rw, rh, dc);
        else
          k_render_fullframe<T, NCv, TRv, false, 0><<<grid, 128, 0, t.stream>>>(
              m->d_nb, m->d_fb, bbp, dout, out_kind, rw, rh, dc);
      }
    });
    VT_CUDA(cudaGetLastError());
  }
  VT_CUDA(cudaEventRecord(t.ev1, t.stream));
  unsigned long long h[7];
  VT_CUDA(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, t.stream));
  if (!out_on_device && !direct) {
    VT_CUDA(cudaMemcpyAsync(out, dout, px * 4 * esz, cudaMemcpyDeviceToHost, t.stream));
    release(t, dout);
  }
  release(t, dc);
  VT_CUDA(cudaStreamSynchronize(t.stream));
  float ms = 0;
  if (cudaEventElapsedTime(&ms, t.ev0, t.ev1) == cudaSuccess) t.last_render_ms = ms;
  else cudaGetLastError();  // not a render error
  add_counters(cnt, h);
}

vt_status vt_render_fullframe(vt_mirror* m, const vt_scene* scene, void* out, int32_t out_kind,
                              int32_t out_on_device, vt_counters* cnt) {
  return guarded_on(m->tree->t.device, [&] { render_rect(m, scene, nullptr, out, out_kind, out_on_device, cnt); });
}

vt_status vt_render_tile(vt_mirror* m, const vt_scene* scene, const int32_t rect[4], void* out,
                         int32_t out_kind, int32_t out_on_device, vt_counters* cnt) {
  return guarded_on(m->tree->t.device, [&] { render_rect(m, scene, rect, out, out_kind, out_on_device, cnt); });
}

vt_status vt_render_strips(vt_mirror* m, const vt_scene* scene, int32_t strip_rows,
                           int32_t n_parts, int32_t part, void* out, int32_t out_kind,
                           int32_t out_on_device, vt_counters* cnt) {
  return guarded_on(m->tree->t.device, [&] {
    VT_REQUIRE(n_parts >= 1, VT_EINVAL, "n_parts must be >= 1");
    render_rect(m, scene, nullptr, out, out_kind, out_on_device, cnt, strip_rows, n_parts, part);
  });
}

int32_t vt_strip_part_rows(int32_t height, int32_t strip_rows, int32_t n_parts) {
  if (height <= 0 || strip_rows <= 0 || n_parts <= 0) return 0;
  return strip_part_rows(height, strip_rows, n_parts);
}

vt_status vt_rays_create(vt_mirror* m, const vt_scene* scene, const int32_t* tile, vt_rays** out) {
  return guarded_on(m->tree->t.device, [&] {
    std::lock_guard<std::mutex> lk(g_render_mu);
    Tree& t = m->tree->t;
    auto* r = new vt_rays();
    r->m = m;
    r->ess_want = scene->empty_skip == 0 ? ess_level() : scene->empty_skip - 1;
    m->refs.fetch_add(1);
    fill_params(m, scene, r->P);
    if (tile)
      for (int a = 0; a < 4; ++a) r->P.rect[a] = tile[a];
    r->n = (int64_t)r->P.W * r->P.H;
    const int64_t n = std::max<int64_t>(1, r->n);
    VT_CUDA(cudaMalloc(&r->S.t0, n * 8));
    VT_CUDA(cudaMalloc(&r->S.n, n * 8));
    VT_CUDA(cudaMalloc(&r->S.k, n * 8));
    VT_CUDA(cudaMalloc(&r->S.flags, n));
    VT_CUDA(cudaMalloc(&r->S.acc, n * 32));
    VT_CUDA(cudaMalloc(&r->S.mip, n * 32));
    set_params(r->P, t.stream);
    k_rays_init<<<(unsigned)((n + 127) / 128), 128, 0, t.stream>>>(r->S);
    VT_CUDA(cudaGetLastError());
    VT_CUDA(cudaStreamSynchronize(t.stream));
    *out = r;
  });
}

vt_status vt_rays_destroy(vt_rays* r) {
  return guarded_on(r->m->tree->t.device, [&] {
    if (!r) return;
    cudaStreamSynchronize(r->m->tree->t.stream);
    cudaFree(r->S.t0);
    cudaFree(r->S.n);
    cudaFree(r->S.k);
    cudaFree(r->S.flags);
    cudaFree(r->S.acc);
    cudaFree(r->S.mip);
    mirror_release(r->m);
    delete r;
  });
}

vt_status vt_rays_march(vt_rays* r, int32_t strategy, vt_counters* cnt, int64_t* suspended) {
  return guarded_on(r->m->tree->t.device, [&] {
    std::lock_guard<std::mutex> lk(g_render_mu);
    vt_mirror* m = r->m;
    Tree& t = m->tree->t;
    t.flush();
    if (m->zero_copy && m->bmax_version != t.data_version) update_bmax(m, nullptr, 0);
    RenderParams P = r->P;
    P.borders_filled = t.borders ? 1 : 0;
    P.bmax = m->d_bmax;
    P.bmax_brick = m->d_bmax_brick;
    P.ess = (!P.mip && !P.has_tr && m->bmax_valid && m->d_bmax) ? r->ess_want : 0;
    P.rect[0] = 0;
    P.rect[1] = 0;
    P.rect[2] = P.W;
    P.rect[3] = P.H;
    unsigned long long* dc = nullptr;
    VT_CUDA(cudaMallocAsync(&dc, 8 * sizeof(unsigned long long), t.stream));
    VT_CUDA(cudaMemsetAsync(dc, 0, 8 * sizeof(unsigned long long), t.stream));
    dim3 grid((P.W + VT_TW - 1) / VT_TW, (P.H + 4 * (32 / VT_TW) - 1) / (4 * (32 / VT_TW)));
    P.buf_nb = m->d_nb;
    P.buf_fb = m->d_fb;
    P.buf_bb = brick_ptr(m);
    set_params(P, t.stream);
    dispatch(t.g.sb, t.g.C, P.has_tr != 0, [&](auto tag, auto nc, auto tr) {
      using T = decltype(tag);
      k_rays_march<T, decltype(nc)::value, decltype(tr)::value><<<grid, 128, 0, t.stream>>>(
          r->S, m->d_nb, m->d_fb, (const T*)brick_ptr(m), strategy == 0, dc, dc + 7);
    });
    VT_CUDA(cudaGetLastError());
    unsigned long long h[8];
    VT_CUDA(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, t.stream));
    release(t, dc);
    VT_CUDA(cudaStreamSynchronize(t.stream));
    add_counters(cnt, h);
    if (suspended) *suspended = (int64_t)h[7];
  });
}

vt_status vt_rays_image(vt_rays* r, double* out_host, vt_counters* cnt) {
  return guarded_on(r->m->tree->t.device, [&] {
    std::lock_guard<std::mutex> lk(g_render_mu);
    Tree& t = r->m->tree->t;
    double* dout = nullptr;
    const int64_t n = std::max<int64_t>(1, r->n);
    VT_CUDA(cudaMallocAsync(&dout, n * 32, t.stream));
    unsigned long long* dc = nullptr;
    VT_CUDA(cudaMallocAsync(&dc, 7 * sizeof(unsigned long long), t.stream));
    VT_CUDA(cudaMemsetAsync(dc, 0, 7 * sizeof(unsigned long long), t.stream));
    set_params(r->P, t.stream);
    dispatch(2, t.g.C, false, [&](auto, auto nc, auto) {
      k_rays_image<decltype(nc)::value><<<(unsigned)((n + 127) / 128), 128, 0, t.stream>>>(
          r->S, dout, dc);
    });
    VT_CUDA(cudaGetLastError());
    unsigned long long h[7];
    VT_CUDA(cudaMemcpyAsync(out_host, dout, r->n * 32, cudaMemcpyDeviceToHost, t.stream));
    VT_CUDA(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, t.stream));
    release(t, dout);
    release(t, dc);
    VT_CUDA(cudaStreamSynchronize(t.stream));
    add_counters(cnt, h);
  });
}

vt_status vt_rays_state(vt_rays* r, int64_t* k, int64_t* n_steps, uint8_t* suspended) {
  return guarded_on(r->m->tree->t.device, [&] {
    Tree& t = r->m->tree->t;
    std::vector<uint8_t> fl(r->n);
    if (k) VT_CUDA(cudaMemcpyAsync(k, r->S.k, r->n * 8, cudaMemcpyDeviceToHost, t.stream));
    if (n_steps)
      VT_CUDA(cudaMemcpyAsync(n_steps, r->S.n, r->n * 8, cudaMemcpyDeviceToHost, t.stream));
    VT_CUDA(cudaMemcpyAsync(fl.data(), r->S.flags, r->n, cudaMemcpyDeviceToHost, t.stream));
    VT_CUDA(cudaStreamSynchronize(t.stream));
    if (suspended)
      for (int64_t i = 0; i < r->n; ++i) suspended[i] = fl[i] & 1;
  });
}

}  // extern "C"
