// Dense (pyramid) build kernels for homogeneity threshold 0.
//
// At tau == 0 nothing is ever pruned and every brick whose in-volume leaves
// are fully covered by inserted data is a pure function of that data
// (SURVEY 7.3.1): a leaf brick is the block copied at +1 with a background
// shell, a parent brick the 2x2x2 integer half-sample of its children
// (halfsample_block, octree.py:58-92).  When an insertion covers whole brick
// layers over the full x/y extent (ingest_bulk's z-slabs, ingest.py:182-224,
// or a VSTR layer), the tree control plane (tree.cu) routes its device work
// here instead of the general seed -> scatter -> octant-job pipeline:
//
//   k_dense_leaf   one CTA per leaf brick: writes the WHOLE stored brick
//                  (shell + interior, one coalesced pass), the per-plane
//                  partial statistics and the leaf's final statistics
//                  (_write_leaf + _ensure_brick + _recompute_stats,
//                  octree.py:225-263, 420-442)
//   k_dense_level  one CTA per parent whose in-volume children are all
//                  complete: its whole interior from the children
//                  (_update_parent_octant for every real octant,
//                  octree.py:281-319), plane partials, final statistics and
//                  _aggregate_subtree_extrema (octree.py:265-277)
//
// Results are byte-identical to the general path (tests/test_gpu_dense.py);
// the host emits the same events, slots and structure either way.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cuda.h>

#include "tree.cuh"

namespace vtx {

namespace {

template <int C>
struct Acc {
  int mn[C], mx[C];
  unsigned long long sm[C];
  __device__ void init() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      mn[c] = INT_MAX;
      mx[c] = INT_MIN;
      sm[c] = 0;
    }
  }
  __device__ void add(int c, int v) {
#pragma unroll
    for (int q = 0; q < C; ++q)
      if (q == c) {
        mn[q] = min(mn[q], v);
        mx[q] = max(mx[q], v);
        sm[q] += (unsigned)v;
      }
  }
  __device__ void add_all(const int* v) {
#pragma unroll
    for (int q = 0; q < C; ++q) {
      mn[q] = min(mn[q], v[q]);
      mx[q] = max(mx[q], v[q]);
      sm[q] += (unsigned)v[q];
    }
  }
  __device__ void warp_reduce() {
#pragma unroll
    for (int c = 0; c < C; ++c)
      for (int o = 16; o > 0; o >>= 1) {
        mn[c] = min(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
        mx[c] = max(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], o);
      }
  }
  __device__ void merge(const Acc& o) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      mn[c] = min(mn[c], o.mn[c]);
      mx[c] = max(mx[c], o.mx[c]);
      sm[c] += o.sm[c];
    }
  }
};

constexpr int kMaxWarps = 17;

// CTA-wide reduction of the per-warp totals (held by lane 0 of each warp),
// then the node's final statistics: avg (round_mean, octree.py:53-55),
// smin, smax; sub extrema = own for leaves / childless nodes, else the
// aggregate over existing in-volume children (octree.py:265-277)
template <int C>
__device__ void finish_stats(Acc<C>& tot, int64_t node, int64_t nvox, bool leafish, const Geo& g,
                             const uint8_t* __restrict__ flags, int32_t* stats) {
  __shared__ int s_mn[kMaxWarps][C], s_mx[kMaxWarps][C];
  __shared__ unsigned long long s_sm[kMaxWarps][C];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      s_mn[warp][c] = tot.mn[c];
      s_mx[warp][c] = tot.mx[c];
      s_sm[warp][c] = tot.sm[c];
    }
  __syncthreads();
  if (threadIdx.x >= C) return;
  const int c = threadIdx.x;
  if (nvox > 0) {
    int a = INT_MAX, b = INT_MIN;
    unsigned long long s = 0;
    for (int w = 0; w < nw; ++w) {
      a = min(a, s_mn[w][c]);
      b = max(b, s_mx[w][c]);
      s += s_sm[w][c];
    }
    const long long avg = (2 * (long long)s + nvox) / (2 * nvox);
    stats[st_index(node, ST_AVG, c)] = (int)avg;
    stats[st_index(node, ST_MIN, c)] = a;
    stats[st_index(node, ST_MAX, c)] = b;
    if (leafish) {
      stats[st_index(node, ST_SUBMIN, c)] = a;
      stats[st_index(node, ST_SUBMAX, c)] = b;
    }
  }
  if (!leafish) {
    bool any = false;
    int lo = 0, hi = 0;
    for (int k = 0; k < 8; ++k) {
      if (!g.octant_real(k)) continue;
      const int64_t ch = 8 * node + 1 + k;
      const uint8_t f = flags[ch];
      if (!(f & NF_EXISTS) || !(f & NF_INVOL)) continue;
      const int a = stats[st_index(ch, ST_SUBMIN, c)], b = stats[st_index(ch, ST_SUBMAX, c)];
      lo = any ? min(lo, a) : a;
      hi = any ? max(hi, b) : b;
      any = true;
    }
    if (any) {
      stats[st_index(node, ST_SUBMIN, c)] = lo;
      stats[st_index(node, ST_SUBMAX, c)] = hi;
    }
  }
}

// lane 0 of a warp: write one plane's partials (layout of k_plane) and fold
// them into the warp's running total
template <int C>
__device__ void emit_plane(Acc<C>& pl, Acc<C>& tot, int64_t slot, int mz, int z, int32_t* pmin,
                           int32_t* pmax, unsigned long long* psum) {
  pl.warp_reduce();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int64_t off = (slot * mz + z) * C + c;
      pmin[off] = pl.mn[c];
      pmax[off] = pl.mx[c];
      psum[off] = pl.sm[c];
    }
    tot.merge(pl);
  }
}

// ---------------------------------------------------------------------------
// leaves
// ---------------------------------------------------------------------------
// One CTA per leaf brick of a block that spans the volume's full x/y extent
// and whole brick layers in z.  Warps own stored planes; a plane is written
// as one linear run (rows are contiguous in the stored brick), so stores are
// fully coalesced.  Generic per-sample version (8-bit samples, odd rows).
template <class T, int C>
__global__ void __launch_bounds__(384, 2) k_dense_leaf(const T* __restrict__ src, int oz,
                                                    const DenseJob* __restrict__ jobs, int gnx,
                                                    int gny, int g0z, Geo g, T* __restrict__ pool,
                                                    int32_t* pmin, int32_t* pmax,
                                                    unsigned long long* psum, int32_t* stats,
                                                    const uint8_t* __restrict__ flags,
                                                    int planes_per_warp) {
  const DenseJob j = jobs[blockIdx.x];
  const int gx = (int)(blockIdx.x % gnx);
  const int gy = (int)((blockIdx.x / gnx) % gny);
  const int gz = g0z + (int)(blockIdx.x / (gnx * gny));
  const int Mx = g.brick[0], My = g.brick[1], Mz = g.brick[2];
  const int Sx = g.stored[0], Sy = g.stored[1], Sz = g.stored[2];
  const int X = g.dims[0], Y = g.dims[1];
  const int cx = min(Mx, X - gx * Mx), cy = min(My, Y - gy * My), cz = min(Mz, g.dims[2] - gz * Mz);
  const int rowlen = Sx * C;  // samples per stored row
  T* brick = pool + (int64_t)j.slot * g.brick_elems;
  const T bg = (T)g.bg;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Acc<C> tot;
  tot.init();
  const int zp0 = warp * planes_per_warp;
  for (int zs = zp0; zs < min(Sz, zp0 + planes_per_warp); ++zs) {
    const int zi = zs - 1;
    const bool zdata = zi >= 0 && zi < cz;
    // block row of stored row ys: sample s of the stored row <-> block sample
    // rb + s - C, rb = first sample of voxel x = gx*Mx in that block row
    const int64_t zrow = zdata ? (int64_t)(gz * Mz + zi - oz) * Y : 0;
    T* plane = brick + (int64_t)zs * Sy * rowlen;
    Acc<C> pl;
    pl.init();
    const int n = Sy * rowlen;
#pragma unroll 4
    for (int e = lane; e < n; e += 32) {
      const int ys = e / rowlen;
      const int s = e - ys * rowlen;
      const int x = s / C;
      const bool v = zdata && ys >= 1 && ys <= cy && x >= 1 && x <= cx;
      T val = bg;
      if (v) {
        val = __ldg(src + ((zrow + gy * My + ys - 1) * X + (int64_t)gx * Mx) * C + s - C);
        pl.add(s % C, (int)val);
      }
      plane[e] = val;
    }
    if (zdata) emit_plane<C>(pl, tot, j.slot, Mz, zi, pmin, pmax, psum);
  }
  finish_stats<C>(tot, j.node, (int64_t)cx * cy * cz, true, g, flags, stats);
}

// 16-bit samples, rows of an even number of samples: 32-bit words.  A warp
// owns a stored plane and walks its rows; lane l owns words l, l+32, ... of
// every row, so each lane's x positions, channels and halo flags are
// constants and the per-word work is two aligned loads (one when the row is
// even-aligned in the block), a byte permute, one store and the statistics.
// A stored row is the run of block samples starting one voxel left of the
// brick (+1 interior offset, octree.py:420-442); halo / out-of-volume samples
// are the background (fresh-brick seeding, octree.py:225-241).
template <int C, int WPL>
__global__ void __launch_bounds__(544, 1) k_dense_leaf16(
    const uint16_t* __restrict__ src, int oz, const DenseJob* __restrict__ jobs, int gnx, int gny,
    int g0z, Geo g, uint16_t* __restrict__ pool, int32_t* pmin, int32_t* pmax,
    unsigned long long* psum, int32_t* stats, const uint8_t* __restrict__ flags,
    int planes_per_warp, int64_t nsrc) {
  constexpr int R = 2;  // rows per iteration (all their loads in flight together)
  const DenseJob j = jobs[blockIdx.x];
  const int gx = (int)(blockIdx.x % gnx);
  const int gy = (int)((blockIdx.x / gnx) % gny);
  const int gz = g0z + (int)(blockIdx.x / (gnx * gny));
  const int Mx = g.brick[0], My = g.brick[1], Mz = g.brick[2];
  const int Sx = g.stored[0], Sy = g.stored[1], Sz = g.stored[2];
  const int X = g.dims[0], Y = g.dims[1];
  const int cx = min(Mx, X - gx * Mx), cy = min(My, Y - gy * My), cz = min(Mz, g.dims[2] - gz * Mz);
  const int wpr = Sx * C / 2;  // words per stored row
  const uint32_t* src32 = reinterpret_cast<const uint32_t*>(src);
  uint32_t* brick = reinterpret_cast<uint32_t*>(pool + (int64_t)j.slot * g.brick_elems);
  const uint32_t bgw = (uint32_t)g.bg | ((uint32_t)g.bg << 16);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // lane constants
  bool has[WPL], in0[WPL], in1[WPL];
  int ch[2 * WPL];
#pragma unroll
  for (int q = 0; q < WPL; ++q) {
    const int wl = lane + 32 * q;
    const int s0 = 2 * wl;
    has[q] = wl < wpr;
    const int x0 = s0 / C, x1 = (s0 + 1) / C;
    in0[q] = has[q] && x0 >= 1 && x0 <= cx;
    in1[q] = has[q] && x1 >= 1 && x1 <= cx;
    ch[2 * q] = s0 % C;
    ch[2 * q + 1] = (s0 + 1) % C;
  }
  Acc<C> tot;
  tot.init();
  const int zp0 = warp * planes_per_warp;
  for (int zs = zp0; zs < min(Sz, zp0 + planes_per_warp); ++zs) {
    const int zi = zs - 1;
    const bool zdata = zi >= 0 && zi < cz;
    const int64_t zrow = zdata ? (int64_t)(gz * Mz + zi - oz) * Y : 0;
    uint32_t* plane = brick + (int64_t)zs * Sy * wpr;
    unsigned smn[2 * WPL], smx[2 * WPL], ssm[2 * WPL];
#pragma unroll
    for (int q = 0; q < 2 * WPL; ++q) {
      smn[q] = 0xFFFFFFFFu;
      smx[q] = 0;
      ssm[q] = 0;
    }
    for (int y0 = 0; y0 < Sy; y0 += R) {
      uint32_t A[R][WPL], B[R][WPL];
      bool full[R], odd[R], rd[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        rd[r] = zdata && y >= 1 && y <= cy;
        // block sample index of stored sample 0 of this row (x = gx*Mx - 1)
        const int64_t rb = ((zrow + gy * My + y - 1) * X + (int64_t)gx * Mx - 1) * C;
        odd[r] = rb & 1;
        const int64_t ib = (rb - (rb & 1)) >> 1;
        full[r] = rd[r] && rb + 2 * wpr + 1 < nsrc;
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
          const int wl = lane + 32 * q;
          if (full[r] && in0[q] && in1[q]) {
            A[r][q] = __ldg(src32 + ib + wl);
            B[r][q] = odd[r] ? __ldg(src32 + ib + wl + 1) : 0u;
          } else {
            A[r][q] = (rd[r] && in0[q]) ? (uint32_t)__ldg(src + rb + 2 * wl) : bgw & 0xFFFFu;
            B[r][q] = (rd[r] && in1[q]) ? (uint32_t)__ldg(src + rb + 2 * wl + 1) : bgw & 0xFFFFu;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        if (y >= Sy) break;
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
          if (!has[q]) continue;
          uint32_t out;
          if (full[r] && in0[q] && in1[q])
            out = odd[r] ? __byte_perm(A[r][q], B[r][q], 0x5432) : A[r][q];
          else
            out = A[r][q] | (B[r][q] << 16);
          plane[y * wpr + lane + 32 * q] = out;
          if (rd[r] && in0[q]) {
            const unsigned v = out & 0xFFFFu;
            smn[2 * q] = min(smn[2 * q], v);
            smx[2 * q] = max(smx[2 * q], v);
            ssm[2 * q] += v;
          }
          if (rd[r] && in1[q]) {
            const unsigned v = out >> 16;
            smn[2 * q + 1] = min(smn[2 * q + 1], v);
            smx[2 * q + 1] = max(smx[2 * q + 1], v);
            ssm[2 * q + 1] += v;
          }
        }
      }
    }
    if (zdata) {
      Acc<C> pl;
      pl.init();
#pragma unroll
      for (int q = 0; q < 2 * WPL; ++q)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (ch[q] == c && smx[q] >= smn[q]) {
            pl.mn[c] = min(pl.mn[c], (int)smn[q]);
            pl.mx[c] = max(pl.mx[c], (int)smx[q]);
            pl.sm[c] += ssm[q];
          }
      emit_plane<C>(pl, tot, j.slot, Mz, zi, pmin, pmax, psum);
    }
  }
  finish_stats<C>(tot, j.node, (int64_t)cx * cy * cz, true, g, flags, stats);
}

// ---------------------------------------------------------------------------
// TMA-staged leaves (16-bit samples, 16-byte aligned block rows)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "VT_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra VT_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// 3-D tensor tile (TMA) global -> shared, completion on an mbarrier
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_addr(b))
      : "memory");
}
// One CTA (8 warps) per leaf brick, stored planes in stages of P = 2.  The
// TMA engine streams the block region a stage needs — one 3-D tensor tile of
// the brick's P stored planes WITH their one-voxel x/y/z halo, zero-filled
// outside the block — into a 3-deep shared-memory ring (data in flight lives
// in shared memory, not registers).  Four warps per plane then write the
// stored plane straight to HBM as coalesced 32-bit words (a stored row is
// one contiguous run of block samples starting one voxel left of the brick:
// a byte permute of two aligned shared words when that start is odd) and
// reduce the interior's per-plane statistics.
//
// Shell voxels: with `prefill` they receive the value fill_borders will give
// them at threshold 0 once every in-volume leaf is complete — the block
// voxel when it lies inside the volume (the same-level neighbour's interior,
// octree.py:593-605), else the background (outside the virtual extent, or an
// out-of-volume neighbour whose AVG is the background) — except z-shell
// planes whose block plane lies outside this insertion (owed: background
// now, copied from the neighbour brick by fill_borders).  The tree keeps
// such shells logically background until fill_borders (Tree::halo_prefill).
// Without `prefill` every shell voxel is the background (_ensure_brick,
// octree.py:234-237).
// ring slots: the stage being built, the previous one (its second plane
// pairs with this stage's first for the fused parent octant) and two in flight
constexpr int kTmaStages = 4;
constexpr int kTmaAhead = 3;  // stages in flight ahead of the one being built
constexpr int kTmaWarps = 8;
constexpr int kTmaP = 2;

// staged row: the stored row's (Mx+2)*C samples from a 16-byte aligned start
// (the TMA inner coordinate must be a multiple of 8 samples), <= 7 leading
__host__ __device__ inline int tma_box_row(int mx, int C) { return ((mx + 2) * C + 7 + 7) / 8 * 8; }
__host__ __device__ inline uint32_t tma_in_bytes(int mx, int my, int C) {
  return ((uint32_t)kTmaP * (my + 2) * tma_box_row(mx, C) * 2 + 127) / 128 * 128;
}

// MX, MY: brick x/y edge fixed at compile time (0 = from g) — with them the
// stored-row word copy has constant strides and trip counts (immediate
// offsets, full unrolling)
// ST: input stages in the shared-memory ring (4, or 3 for large bricks)
template <int C, int MX = 0, int MY = 0, int ST = kTmaStages>
__global__ void __launch_bounds__(kTmaWarps * 32) k_dense_leaf_tma(
    const __grid_constant__ CUtensorMap map, int oz, int dz, int prefill,
    const DenseJob* __restrict__ jobs, int gnx, int gny, int g0z, Geo g,
    uint16_t* __restrict__ pool, int32_t* stats, int32_t* nmin, int32_t* nmax,
    unsigned long long* nsum, int pshell) {
  constexpr int P = kTmaP;
  constexpr int WPP = kTmaWarps / P;  // warps per plane
  constexpr int NT = WPP * 32;        // threads per plane
  extern __shared__ __align__(128) unsigned char s_in[];
  __shared__ uint64_t s_bar[ST];
  __shared__ int s_mn[2][kTmaWarps][C], s_mx[2][kTmaWarps][C];
  __shared__ unsigned long long s_sm[2][kTmaWarps][C];
  const DenseJob j = jobs[blockIdx.x];
  const int gx = (int)(blockIdx.x % gnx);
  const int gy = (int)((blockIdx.x / gnx) % gny);
  const int gz = g0z + (int)(blockIdx.x / (gnx * gny));
  const int Mx = MX ? MX : g.brick[0], My = MY ? MY : g.brick[1], Mz = g.brick[2];
  const int Sx = Mx + 2, Sy = My + 2, Sz = g.stored[2];
  const int X = g.dims[0], Y = g.dims[1], Z = g.dims[2];
  const int cx = min(Mx, X - gx * Mx), cy = min(My, Y - gy * My), cz = min(Mz, Z - gz * Mz);
  const int brow = tma_box_row(Mx, C);                  // staged row (samples)
  const int RS = My + 2;  // staged rows per plane
  const uint32_t in_bytes = tma_in_bytes(Mx, My, C);    // one input stage
  const uint32_t plane_elems = (uint32_t)Sx * Sy * C;   // one stored plane
  const int wpr = Sx * C / 2;                           // 32-bit words per stored row
  const int nstages = Sz / P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint16_t* brick = pool + (int64_t)j.slot * g.brick_elems;
  const uint16_t bg = (uint16_t)g.bg;
  const uint32_t bgw = (uint32_t)bg | ((uint32_t)bg << 16);
  const int x0 = gx * Mx - 1, y0 = gy * My - 1;     // block voxel of stored (0, 0)
  const int xa = x0 * C - (((x0 * C) % 8 + 8) % 8);  // 16-byte aligned tile start (samples)
  const int xoff = x0 * C - xa;                     // leading samples of a staged row
  // every stored x / row inside the volume — or a zero background, which the
  // TMA tile's zero fill outside the volume reproduces
  const bool xfull = prefill && (bg == 0 || (x0 >= 0 && x0 + Sx <= X));
  const bool yfull = bg == 0 || (y0 >= 0 && y0 + Sy <= Y);
  // e / (Sx * C) and e / C by multiply-high (e < 2^16; a divisor of 1 has no
  // 32-bit magic)
  const uint32_t rowmagic = (uint32_t)((((uint64_t)1 << 32) + Sx * C - 1) / (Sx * C));
  const uint32_t cmagic = C == 1 ? 0u : (uint32_t)((((uint64_t)1 << 32) + C - 1) / C);
  const uint32_t cxmagic = (uint32_t)((((uint64_t)1 << 32) + cx - 1) / cx);  // v / cx by mul-high

  if (tid == 0) {
    for (int b = 0; b < ST; ++b) mbar_init(&s_bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int s) {  // one thread: one tensor tile per stage
    const int b = s % ST;
    mbar_expect_tx(&s_bar[b], (uint32_t)P * RS * brow * 2);
    tma_load_3d(s_in + (size_t)b * in_bytes, &map, xa, y0, gz * Mz - oz + P * s - 1, &s_bar[b]);
  };
  if (tid == 0)
    for (int s = 0; s < min((ST - 1), nstages); ++s) issue(s);

  // fused parent octant (j.pad = parent slot, else -1): the 2x2x2 integer
  // half-sample of this leaf (halfsample_block, octree.py:58-92) written into
  // the parent's octant (_update_parent_octant, octree.py:308-319).  That
  // pass visits every interior voxel exactly once, so it also carries the
  // leaf's statistics; the parent's are folded into its accumulators
  // (nmin, nmax, nsum) with one atomic per channel per CTA.
  const int pslot = j.pad;
  const int hx = Mx / 2, hy = My / 2;
  const int offx = (gx & 1) * hx, offy = (gy & 1) * hy, offz = (gz & 1) * (Mz / 2);
  int pcx, pcy, pcz;  // the parent's in-volume extent (octree.py:190-199)
  {
    const int plx = (gx >> 1) * 2 * Mx, ply = (gy >> 1) * 2 * My, plz = (gz >> 1) * 2 * Mz;
    pcx = min(Mx, max(0, (X - plx + 1) / 2));
    pcy = min(My, max(0, (Y - ply + 1) / 2));
    pcz = min(Mz, max(0, (Z - plz + 1) / 2));
  }
  uint16_t* parent = pslot >= 0 ? pool + (int64_t)pslot * g.brick_elems : nullptr;
  // interior level-1 parent: its x-face shell rows on this child's side,
  // from the staged x halo (as k_dense_leaf_tma_planar; Tree::parent_interior
  // mirrors the rule)
  const bool pxy = parent && pshell && (gx >> 1) >= 1 && (gy >> 1) >= 1 &&
                   ((gx >> 1) + 1) * 2 * Mx + 2 <= X && ((gy >> 1) + 1) * 2 * My + 2 <= Y &&
                   xoff >= C && (Mx + 3) * C + xoff <= brow;

  // per-thread totals over the whole brick: the leaf (l*) and the octant (o*)
  int lmn[C], lmx[C], omn[C], omx[C];
  unsigned long long lsm[C], osm[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    lmn[c] = omn[c] = INT_MAX;
    lmx[c] = omx[c] = INT_MIN;
    lsm[c] = osm[c] = 0;
  }

  // word mapping: thread pt of a plane group owns word wr of rows rr, rr+R, ..
  const int pw = warp / WPP;                // plane of the stage this warp group builds
  const int pt = (warp % WPP) * 32 + lane;  // thread within the plane group
  const int R = wpr <= NT ? NT / wpr : 1;   // rows per pass of the group
  const int rr = wpr <= NT ? pt / wpr : 0;
  const int wr0 = wpr <= NT ? pt % wpr : pt;
  const int wstep = wpr <= NT ? wpr : NT;
  const bool wact = rr < R;
  const int xo = (xoff >> 1) + wr0;  // staged word of this thread's first word

  const int toy = hx > 0 ? tid / hx : 0;  // octant row of this thread's first octant voxel
  for (int s = 0; s < nstages; ++s) {
    const int b = (unsigned)s % ST;
    const int zs = P * s + pw;
    const int zi = zs - 1;
    const int rz = gz * Mz + zi;  // volume z of this stored plane
    // 1: interior data plane, 2: shell plane taken from the block, 0: background
    const int mode = (zi >= 0 && zi < cz) ? 1
                     : (prefill && zs < Sz && rz >= 0 && rz < Z && rz - oz >= 0 && rz - oz < dz) ? 2
                                                                                               : 0;
    const uint16_t* iplane = reinterpret_cast<const uint16_t*>(s_in + (size_t)b * in_bytes) +
                             (size_t)pw * RS * brow;
    uint32_t* oplane = reinterpret_cast<uint32_t*>(brick + (size_t)zs * plane_elems);
    // every thread waits, so the slot's phase is complete before it is re-armed
    mbar_wait(&s_bar[b], (uint32_t)(s / ST) & 1u);
    if (zs < Sz) {
      if (mode != 0 && xfull) {
        // the common case: stored sample e of a row <-> staged sample xoff+e
        // of the same row (rows outside the volume: background)
        if (wact) {
          const uint32_t* iw = reinterpret_cast<const uint32_t*>(iplane) + xo;
          const int qs = brow >> 1;
          if (wpr <= NT && yfull) {
            // one word per row per thread, every stored row inside the
            // volume: a flat loop of load(s), permute, store with running
            // 32-bit offsets (the parity of the row start is per brick)
            uint32_t* o = oplane + wr0 + rr * wpr;
            const uint32_t* q = iw + rr * qs;
            if (MX && MY) {
              // constant strides: rows rr, rr + R, ... (the last pass may
              // hold one row fewer for some threads)
              constexpr int kWpr = (MX + 2) * C / 2, kQs = ((MX + 2) * C + 14) / 8 * 8 / 2;
              constexpr int kR = kWpr <= NT ? NT / kWpr : 1, kN = (MY + 2 + kR - 1) / kR;
              const int nrow = (Sy - rr + kR - 1) / kR;
              if (xoff & 1) {
#pragma unroll
                for (int t = 0; t < kN; ++t)
                  if (t < nrow) o[t * kR * kWpr] = __byte_perm(q[t * kR * kQs], q[t * kR * kQs + 1], 0x5432);
              } else {
#pragma unroll
                for (int t = 0; t < kN; ++t)
                  if (t < nrow) o[t * kR * kWpr] = q[t * kR * kQs];
              }
            } else {
              int oo = 0, qo = 0;
              const int ostep = R * wpr, qstep = R * qs;
              if (xoff & 1) {
#pragma unroll 4
                for (int ys = rr; ys < Sy; ys += R, oo += ostep, qo += qstep)
                  o[oo] = __byte_perm(q[qo], q[qo + 1], 0x5432);
              } else {
#pragma unroll 4
                for (int ys = rr; ys < Sy; ys += R, oo += ostep, qo += qstep) o[oo] = q[qo];
              }
            }
          } else if (wpr <= NT) {
            // one word per row per thread: a flat, unrollable row loop
            uint32_t* o = oplane + wr0;
            const bool odd = xoff & 1;
#pragma unroll 4
            for (int ys = rr; ys < Sy; ys += R) {
              const uint32_t* q = iw + ys * qs;
              const uint32_t out = odd ? __byte_perm(q[0], q[1], 0x5432) : q[0];
              o[ys * wpr] = (unsigned)(y0 + ys) < (unsigned)Y ? out : bgw;
            }
          } else {
            for (int ys = rr; ys < Sy; ys += R) {
              const bool rin = (unsigned)(y0 + ys) < (unsigned)Y;
              const uint32_t* q = iw + ys * qs;
              uint32_t* o = oplane + ys * wpr + wr0;
              for (int w = 0; w < wpr - wr0; w += wstep) {
                const uint32_t out = (xoff & 1) ? __byte_perm(q[w], q[w + 1], 0x5432) : q[w];
                o[w] = rin ? out : bgw;
              }
            }
          }
        }
      } else if (mode == 0) {
        if (wact)
          for (int ys = rr; ys < Sy; ys += R)
            for (int w = wr0; w < wpr; w += wstep) oplane[ys * wpr + w] = bgw;
      } else {
        // bricks on the volume's x boundary, or shells not prefilled
        uint16_t* o16 = reinterpret_cast<uint16_t*>(oplane);
        for (int e = pt; e < (int)plane_elems; e += NT) {
          const int ys = (int)__umulhi((uint32_t)e, rowmagic);
          const int es = e - ys * Sx * C;
          const int xs = C == 1 ? es : (int)__umulhi((uint32_t)es, cmagic);
          const int rx = x0 + xs, ry = y0 + ys;
          const bool take = prefill ? (rx >= 0 && rx < X && ry >= 0 && ry < Y)
                                    : (mode == 1 && xs >= 1 && xs <= cx && ys >= 1 && ys <= cy);
          o16[e] = take ? iplane[(size_t)ys * brow + xoff + es] : bg;
        }
      }
      if (mode == 1 && !parent) {
        // interior statistics of an unfused leaf: voxel v of the interior plane
        for (int v = pt; v < cx * cy; v += NT) {
          const int y = (int)__umulhi((uint32_t)v, cxmagic);
          const int x = v - y * cx;
          const uint16_t* iv = iplane + (size_t)(y + 1) * brow + xoff + (x + 1) * C;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int val = iv[c];
            lmn[c] = min(lmn[c], val);
            lmx[c] = max(lmx[c], val);
            lsm[c] += (unsigned)val;
          }
        }
      }
    }
    // fused octant plane k = s - 1 from interior planes 2k (previous stage,
    // second plane) and 2k + 1 (this stage, first plane)
    if (parent && s >= 1 && 2 * (s - 1) < cz) {
      const int k = s - 1;
      const uint16_t* pa = reinterpret_cast<const uint16_t*>(
                               s_in + (size_t)((unsigned)(s - 1) % ST) * in_bytes) +
                           (size_t)RS * brow;  // previous stage, plane 1
      const uint16_t* pb = reinterpret_cast<const uint16_t*>(s_in + (size_t)b * in_bytes);
      const bool zfull = 2 * k + 1 < cz;
      const bool pin = offz + k < pcz;
      for (int v = tid; v < hx * hy; v += kTmaWarps * 32) {
        // the first pass (all of it for 32x32 leaves) uses the hoisted split
        const int oy = v == tid ? toy : v / hx, ox = v - oy * hx;
        int val[C];
        if (zfull && 2 * ox + 1 < cx && 2 * oy + 1 < cy) {
          const int o00 = (1 + 2 * oy) * brow + xoff + (1 + 2 * ox) * C;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int a0 = pa[o00 + c], a1 = pa[o00 + C + c], a2 = pa[o00 + brow + c],
                      a3 = pa[o00 + brow + C + c], b0 = pb[o00 + c], b1 = pb[o00 + C + c],
                      b2 = pb[o00 + brow + c], b3 = pb[o00 + brow + C + c];
            const unsigned sum = (unsigned)(a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3);
            val[c] = (int)((2 * sum + 8) / 16);
            lmn[c] = min(lmn[c], min(min(min(a0, a1), min(a2, a3)), min(min(b0, b1), min(b2, b3))));
            lmx[c] = max(lmx[c], max(max(max(a0, a1), max(a2, a3)), max(max(b0, b1), max(b2, b3))));
            lsm[c] += sum;
          }
        } else {
          // partial leaf: mean over its in-volume voxels, background if none
          unsigned sum[C];
#pragma unroll
          for (int c = 0; c < C; ++c) sum[c] = 0;
          int cnt = 0;
          for (int dz = 0; dz < 2; ++dz) {
            if (2 * k + dz >= cz) continue;
            const uint16_t* pl = dz ? pb : pa;
            for (int dy = 0; dy < 2; ++dy) {
              if (2 * oy + dy >= cy) continue;
              for (int dx = 0; dx < 2; ++dx) {
                if (2 * ox + dx >= cx) continue;
                const int o = (1 + 2 * oy + dy) * brow + xoff + (1 + 2 * ox + dx) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                  const int x = pl[o + c];
                  sum[c] += x;
                  lmn[c] = min(lmn[c], x);
                  lmx[c] = max(lmx[c], x);
                }
                ++cnt;
              }
            }
          }
#pragma unroll
          for (int c = 0; c < C; ++c) {
            lsm[c] += sum[c];
            val[c] = cnt ? (int)((2 * (unsigned long long)sum[c] + cnt) / (2 * cnt)) : (int)bg;
          }
        }
        uint16_t* dst = parent + g.voxel_offset(1 + offz + k, 1 + offy + oy, 1 + offx + ox);
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c] = (uint16_t)val[c];
        if (pin && offx + ox < pcx && offy + oy < pcy) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            omn[c] = min(omn[c], val[c]);
            omx[c] = max(omx[c], val[c]);
            osm[c] += (unsigned)val[c];
          }
        }
      }
      if (pxy) {
        // x-face voxel of parent row 1 + offy + v
        const int lx = (gx & 1) ? Mx : -2;         // child-local raw x of the footprint
        const int dxs = (gx & 1) ? Mx + 1 : 0;     // stored x of the shell
        for (int v = tid; v < hy; v += kTmaWarps * 32) {
          const int ly = 2 * v, dys = 1 + offy + v;
          unsigned sum[C];
#pragma unroll
          for (int c = 0; c < C; ++c) sum[c] = 0;
          int cnt = 0;
          for (int dz2 = 0; dz2 < 2; ++dz2) {
            if (2 * k + dz2 >= cz) continue;
            const uint16_t* pl = dz2 ? pb : pa;
#pragma unroll
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll
              for (int dx = 0; dx < 2; ++dx) {
                const int o = (1 + ly + dy) * brow + xoff + (1 + lx + dx) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) sum[c] += pl[o + c];
                ++cnt;
              }
          }
          uint16_t* dst = parent + g.voxel_offset(1 + offz + k, dys, dxs);
#pragma unroll
          for (int c = 0; c < C; ++c)
            dst[c] = (uint16_t)(cnt ? (2 * (unsigned long long)sum[c] + cnt) / (2 * cnt) : bg);
        }
      }
    }
    __syncthreads();  // input slots consumed
    // the previous stage's slot is free now: refill it (ST - 1) stages ahead
    if (tid == 0 && s + (ST - 1) < nstages) issue(s + (ST - 1));
  }

  // CTA totals: warp shuffles, then one thread per channel
#pragma unroll
  for (int c = 0; c < C; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lmn[c] = min(lmn[c], __shfl_xor_sync(0xffffffffu, lmn[c], o));
      lmx[c] = max(lmx[c], __shfl_xor_sync(0xffffffffu, lmx[c], o));
      lsm[c] += __shfl_xor_sync(0xffffffffu, lsm[c], o);
      omn[c] = min(omn[c], __shfl_xor_sync(0xffffffffu, omn[c], o));
      omx[c] = max(omx[c], __shfl_xor_sync(0xffffffffu, omx[c], o));
      osm[c] += __shfl_xor_sync(0xffffffffu, osm[c], o);
    }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      s_mn[0][warp][c] = lmn[c];
      s_mx[0][warp][c] = lmx[c];
      s_sm[0][warp][c] = lsm[c];
      s_mn[1][warp][c] = omn[c];
      s_mx[1][warp][c] = omx[c];
      s_sm[1][warp][c] = osm[c];
    }
  __syncthreads();
  if (tid < C) {
    const int c = tid;
    int a = INT_MAX, bmx = INT_MIN, pa = INT_MAX, pb = INT_MIN;
    unsigned long long t = 0, pt2 = 0;
    for (int w = 0; w < kTmaWarps; ++w) {
      a = min(a, s_mn[0][w][c]);
      bmx = max(bmx, s_mx[0][w][c]);
      t += s_sm[0][w][c];
      pa = min(pa, s_mn[1][w][c]);
      pb = max(pb, s_mx[1][w][c]);
      pt2 += s_sm[1][w][c];
    }
    const long long n = (long long)cx * cy * cz;
    stats[st_index(j.node, ST_AVG, c)] = (int)((2 * (long long)t + n) / (2 * n));
    stats[st_index(j.node, ST_MIN, c)] = a;
    stats[st_index(j.node, ST_MAX, c)] = bmx;
    stats[st_index(j.node, ST_SUBMIN, c)] = a;
    stats[st_index(j.node, ST_SUBMAX, c)] = bmx;
    if (parent && pb != INT_MIN) {
      const int64_t pnode = (j.node - 1) >> 3;
      atomicMin(nmin + pnode * C + c, pa);
      atomicMax(nmax + pnode * C + c, pb);
      atomicAdd(nsum + pnode * C + c, pt2);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-staged leaves from a PLANAR source (16-bit samples)
// ---------------------------------------------------------------------------
// The layer of a slice stream arrives channel by channel (ingest_stream's
// VSTR order: per z one single-channel frame per channel), so its natural
// device layout is planar: sample (x, y, z, c) at
// base + c*cstride + (z - oz)*zstride + (y*X + x)*2 bytes.  The TMA engine
// streams one 4-D tensor tile per stage — P stored planes x (My+2) rows x
// the aligned row span, for every channel — into [C][P][Sy][bx] shared
// memory, and the warps interleave channels on the way out: thread v of a
// plane group owns stored voxel v of the plane (consecutive lanes read
// consecutive x of a channel row: no bank conflicts), loads its C samples
// and writes them as 32-bit words of the channel-fastest stored row; for odd
// C an even voxel completes its last word with the next voxel's first sample
// (one shuffle, the pair is always in the same warp since rows are even).
// The stored brick, statistics and fused parent octant are exactly those of
// k_dense_leaf_tma (same shells, prefill rules and rounding); only the
// source layout differs.  Reference: _write_leaf + _ensure_brick +
// _recompute_stats (octree.py:225-263, 420-442), halfsample_block
// (octree.py:58-92), _update_parent_octant (octree.py:308-319).
constexpr int kPStages = 3;  // planar ring: building, previous (fused octant), one in flight
constexpr int kPAhead = 2;
__host__ __device__ inline int tma_box_row_planar(int mx) { return (mx + 2 + 7 + 7) / 8 * 8; }
__host__ __device__ inline uint32_t tma_in_bytes_planar(int mx, int my, int C) {
  return ((uint32_t)C * kTmaP * (my + 2) * tma_box_row_planar(mx) * 2 + 127) / 128 * 128;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            int c, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_addr(b))
      : "memory");
}

template <int C, int MX = 0, int MY = 0>
__global__ void __launch_bounds__(kTmaWarps * 32) k_dense_leaf_tma_planar(
    const __grid_constant__ CUtensorMap map, int oz, int dz, int prefill,
    const DenseJob* __restrict__ jobs, int gnx, int gny, int g0z, Geo g,
    uint16_t* __restrict__ pool, int32_t* stats, int32_t* nmin, int32_t* nmax,
    unsigned long long* nsum, uint16_t* __restrict__ bmax_sub, uint16_t* __restrict__ bmax_brick,
    int nsb, uint8_t* __restrict__ dflags, int32_t* __restrict__ dslot, int pshell) {
  constexpr int P = kTmaP;
  constexpr int WPP = kTmaWarps / P;  // warps per plane
  constexpr int NT = WPP * 32;        // threads per plane
  extern __shared__ __align__(128) unsigned char s_in[];
  __shared__ uint64_t s_bar[kPStages];
  __shared__ int s_mn[2][kTmaWarps][C], s_mx[2][kTmaWarps][C];
  __shared__ unsigned long long s_sm[2][kTmaWarps][C];
  const DenseJob j = jobs[blockIdx.x];
  const int gx = (int)(blockIdx.x % gnx);
  const int gy = (int)((blockIdx.x / gnx) % gny);
  const int gz = g0z + (int)(blockIdx.x / (gnx * gny));
  const int Mx = MX ? MX : g.brick[0], My = MY ? MY : g.brick[1], Mz = g.brick[2];
  const int Sx = MX ? MX + 2 : Mx + 2, Sy = MY ? MY + 2 : My + 2, Sz = g.stored[2];
  const int X = g.dims[0], Y = g.dims[1], Z = g.dims[2];
  const int cx = min(Mx, X - gx * Mx), cy = min(My, Y - gy * My), cz = min(Mz, Z - gz * Mz);
  const int bx = tma_box_row_planar(Mx);             // staged row (samples, one channel)
  const int RS = Sy;  // staged rows per plane
  const int rows = P * RS;                           // staged rows per channel
  const uint32_t in_bytes = tma_in_bytes_planar(Mx, My, C);
  const uint32_t plane_elems = (uint32_t)Sx * Sy * C;
  const int nvox = Sx * Sy;                          // stored voxels per plane
  const int nstages = Sz / P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint16_t* brick = pool + (int64_t)j.slot * g.brick_elems;
  const uint16_t bg = (uint16_t)g.bg;
  const int x0 = gx * Mx - 1, y0 = gy * My - 1;  // block voxel of stored (0, 0)
  const int xa = x0 - ((x0 % 8 + 8) % 8);        // 16-byte aligned tile start (samples)
  const int xoff = x0 - xa;                      // leading samples of a staged row (odd)
  // every stored voxel of a block plane inside the volume (prefilled shells)
  // (with a zero background the TMA tile's zero fill outside the volume IS
  // the background, so bricks on the volume's x/y faces take this path too)
  const bool xyfull =
      prefill && (bg == 0 || (x0 >= 0 && x0 + Sx <= X && y0 >= 0 && y0 + Sy <= Y));

  if (tid == 0) {
    for (int b = 0; b < kPStages; ++b) mbar_init(&s_bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (dflags) {  // structure mirror of this in-volume leaf (held pairs)
      dflags[j.node] = NF_EXISTS | NF_INVOL | NF_BRICK;
      dslot[j.node] = j.slot;
    }
  }
  __syncthreads();

  auto issue = [&](int s) {  // one thread: one 4-D tensor tile per stage
    const int b = s % kPStages;
    mbar_expect_tx(&s_bar[b], (uint32_t)C * rows * bx * 2);
    tma_load_4d(s_in + (size_t)b * in_bytes, &map, xa, y0, gz * Mz - oz + P * s - 1, 0, &s_bar[b]);
  };
  if (tid == 0)
    for (int s = 0; s < min(kPAhead, nstages); ++s) issue(s);

  const int pslot = j.pad;
  const int hx = Mx / 2, hy = My / 2;
  const int offx = (gx & 1) * hx, offy = (gy & 1) * hy, offz = (gz & 1) * (Mz / 2);
  int pcx, pcy, pcz;  // the parent's in-volume extent (octree.py:190-199)
  {
    const int plx = (gx >> 1) * 2 * Mx, ply = (gy >> 1) * 2 * My, plz = (gz >> 1) * 2 * Mz;
    pcx = min(Mx, max(0, (X - plx + 1) / 2));
    pcy = min(My, max(0, (Y - ply + 1) / 2));
    pcz = min(Mz, max(0, (Z - plz + 1) / 2));
  }
  uint16_t* parent = pslot >= 0 ? pool + (int64_t)pslot * g.brick_elems : nullptr;
  // interior level-1 parent (its x/y neighbour parents' footprints lie in
  // the volume): this child also writes the parent's x-face shell rows on
  // its side — the neighbour parent's edge voxels, half-sampled from the two
  // raw voxels beyond the child's edge that the staged x halo holds (the
  // strided x faces are k_borders' costly segments; it skips them)
  const bool pxy = parent && pshell && (gx >> 1) >= 1 && (gy >> 1) >= 1 &&
                   ((gx >> 1) + 1) * 2 * Mx + 2 <= X && ((gy >> 1) + 1) * 2 * My + 2 <= Y;

  int lmn[C], lmx[C], omn[C], omx[C];
  unsigned long long lsm[C], osm[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    lmn[c] = omn[c] = INT_MAX;
    lmx[c] = omx[c] = INT_MIN;
    lsm[c] = osm[c] = 0;
  }
  const int pw = warp / WPP;                // plane of the stage this warp group builds
  const int cstr = rows * bx;               // staged channel stride (samples)

  for (int s = 0; s < nstages; ++s) {
    const int b = (unsigned)s % kPStages;
    const int zs = P * s + pw;
    const int zi = zs - 1;
    const int rz = gz * Mz + zi;
    const int mode = (zi >= 0 && zi < cz) ? 1
                     : (prefill && zs < Sz && rz >= 0 && rz < Z && rz - oz >= 0 && rz - oz < dz) ? 2
                                                                                               : 0;
    const uint16_t* stage = reinterpret_cast<const uint16_t*>(s_in + (size_t)b * in_bytes);
    const uint16_t* iplane = stage + (size_t)pw * RS * bx + xoff;  // channel 0, stored (0, 0)
    uint32_t* oplane = reinterpret_cast<uint32_t*>(brick + (size_t)zs * plane_elems);
    mbar_wait(&s_bar[b], (uint32_t)(s / kPStages) & 1u);
    if (zs < Sz && mode != 0 && xyfull) {
      // the common case: every stored voxel of the plane comes from the
      // block.  Thread q builds voxel pair (2q, 2q + 1) of the plane (Sx is
      // even): per channel two aligned 32-bit shared loads and a byte
      // permute give both voxels (the staged row starts at an odd xoff, so
      // stored x = 2k - 1 sits at an even sample), then the pair's C words
      // of the channel-fastest stored row are assembled and stored.
      const bool stat_plane = mode == 1 && !parent;
      const uint32_t* s32 =
          reinterpret_cast<const uint32_t*>(stage) + (pw * RS * bx + xoff - 1) / 2;
      const int pt = (warp % WPP) * 32 + lane;
      const int SP = Sx / 2;  // voxel pairs per stored row
      auto pair = [&](int ys, int xs, const uint32_t* w, uint32_t* o) {
        uint32_t pv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) pv[c] = __byte_perm(w[c * cstr / 2], w[c * cstr / 2 + 1], 0x5432);
        if (stat_plane) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int x = xs + h;
            if (x >= 1 && x <= cx && ys >= 1 && ys <= cy) {
#pragma unroll
              for (int c = 0; c < C; ++c) {
                const int v = (int)((pv[c] >> (16 * h)) & 0xFFFFu);
                lmn[c] = min(lmn[c], v);
                lmx[c] = max(lmx[c], v);
                lsm[c] += (unsigned)v;
              }
            }
          }
        }
        if (C == 3) {
          // (v0c0 | v0c1), (v0c2 | v1c0), (v1c1 | v1c2): one byte permute each
          o[0] = __byte_perm(pv[0], pv[1 % C], 0x5410);
          o[1] = __byte_perm(pv[2 % C], pv[0], 0x7610);
          o[2] = __byte_perm(pv[1 % C], pv[2 % C], 0x7632);
        } else {
#pragma unroll
          for (int j2 = 0; j2 < C; ++j2) {
            // samples 2 j2 and 2 j2 + 1 of the pair: voxel k / C, channel k % C
            const int k0 = 2 * j2, k1 = 2 * j2 + 1;
            const uint32_t a0 = k0 / C ? (pv[k0 % C] >> 16) : (pv[k0 % C] & 0xFFFFu);
            const uint32_t a1 = k1 / C ? (pv[k1 % C] >> 16) : (pv[k1 % C] & 0xFFFFu);
            o[j2] = a0 | (a1 << 16);
          }
        }
      };
      // Each thread owns one pair column xp of rows y0, y0 + RSTEP, ...
      // (RSTEP = NT / SP rows per pass: 7 x 17 of the 128 threads for 32^3
      // bricks), so the per-pair index arithmetic reduces to two pointer
      // increments; the staged row stride bx is even
      const int RSTEP = NT / SP;
      if (RSTEP > 0) {
        if (pt < RSTEP * SP) {
          const int y0 = pt / SP, xp = pt - y0 * SP;
          const uint32_t* w = s32 + y0 * (bx / 2) + xp;
          uint32_t* o = oplane + (size_t)(y0 * SP + xp) * C;
          for (int ys = y0; ys < Sy; ys += RSTEP, w += RSTEP * (bx / 2), o += RSTEP * SP * C)
            pair(ys, 2 * xp, w, o);
        }
      } else {
        for (int q = pt; q < Sy * SP; q += NT) {
          const int ys = q / SP, xs = 2 * (q - ys * SP);
          pair(ys, xs, s32 + (ys * bx + xs) / 2, oplane + (size_t)q * C);
        }
      }
    } else if (zs < Sz && mode == 0) {
      // a shell plane outside the volume or the insertion: background words
      const uint32_t bgw = (uint32_t)bg | ((uint32_t)bg << 16);
      const int words = (int)(plane_elems / 2);
      for (int w = (warp % WPP) * 32 + lane; w < words; w += NT) oplane[w] = bgw;
    } else if (zs < Sz) {
      const bool stat_plane = mode == 1 && !parent;
      // every lane runs the same trip count (shuffles below)
      for (int v0 = (warp % WPP) * 32; v0 < nvox; v0 += NT) {
        const int v = v0 + lane;
        const bool act = v < nvox;
        const int ys = v / Sx, xs = v - ys * Sx;
        const int rx = x0 + xs, ry = y0 + ys;
        const bool take = act && mode != 0 &&
                          (prefill ? ((unsigned)rx < (unsigned)X && (unsigned)ry < (unsigned)Y)
                                   : (xs >= 1 && xs <= cx && ys >= 1 && ys <= cy));
        uint32_t val[C];
        const uint16_t* q = iplane + ys * bx + xs;
#pragma unroll
        for (int c = 0; c < C; ++c) val[c] = take ? (uint32_t)q[c * cstr] : (uint32_t)bg;
        if (stat_plane && xs >= 1 && xs <= cx && ys >= 1 && ys <= cy && act) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            lmn[c] = min(lmn[c], (int)val[c]);
            lmx[c] = max(lmx[c], (int)val[c]);
            lsm[c] += val[c];
          }
        }
        if ((C & 1) == 0) {
          if (act) {
            uint32_t* o = oplane + (size_t)v * (C / 2);
#pragma unroll
            for (int w = 0; w < C / 2; ++w) o[w] = val[2 * w] | (val[2 * w + 1] << 16);
          }
        } else {
          const uint32_t nb = __shfl_down_sync(0xffffffffu, val[0], 1);
          if (act) {
            const uint32_t e = (uint32_t)v * C;  // first sample of this voxel
            if ((v & 1) == 0) {
              // even voxel: its samples start a word; the last pairs with nb
#pragma unroll
              for (int w = 0; w < C / 2; ++w) oplane[e / 2 + w] = val[2 * w] | (val[2 * w + 1] << 16);
              oplane[e / 2 + C / 2] = val[C - 1] | (nb << 16);
            } else {
              // odd voxel: sample 0 completed the previous voxel's word
#pragma unroll
              for (int w = 0; w < C / 2; ++w)
                oplane[(e + 1) / 2 + w] = val[2 * w + 1] | (val[2 * w + 2] << 16);
            }
          }
        }
      }
    }
    // fused octant plane k = s - 1 from interior planes 2k (previous stage,
    // second plane) and 2k + 1 (this stage, first plane)
    if (parent && s >= 1 && 2 * (s - 1) < cz) {
      const int k = s - 1;
      const uint16_t* pa = reinterpret_cast<const uint16_t*>(
                               s_in + (size_t)((unsigned)(s - 1) % kPStages) * in_bytes) +
                           (size_t)RS * bx + xoff;  // previous stage, plane 1
      const uint16_t* pb = stage + xoff;             // this stage, plane 0
      const bool zfull = 2 * k + 1 < cz;
      const bool pin = offz + k < pcz;
      for (int v = tid; v < hx * hy; v += kTmaWarps * 32) {
        const int oy = v / hx, ox = v - oy * hx;
        int val[C];
        if (zfull && 2 * ox + 1 < cx && 2 * oy + 1 < cy) {
          const int o00 = (1 + 2 * oy) * bx + 1 + 2 * ox;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int oc = o00 + c * cstr;
            const int a0 = pa[oc], a1 = pa[oc + 1], a2 = pa[oc + bx], a3 = pa[oc + bx + 1];
            const int b0 = pb[oc], b1 = pb[oc + 1], b2 = pb[oc + bx], b3 = pb[oc + bx + 1];
            const unsigned sum = (unsigned)(a0 + a1 + a2 + a3 + b0 + b1 + b2 + b3);
            val[c] = (int)((2 * sum + 8) / 16);
            lmn[c] = min(lmn[c], min(min(min(a0, a1), min(a2, a3)), min(min(b0, b1), min(b2, b3))));
            lmx[c] = max(lmx[c], max(max(max(a0, a1), max(a2, a3)), max(max(b0, b1), max(b2, b3))));
            lsm[c] += sum;
          }
        } else {
          unsigned sum[C];
#pragma unroll
          for (int c = 0; c < C; ++c) sum[c] = 0;
          int cnt = 0;
          for (int dz2 = 0; dz2 < 2; ++dz2) {
            if (2 * k + dz2 >= cz) continue;
            const uint16_t* pl = dz2 ? pb : pa;
            for (int dy = 0; dy < 2; ++dy) {
              if (2 * oy + dy >= cy) continue;
              for (int dx = 0; dx < 2; ++dx) {
                if (2 * ox + dx >= cx) continue;
                const int o = (1 + 2 * oy + dy) * bx + 1 + 2 * ox + dx;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                  const int x = pl[o + c * cstr];
                  sum[c] += x;
                  lmn[c] = min(lmn[c], x);
                  lmx[c] = max(lmx[c], x);
                }
                ++cnt;
              }
            }
          }
#pragma unroll
          for (int c = 0; c < C; ++c) {
            lsm[c] += sum[c];
            val[c] = cnt ? (int)((2 * (unsigned long long)sum[c] + cnt) / (2 * cnt)) : (int)bg;
          }
        }
        uint16_t* dst = parent + g.voxel_offset(1 + offz + k, 1 + offy + oy, 1 + offx + ox);
#pragma unroll
        for (int c = 0; c < C; ++c) dst[c] = (uint16_t)val[c];
        if (pin && offx + ox < pcx && offy + oy < pcy) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            omn[c] = min(omn[c], val[c]);
            omx[c] = max(omx[c], val[c]);
            osm[c] += (unsigned)val[c];
          }
        }
      }
      if (pxy) {
        // x-face voxel of parent row 1 + offy + v
        const int lx = (gx & 1) ? Mx : -2;         // child-local raw x of the footprint
        const int dxs = (gx & 1) ? Mx + 1 : 0;     // stored x of the shell
        for (int v = tid; v < hy; v += kTmaWarps * 32) {
          const int ly = 2 * v, dys = 1 + offy + v;
          unsigned sum[C];
#pragma unroll
          for (int c = 0; c < C; ++c) sum[c] = 0;
          int cnt = 0;
          for (int dz2 = 0; dz2 < 2; ++dz2) {
            if (2 * k + dz2 >= cz) continue;
            const uint16_t* pl = dz2 ? pb : pa;
#pragma unroll
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll
              for (int dx = 0; dx < 2; ++dx) {
                const int o = (1 + ly + dy) * bx + 1 + lx + dx;
#pragma unroll
                for (int c = 0; c < C; ++c) sum[c] += pl[o + c * cstr];
                ++cnt;
              }
          }
          uint16_t* dst = parent + g.voxel_offset(1 + offz + k, dys, dxs);
#pragma unroll
          for (int c = 0; c < C; ++c)
            dst[c] = (uint16_t)(cnt ? (2 * (unsigned long long)sum[c] + cnt) / (2 * cnt) : bg);
        }
      }
    }
    __syncthreads();  // input slots consumed
    if (tid == 0 && s + kPAhead < nstages) issue(s + kPAhead);
  }

#pragma unroll
  for (int c = 0; c < C; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lmn[c] = min(lmn[c], __shfl_xor_sync(0xffffffffu, lmn[c], o));
      lmx[c] = max(lmx[c], __shfl_xor_sync(0xffffffffu, lmx[c], o));
      lsm[c] += __shfl_xor_sync(0xffffffffu, lsm[c], o);
      omn[c] = min(omn[c], __shfl_xor_sync(0xffffffffu, omn[c], o));
      omx[c] = max(omx[c], __shfl_xor_sync(0xffffffffu, omx[c], o));
      osm[c] += __shfl_xor_sync(0xffffffffu, osm[c], o);
    }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      s_mn[0][warp][c] = lmn[c];
      s_mx[0][warp][c] = lmx[c];
      s_sm[0][warp][c] = lsm[c];
      s_mn[1][warp][c] = omn[c];
      s_mx[1][warp][c] = omx[c];
      s_sm[1][warp][c] = osm[c];
    }
  __syncthreads();
  if (tid < C) {
    const int c = tid;
    int a = INT_MAX, bmx = INT_MIN, pa = INT_MAX, pb = INT_MIN;
    unsigned long long t = 0, pt2 = 0;
    for (int w = 0; w < kTmaWarps; ++w) {
      a = min(a, s_mn[0][w][c]);
      bmx = max(bmx, s_mx[0][w][c]);
      t += s_sm[0][w][c];
      pa = min(pa, s_mn[1][w][c]);
      pb = max(pb, s_mx[1][w][c]);
      pt2 += s_sm[1][w][c];
    }
    const long long n = (long long)cx * cy * cz;
    stats[st_index(j.node, ST_AVG, c)] = (int)((2 * (long long)t + n) / (2 * n));
    stats[st_index(j.node, ST_MIN, c)] = a;
    stats[st_index(j.node, ST_MAX, c)] = bmx;
    stats[st_index(j.node, ST_SUBMIN, c)] = a;
    stats[st_index(j.node, ST_SUBMAX, c)] = bmx;
    // brick maxima for the empty-space skip: before fill_borders a sample's
    // trilinear weights on shell voxels are exactly 0 (the sampler clamps to
    // interior centres, render/raycast.py:141-144), so the interior maximum
    // (background for interior voxels outside the volume) bounds it;
    // fill_borders re-derives every brick's maxima with its shells
    if (bmax_brick) bmax_brick[(int64_t)j.slot * kMaxC + c] = (uint16_t)max(bmx, (int)bg);
    if (parent && pb != INT_MIN) {
      const int64_t pnode = (j.node - 1) >> 3;
      atomicMin(nmin + pnode * C + c, pa);
      atomicMax(nmax + pnode * C + c, pb);
      atomicAdd(nsum + pnode * C + c, pt2);
    }
  }
  if (bmax_brick) {
    if (tid >= C && tid < kMaxC) bmax_brick[(int64_t)j.slot * kMaxC + tid] = 0;
    // sub-brick maxima unknown: never skip at sub-brick granularity
    for (int i = tid; i < nsb * kMaxC; i += kTmaWarps * 32)
      bmax_sub[(int64_t)j.slot * nsb * kMaxC + i] = 0xFFFFu;
  }
}

// ---------------------------------------------------------------------------
// parents
// ---------------------------------------------------------------------------
// One CTA per parent; warps own interior planes, lanes the voxels of a row.
// Every interior voxel is the half-sample of its child octant (counts over
// the child's in-volume voxels, background where none, octree.py:83-92); an
// out-of-volume child contributes background (its AVG is the background and
// it covers no in-volume parent voxel, octree.py:296-306).
template <class T, int C>
__global__ void __launch_bounds__(256) k_dense_level(const int64_t* __restrict__ nodes, Geo g,
                                                     T* pool, const int32_t* __restrict__ slots,
                                                     const uint8_t* __restrict__ flags,
                                                     int32_t* pmin, int32_t* pmax,
                                                     unsigned long long* psum, int32_t* stats,
                                                     int zsplit) {
  // zsplit > 1 (small levels): CTA part p of a node builds interior planes
  // [p*Mz/zsplit, (p+1)*Mz/zsplit); the statistics come from a k_reduce pass
  const int64_t node = nodes[blockIdx.x / zsplit];
  const int part = blockIdx.x % zsplit;
  const int level = g.level_of(node);
  const int Mx = g.brick[0], My = g.brick[1], Mz = g.brick[2];
  __shared__ int s_cslot[8];
  __shared__ int s_cext[8][3];
  __shared__ int s_pext[3];
  __shared__ int s_pslot;
  if (threadIdx.x < 8) {
    const int k = threadIdx.x;
    int sl = -1, ce[3] = {0, 0, 0};
    if (g.octant_real(k)) {
      const int64_t ch = 8 * node + 1 + k;
      if ((flags[ch] & NF_EXISTS) && (flags[ch] & NF_BRICK)) sl = slots[ch];
      int lo[3];
      g.box_lo(ch, lo);
      g.in_extent(lo, level - 1, ce);
    }
    s_cslot[k] = sl;
    for (int a = 0; a < 3; ++a) s_cext[k][a] = ce[a];
  } else if (threadIdx.x == 8) {
    int lo[3], ce[3];
    g.box_lo(node, lo);
    g.in_extent(lo, level, ce);
    for (int a = 0; a < 3; ++a) s_pext[a] = ce[a];
    s_pslot = slots[node];
  }
  __syncthreads();
  const int kx = g.split[0] ? 2 : 1, ky = g.split[1] ? 2 : 1, kz = g.split[2] ? 2 : 1;
  const int hx = Mx / kx, hy = My / ky, hz = Mz / kz;  // octant extents
  const int pcx = s_pext[0], pcy = s_pext[1], pcz = s_pext[2];
  T* parent = pool + (int64_t)s_pslot * g.brick_elems;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Acc<C> tot;
  tot.init();
  const int64_t rs = (int64_t)g.stored[0] * C, ps = rs * g.stored[1];  // row / plane stride
  // value of parent interior voxel (x, y, z): loads only, no stores, so the
  // two rows of an iteration keep all their gathers in flight together
  struct Vox {
    int v[C];
  };
  auto voxel = [&](int x, int y, int z) -> Vox {
    Vox r;
    int* v = r.v;
    // coordinates are below 2 * half-extent: the octant bit is a compare
    const int bz = z >= hz ? 1 : 0, oz = z - bz * hz;
    const int by = y >= hy ? 1 : 0, oy = y - by * hy;
    const int bx = x >= hx ? 1 : 0, ox = x - bx * hx;
    const int k = bx | (by << 1) | (bz << 2);
    const int cs = s_cslot[k];
    if (cs < 0) {
#pragma unroll
      for (int c = 0; c < C; ++c) v[c] = g.bg;
      return r;
    }
    const T* child = pool + (int64_t)cs * g.brick_elems;
    const int ex = s_cext[k][0], ey = s_cext[k][1], ez = s_cext[k][2];
    if (kx == 2 && ky == 2 && kz == 2 && 2 * ox + 1 < ex && 2 * oy + 1 < ey && 2 * oz + 1 < ez) {
      // full 2x2x2 block: 8 voxels = 4 runs of 2*C contiguous samples
      const T* q = child + g.voxel_offset(1 + 2 * oz, 1 + 2 * oy, 1 + 2 * ox);
      unsigned sum[C];
#pragma unroll
      for (int c = 0; c < C; ++c)
        sum[c] = (unsigned)__ldg(q + c) + __ldg(q + C + c) + __ldg(q + rs + c) +
                 __ldg(q + rs + C + c) + __ldg(q + ps + c) + __ldg(q + ps + C + c) +
                 __ldg(q + ps + rs + c) + __ldg(q + ps + rs + C + c);
#pragma unroll
      for (int c = 0; c < C; ++c) v[c] = (int)((2 * sum[c] + 8) / 16);
      return r;
    }
    long long sum[C];
#pragma unroll
    for (int c = 0; c < C; ++c) sum[c] = 0;
    int cnt = 0;
    for (int dz = 0; dz < kz; ++dz) {
      const int sz = kz * oz + dz;
      if (sz >= ez) continue;
      for (int dy = 0; dy < ky; ++dy) {
        const int sy = ky * oy + dy;
        if (sy >= ey) continue;
        const T* row = child + g.voxel_offset(1 + sz, 1 + sy, 1);
        for (int dx = 0; dx < kx; ++dx) {
          const int sx = kx * ox + dx;
          if (sx >= ex) continue;
#pragma unroll
          for (int c = 0; c < C; ++c) sum[c] += __ldg(row + sx * C + c);
          ++cnt;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = cnt ? (int)((2 * sum[c] + cnt) / (2 * cnt)) : g.bg;
    return r;
  };
  const int zb0 = part * Mz / zsplit, zb1 = (part + 1) * Mz / zsplit;
  // fewer planes than warps (small levels split finely): wpp warps share a
  // plane, each taking every wpp-th group of rows; their plane partials are
  // combined in shared memory before the first of them emits the plane
  const int nplanes = zb1 - zb0;
  const int wpp = nplanes >= nw ? 1 : nw / nplanes;
  const int pz = warp / wpp, wy = warp % wpp, ppass = nw / wpp;
  __shared__ int s_pmn[kMaxWarps][C], s_pmx[kMaxWarps][C];
  __shared__ unsigned long long s_psm[kMaxWarps][C];
  const int zend = zb0 + (nplanes + ppass - 1) / ppass * ppass;  // uniform trip count
  for (int z = zb0 + pz; z < zend; z += ppass) {
    Acc<C> pl;
    pl.init();
    // kRows rows per iteration: their gathers are all in flight together
    // (the small top levels are latency bound: few CTAs, a serial row chain)
    constexpr int kRows = 4;
    for (int y = wy * kRows; y < My && z < zb1; y += kRows * wpp) {
      for (int x = lane; x < Mx; x += 32) {
        Vox vv[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (y + r < My) vv[r] = voxel(x, y + r, z);
        T* dst = parent + g.voxel_offset(1 + z, 1 + y, 1 + x);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
          if (y + r >= My) continue;
#pragma unroll
          for (int c = 0; c < C; ++c) dst[r * rs + c] = (T)vv[r].v[c];
          if (x < pcx && y + r < pcy && z < pcz) pl.add_all(vv[r].v);
        }
      }
    }
    if (wpp > 1) {
      pl.warp_reduce();
      if (lane == 0)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          s_pmn[warp][c] = pl.mn[c];
          s_pmx[warp][c] = pl.mx[c];
          s_psm[warp][c] = pl.sm[c];
        }
      __syncthreads();
      pl.init();
      if (wy == 0 && lane == 0)
        for (int w = warp; w < warp + wpp; ++w)
#pragma unroll
          for (int c = 0; c < C; ++c) {
            pl.mn[c] = min(pl.mn[c], s_pmn[w][c]);
            pl.mx[c] = max(pl.mx[c], s_pmx[w][c]);
            pl.sm[c] += s_psm[w][c];
          }
      __syncthreads();
    }
    if (wy == 0 && z < zb1 && z < pcz && pcx > 0 && pcy > 0)
      emit_plane<C>(pl, tot, s_pslot, Mz, z, pmin, pmax, psum);
  }
  finish_stats<C>(tot, node, (int64_t)pcx * pcy * pcz, false, g, flags, stats);
}

// fill_borders' z-shell fix-up for prefilled leaves (Tree::fill_borders):
// job = (dst slot, dst stored plane, src slot, src stored plane); a stored
// plane is contiguous, so this is a straight 32-bit word copy
__global__ void k_plane_copy(const int32_t* __restrict__ jobs, int n, int64_t brick_words,
                             int plane_words, uint32_t* pool) {
  const int32_t* j = jobs + 4 * blockIdx.x;
  uint32_t* dst = pool + (int64_t)j[0] * brick_words + (int64_t)j[1] * plane_words;
  const uint32_t* src = pool + (int64_t)j[2] * brick_words + (int64_t)j[3] * plane_words;
  for (int i = threadIdx.x; i < plane_words; i += blockDim.x) dst[i] = src[i];
}

// fused level-1 parents: min / max / sum accumulators (nmin, nmax, nsum)
__global__ void k_init_fused(const int64_t* __restrict__ nodes, int n, int C, int32_t* nmin,
                             int32_t* nmax, unsigned long long* nsum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * C) return;
  const int64_t node = nodes[i / C];
  const int c = i % C;
  nmin[node * C + c] = INT_MAX;
  nmax[node * C + c] = INT_MIN;
  nsum[node * C + c] = 0;
}

// fused level-1 parents after their leaves: AVG = round_mean(sum, n)
// (octree.py:53-55) and the subtree extrema (octree.py:265-277)
__global__ void k_finish_fused(const int64_t* __restrict__ nodes, int n, Geo g,
                               const uint8_t* __restrict__ flags, int32_t* stats,
                               const int32_t* __restrict__ nmin, const int32_t* __restrict__ nmax,
                               const unsigned long long* __restrict__ nsum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * g.C) return;
  const int64_t node = nodes[i / g.C];
  const int c = i % g.C;
  int lo[3], ce[3];
  g.box_lo(node, lo);
  g.in_extent(lo, 1, ce);
  const long long cnt = (long long)ce[0] * ce[1] * ce[2];
  stats[st_index(node, ST_AVG, c)] = (int)((2 * (long long)nsum[node * g.C + c] + cnt) / (2 * cnt));
  stats[st_index(node, ST_MIN, c)] = nmin[node * g.C + c];
  stats[st_index(node, ST_MAX, c)] = nmax[node * g.C + c];
  bool any = false;
  int a = 0, b = 0;
  for (int k = 0; k < 8; ++k) {
    if (!g.octant_real(k)) continue;
    const int64_t ch = 8 * node + 1 + k;
    if (!(flags[ch] & NF_EXISTS) || !(flags[ch] & NF_INVOL)) continue;
    const int x = stats[st_index(ch, ST_SUBMIN, c)], y = stats[st_index(ch, ST_SUBMAX, c)];
    a = any ? min(a, x) : x;
    b = any ? max(b, y) : y;
    any = true;
  }
  if (any) {
    stats[st_index(node, ST_SUBMIN, c)] = a;
    stats[st_index(node, ST_SUBMAX, c)] = b;
  }
}

// every shell voxel of a brick <- background (publishing prefilled shells as
// the reference's pre-fill_borders state, Tree::publish_halos)
template <class T>
__global__ void k_clear_shells(const int32_t* __restrict__ slots, Geo g, T* pool) {
  T* b = pool + (int64_t)slots[blockIdx.x] * g.brick_elems;
  const int Sx = g.stored[0], Sy = g.stored[1], Sz = g.stored[2], C = g.C;
  const int n = Sx * Sy * Sz;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    const int x = v % Sx, y = (v / Sx) % Sy, z = v / (Sx * Sy);
    if (x == 0 || y == 0 || z == 0 || x == Sx - 1 || y == Sy - 1 || z == Sz - 1)
      for (int c = 0; c < C; ++c) b[(int64_t)v * C + c] = (T)g.bg;
  }
}

int planes_per_warp(int sz) { return (sz + 11) / 12; }  // <= 12 warps per CTA

}  // namespace

#define VT_CHECK_LAUNCH() VT_CUDA(cudaGetLastError())

// TMA tensor tiles need a 16-byte aligned block and row pitch, a box row of
// at most 256 samples, and the rings must fit in shared memory
static size_t tma_smem(const Geo& g, int stages = kTmaStages) {
  return (size_t)stages * tma_in_bytes(g.brick[0], g.brick[1], g.C);
}
// ring depth of the interleaved leaf kernel: 4 stages, 3 when 4 do not fit
static int tma_stages(const Geo& g) { return tma_smem(g) <= 200 * 1024 ? kTmaStages : 3; }
static bool tma_ok(const Tree& t, const void* src) {
  if (std::getenv("VT_DENSE_TMA") && std::getenv("VT_DENSE_TMA")[0] == '0') return false;
  const int64_t stride = (int64_t)t.g.dims[0] * t.g.C * 2;
  return t.g.sb == 2 && ((uintptr_t)src & 15) == 0 && stride % 16 == 0 &&
         tma_box_row(t.g.brick[0], t.g.C) <= 256 && t.g.brick[1] + 2 <= 256 &&
         tma_smem(t.g, tma_stages(t.g)) <= 200 * 1024;
}

// 3-D tensor map of a (dz, Y, X*C) u16 block for the TMA unit, box = one
// stage of stored planes with their halo; the encoder comes from the driver
// through the runtime (no libcuda link)
static bool encode_block_map(const Tree& t, const void* src, int64_t dz, CUtensorMap* map) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = (Encode)fn;
    cudaGetLastError();
  }
  if (!enc) return false;
  const int C = t.g.C;
  const int64_t row = (int64_t)t.g.dims[0] * C;
  cuuint64_t dims[3] = {(cuuint64_t)row, (cuuint64_t)t.g.dims[1], (cuuint64_t)dz};
  cuuint64_t strides[2] = {(cuuint64_t)row * 2, (cuuint64_t)row * 2 * t.g.dims[1]};
  cuuint32_t box[3] = {(cuuint32_t)tma_box_row(t.g.brick[0], C), (cuuint32_t)(t.g.brick[1] + 2),
                       (cuuint32_t)kTmaP};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(src), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns kLeafPrefilled | kLeafTma as applicable
template <class T, int C>
static int leaf_launch(const Tree& t, const void* src, int64_t nsrc, int oz, int prefill,
                        const DenseJob* jobs, int n, const int gn[3], int g0z) {
  const int sz = t.g.stored[2];
  const int rowlen = t.g.stored[0] * C;
  const int wpl = (rowlen / 2 + 31) / 32;
  const int64_t dz = nsrc / ((int64_t)t.g.dims[0] * t.g.dims[1] * C);
  CUtensorMap map;
  if (sizeof(T) == 2 && tma_ok(t, src) && encode_block_map(t, src, dz, &map)) {
    const int st = tma_stages(t.g);
    const size_t smem = tma_smem(t.g, st);
    auto k = t.g.brick[0] == 32 && t.g.brick[1] == 32 ? k_dense_leaf_tma<C, 32, 32>
             : st == kTmaStages                       ? k_dense_leaf_tma<C>
                                                      : k_dense_leaf_tma<C, 0, 0, 3>;
    VT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int ps = t.parent_shells_next && prefill ? 1 : 0;
    k<<<n, kTmaWarps * 32, smem, t.stream>>>(map, oz, (int)dz, prefill, jobs, gn[0], gn[1], g0z,
                                            t.g, (uint16_t*)t.d_pool, t.d_stats, t.d_nmin,
                                            t.d_nmax, t.d_nsum, ps);
    VT_CHECK_LAUNCH();
    return kLeafTma | (prefill ? kLeafPrefilled : 0) | (ps ? kLeafParentShells : 0);
  }
  if (sizeof(T) == 2 && rowlen % 2 == 0 && wpl <= 4) {
    // warps own ceil(Sz / 17) planes each (<= 17 warps)
    const int ppw = (sz + 16) / 17;
    const int warps = (sz + ppw - 1) / ppw;
    auto* p = (const uint16_t*)src;
    auto* pool = (uint16_t*)t.d_pool;
#define VT_LEAF16(W)                                                                      \
  k_dense_leaf16<C, W><<<n, 32 * warps, 0, t.stream>>>(p, oz, jobs, gn[0], gn[1], g0z, t.g, \
                                                       pool, t.d_pmin, t.d_pmax, t.d_psum, \
                                                       t.d_stats, t.d_flags, ppw, nsrc)
    switch (wpl) {
      case 1: VT_LEAF16(1); break;
      case 2: VT_LEAF16(2); break;
      case 3: VT_LEAF16(3); break;
      default: VT_LEAF16(4); break;
    }
#undef VT_LEAF16
    VT_CHECK_LAUNCH();
    return 0;
  }
  const int ppw = planes_per_warp(sz);
  const int warps = (sz + ppw - 1) / ppw;
  k_dense_leaf<T, C><<<n, 32 * warps, 0, t.stream>>>(
      (const T*)src, oz, jobs, gn[0], gn[1], g0z, t.g, (T*)t.d_pool, t.d_pmin, t.d_pmax, t.d_psum,
      t.d_stats, t.d_flags, ppw);
  VT_CHECK_LAUNCH();
  return 0;
}

template <class T>
static int leaf_dispatch(const Tree& t, const void* src, int64_t nsrc, int oz, int prefill,
                          const DenseJob* jobs, int n, const int gn[3], int g0z) {
  switch (t.g.C) {
    case 1: return leaf_launch<T, 1>(t, src, nsrc, oz, prefill, jobs, n, gn, g0z);
    case 2: return leaf_launch<T, 2>(t, src, nsrc, oz, prefill, jobs, n, gn, g0z);
    case 3: return leaf_launch<T, 3>(t, src, nsrc, oz, prefill, jobs, n, gn, g0z);
    default: return leaf_launch<T, 4>(t, src, nsrc, oz, prefill, jobs, n, gn, g0z);
  }
}

void launch_plane_copy(const Tree& t, const int32_t* d_jobs, int n) {
  if (n <= 0) return;
  const int64_t bw = t.g.brick_elems * t.g.sb / 4;
  const int pw = t.g.stored[0] * t.g.stored[1] * t.g.C * t.g.sb / 4;
  k_plane_copy<<<n, 256, 0, t.stream>>>(d_jobs, n, bw, pw, (uint32_t*)t.d_pool);
  VT_CHECK_LAUNCH();
}

template <class T>
__global__ void k_interleave(const T* __restrict__ src, int64_t n, int C, int c, T* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i * C + c] = src[i];
}

void launch_interleave(const Tree& t, const void* src, int64_t n, int c, void* dst) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  if (t.g.sb == 1)
    k_interleave<uint8_t><<<grid, 256, 0, t.stream>>>((const uint8_t*)src, n, t.g.C, c,
                                                       (uint8_t*)dst);
  else
    k_interleave<uint16_t><<<grid, 256, 0, t.stream>>>((const uint16_t*)src, n, t.g.C, c,
                                                        (uint16_t*)dst);
  VT_CHECK_LAUNCH();
}

void launch_init_fused(const Tree& t, const int64_t* d_nodes, int n) {
  if (n <= 0) return;
  const int work = n * t.g.C;
  k_init_fused<<<(work + 255) / 256, 256, 0, t.stream>>>(d_nodes, n, t.g.C, t.d_nmin, t.d_nmax,
                                                        t.d_nsum);
  VT_CHECK_LAUNCH();
}

void launch_finish_fused(const Tree& t, const int64_t* d_nodes, int n) {
  if (n <= 0) return;
  const int work = n * t.g.C;
  k_finish_fused<<<(work + 255) / 256, 256, 0, t.stream>>>(d_nodes, n, t.g, t.d_flags, t.d_stats,
                                                          t.d_nmin, t.d_nmax, t.d_nsum);
  VT_CHECK_LAUNCH();
}

void launch_clear_shells(const Tree& t, const int32_t* d_slots, int n) {
  if (n <= 0) return;
  if (t.g.sb == 1)
    k_clear_shells<uint8_t><<<n, 256, 0, t.stream>>>(d_slots, t.g, t.d_pool);
  else
    k_clear_shells<uint16_t><<<n, 256, 0, t.stream>>>(d_slots, t.g, (uint16_t*)t.d_pool);
  VT_CHECK_LAUNCH();
}

static size_t tma_smem_planar(const Geo& g) {
  return (size_t)kPStages * tma_in_bytes_planar(g.brick[0], g.brick[1], g.C);
}

bool planar_leaf_ok(const Tree& t, const void* base, int64_t zstride, int64_t cstride) {
  if (std::getenv("VT_DENSE_TMA") && std::getenv("VT_DENSE_TMA")[0] == '0') return false;
  const Geo& g = t.g;
  return g.sb == 2 && ((uintptr_t)base & 15) == 0 && ((int64_t)g.dims[0] * 2) % 16 == 0 &&
         zstride > 0 && zstride % 16 == 0 && (g.C == 1 || (cstride > 0 && cstride % 16 == 0)) &&
         tma_box_row_planar(g.brick[0]) <= 256 && g.brick[1] + 2 <= 256 &&
         g.brick[0] % 2 == 0 && tma_smem_planar(g) <= 200 * 1024;
}

// 4-D tensor map (x, y, z, c) of a planar u16 block of dz planes per channel
static bool encode_planar_map(const Tree& t, const void* base, int64_t zstride, int64_t cstride,
                              int64_t dz, CUtensorMap* map) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = (Encode)fn;
    cudaGetLastError();
  }
  if (!enc) return false;
  const Geo& g = t.g;
  cuuint64_t dims[4] = {(cuuint64_t)g.dims[0], (cuuint64_t)g.dims[1], (cuuint64_t)dz,
                        (cuuint64_t)g.C};
  cuuint64_t strides[3] = {(cuuint64_t)g.dims[0] * 2, (cuuint64_t)zstride,
                           (cuuint64_t)(g.C == 1 ? zstride * dz : cstride)};
  cuuint32_t box[4] = {(cuuint32_t)tma_box_row_planar(g.brick[0]), (cuuint32_t)(g.brick[1] + 2),
                       (cuuint32_t)kTmaP, (cuuint32_t)g.C};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C>
static int leaf_launch_planar(const Tree& t, const void* base, int64_t zstride, int64_t cstride,
                              int oz, int64_t dz, int prefill, const DenseJob* jobs, int n,
                              const int gn[3], int g0z, bool write_struct, bool pshell) {
  CUtensorMap map;
  if (!encode_planar_map(t, base, zstride, cstride, dz, &map)) return -1;
  const size_t smem = tma_smem_planar(t.g);
  auto k = t.g.brick[0] == 32 && t.g.brick[1] == 32 ? k_dense_leaf_tma_planar<C, 32, 32>
                                                    : k_dense_leaf_tma_planar<C>;
  VT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  uint16_t* bb = t.bmax_brick();
  k<<<n, kTmaWarps * 32, smem, t.stream>>>(map, oz, (int)dz, prefill, jobs, gn[0], gn[1], g0z, t.g,
                                          (uint16_t*)t.d_pool, t.d_stats, t.d_nmin, t.d_nmax,
                                          t.d_nsum, t.d_bmax, bb, t.bmax_nsb,
                                          write_struct ? t.d_flags : nullptr,
                                          write_struct ? t.d_slot : nullptr,
                                          (pshell && prefill) ? 1 : 0);
  VT_CHECK_LAUNCH();
  return kLeafTma | (prefill ? kLeafPrefilled : 0) | (bb ? kLeafBmax : 0) |
         ((pshell && prefill) ? kLeafParentShells : 0);
}

int launch_dense_leaf_planar(const Tree& t, const void* base, int64_t zstride, int64_t cstride,
                             int oz, int64_t dz, int prefill, const DenseJob* jobs, int n,
                             const int gn[3], int g0z, bool ws, bool ps) {
  if (n <= 0) return 0;
  if (!planar_leaf_ok(t, base, zstride, cstride)) return -1;
  switch (t.g.C) {
    case 1: return leaf_launch_planar<1>(t, base, zstride, cstride, oz, dz, prefill, jobs, n, gn, g0z, ws, ps);
    case 2: return leaf_launch_planar<2>(t, base, zstride, cstride, oz, dz, prefill, jobs, n, gn, g0z, ws, ps);
    case 3: return leaf_launch_planar<3>(t, base, zstride, cstride, oz, dz, prefill, jobs, n, gn, g0z, ws, ps);
    default: return leaf_launch_planar<4>(t, base, zstride, cstride, oz, dz, prefill, jobs, n, gn, g0z, ws, ps);
  }
}

// planar (c, z, y, x) block -> interleaved (z, y, x, c) (fallback for the
// kernels that read interleaved blocks)
template <class T>
__global__ void k_planar_to_interleaved(const unsigned char* __restrict__ base, int64_t zstride,
                                        int64_t cstride, int64_t plane, int dz, int C, T* dst) {
  const int64_t n = plane * dz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i / plane, r = i - z * plane;
    for (int c = 0; c < C; ++c)
      dst[i * C + c] = *reinterpret_cast<const T*>(base + c * cstride + z * zstride + r * sizeof(T));
  }
}

void launch_planar_to_interleaved(const Tree& t, const void* base, int64_t zstride,
                                  int64_t cstride, int dz, void* dst) {
  const int64_t plane = (int64_t)t.g.dims[0] * t.g.dims[1];
  const int64_t n = plane * dz;
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
  if (t.g.sb == 1)
    k_planar_to_interleaved<uint8_t><<<grid, 256, 0, t.stream>>>(
        (const unsigned char*)base, zstride, cstride, plane, dz, t.g.C, (uint8_t*)dst);
  else
    k_planar_to_interleaved<uint16_t><<<grid, 256, 0, t.stream>>>(
        (const unsigned char*)base, zstride, cstride, plane, dz, t.g.C, (uint16_t*)dst);
  VT_CHECK_LAUNCH();
}

template <class T>
__global__ void k_fill_value(T* dst, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

void launch_fill_bg(const Tree& t, void* dst, int64_t n) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (t.g.sb == 1)
    k_fill_value<uint8_t><<<grid, 256, 0, t.stream>>>((uint8_t*)dst, n, (uint8_t)t.g.bg);
  else
    k_fill_value<uint16_t><<<grid, 256, 0, t.stream>>>((uint16_t*)dst, n, (uint16_t)t.g.bg);
  VT_CHECK_LAUNCH();
}

// background into planes base + idx[k] * plane (samples), one launch for
// up to kMaxFillPlanes planes: 16-byte stores, grid.y = plane
struct FillPlanes {
  int32_t idx[kMaxFillPlanes];
};
__global__ void k_fill_planes(uint8_t* base, int64_t plane_bytes, FillPlanes fp, uint32_t word) {
  uint4* dst = reinterpret_cast<uint4*>(base + (int64_t)fp.idx[blockIdx.y] * plane_bytes);
  const int64_t n = plane_bytes / 16;
  const uint4 v = make_uint4(word, word, word, word);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

void launch_fill_planes(const Tree& t, void* base, int64_t plane, const int32_t* idx, int n) {
  const int64_t pb = plane * t.g.sb;
  if (pb % 16 != 0 || ((uintptr_t)base & 15) != 0) {
    for (int k = 0; k < n; ++k) launch_fill_bg(t, (uint8_t*)base + (int64_t)idx[k] * pb, plane);
    return;
  }
  const uint32_t bg = (uint32_t)t.g.bg;
  const uint32_t word = t.g.sb == 1 ? bg * 0x01010101u : (bg | (bg << 16));
  for (int k0 = 0; k0 < n; k0 += kMaxFillPlanes) {
    FillPlanes fp{};
    const int m = std::min(kMaxFillPlanes, n - k0);
    for (int k = 0; k < m; ++k) fp.idx[k] = idx[k0 + k];
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(pb / 16 / 256, 64));
    k_fill_planes<<<dim3(gx, m), 256, 0, t.stream>>>((uint8_t*)base, pb, fp, word);
    VT_CHECK_LAUNCH();
  }
}

int launch_dense_leaf(const Tree& t, const void* src, int64_t nsrc, int oz, int prefill,
                      const DenseJob* jobs, int n, const int gn[3], int g0z) {
  if (n <= 0) return 0;
  if (t.g.sb == 1) return leaf_dispatch<uint8_t>(t, src, nsrc, oz, 0, jobs, n, gn, g0z);
  return leaf_dispatch<uint16_t>(t, src, nsrc, oz, prefill, jobs, n, gn, g0z);
}

// Shared-memory variant for 16-bit pools, all axes split, every child a
// full in-volume brick (the bulk of every dense level): per parent interior
// plane z, the two child planes it half-samples from each of the 4
// children of that z-half (contiguous in the stored brick) are staged into
// shared memory with 16-byte cp.async copies — double buffered, so the next
// plane's copies overlap this plane's arithmetic — then every parent voxel
// is the 2x2x2 round_mean of 8 shared samples per channel.  Same values,
// plane partials and statistics as k_dense_level.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

inline int64_t level_s_span(const Geo& g) {
  const int64_t pair = 2LL * g.stored[0] * g.stored[1] * g.C * 2;
  return ((pair + 15) & ~15LL) + 16;
}
constexpr int64_t kLevelSmemMax = 112 * 1024;

template <int C>
__global__ void __launch_bounds__(256, 2) k_dense_level_s(
    const int64_t* __restrict__ nodes, Geo g, uint16_t* pool, const int32_t* __restrict__ slots,
    const uint8_t* __restrict__ flags, int32_t* pmin, int32_t* pmax, unsigned long long* psum,
    int32_t* stats, int zsplit, int span) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int64_t node = nodes[blockIdx.x / zsplit];
  const int part = blockIdx.x % zsplit;
  const int Mx = g.brick[0], My = g.brick[1], Mz = g.brick[2];
  const int hx = Mx / 2, hy = My / 2, hz = Mz / 2;
  const int Sx = g.stored[0], Sy = g.stored[1];
  const int64_t plane_elems = (int64_t)Sx * Sy * C;
  const int64_t pair_bytes = 2 * plane_elems * 2;
  __shared__ const uint16_t* s_child[8];
  __shared__ int s_pslot;
  __shared__ int s_pmn[8][C], s_pmx[8][C];
  __shared__ unsigned long long s_psm[8][C];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid < 8) s_child[tid] = pool + (int64_t)slots[8 * node + 1 + tid] * g.brick_elems;
  if (tid == 8) s_pslot = slots[node];
  __syncthreads();
  uint16_t* parent = pool + (int64_t)s_pslot * g.brick_elems;
  const int zb0 = part * Mz / zsplit, zb1 = (part + 1) * Mz / zsplit;
  // copy the child plane pairs of parent plane z into buffer b
  auto issue = [&](int z, int b) {
    const int bz = z >= hz ? 1 : 0, oz = z - bz * hz;
    for (int q = 0; q < 4; ++q) {
      const uintptr_t src = (uintptr_t)(s_child[q | (bz << 2)] + (1 + 2 * oz) * plane_elems);
      const uintptr_t a0 = src & ~(uintptr_t)15, a1 = (src + pair_bytes + 15) & ~(uintptr_t)15;
      const int nvec = (int)((a1 - a0) / 16);
      unsigned char* dst = s_raw + (size_t)(b * 4 + q) * span;
      for (int i = tid; i < nvec; i += blockDim.x)
        cp_async16(dst + 16 * i, (const void*)(a0 + 16 * (uintptr_t)i));
    }
    cp_async_commit();
  };
  Acc<C> tot;
  tot.init();
  if (zb0 < zb1) issue(zb0, 0);
  for (int z = zb0; z < zb1; ++z) {
    const int b = (z - zb0) & 1;
    if (z + 1 < zb1) {
      issue(z + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int bz = z >= hz ? 1 : 0, oz = z - bz * hz;
    Acc<C> pl;
    pl.init();
    for (int v = tid; v < Mx * My; v += blockDim.x) {
      const int y = v / Mx, x = v - y * Mx;
      const int bx = x >= hx ? 1 : 0, by = y >= hy ? 1 : 0;
      const int ox = x - bx * hx, oy = y - by * hy;
      const int q = bx | (by << 1);
      const uintptr_t src = (uintptr_t)(s_child[q | (bz << 2)] + (1 + 2 * oz) * plane_elems);
      const uint16_t* base =
          reinterpret_cast<const uint16_t*>(s_raw + (size_t)(b * 4 + q) * span + (src & 15));
      const uint16_t* p0 = base + ((1 + 2 * oy) * Sx + 1 + 2 * ox) * C;
      const uint16_t* p1 = p0 + plane_elems;
      int val[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const unsigned sum = (unsigned)p0[c] + p0[C + c] + p0[Sx * C + c] + p0[Sx * C + C + c] +
                             p1[c] + p1[C + c] + p1[Sx * C + c] + p1[Sx * C + C + c];
        val[c] = (int)((2 * sum + 8) / 16);
      }
      uint16_t* dst = parent + g.voxel_offset(1 + z, 1 + y, 1 + x);
#pragma unroll
      for (int c = 0; c < C; ++c) dst[c] = (uint16_t)val[c];
      pl.add_all(val);
    }
    pl.warp_reduce();
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        s_pmn[warp][c] = pl.mn[c];
        s_pmx[warp][c] = pl.mx[c];
        s_psm[warp][c] = pl.sm[c];
      }
    __syncthreads();  // plane partials visible; buffer b free for reuse
    if (tid == 0) {
      Acc<C> a;
      a.init();
      for (int w = 0; w < nw; ++w)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          a.mn[c] = min(a.mn[c], s_pmn[w][c]);
          a.mx[c] = max(a.mx[c], s_pmx[w][c]);
          a.sm[c] += s_psm[w][c];
        }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int64_t off = ((int64_t)s_pslot * Mz + z) * C + c;
        pmin[off] = a.mn[c];
        pmax[off] = a.mx[c];
        psum[off] = a.sm[c];
      }
      tot.merge(a);
    }
  }
  finish_stats<C>(tot, node, (int64_t)Mx * My * Mz, false, g, flags, stats);
}

template <class T, int C>
static void level_launch_s(const Tree& t, const int64_t* nodes, int n, int zsplit) {
  const int span = (int)level_s_span(t.g);
  const int smem = 8 * span;
  static bool attr = false;
  if (!attr) {
    VT_CUDA(cudaFuncSetAttribute(k_dense_level_s<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kLevelSmemMax));
    attr = true;
  }
  k_dense_level_s<C><<<n * zsplit, 256, smem, t.stream>>>(
      nodes, t.g, (uint16_t*)t.d_pool, t.d_slot, t.d_flags, t.d_pmin, t.d_pmax, t.d_psum,
      t.d_stats, zsplit, span);
  VT_CHECK_LAUNCH();
}

template <class T, int C>
static void level_launch(const Tree& t, const int64_t* nodes, int n, int zsplit) {
  const int warps = std::min(8, std::max(1, t.g.brick[2]));
  k_dense_level<T, C><<<n * zsplit, 32 * warps, 0, t.stream>>>(
      nodes, t.g, (T*)t.d_pool, t.d_slot, t.d_flags, t.d_pmin, t.d_pmax, t.d_psum, t.d_stats,
      zsplit);
  VT_CHECK_LAUNCH();
}

template <class T>
static void level_dispatch(const Tree& t, const int64_t* nodes, int n, int zs) {
  switch (t.g.C) {
    case 1: level_launch<T, 1>(t, nodes, n, zs); break;
    case 2: level_launch<T, 2>(t, nodes, n, zs); break;
    case 3: level_launch<T, 3>(t, nodes, n, zs); break;
    default: level_launch<T, 4>(t, nodes, n, zs); break;
  }
}

int dense_level_split(const Tree& t, int n) {
  // few parents: split each over CTAs of fewer planes (down to one plane per
  // CTA, its warps sharing the rows) so the level is not the latency of a
  // single CTA walking a whole brick
  static const int target = [] {
    const char* e = std::getenv("VT_LEVEL_CTAS");
    return e ? std::max(1, atoi(e)) : 2 * 148;
  }();
  const int mz = t.g.brick[2];
  int k = 1;
  while (k * 2 <= mz && (int64_t)n * k * 2 <= target) k *= 2;
  return k;
}

// the shared-memory level kernel applies: 16-bit samples, all axes split,
// even brick edges, the staged plane pairs fit
bool level_smem_ok(const Tree& t) {
  static const bool off = [] {
    const char* e = std::getenv("VT_LEVEL_SMEM");
    return e && e[0] == '0';
  }();
  const Geo& g = t.g;
  return !off && g.sb == 2 && g.split[0] && g.split[1] && g.split[2] && g.brick[0] % 2 == 0 &&
         g.brick[1] % 2 == 0 && g.brick[2] % 2 == 0 && 8 * level_s_span(g) <= kLevelSmemMax;
}

void launch_dense_level(const Tree& t, const int64_t* nodes, int n, int zsplit, bool smem) {
  if (n <= 0) return;
  if (smem && level_smem_ok(t)) {
    switch (t.g.C) {
      case 1: level_launch_s<uint16_t, 1>(t, nodes, n, zsplit); break;
      case 2: level_launch_s<uint16_t, 2>(t, nodes, n, zsplit); break;
      case 3: level_launch_s<uint16_t, 3>(t, nodes, n, zsplit); break;
      default: level_launch_s<uint16_t, 4>(t, nodes, n, zsplit); break;
    }
    return;
  }
  if (t.g.sb == 1)
    level_dispatch<uint8_t>(t, nodes, n, zsplit);
  else
    level_dispatch<uint16_t>(t, nodes, n, zsplit);
}

}  // namespace vtx
