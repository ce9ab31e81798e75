// Octree build kernels for sm_100a: node-structure mirror updates, child
// creation, brick seeding, block scatter into leaf bricks, per-plane brick
// statistics, 2x2x2 integer half-sampling, border fill and bulk gathers.
// All integer arithmetic reproduces voxtree bit-exactly:
//   means (2*sum + n) // (2n)     octree.py:53-55, 82, 91
//   homogeneity / extents         octree.py:95-99, 190-199
#include <algorithm>
#include <climits>

#include "tree.cuh"

namespace vtx {

namespace {

constexpr int kThreads = 256;


__global__ void k_struct_update(const StructUpd* __restrict__ u, int n, uint8_t* flags,
                                int32_t* slot) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    flags[u[i].node] = (uint8_t)u[i].flags;
    slot[u[i].node] = u[i].slot;
  }
}

// _ensure_children (octree.py:209-223): seed = parent AVG when in volume
__global__ void k_create(const CreateJob* __restrict__ jobs, int n, Geo g,
                         const uint8_t* __restrict__ flags, int32_t* stats) {
  int job = blockIdx.x;
  int t = threadIdx.x;
  if (job >= n || t >= 8 * g.C) return;
  int k = t / g.C, c = t % g.C;
  if (!g.octant_real(k)) return;
  int64_t child = 8 * jobs[job].parent + 1 + k;
  bool inv = flags[child] & NF_INVOL;
  if (inv && jobs[job].skip_z1 >= jobs[job].skip_z0 && g.level_of(child) == 0) {
    int lo[3];
    g.box_lo(child, lo);
    const int gz = lo[2] / g.brick[2];
    if (gz >= jobs[job].skip_z0 && gz <= jobs[job].skip_z1) return;
  }
  int v = inv ? stats[st_index(jobs[job].seed_src, ST_AVG, c)] : g.bg;
  stats[st_index(child, ST_AVG, c)] = v;
  stats[st_index(child, ST_MIN, c)] = v;
  stats[st_index(child, ST_MAX, c)] = v;
  stats[st_index(child, ST_SUBMIN, c)] = inv ? v : 0;
  stats[st_index(child, ST_SUBMAX, c)] = inv ? v : 0;
}

// _ensure_brick (octree.py:225-241): bg everywhere, node AVG on the
// in-volume interior — except the cover box, which later work of the same
// insertion overwrites with every channel.  One warp per stored row.
template <class T>
__global__ void k_seed(const SeedJob* __restrict__ jobs, int n, Geo g, T* pool,
                       const int32_t* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int C = g.C;
  const int sx = g.stored[0], sy = g.stored[1], sz = g.stored[2];
  const int rowlen = sx * C;
  // x = e / C by multiply-shift (e < 2^12, C <= 4)
  const uint32_t inv = (65536u + (uint32_t)C - 1) / (uint32_t)C;
  for (int job = blockIdx.x; job < n; job += gridDim.x) {
    const SeedJob j = jobs[job];
    T* b = pool + (int64_t)j.slot * g.brick_elems;
    T avg[kMaxC];
#pragma unroll
    for (int c = 0; c < kMaxC; ++c) avg[c] = c < C ? (T)stats[st_index(j.node, ST_AVG, c)] : (T)0;
    const T bg = (T)g.bg;
    auto val = [&](int x, int c, bool yz_in) {
      const bool in = yz_in && x >= 1 && x <= j.cext[0];
      T v = bg;
#pragma unroll
      for (int q = 0; q < kMaxC; ++q)
        if (in && q == c) v = avg[q];
      return v;
    };
    const bool cov = j.cov_hi[0] > j.cov_lo[0] && j.cov_hi[1] > j.cov_lo[1] &&
                     j.cov_hi[2] > j.cov_lo[2];
    if (cov && j.cov_lo[0] == 0 && j.cov_lo[1] == 0 && j.cov_lo[2] == 0 &&
        j.cov_hi[0] == g.brick[0] && j.cov_hi[1] == g.brick[1] && j.cov_hi[2] == g.brick[2]) {
      // the whole interior is rewritten later (fresh parent): the seed is the
      // background shell only — two full planes, two rows per inner plane,
      // two voxels per inner row, as flat coalesced runs
      const int plane = sx * sy * C, inner = sz - 2;
      const int n1 = 2 * plane, n2 = n1 + inner * 2 * rowlen, n3 = n2 + inner * (sy - 2) * 2 * C;
      for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < n3; e += blockDim.x * gridDim.y) {
        int64_t off;
        if (e < n1) {
          off = e < plane ? e : (int64_t)(sz - 1) * plane + (e - plane);
        } else if (e < n2) {
          const int r = (e - n1) / rowlen, q = (e - n1) - r * rowlen;
          off = (int64_t)(1 + r / 2) * plane + (int64_t)((r & 1) ? sy - 1 : 0) * rowlen + q;
        } else {
          const int r = (e - n2) / (2 * C), q = (e - n2) - r * 2 * C;
          const int z = 1 + r / (sy - 2), y = 1 + r % (sy - 2);
          off = (int64_t)z * plane + (int64_t)y * rowlen + (q < C ? q : (sx - 1) * C + (q - C));
        }
        b[off] = bg;
      }
      continue;
    }
    // rows outside the cover: whole rows, one warp each
    for (int row = (threadIdx.x >> 5) + blockIdx.y * (blockDim.x >> 5); row < sy * sz;
         row += (blockDim.x >> 5) * gridDim.y) {
      const int y = row % sy, z = row / sy;
      const bool yz_cov = cov && y >= 1 + j.cov_lo[1] && y < 1 + j.cov_hi[1] &&
                          z >= 1 + j.cov_lo[2] && z < 1 + j.cov_hi[2];
      if (yz_cov) continue;
      const bool yz_in = y >= 1 && y <= j.cext[1] && z >= 1 && z <= j.cext[2];
      T* dst = b + (int64_t)row * rowlen;
      for (int e = lane; e < rowlen; e += 32) {
        const int x = (int)(((uint32_t)e * inv) >> 16);
        dst[e] = val(x, e - x * C, yz_in);
      }
    }
    if (!cov) continue;
    // covered rows: only the x ends outside the cover, one thread per row
    const int cy = j.cov_hi[1] - j.cov_lo[1], cz = j.cov_hi[2] - j.cov_lo[2];
    for (int r = threadIdx.x; r < cy * cz; r += blockDim.x) {
      const int y = 1 + j.cov_lo[1] + r % cy, z = 1 + j.cov_lo[2] + r / cy;
      const bool yz_in = y <= j.cext[1] && z <= j.cext[2];
      T* dst = b + ((int64_t)z * sy + y) * rowlen;
      for (int x = 0; x < 1 + j.cov_lo[0]; ++x)
        for (int c = 0; c < C; ++c) dst[x * C + c] = val(x, c, yz_in);
      for (int x = 1 + j.cov_hi[0]; x < sx; ++x)
        for (int c = 0; c < C; ++c) dst[x * C + c] = val(x, c, yz_in);
    }
  }
}

// _write_leaf (octree.py:420-442): block (dz,dy,dx[,C]) -> leaf bricks at +1.
// One CTA per (brick column, block z): warps over rows, lanes over the
// contiguous samples of a row (coalesced on both sides).  When the block
// holds every channel and covers the brick's whole in-volume plane, the CTA
// also emits that plane's partial stats (_recompute_stats, octree.py:248-263)
// so the plane is never re-read.
__device__ __forceinline__ bool owns_stats(const Geo& g, int channel, int ox, int oy, int dx,
                                           int dy, int gx, int gy) {
  if (!(channel < 0 || g.C == 1)) return false;
  const int bx0 = gx * g.brick[0], by0 = gy * g.brick[1];
  const int ix1 = min(g.dims[0], bx0 + g.brick[0]), iy1 = min(g.dims[1], by0 + g.brick[1]);
  return ox <= bx0 && ox + dx >= ix1 && oy <= by0 && oy + dy >= iy1;
}

template <class T>
__global__ void __launch_bounds__(256) k_scatter(const T* __restrict__ src, int channel,
                                                 int src_stride, int src_off, int ox, int oy,
                                                 int oz, int zb, int dx, int dy, int g0x, int g0y,
                                                 int g0z, int gnx, int gny,
                                                 const int32_t* __restrict__ leaf_slots, Geo g,
                                                 T* pool, int32_t* pmin, int32_t* pmax,
                                                 unsigned long long* psum) {
  const int mx = g.brick[0], my = g.brick[1], mz = g.brick[2], C = g.C;
  const int gx = g0x + (int)(blockIdx.x % gnx), gy = g0y + (int)(blockIdx.x / gnx);
  const int Z = oz + zb + (int)blockIdx.y;
  const int gz = Z / mz, lz = Z - gz * mz;
  const int32_t s = leaf_slots[((int64_t)(gz - g0z) * gny + (gy - g0y)) * gnx + (gx - g0x)];
  const int X0 = max(ox, gx * mx), X1 = min(ox + dx, (gx + 1) * mx);
  const int Y0 = max(oy, gy * my), Y1 = min(oy + dy, (gy + 1) * my);
  const bool fused = channel < 0;
  T* brick = pool + (int64_t)s * g.brick_elems;
  const bool stats = owns_stats(g, channel, ox, oy, dx, dy, gx, gy);
  int mn[kMaxC], mxv[kMaxC];
  unsigned long long sm[kMaxC];
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) {
    mn[c] = INT_MAX;
    mxv[c] = INT_MIN;
    sm[c] = 0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t zrow = (int64_t)(Z - oz) * dy;
  const int nvox = X1 - X0;
  unsigned int sm32[kMaxC] = {0, 0, 0, 0};
  for (int y = Y0 + warp; y < Y1; y += nw) {
    const int64_t svox = (zrow + (y - oy)) * dx + (X0 - ox);
    T* drow = brick + g.voxel_offset(lz + 1, y - gy * my + 1, X0 - gx * mx + 1);
    if (fused) {
      // lane per voxel: its C samples are contiguous on both sides
      const T* srow = src + svox * C;
      for (int v = lane; v < nvox; v += 32) {
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) {
          if (c < C) {
            const T val = srow[v * C + c];
            drow[v * C + c] = val;
            mn[c] = min(mn[c], (int)val);
            mxv[c] = max(mxv[c], (int)val);
            sm32[c] += val;
          }
        }
      }
    } else {
      for (int v = lane; v < nvox; v += 32) {
        const T val = src[(svox + v) * src_stride + src_off];
        drow[(int64_t)v * C + channel] = val;
        mn[0] = min(mn[0], (int)val);
        mxv[0] = max(mxv[0], (int)val);
        sm32[0] += val;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) sm[c] = sm32[c];
  if (!stats) return;
  __shared__ int s_mn[8][kMaxC], s_mx[8][kMaxC];
  __shared__ unsigned long long s_sm[8][kMaxC];
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[c] = min(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mxv[c] = max(mxv[c], __shfl_xor_sync(0xffffffffu, mxv[c], o));
      sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], o);
    }
    if (lane == 0) {
      s_mn[warp][c] = mn[c];
      s_mx[warp][c] = mxv[c];
      s_sm[warp][c] = sm[c];
    }
  }
  __syncthreads();
  if (threadIdx.x < C) {
    const int c = threadIdx.x;
    int a = INT_MAX, b = INT_MIN;
    unsigned long long t = 0;
    for (int w = 0; w < nw; ++w) {
      a = min(a, s_mn[w][c]);
      b = max(b, s_mx[w][c]);
      t += s_sm[w][c];
    }
    const int64_t off = ((int64_t)s * mz + lz) * C + c;
    pmin[off] = a;
    pmax[off] = b;
    psum[off] = t;
  }
}

// per-plane partial statistics of the in-volume interior (feeds
// _recompute_stats, octree.py:248-263): one warp per plane of a brick job,
// one lane per voxel of a row, warp-shuffle reductions per channel
template <class T>
__global__ void __launch_bounds__(128) k_plane(const PlaneJob* __restrict__ jobs, int n, Geo g,
                                               const T* __restrict__ pool, int32_t* pmin,
                                               int32_t* pmax, unsigned long long* psum) {
  // one CTA per (job, plane): its 4 warps split the plane's rows, lanes the
  // voxels of a row; warp partials combine in shared memory.  Small
  // per-insertion launches (a slice at threshold > 0) are latency bound, so
  // every plane's rows are in flight at once rather than walked by one warp.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int C = g.C;
  const int64_t rowstride = (int64_t)g.stored[0] * C;
  __shared__ int s_mn[4][kMaxC], s_mx[4][kMaxC];
  __shared__ unsigned long long s_sm[4][kMaxC];
  for (int job = blockIdx.x; job < n; job += gridDim.x) {
    const PlaneJob j = jobs[job];
    for (int z = j.z0 + blockIdx.y; z < j.z1; z += gridDim.y) {
      const T* base = pool + (int64_t)j.slot * g.brick_elems + g.voxel_offset(z + 1, 1, 1);
      int mn[kMaxC], mx[kMaxC];
      unsigned long long sm[kMaxC];
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) {
        mn[c] = INT_MAX;
        mx[c] = INT_MIN;
        sm[c] = 0;
      }
#pragma unroll 4
      for (int y = warp; y < j.cy; y += nw) {
        const T* row = base + y * rowstride;
        for (int x = lane; x < j.cx; x += 32) {
#pragma unroll
          for (int c = 0; c < kMaxC; ++c) {
            if (c < C) {
              const int v = row[x * C + c];
              mn[c] = min(mn[c], v);
              mx[c] = max(mx[c], v);
              sm[c] += (unsigned)v;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) {
        if (c >= C) continue;
        for (int o = 16; o > 0; o >>= 1) {
          mn[c] = min(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
          mx[c] = max(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
          sm[c] += __shfl_xor_sync(0xffffffffu, sm[c], o);
        }
        if (lane == 0) {
          s_mn[warp][c] = mn[c];
          s_mx[warp][c] = mx[c];
          s_sm[warp][c] = sm[c];
        }
      }
      __syncthreads();
      if (threadIdx.x < C) {
        const int c = threadIdx.x;
        int a = INT_MAX, b = INT_MIN;
        unsigned long long t = 0;
        for (int w = 0; w < nw; ++w) {
          a = min(a, s_mn[w][c]);
          b = max(b, s_mx[w][c]);
          t += s_sm[w][c];
        }
        const int64_t off = ((int64_t)j.slot * g.brick[2] + z) * C + c;
        pmin[off] = a;
        pmax[off] = b;
        psum[off] = t;
      }
      __syncthreads();
    }
  }
}

// plane partials -> smin/smax/avg (round_mean), sub extrema for leaves and
// childless nodes, else _aggregate_subtree_extrema (octree.py:265-277)
__global__ void k_reduce(const ReduceJob* __restrict__ jobs, int n, Geo g,
                         const int32_t* __restrict__ pmin, const int32_t* __restrict__ pmax,
                         const unsigned long long* __restrict__ psum,
                         const uint8_t* __restrict__ flags, int32_t* stats) {
  // one warp per (node, channel): lanes take the plane partials and the
  // children's subtree extrema, warp shuffles combine them (tiny launches
  // per insertion at threshold > 0 are latency bound)
  const int lane = threadIdx.x & 31;
  const int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (i >= n * g.C) return;
  const ReduceJob j = jobs[i / g.C];
  const int c = i % g.C;
  const int cx = j.cext[0], cy = j.cext[1], cz = j.cext[2];
  if (cx > 0 && cy > 0 && cz > 0) {
    int mn = INT_MAX, mx = INT_MIN;
    unsigned long long s = 0;
    for (int z = lane; z < cz; z += 32) {
      const int64_t o = ((int64_t)j.slot * g.brick[2] + z) * g.C + c;
      mn = min(mn, pmin[o]);
      mx = max(mx, pmax[o]);
      s += psum[o];
    }
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) {
      const long long cnt = (long long)cx * cy * cz;
      const long long avg = (2 * (long long)s + cnt) / (2 * cnt);
      stats[st_index(j.node, ST_AVG, c)] = (int)avg;
      stats[st_index(j.node, ST_MIN, c)] = mn;
      stats[st_index(j.node, ST_MAX, c)] = mx;
      if (j.leafish) {
        stats[st_index(j.node, ST_SUBMIN, c)] = mn;
        stats[st_index(j.node, ST_SUBMAX, c)] = mx;
      }
    }
  }
  if (!j.leafish) {
    // lanes 0..7: the children's subtree extrema (existing, in volume)
    bool ok = false;
    int a = INT_MAX, b = INT_MIN;
    if (lane < 8 && g.octant_real(lane)) {
      const int64_t ch = 8 * j.node + 1 + lane;
      const uint8_t f = flags[ch];
      if ((f & NF_EXISTS) && (f & NF_INVOL)) {
        ok = true;
        a = stats[st_index(ch, ST_SUBMIN, c)];
        b = stats[st_index(ch, ST_SUBMAX, c)];
      }
    }
    const bool any = __any_sync(0xffffffffu, ok);
    for (int o = 4; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0 && any) {
      stats[st_index(j.node, ST_SUBMIN, c)] = a;
      stats[st_index(j.node, ST_SUBMAX, c)] = b;
    }
  }
}

// child contribution to its parent's octant: halfsample_block or AVG fill
// (octree.py:58-92, 281-319).  One CTA per job; a thread owns one output
// voxel (all channels) of a plane and walks the planes, so a warp reads
// 2 x 32 consecutive child voxels per (dz, dy) row — coalesced.
template <class T>
__global__ void __launch_bounds__(256) k_octant(const OctJob* __restrict__ jobs, int n, Geo g,
                                                T* pool, const int32_t* __restrict__ stats) {
  const int C = g.C;
  for (int job = blockIdx.x; job < n; job += gridDim.x) {
    const OctJob j = jobs[job];
    int kk[3], off[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      kk[a] = g.split[a] ? 2 : 1;
      off[a] = (((j.k >> a) & 1) && g.split[a]) ? g.brick[a] / 2 : 0;
    }
    const int wx = j.r1[0] - j.r0[0], wy = j.r1[1] - j.r0[1], wz = j.r1[2] - j.r0[2];
    T* parent = pool + (int64_t)j.pslot * g.brick_elems;
    const T* child = j.cslot >= 0 ? pool + (int64_t)j.cslot * g.brick_elems : nullptr;
    const int per_plane = wx * wy;
    int avgv[kMaxC];
    int lim[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) lim[a] = (j.cext[a] + kk[a] - 1) / kk[a];
    if (!child) {
#pragma unroll
      for (int c = 0; c < kMaxC; ++c) avgv[c] = c < C ? stats[st_index(j.child, ST_AVG, c)] : 0;
    }
    // fast path: the 2x2x2 (or 2x2 / 2) source block is fully in volume
    const bool full = child && j.cext[0] >= kk[0] * j.r1[0] && j.cext[1] >= kk[1] * j.r1[1] &&
                      j.cext[2] >= kk[2] * j.r1[2];
    const int n_out = kk[0] * kk[1] * kk[2];
#pragma unroll 2
    for (int e = threadIdx.x + blockIdx.y * blockDim.x; e < per_plane * wz;
         e += blockDim.x * gridDim.y) {
      const int oz = j.r0[2] + e / per_plane;
      const int rem = e - (e / per_plane) * per_plane;
      const int oy = j.r0[1] + rem / wx, ox = j.r0[0] + rem % wx;
      T* dst = parent + g.voxel_offset(1 + off[2] + oz, 1 + off[1] + oy, 1 + off[0] + ox);
      if (!child) {
        const bool in = ox < lim[0] && oy < lim[1] && oz < lim[2];
#pragma unroll
        for (int c = 0; c < kMaxC; ++c)
          if (c < C) dst[c] = (T)(in ? avgv[c] : g.bg);
        continue;
      }
      long long sum[kMaxC] = {0, 0, 0, 0};
      int cnt = 0;
      if (full) {
        for (int dz = 0; dz < kk[2]; ++dz)
          for (int dy = 0; dy < kk[1]; ++dy) {
            const T* row = child + g.voxel_offset(1 + kk[2] * oz + dz, 1 + kk[1] * oy + dy,
                                                  1 + kk[0] * ox);
            for (int dx = 0; dx < kk[0]; ++dx)
#pragma unroll
              for (int c = 0; c < kMaxC; ++c)
                if (c < C) sum[c] += row[dx * C + c];
          }
        cnt = n_out;
      } else {
        for (int dz = 0; dz < kk[2]; ++dz) {
          const int sz = kk[2] * oz + dz;
          if (sz >= j.cext[2]) continue;
          for (int dy = 0; dy < kk[1]; ++dy) {
            const int sy = kk[1] * oy + dy;
            if (sy >= j.cext[1]) continue;
            for (int dx = 0; dx < kk[0]; ++dx) {
              const int sx = kk[0] * ox + dx;
              if (sx >= j.cext[0]) continue;
              const T* v = child + g.voxel_offset(1 + sz, 1 + sy, 1 + sx);
#pragma unroll
              for (int c = 0; c < kMaxC; ++c)
                if (c < C) sum[c] += v[c];
              ++cnt;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kMaxC; ++c)
        if (c < C) dst[c] = (T)(cnt ? (2 * sum[c] + cnt) / (2 * cnt) : g.bg);
    }
  }
}

// fill_borders (octree.py:540-614): 26 segments per brick from same-level
// neighbour interiors, else neighbour AVG, bg outside the virtual extent.
// One CTA per brick: 26 threads resolve the segments' neighbours at once
// (find_node, octree.py:497-505, with exact integer compares), then the
// whole CTA walks every shell voxel of the brick in one flat loop (a
// thread per voxel, all channels), so the small segments do not serialise.
#ifndef VT_BORDER_K
#define VT_BORDER_K 4
#endif
template <class T>
__global__ void __launch_bounds__(256) k_borders(const BorderJob* __restrict__ jobs, Geo g,
                                                 T* pool, const uint8_t* __restrict__ flags,
                                                 const int32_t* __restrict__ slots,
                                                 const int32_t* __restrict__ stats) {
  const BorderJob j = jobs[blockIdx.x];
  const int level = g.level_of(j.node);
  __shared__ int s_mode[27];  // 0 bg, 1 copy, 2 avg
  __shared__ int s_src[27][3];  // copy: neighbour-interior origin of the segment
  __shared__ int s_nslot[27];
  __shared__ int s_avg[27][kMaxC];
  __shared__ int s_start[28];
  __shared__ int s_len[27][3], s_l0[27][3];
  __shared__ uint32_t s_mg[27][2];  // v / lx and v / (lx * ly) by multiply-high
  const int C = g.C;
  if (threadIdx.x < 27) {
    const int seg = threadIdx.x;
    int lo[3], sc[3], mlo[3], mvirt[3];
    g.box_lo(j.node, lo);
    for (int a = 0; a < 3; ++a) {
      sc[a] = g.scale(a, level);
      mlo[a] = lo[a] / sc[a];
      mvirt[a] = (g.virt[a] + sc[a] - 1) / sc[a];
    }
    const int s3[3] = {seg % 3, (seg / 3) % 3, seg / 9};
    int l0[3], len[3], g0[3];
    bool outside = false;
    for (int a = 0; a < 3; ++a) {
      if (s3[a] == 1) {
        l0[a] = 1;
        len[a] = g.brick[a];
        g0[a] = mlo[a];
      } else {
        l0[a] = s3[a] == 0 ? 0 : 1 + g.brick[a];
        len[a] = 1;
        g0[a] = s3[a] == 0 ? mlo[a] - 1 : mlo[a] + g.brick[a];
        if (g0[a] < 0 || g0[a] >= mvirt[a]) outside = true;
      }
    }
    const bool interior = (s3[0] == 1 && s3[1] == 1 && s3[2] == 1) ||
                          (j.skipx && s3[0] != 1 && s3[1] == 1 && s3[2] == 1);
    for (int a = 0; a < 3; ++a) {
      s_len[seg][a] = interior ? 0 : len[a];
      s_l0[seg][a] = l0[a];
    }
    {
      const uint64_t dx = (uint64_t)(len[0] > 0 ? len[0] : 1), dxy = dx * (len[1] > 0 ? len[1] : 1);
      s_mg[seg][0] = (uint32_t)((((uint64_t)1 << 32) + dx - 1) / dx);
      s_mg[seg][1] = (uint32_t)((((uint64_t)1 << 32) + dxy - 1) / dxy);
    }
    int mode = 0;
    if (!interior && !outside) {
      int64_t idx = 0;
      int lvl = g.depth;
      int nlo[3] = {0, 0, 0};
      while (lvl > level && (flags[idx] & NF_CHILDREN)) {
        int k = 0;
        for (int a = 0; a < 3; ++a) {
          const int half = g.extent(a, lvl - 1);
          if (g.split[a] && 2LL * g0[a] * sc[a] + sc[a] >= 2LL * (nlo[a] + half)) {
            k |= 1 << a;
            nlo[a] += half;
          }
        }
        idx = 8 * idx + 1 + k;
        --lvl;
      }
      if (lvl == level && (flags[idx] & NF_BRICK)) {
        mode = 1;
        s_nslot[seg] = slots[idx];
        // stored coords in the neighbour of the segment's first voxel
        for (int a = 0; a < 3; ++a) s_src[seg][a] = 1 + g0[a] - nlo[a] / sc[a];
      } else {
        mode = 2;
        for (int c = 0; c < kMaxC; ++c) s_avg[seg][c] = c < C ? stats[st_index(idx, ST_AVG, c)] : 0;
      }
    }
    s_mode[seg] = mode;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int seg = 0; seg < 27; ++seg) {
      s_start[seg] = acc;
      acc += s_len[seg][0] * s_len[seg][1] * s_len[seg][2];
    }
    s_start[27] = acc;
  }
  __syncthreads();
  T* dst = pool + (int64_t)j.slot * g.brick_elems;
  const int total = s_start[27];
  // batches of K shell voxels per thread: every source of a batch is read
  // before any destination is written (the reads are strided neighbour
  // columns: latency, not bandwidth, bounds this loop)
  constexpr int K = VT_BORDER_K;
  for (int e0 = threadIdx.x; e0 < total; e0 += K * blockDim.x) {
    int64_t doff[K];
    T val[K][kMaxC];
    bool live[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const int e = e0 + q * blockDim.x;
      live[q] = e < total;
      if (!live[q]) continue;
      int seg = 0;  // binary search of the segment prefix sums
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1)
        if (seg + step < 27 && e >= s_start[seg + step]) seg += step;
      const int v = e - s_start[seg];
      const uint32_t lxly = (uint32_t)(s_len[seg][0] * s_len[seg][1]);
      // (a divisor of 1 has no 32-bit magic: 2^32 does not fit)
      const int z = lxly == 1 ? v : (int)__umulhi((uint32_t)v, s_mg[seg][1]);
      const int r = v - z * (int)lxly;
      const int y = s_len[seg][0] == 1 ? r : (int)__umulhi((uint32_t)r, s_mg[seg][0]);
      const int x = r - y * s_len[seg][0];
      doff[q] = g.voxel_offset(s_l0[seg][2] + z, s_l0[seg][1] + y, s_l0[seg][0] + x);
      const int mode = s_mode[seg];
      if (mode == 1) {
        const T* src = pool + (int64_t)s_nslot[seg] * g.brick_elems +
                       g.voxel_offset(s_src[seg][2] + z, s_src[seg][1] + y, s_src[seg][0] + x);
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) val[q][c] = c < C ? src[c] : (T)0;
      } else {
#pragma unroll
        for (int c = 0; c < kMaxC; ++c) val[q][c] = mode == 2 ? (T)s_avg[seg][c] : (T)g.bg;
      }
    }
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (live[q])
#pragma unroll
        for (int c = 0; c < kMaxC; ++c)
          if (c < C) dst[doff[q] + c] = val[q][c];
  }
}

__global__ void k_set_stats(const int64_t* __restrict__ nodes, int n,
                            const int32_t* __restrict__ in, int32_t* stats) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * ST_N * kMaxC) return;
  int r = i / (ST_N * kMaxC), w = i % (ST_N * kMaxC);
  stats[nodes[r] * ST_N * kMaxC + w] = in[i];
}

__global__ void k_gather_stats(const int64_t* __restrict__ nodes, int n,
                               const int32_t* __restrict__ stats, int32_t* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * ST_N * kMaxC) return;
  int r = i / (ST_N * kMaxC), w = i % (ST_N * kMaxC);
  out[i] = stats[nodes[r] * ST_N * kMaxC + w];
}

// position-dependent 64-bit hash of one brick's bytes (sum of mixed words,
// so a parallel reduction gives the same value for any thread order)
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__global__ void __launch_bounds__(256) k_brick_hash(const int32_t* __restrict__ slots, int n,
                                                    const uint8_t* __restrict__ pool, int64_t bytes,
                                                    unsigned long long* out) {
  __shared__ unsigned long long red[8];
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const uint8_t* src = pool + (int64_t)slots[b] * bytes;
    unsigned long long h = 0;
    const int64_t words = bytes / 4;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(src);
    const bool aligned = ((uintptr_t)src & 3) == 0;
    for (int64_t k = threadIdx.x; k < words; k += blockDim.x) {
      uint32_t v;
      if (aligned) {
        v = w[k];
      } else {
        v = (uint32_t)src[4 * k] | ((uint32_t)src[4 * k + 1] << 8) |
            ((uint32_t)src[4 * k + 2] << 16) | ((uint32_t)src[4 * k + 3] << 24);
      }
      h += mix64(((unsigned long long)k << 32) ^ v);
    }
    for (int64_t k = words * 4 + threadIdx.x; k < bytes; k += blockDim.x)
      h += mix64((0xABCDULL << 48) ^ ((unsigned long long)k << 8) ^ src[k]);
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = h;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
      out[b] = t;
    }
    __syncthreads();
  }
}

__global__ void k_copy_bricks(const int32_t* __restrict__ slots, int n, const uint8_t* src_pool,
                              uint8_t* dst_pool, int64_t bytes, int gather) {
  int b = blockIdx.y;
  if (b >= n) return;
  const uint8_t* s = gather ? src_pool + (int64_t)slots[b] * bytes : src_pool + (int64_t)b * bytes;
  uint8_t* d = gather ? dst_pool + (int64_t)b * bytes : dst_pool + (int64_t)slots[b] * bytes;
  if ((bytes & 3) == 0) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(s);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(d);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bytes / 4;
         e += (int64_t)gridDim.x * blockDim.x)
      d4[e] = s4[e];
  } else {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < bytes;
         e += (int64_t)gridDim.x * blockDim.x)
      d[e] = s[e];
  }
}

template <class T>
__global__ void k_pool_fill(T* pool, int64_t n, T v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    pool[e] = v;
}

inline unsigned grid_for(int64_t work, int per_block = kThreads, unsigned cap = 148 * 16) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  return (unsigned)(b > cap ? cap : b);
}

}  // namespace

#define VT_CHECK_LAUNCH() VT_CUDA(cudaGetLastError())

void launch_struct_update(const Tree& t, const StructUpd* d, int n) {
  if (n <= 0) return;
  k_struct_update<<<(n + kThreads - 1) / kThreads, kThreads, 0, t.stream>>>(d, n, t.d_flags,
                                                                             t.d_slot);
  VT_CHECK_LAUNCH();
}

void launch_create(const Tree& t, const CreateJob* d, int n) {
  if (n <= 0) return;
  k_create<<<n, 32, 0, t.stream>>>(d, n, t.g, t.d_flags, t.d_stats);
  VT_CHECK_LAUNCH();
}

constexpr int kMaxGridY = 65535;

// CTAs per job for a launch of n jobs: small per-insertion launches (a
// slice's few dozen bricks at threshold > 0) split each job so every SM works
static unsigned split_for(int n, int max_split) {
  int k = 1;
  while (k < max_split && (int64_t)n * k < 2 * 148) k *= 2;
  return (unsigned)k;
}

void launch_seed(const Tree& t, const SeedJob* d, int n) {
  if (n <= 0) return;
  const dim3 grid((unsigned)std::min<int64_t>(n, 148 * 64), split_for(n, 16));
  if (t.g.sb == 1)
    k_seed<uint8_t><<<grid, 256, 0, t.stream>>>(d, n, t.g, t.d_pool, t.d_stats);
  else
    k_seed<uint16_t><<<grid, 256, 0, t.stream>>>(d, n, t.g, (uint16_t*)t.d_pool, t.d_stats);
  VT_CHECK_LAUNCH();
}

bool scatter_owns_stats(const Geo& g, int channel, const int o[3], const int d[3], int gx,
                        int gy) {
  if (!(channel < 0 || g.C == 1)) return false;
  const int bx0 = gx * g.brick[0], by0 = gy * g.brick[1];
  const int ix1 = std::min(g.dims[0], bx0 + g.brick[0]), iy1 = std::min(g.dims[1], by0 + g.brick[1]);
  return o[0] <= bx0 && o[0] + d[0] >= ix1 && o[1] <= by0 && o[1] + d[1] >= iy1;
}

void launch_scatter(const Tree& t, const void* src, int channel, int ss, int so, const int o[3],
                    const int d[3], const int g0[3], const int gn[3], const int32_t* slots) {
  if ((int64_t)d[0] * d[1] * d[2] == 0) return;
  for (int z = 0; z < d[2]; z += 65535) {
    const int nz = std::min(65535, d[2] - z);
    dim3 grid((unsigned)(gn[0] * gn[1]), (unsigned)nz);
    if (t.g.sb == 1)
      k_scatter<uint8_t><<<grid, 256, 0, t.stream>>>(
          (const uint8_t*)src, channel, ss, so, o[0], o[1], o[2], z, d[0], d[1], g0[0], g0[1],
          g0[2], gn[0], gn[1], slots, t.g, t.d_pool, t.d_pmin, t.d_pmax, t.d_psum);
    else
      k_scatter<uint16_t><<<grid, 256, 0, t.stream>>>(
          (const uint16_t*)src, channel, ss, so, o[0], o[1], o[2], z, d[0], d[1], g0[0], g0[1],
          g0[2], gn[0], gn[1], slots, t.g, (uint16_t*)t.d_pool, t.d_pmin, t.d_pmax, t.d_psum);
    VT_CHECK_LAUNCH();
  }
}

void launch_octant(const Tree& t, const OctJob* d, int n) {
  if (n <= 0) return;
  const dim3 grid((unsigned)std::min<int64_t>(n, 148 * 32), split_for(n, 8));
  if (t.g.sb == 1)
    k_octant<uint8_t><<<grid, 256, 0, t.stream>>>(d, n, t.g, t.d_pool, t.d_stats);
  else
    k_octant<uint16_t><<<grid, 256, 0, t.stream>>>(d, n, t.g, (uint16_t*)t.d_pool, t.d_stats);
  VT_CHECK_LAUNCH();
}

void launch_plane(const Tree& t, const PlaneJob* d, int n) {
  if (n <= 0) return;
  const dim3 grid((unsigned)std::min<int64_t>(n, 148 * 64), split_for(n, 32));
  if (t.g.sb == 1)
    k_plane<uint8_t><<<grid, 128, 0, t.stream>>>(d, n, t.g, t.d_pool, t.d_pmin, t.d_pmax,
                                                  t.d_psum);
  else
    k_plane<uint16_t><<<grid, 128, 0, t.stream>>>(d, n, t.g, (const uint16_t*)t.d_pool, t.d_pmin,
                                                   t.d_pmax, t.d_psum);
  VT_CHECK_LAUNCH();
}

void launch_reduce(const Tree& t, const ReduceJob* d, int n) {
  if (n <= 0) return;
  const int64_t work = (int64_t)n * t.g.C * 32;  // a warp per (node, channel)
  k_reduce<<<(unsigned)((work + 127) / 128), 128, 0, t.stream>>>(
      d, n, t.g, t.d_pmin, t.d_pmax, t.d_psum, t.d_flags, t.d_stats);
  VT_CHECK_LAUNCH();
}

void launch_borders(const Tree& t, const BorderJob* d, int n) {
  if (n <= 0) return;
  if (t.g.sb == 1)
    k_borders<uint8_t><<<n, 256, 0, t.stream>>>(d, t.g, t.d_pool, t.d_flags, t.d_slot, t.d_stats);
  else
    k_borders<uint16_t><<<n, 256, 0, t.stream>>>(d, t.g, (uint16_t*)t.d_pool, t.d_flags,
                                                 t.d_slot, t.d_stats);
  VT_CHECK_LAUNCH();
}

void launch_gather_stats(const Tree& t, const int64_t* d_nodes, int n, int32_t* d_out) {
  if (n <= 0) return;
  int work = n * ST_N * kMaxC;
  k_gather_stats<<<(work + kThreads - 1) / kThreads, kThreads, 0, t.stream>>>(d_nodes, n,
                                                                               t.d_stats, d_out);
  VT_CHECK_LAUNCH();
}

void launch_brick_hash(const Tree& t, const int32_t* d_slots, int n, unsigned long long* d_out) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(n, 148 * 16);
  k_brick_hash<<<grid, 256, 0, t.stream>>>(d_slots, n, t.d_pool, t.g.brick_elems * t.g.sb, d_out);
  VT_CHECK_LAUNCH();
}

void launch_set_stats(const Tree& t, const int64_t* d_nodes, int n, const int32_t* d_rows) {
  if (n <= 0) return;
  const int work = n * ST_N * kMaxC;
  k_set_stats<<<(work + kThreads - 1) / kThreads, kThreads, 0, t.stream>>>(d_nodes, n, d_rows,
                                                                          t.d_stats);
  VT_CHECK_LAUNCH();
}

void launch_gather_bricks(const Tree& t, const int32_t* d_slots, int n, uint8_t* d_out) {
  int64_t bytes = t.g.brick_elems * t.g.sb;
  for (int o = 0; o < n; o += kMaxGridY) {
    int m = n - o < kMaxGridY ? n - o : kMaxGridY;
    dim3 grid(grid_for(bytes / 4 + 1, kThreads, 64), m);
    k_copy_bricks<<<grid, kThreads, 0, t.stream>>>(d_slots + o, m, t.d_pool, d_out + o * bytes,
                                                   bytes, 1);
    VT_CHECK_LAUNCH();
  }
}

void launch_scatter_bricks(const Tree& t, const int32_t* d_slots, int n, const uint8_t* d_in) {
  int64_t bytes = t.g.brick_elems * t.g.sb;
  for (int o = 0; o < n; o += kMaxGridY) {
    int m = n - o < kMaxGridY ? n - o : kMaxGridY;
    dim3 grid(grid_for(bytes / 4 + 1, kThreads, 64), m);
    k_copy_bricks<<<grid, kThreads, 0, t.stream>>>(d_slots + o, m, d_in + o * bytes, t.d_pool,
                                                   bytes, 0);
    VT_CHECK_LAUNCH();
  }
}

void launch_pool_fill(const Tree& t, int64_t first, int64_t n) {
  if (n <= 0) return;
  int64_t elems = n * t.g.brick_elems;
  if (t.g.sb == 1)
    k_pool_fill<uint8_t><<<grid_for(elems), kThreads, 0, t.stream>>>(
        t.d_pool + first * t.g.brick_elems, elems, (uint8_t)t.g.bg);
  else
    k_pool_fill<uint16_t><<<grid_for(elems), kThreads, 0, t.stream>>>(
        (uint16_t*)t.d_pool + first * t.g.brick_elems, elems, (uint16_t)t.g.bg);
  VT_CHECK_LAUNCH();
}

}  // namespace vtx
