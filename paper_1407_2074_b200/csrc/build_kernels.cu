// Octree build kernels for sm_100a: node-structure mirror updates, child
// creation, brick seeding, block scatter into leaf bricks, per-plane brick
// statistics, 2x2x2 integer half-sampling, border fill and bulk gathers.
// All integer arithmetic reproduces voxtree bit-exactly:
//   means (2*sum + n) // (2n)     octree.py:53-55, 82, 91
//   homogeneity / extents         octree.py:95-99, 190-199
#include <climits>

#include "tree.cuh"

namespace vtx {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int div_up(int a, int b) { return (a + b - 1) / b; }

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
  int v = inv ? stats[st_index(jobs[job].seed_src, ST_AVG, c)] : g.bg;
  stats[st_index(child, ST_AVG, c)] = v;
  stats[st_index(child, ST_MIN, c)] = v;
  stats[st_index(child, ST_MAX, c)] = v;
  stats[st_index(child, ST_SUBMIN, c)] = inv ? v : 0;
  stats[st_index(child, ST_SUBMAX, c)] = inv ? v : 0;
}

// _ensure_brick (octree.py:225-241): bg everywhere, node AVG on the
// in-volume interior
template <class T>
__global__ void k_seed(const SeedJob* __restrict__ jobs, Geo g, T* pool,
                       const int32_t* __restrict__ stats) {
  const SeedJob j = jobs[blockIdx.y];
  T* b = pool + (int64_t)j.slot * g.brick_elems;
  T avg[kMaxC];
  for (int c = 0; c < g.C; ++c) avg[c] = (T)stats[st_index(j.node, ST_AVG, c)];
  const int sx = g.stored[0], sy = g.stored[1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.brick_elems;
       e += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(e % g.C);
    int64_t v = e / g.C;
    int x = (int)(v % sx);
    int y = (int)((v / sx) % sy);
    int z = (int)(v / ((int64_t)sx * sy));
    bool in = x >= 1 && x <= j.cext[0] && y >= 1 && y <= j.cext[1] && z >= 1 && z <= j.cext[2];
    b[e] = in ? avg[c] : (T)g.bg;
  }
}

// _write_leaf (octree.py:420-442): block (dz,dy,dx[,C]) -> leaf bricks at +1
template <class T>
__global__ void k_scatter(const T* __restrict__ src, int channel, int src_stride, int src_off,
                          int ox, int oy, int oz, int dx,
                          int dy, int dz, int g0x, int g0y, int g0z, int gnx, int gny,
                          const int32_t* __restrict__ leaf_slots, Geo g, T* pool) {
  const int64_t rows = (int64_t)dy * dz;
  const int mx = g.brick[0], my = g.brick[1], mz = g.brick[2];
  for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
    int y = (int)(row % dy), z = (int)(row / dy);
    int Y = oy + y, Z = oz + z;
    int gy = Y / my, gz = Z / mz;
    int ly = Y - gy * my, lz = Z - gz * mz;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < dx; x += gridDim.x * blockDim.x) {
      int X = ox + x;
      int gx = X / mx, lx = X - gx * mx;
      int32_t s = leaf_slots[((int64_t)(gz - g0z) * gny + (gy - g0y)) * gnx + (gx - g0x)];
      T* dst = pool + (int64_t)s * g.brick_elems + g.voxel_offset(lz + 1, ly + 1, lx + 1);
      if (channel >= 0) {
        dst[channel] = src[(row * dx + x) * src_stride + src_off];
      } else {
        const T* sp = src + (row * dx + x) * g.C;
        for (int c = 0; c < g.C; ++c) dst[c] = sp[c];
      }
    }
  }
}

// per-plane partial statistics of the in-volume interior (feeds
// _recompute_stats, octree.py:248-263); blockDim multiple of C
template <class T>
__global__ void __launch_bounds__(192) k_plane(const PlaneJob* __restrict__ jobs, Geo g,
                                               const T* __restrict__ pool, int32_t* pmin,
                                               int32_t* pmax, unsigned long long* psum) {
  const PlaneJob j = jobs[blockIdx.x];
  const int C = g.C;
  const int t = threadIdx.x;
  const int c = t % C;
  const T* base = pool + (int64_t)j.slot * g.brick_elems + g.voxel_offset(j.z + 1, 1, 1);
  const int rowlen = j.cx * C;
  const int64_t rowstride = (int64_t)g.stored[0] * C;
  const int n = j.cy * rowlen;
  int mn = INT_MAX, mx = INT_MIN;
  unsigned long long s = 0;
  for (int e = t; e < n; e += blockDim.x) {
    int y = e / rowlen;
    int r = e - y * rowlen;
    int v = base[y * rowstride + r];
    mn = min(mn, v);
    mx = max(mx, v);
    s += (unsigned)v;
  }
  __shared__ int smn[192], smx[192];
  __shared__ unsigned long long ss[192];
  smn[t] = mn;
  smx[t] = mx;
  ss[t] = s;
  __syncthreads();
  if (t < C) {
    for (int u = t + C; u < blockDim.x; u += C) {
      mn = min(mn, smn[u]);
      mx = max(mx, smx[u]);
      s += ss[u];
    }
    int64_t o = ((int64_t)j.slot * g.brick[2] + j.z) * C + t;
    pmin[o] = mn;
    pmax[o] = mx;
    psum[o] = s;
  }
}

// plane partials -> smin/smax/avg (round_mean), sub extrema for leaves and
// childless nodes, else _aggregate_subtree_extrema (octree.py:265-277)
__global__ void k_reduce(const ReduceJob* __restrict__ jobs, int n, Geo g,
                         const int32_t* __restrict__ pmin, const int32_t* __restrict__ pmax,
                         const unsigned long long* __restrict__ psum,
                         const uint8_t* __restrict__ flags, int32_t* stats) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * g.C) return;
  const ReduceJob j = jobs[i / g.C];
  const int c = i % g.C;
  const int cx = j.cext[0], cy = j.cext[1], cz = j.cext[2];
  if (cx > 0 && cy > 0 && cz > 0) {
    int mn = INT_MAX, mx = INT_MIN;
    unsigned long long s = 0;
    for (int z = 0; z < cz; ++z) {
      int64_t o = ((int64_t)j.slot * g.brick[2] + z) * g.C + c;
      mn = min(mn, pmin[o]);
      mx = max(mx, pmax[o]);
      s += psum[o];
    }
    long long cnt = (long long)cx * cy * cz;
    long long avg = (2 * (long long)s + cnt) / (2 * cnt);
    stats[st_index(j.node, ST_AVG, c)] = (int)avg;
    stats[st_index(j.node, ST_MIN, c)] = mn;
    stats[st_index(j.node, ST_MAX, c)] = mx;
    if (j.leafish) {
      stats[st_index(j.node, ST_SUBMIN, c)] = mn;
      stats[st_index(j.node, ST_SUBMAX, c)] = mx;
    }
  }
  if (!j.leafish) {
    bool any = false;
    int lo = 0, hi = 0;
    for (int k = 0; k < 8; ++k) {
      if (!g.octant_real(k)) continue;
      int64_t ch = 8 * j.node + 1 + k;
      uint8_t f = flags[ch];
      if (!(f & NF_EXISTS) || !(f & NF_INVOL)) continue;
      int a = stats[st_index(ch, ST_SUBMIN, c)], b = stats[st_index(ch, ST_SUBMAX, c)];
      lo = any ? min(lo, a) : a;
      hi = any ? max(hi, b) : b;
      any = true;
    }
    if (any) {
      stats[st_index(j.node, ST_SUBMIN, c)] = lo;
      stats[st_index(j.node, ST_SUBMAX, c)] = hi;
    }
  }
}

// child contribution to its parent's octant: halfsample_block or AVG fill
// (octree.py:58-92, 281-319)
template <class T>
__global__ void k_octant(const OctJob* __restrict__ jobs, Geo g, T* pool,
                         const int32_t* __restrict__ stats) {
  const OctJob j = jobs[blockIdx.y];
  const int C = g.C;
  int kk[3], off[3];
  for (int a = 0; a < 3; ++a) {
    kk[a] = g.split[a] ? 2 : 1;
    off[a] = (((j.k >> a) & 1) && g.split[a]) ? g.brick[a] / 2 : 0;
  }
  const int wx = j.r1[0] - j.r0[0], wy = j.r1[1] - j.r0[1], wz = j.r1[2] - j.r0[2];
  const int64_t n = (int64_t)wx * wy * wz * C;
  T* parent = pool + (int64_t)j.pslot * g.brick_elems;
  const T* child = j.cslot >= 0 ? pool + (int64_t)j.cslot * g.brick_elems : nullptr;
  int lim[3];
  for (int a = 0; a < 3; ++a) lim[a] = div_up(j.cext[a], kk[a]);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(e % C);
    int64_t v = e / C;
    int ox = j.r0[0] + (int)(v % wx);
    int oy = j.r0[1] + (int)((v / wx) % wy);
    int oz = j.r0[2] + (int)(v / ((int64_t)wx * wy));
    int val;
    if (child) {
      long long s = 0;
      int cnt = 0;
      for (int dz = 0; dz < kk[2]; ++dz) {
        int sz = kk[2] * oz + dz;
        if (sz >= j.cext[2]) continue;
        for (int dy = 0; dy < kk[1]; ++dy) {
          int sy = kk[1] * oy + dy;
          if (sy >= j.cext[1]) continue;
          for (int dx = 0; dx < kk[0]; ++dx) {
            int sx = kk[0] * ox + dx;
            if (sx >= j.cext[0]) continue;
            s += child[g.voxel_offset(1 + sz, 1 + sy, 1 + sx) + c];
            ++cnt;
          }
        }
      }
      val = cnt ? (int)((2 * s + cnt) / (2 * cnt)) : g.bg;
    } else {
      bool in = ox < lim[0] && oy < lim[1] && oz < lim[2];
      val = in ? stats[st_index(j.child, ST_AVG, c)] : g.bg;
    }
    parent[g.voxel_offset(1 + off[2] + oz, 1 + off[1] + oy, 1 + off[0] + ox) + c] = (T)val;
  }
}

// fill_borders (octree.py:540-614): 26 segments per brick from same-level
// neighbour interiors, else neighbour AVG, bg outside the virtual extent
template <class T>
__global__ void k_borders(const BorderJob* __restrict__ jobs, Geo g, T* pool,
                          const uint8_t* __restrict__ flags, const int32_t* __restrict__ slots,
                          const int32_t* __restrict__ stats) {
  const BorderJob j = jobs[blockIdx.x];
  const int level = g.level_of(j.node);
  int lo[3], sc[3], mlo[3], mvirt[3];
  g.box_lo(j.node, lo);
  for (int a = 0; a < 3; ++a) {
    sc[a] = g.scale(a, level);
    mlo[a] = lo[a] / sc[a];
    mvirt[a] = (g.virt[a] + sc[a] - 1) / sc[a];
  }
  T* dst = pool + (int64_t)j.slot * g.brick_elems;
  __shared__ int64_t s_nb;
  __shared__ int s_mode;  // 0 bg, 1 copy, 2 avg
  __shared__ int s_nlo[3];
  __shared__ int s_nslot;
  for (int seg = 0; seg < 27; ++seg) {
    int s3[3] = {seg % 3, (seg / 3) % 3, seg / 9};
    if (s3[0] == 1 && s3[1] == 1 && s3[2] == 1) continue;
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
    if (threadIdx.x == 0) {
      if (outside) {
        s_mode = 0;
      } else {
        // find_node((g0 + 0.5) * scale, level) with exact integer compares
        int64_t idx = 0;
        int lvl = g.depth;
        int nlo[3] = {0, 0, 0};
        while (lvl > level && (flags[idx] & NF_CHILDREN)) {
          int k = 0;
          for (int a = 0; a < 3; ++a) {
            int half = g.extent(a, lvl - 1);
            if (g.split[a] && 2LL * g0[a] * sc[a] + sc[a] >= 2LL * (nlo[a] + half)) {
              k |= 1 << a;
              nlo[a] += half;
            }
          }
          idx = 8 * idx + 1 + k;
          --lvl;
        }
        s_nb = idx;
        if (lvl == level && (flags[idx] & NF_BRICK)) {
          s_mode = 1;
          s_nslot = slots[idx];
          for (int a = 0; a < 3; ++a) s_nlo[a] = nlo[a] / sc[a];
        } else {
          s_mode = 2;
        }
      }
    }
    __syncthreads();
    const int mode = s_mode;
    const int n = len[0] * len[1] * len[2] * g.C;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      int c = e % g.C;
      int v = e / g.C;
      int x = v % len[0], y = (v / len[0]) % len[1], z = v / (len[0] * len[1]);
      T val;
      if (mode == 0) {
        val = (T)g.bg;
      } else if (mode == 1) {
        const T* src = pool + (int64_t)s_nslot * g.brick_elems;
        val = src[g.voxel_offset(1 + g0[2] + z - s_nlo[2], 1 + g0[1] + y - s_nlo[1],
                                 1 + g0[0] + x - s_nlo[0]) + c];
      } else {
        val = (T)stats[st_index(s_nb, ST_AVG, c)];
      }
      dst[g.voxel_offset(l0[2] + z, l0[1] + y, l0[0] + x) + c] = val;
    }
    __syncthreads();
  }
}

__global__ void k_gather_stats(const int64_t* __restrict__ nodes, int n,
                               const int32_t* __restrict__ stats, int32_t* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * ST_N * kMaxC) return;
  int r = i / (ST_N * kMaxC), w = i % (ST_N * kMaxC);
  out[i] = stats[nodes[r] * ST_N * kMaxC + w];
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

void launch_seed(const Tree& t, const SeedJob* d_all, int n_all) {
  for (int o = 0; o < n_all; o += kMaxGridY) {
  const SeedJob* d = d_all + o;
  int n = n_all - o < kMaxGridY ? n_all - o : kMaxGridY;
  dim3 grid(grid_for(t.g.brick_elems, kThreads, 64), n);
  if (t.g.sb == 1)
    k_seed<uint8_t><<<grid, kThreads, 0, t.stream>>>(d, t.g, t.d_pool, t.d_stats);
  else
    k_seed<uint16_t><<<grid, kThreads, 0, t.stream>>>(d, t.g, (uint16_t*)t.d_pool, t.d_stats);
  VT_CHECK_LAUNCH();
  }
}

void launch_scatter(const Tree& t, const void* src, int channel, int ss, int so, const int o[3],
                    const int d[3],
                    const int g0[3], const int gn[3], const int32_t* slots) {
  int64_t rows = (int64_t)d[1] * d[2];
  dim3 grid((d[0] + kThreads - 1) / kThreads, (unsigned)(rows > 65535 ? 65535 : rows));
  if (t.g.sb == 1)
    k_scatter<uint8_t><<<grid, kThreads, 0, t.stream>>>((const uint8_t*)src, channel, ss, so, o[0], o[1],
                                                        o[2], d[0], d[1], d[2], g0[0], g0[1],
                                                        g0[2], gn[0], gn[1], slots, t.g, t.d_pool);
  else
    k_scatter<uint16_t><<<grid, kThreads, 0, t.stream>>>(
        (const uint16_t*)src, channel, ss, so, o[0], o[1], o[2], d[0], d[1], d[2], g0[0], g0[1], g0[2],
        gn[0], gn[1], slots, t.g, (uint16_t*)t.d_pool);
  VT_CHECK_LAUNCH();
}

void launch_octant(const Tree& t, const OctJob* d_all, int n_all) {
  for (int o = 0; o < n_all; o += kMaxGridY) {
  const OctJob* d = d_all + o;
  int n = n_all - o < kMaxGridY ? n_all - o : kMaxGridY;
  int64_t per = (int64_t)t.g.brick[0] * t.g.brick[1] * t.g.brick[2] * t.g.C / 8;
  dim3 grid(grid_for(per, kThreads, 32), n);
  if (t.g.sb == 1)
    k_octant<uint8_t><<<grid, kThreads, 0, t.stream>>>(d, t.g, t.d_pool, t.d_stats);
  else
    k_octant<uint16_t><<<grid, kThreads, 0, t.stream>>>(d, t.g, (uint16_t*)t.d_pool, t.d_stats);
  VT_CHECK_LAUNCH();
  }
}

void launch_plane(const Tree& t, const PlaneJob* d, int n) {
  if (n <= 0) return;
  if (t.g.sb == 1)
    k_plane<uint8_t><<<n, 192, 0, t.stream>>>(d, t.g, t.d_pool, t.d_pmin, t.d_pmax, t.d_psum);
  else
    k_plane<uint16_t><<<n, 192, 0, t.stream>>>(d, t.g, (const uint16_t*)t.d_pool, t.d_pmin,
                                               t.d_pmax, t.d_psum);
  VT_CHECK_LAUNCH();
}

void launch_reduce(const Tree& t, const ReduceJob* d, int n) {
  if (n <= 0) return;
  int work = n * t.g.C;
  k_reduce<<<(work + kThreads - 1) / kThreads, kThreads, 0, t.stream>>>(
      d, n, t.g, t.d_pmin, t.d_pmax, t.d_psum, t.d_flags, t.d_stats);
  VT_CHECK_LAUNCH();
}

void launch_borders(const Tree& t, const BorderJob* d, int n) {
  if (n <= 0) return;
  if (t.g.sb == 1)
    k_borders<uint8_t><<<n, 128, 0, t.stream>>>(d, t.g, t.d_pool, t.d_flags, t.d_slot, t.d_stats);
  else
    k_borders<uint16_t><<<n, 128, 0, t.stream>>>(d, t.g, (uint16_t*)t.d_pool, t.d_flags,
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
