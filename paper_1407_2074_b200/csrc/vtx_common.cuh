// Internal shared definitions for libvtx (octree build + ray casting on sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/vtx.h"

namespace vtx {

// ---------------------------------------------------------------------------
// error plumbing: C++ exceptions inside, vt_status at the ABI edge
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  vt_status code;
  Error(vt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define VT_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw ::vtx::Error(_e == cudaErrorMemoryAllocation ? VT_ENOMEM : VT_ECUDA,        \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));           \
  } while (0)

#define VT_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) throw ::vtx::Error((code), (msg)); \
  } while (0)

template <class F>
vt_status guarded(F&& f) {
  try {
    f();
    return VT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return VT_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return VT_ESTATE;
  }
}

// the calling thread's current device is restored on exit from every ABI
// entry point that works on a tree's device (Octree(device=k) with k not the
// current device must neither fail nor leave k current)
struct DeviceScope {
  int prev = -1;
  bool changed = false;
  explicit DeviceScope(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      if (cudaSetDevice(dev) != cudaSuccess) throw Error(VT_ECUDA, "cudaSetDevice failed");
      changed = true;
    }
  }
  ~DeviceScope() {
    if (changed) cudaSetDevice(prev);
  }
};

template <class F>
vt_status guarded_on(int device, F&& f) {
  return guarded([&] {
    DeviceScope ds(device);
    f();
  });
}

constexpr int kMaxDepth = 8;   // volume.py:23-25 (22-bit child pointers)
constexpr int kMaxC = 4;

// ---------------------------------------------------------------------------
// tree geometry, passed by value to kernels (volume.py:155-260)
// ---------------------------------------------------------------------------
struct Geo {
  int dims[3];      // original extent (x, y, z)
  int brick[3];     // M per axis
  int stored[3];    // M + 2
  int virt[3];      // virtual extent
  int split[3];     // axis splits (virtual > M)
  int depth;        // N (leaves level 0, root level N)
  int C;            // channels
  int sb;           // sample bytes (1 | 2)
  int bg;           // background value
  int64_t level_start[kMaxDepth + 2];  // first BFS index at tree depth d
  int64_t capacity;
  int64_t brick_elems;  // stored voxels * C

  __host__ __device__ int level_of(int64_t idx) const {
    int d = 0;
    while (d < depth && idx >= level_start[d + 1]) ++d;
    return depth - d;
  }
  __host__ __device__ int extent(int a, int level) const { return split[a] ? brick[a] << level : brick[a]; }
  __host__ __device__ int scale(int a, int level) const { return split[a] ? 1 << level : 1; }
  __host__ __device__ bool octant_real(int k) const {
    for (int a = 0; a < 3; ++a)
      if (((k >> a) & 1) && !split[a]) return false;
    return true;
  }
  // box origin (level-0 virtual voxels) of a node from its BFS index
  __host__ __device__ void box_lo(int64_t idx, int lo[3]) const {
    lo[0] = lo[1] = lo[2] = 0;
    int level = level_of(idx);
    while (idx > 0) {
      int k = (int)((idx - 1) & 7);
      for (int a = 0; a < 3; ++a)
        if ((k >> a) & 1) lo[a] += extent(a, level);
      idx = (idx - 1) >> 3;
      ++level;
    }
  }
  // in-volume interior voxel counts (octree.py:190-199)
  __host__ __device__ void in_extent(const int lo[3], int level, int c[3]) const {
    for (int a = 0; a < 3; ++a) {
      int s = scale(a, level);
      int rem = dims[a] - lo[a];
      int v = rem <= 0 ? 0 : (rem + s - 1) / s;
      c[a] = v > brick[a] ? brick[a] : v;
    }
  }
  __host__ __device__ int64_t voxel_offset(int z, int y, int x) const {
    return (((int64_t)z * stored[1] + y) * stored[0] + x) * C;
  }
};

// node flag bits (host + device mirror), identical to the ABI VT_NODE_*
constexpr uint8_t NF_EXISTS = 1, NF_CHILDREN = 2, NF_INVOL = 4, NF_BRICK = 8;

// stats layout on device: [node][stat][channel], stat = avg, smin, smax, submin, submax
constexpr int ST_AVG = 0, ST_MIN = 1, ST_MAX = 2, ST_SUBMIN = 3, ST_SUBMAX = 4, ST_N = 5;
__host__ __device__ inline int64_t st_index(int64_t node, int stat, int c) {
  return (node * ST_N + stat) * kMaxC + c;
}

// ---------------------------------------------------------------------------
// build job records (host builds them, kernels consume them)
// ---------------------------------------------------------------------------
struct StructUpd { int64_t node; int32_t flags; int32_t slot; };
// seed children of parent; leaves in grid layers [skip_z0, skip_z1] are left
// alone (a dense insertion's leaf kernel writes their statistics)
struct CreateJob { int64_t parent; int64_t seed_src; int32_t skip_z0, skip_z1; };
// cov_lo/cov_hi: interior box [lo, hi) that later work of the same insertion
// overwrites with every channel (scatter of a fused all-channel block, or the
// octant rewrite of a fresh parent) — the seed skips it
struct SeedJob { int64_t node; int32_t slot; int32_t cext[3]; int32_t cov_lo[3], cov_hi[3]; };
struct OctJob {
  int32_t pslot, cslot;  // cslot < 0: brickless child, AVG fill
  int64_t child;
  int32_t k;
  int32_t cext[3];       // child in-volume extent
  int32_t r0[3], r1[3];  // region in octant-local output voxels
};
struct PlaneJob { int32_t slot, z0, z1, cx, cy; };  // planes [z0, z1) of one brick
struct ReduceJob { int64_t node; int32_t slot; int32_t cext[3]; int32_t leafish; };
// skipx: the two x-face segments (x = 0 and x = M + 1 over the interior y/z
// rows) were written by the leaf kernel (interior level-1 parents)
struct BorderJob { int64_t node; int32_t slot; int32_t skipx = 0; };
// dense (tau == 0) build: one leaf brick of a full-layer block
struct DenseJob { int64_t node; int32_t slot; int32_t pad; };

}  // namespace vtx
