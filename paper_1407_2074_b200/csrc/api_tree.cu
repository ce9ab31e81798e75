// extern "C" surface for the octree build side of libvtx (include/vtx.h).
#include <algorithm>
#include <cstring>

#include "tree.cuh"

using namespace vtx;

namespace vtx {
const char* last_error();
}

namespace {

// standalone halfsample_block (octree.py:58-92) on int32 values
__global__ void k_halfsample(const int32_t* __restrict__ v, int mz, int my, int mx, int C, int cx,
                             int cy, int cz, int kx, int ky, int kz, int bg, int32_t* out) {
  int oz = mz / kz, oy = my / ky, ox = mx / kx;
  int64_t n = (int64_t)oz * oy * ox * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(e % C);
    int64_t p = e / C;
    int x = (int)(p % ox), y = (int)((p / ox) % oy), z = (int)(p / ((int64_t)ox * oy));
    long long s = 0;
    int cnt = 0;
    for (int dz = 0; dz < kz; ++dz)
      for (int dy = 0; dy < ky; ++dy)
        for (int dx = 0; dx < kx; ++dx) {
          int sz = kz * z + dz, sy = ky * y + dy, sx = kx * x + dx;
          if (sx < cx && sy < cy && sz < cz) {
            s += v[(((int64_t)sz * my + sy) * mx + sx) * C + c];
            ++cnt;
          }
        }
    out[e] = cnt ? (int32_t)((2 * s + cnt) / (2 * cnt)) : bg;
  }
}

// synthetic volumes: bit-identical twins of oracle/voxtree_oracle.py
__device__ __forceinline__ uint32_t hash4(uint32_t x, uint32_t y, uint32_t z, uint32_t c,
                                          uint32_t seed) {
  uint32_t h = x * 0x9E3779B1u;
  h ^= y * 0x85EBCA77u;
  h *= 0xC2B2AE3Du;
  h ^= z * 0x27D4EB2Fu;
  h ^= c * 0x165667B1u + seed;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  h *= 0x297A2D39u;
  h ^= h >> 15;
  return h;
}

template <class T>
__global__ void k_synth(T* out, int kind, int dx, int dy, int dz, int C, int fmax, uint32_t seed,
                        int z0, int z1) {
  const int64_t n = (int64_t)(z1 - z0) * dy * dx;
  const bool big = fmax > 255;
  const int amp = big ? 40000 : 220, base = big ? 100 : 8, nmask = big ? 15 : 3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(e % dx);
    int y = (int)((e / dx) % dy);
    int z = z0 + (int)(e / ((int64_t)dx * dy));
    T* o = out + e * C;
    if (kind == 0) {
      for (int c = 0; c < C; ++c) o[c] = (T)(hash4(x, y, z, c, seed) % (uint32_t)(fmax + 1));
      continue;
    }
    long long ex = (long long)(2 * x - dx) * (2 * x - dx) * 10000 / max((long long)dx * dx, 1LL);
    long long ey = (long long)(2 * y - dy) * (2 * y - dy) * 10000 / max((long long)dy * dy, 1LL);
    long long ez = (long long)(2 * z - dz) * (2 * z - dz) * 10000 / max((long long)dz * dz, 1LL);
    bool inside = ex + ey + ez <= 8100;
    int lx = (x & 31) - 16, ly = (y & 31) - 16, lz = (z & 31) - 16;
    int d2 = lx * lx + ly * ly + lz * lz;
    for (int c = 0; c < C; ++c) {
      long long v = base + (hash4(x, y, z, c, seed) & (uint32_t)nmask);
      uint32_t hc = hash4(x >> 5, y >> 5, z >> 5, c + 7, seed);
      if (inside && (hc % 4u) == 0) {
        long long r = 4 + (hc >> 8) % 9u;
        long long r2 = r * r;
        long long b = r2 - d2;
        v += b > 0 ? (long long)amp * b / r2 : 0;
      }
      o[c] = (T)(v < 0 ? 0 : (v > fmax ? fmax : v));
    }
  }
}

}  // namespace

extern "C" {

const char* vt_last_error(void) { return vtx::last_error(); }
int32_t vt_abi_version(void) { return 1; }

vt_status vt_tree_create(const vt_tree_desc* desc, vt_tree** out) {
  return guarded([&] {
    VT_REQUIRE(desc && out, VT_EINVAL, "null argument");
    *out = new vt_tree(*desc);
  });
}

vt_status vt_tree_destroy(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { vt_tree_release(tree); });
}

vt_status vt_tree_set_stream(vt_tree* tree, void* stream) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    VT_CUDA(cudaStreamSynchronize(t.stream));
    if (t.own_stream) VT_CUDA(cudaStreamDestroy(t.stream));
    t.own_stream = false;
    t.stream = (cudaStream_t)stream;
  });
}

vt_status vt_tree_insert(vt_tree* tree, int32_t channel, const int32_t origin[3],
                         const int32_t dims[3], const void* samples, int32_t mem_kind) {
  return guarded_on(tree->t.device, [&] {
    VT_REQUIRE(channel >= 0, VT_EINVAL, "channel " + std::to_string(channel) + " out of range");
    tree->t.insert(channel, origin, dims, samples, mem_kind);
  });
}

// one call per insertion (B200 extension): caller-stream ordering of a
// device block, the insertion, and the first `cap` change events
vt_status vt_tree_insert_ev(vt_tree* tree, int32_t channel, const int32_t origin[3],
                            const int32_t dims[3], const void* samples, int32_t mem_kind,
                            void* caller_stream, int32_t* kinds, int64_t* indices, int64_t cap,
                            int64_t* n_events) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    VT_REQUIRE(channel >= -1, VT_EINVAL, "channel " + std::to_string(channel) + " out of range");
    // a device block is ordered against the caller's stream; a null handle
    // is the legacy default stream (torch's default), not "no stream"
    cudaStream_t cs = (cudaStream_t)caller_stream;
    const bool order = mem_kind == VT_MEM_DEVICE && cs != t.stream;
    if (order) {
      if (!t.ev_wait) VT_CUDA(cudaEventCreateWithFlags(&t.ev_wait, cudaEventDisableTiming));
      VT_CUDA(cudaEventRecord(t.ev_wait, cs));
      VT_CUDA(cudaStreamWaitEvent(t.stream, t.ev_wait, 0));
    }
    const int64_t before = t.event_total();
    t.insert(channel, origin, dims, samples, mem_kind);
    if (order) {
      // the caller's allocator may recycle the block only after our reads
      if (!t.ev_signal) VT_CUDA(cudaEventCreateWithFlags(&t.ev_signal, cudaEventDisableTiming));
      VT_CUDA(cudaEventRecord(t.ev_signal, t.stream));
      VT_CUDA(cudaStreamWaitEvent(cs, t.ev_signal, 0));
    }
    // this insertion's events, copied; they stay queued for drain_events
    *n_events = t.event_total() - before;
    if (*n_events > cap) return;  // too many: the caller copies them with vt_tree_copy_events
    t.copy_events(before, *n_events, kinds, indices);
  });
}

vt_status vt_tree_insert_many(vt_tree* tree, int64_t n, const vt_block* blocks, int32_t mem_kind,
                              void* caller_stream) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    VT_REQUIRE(n >= 0 && (n == 0 || blocks), VT_EINVAL, "null block list");
    VT_REQUIRE(mem_kind == VT_MEM_HOST || mem_kind == VT_MEM_DEVICE, VT_EINVAL, "bad memory kind");
    VT_CUDA(cudaSetDevice(t.device));
    cudaStream_t cs = (cudaStream_t)caller_stream;
    const bool order = mem_kind == VT_MEM_DEVICE && cs != t.stream;
    if (order) {
      if (!t.ev_wait) VT_CUDA(cudaEventCreateWithFlags(&t.ev_wait, cudaEventDisableTiming));
      VT_CUDA(cudaEventRecord(t.ev_wait, cs));
      VT_CUDA(cudaStreamWaitEvent(t.stream, t.ev_wait, 0));
    }
    struct Signal {  // also on error: blocks inserted before it were read
      Tree& t;
      cudaStream_t cs;
      bool on;
      ~Signal() {
        if (!on) return;
        if (!t.ev_signal && cudaEventCreateWithFlags(&t.ev_signal, cudaEventDisableTiming) != cudaSuccess)
          return;
        cudaEventRecord(t.ev_signal, t.stream);
        cudaStreamWaitEvent(cs, t.ev_signal, 0);
      }
    } sig{t, cs, order};
    t.insert_many(n, blocks, mem_kind);
    if (mem_kind == VT_MEM_HOST) VT_CUDA(cudaStreamSynchronize(t.stream));  // host borrow
  });
}

vt_status vt_tree_insert_channels(vt_tree* tree, const int32_t origin[3], const int32_t dims[3],
                                  const void* samples, int32_t mem_kind) {
  return guarded_on(tree->t.device, [&] { tree->t.insert(-1, origin, dims, samples, mem_kind); });
}

vt_status vt_tree_take_events(vt_tree* tree, int32_t* kinds, int64_t* indices, int64_t cap,
                              int64_t* n, int32_t* more) {
  return guarded_on(tree->t.device, [&] {
    *n = tree->t.take_events(kinds, indices, cap);
    *more = tree->t.event_total() > 0 ? 1 : 0;
  });
}

vt_status vt_tree_copy_events(vt_tree* tree, int64_t from, int64_t n, int32_t* kinds,
                              int64_t* indices) {
  return guarded_on(tree->t.device, [&] {
    VT_REQUIRE(from >= 0 && n >= 0 && from + n <= tree->t.event_total(), VT_EINVAL,
               "event range outside the queue");
    tree->t.copy_events(from, n, kinds, indices);
  });
}

vt_status vt_tree_wait_stream(vt_tree* tree, void* stream) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    if ((cudaStream_t)stream == t.stream) return;
    if (!t.ev_wait) VT_CUDA(cudaEventCreateWithFlags(&t.ev_wait, cudaEventDisableTiming));
    VT_CUDA(cudaEventRecord(t.ev_wait, (cudaStream_t)stream));
    VT_CUDA(cudaStreamWaitEvent(t.stream, t.ev_wait, 0));
  });
}

vt_status vt_tree_signal_stream(vt_tree* tree, void* stream) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    if ((cudaStream_t)stream == t.stream) return;
    if (!t.ev_signal) VT_CUDA(cudaEventCreateWithFlags(&t.ev_signal, cudaEventDisableTiming));
    VT_CUDA(cudaEventRecord(t.ev_signal, t.stream));
    VT_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, t.ev_signal, 0));
  });
}

vt_status vt_tree_event_count(vt_tree* tree, int64_t* n) {
  return guarded_on(tree->t.device, [&] { *n = tree->t.event_total(); });
}

vt_status vt_tree_set_dense(vt_tree* tree, int32_t enabled) {
  return guarded_on(tree->t.device, [&] {
    tree->t.flush();
    tree->t.dense_enabled = enabled != 0;
  });
}

vt_status vt_tree_dense_counts(vt_tree* tree, int64_t* leaf_inserts, int64_t* level_nodes,
                               int64_t* fast_borders) {
  return guarded_on(tree->t.device, [&] {
    if (leaf_inserts) *leaf_inserts = tree->t.dense_leaf_inserts;
    if (level_nodes) *level_nodes = tree->t.dense_level_nodes;
    if (fast_borders) *fast_borders = tree->t.fast_borders;
  });
}

vt_status vt_tree_stream_counts(vt_tree* tree, int64_t* layer_groups, int64_t* zero_copy_layers,
                                int64_t* deferred_layers) {
  return guarded_on(tree->t.device, [&] {
    if (layer_groups) *layer_groups = tree->t.layer_groups;
    if (zero_copy_layers) *zero_copy_layers = tree->t.zero_copy_layers;
    if (deferred_layers) *deferred_layers = tree->t.deferred_layers;
  });
}

vt_status vt_tree_publish_halos(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { tree->t.publish_halos(); });
}

vt_status vt_tree_finalize(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { tree->t.finished = true; });
}

vt_status vt_tree_fill_borders(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { tree->t.fill_borders(); });
}

vt_status vt_tree_sync(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { tree->t.sync(); });
}

vt_status vt_tree_flush(vt_tree* tree) {
  return guarded_on(tree->t.device, [&] { tree->t.flush(); });
}

vt_status vt_tree_info_get(vt_tree* tree, vt_tree_info* o) {
  return guarded_on(tree->t.device, [&] {
    const Tree& t = tree->t;
    o->node_count = t.node_count;
    o->brick_count = t.brick_count;
    o->pruned_bricks = t.pruned;
    o->inserted_voxels = t.inserted;
    o->capacity = t.g.capacity;
    o->pool_slots = t.pool_slots;
    o->depth = t.g.depth;
    for (int a = 0; a < 3; ++a) o->virtual_dims[a] = t.g.virt[a];
    o->finished = t.finished;
    o->borders_filled = t.borders;
  });
}

vt_status vt_tree_node(vt_tree* tree, int64_t index, vt_node* out, int32_t* exists) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    *exists = 0;
    if (index < 0 || index >= t.g.capacity || !(t.flags[index] & NF_EXISTS)) return;
    t.flush();
    t.gather_stats({index});
    *exists = 1;
    out->flags = t.flags[index];
    out->level = t.g.level_of(index);
    t.g.box_lo(index, out->box_lo);
    out->slot = t.slot[index];
    for (int c = 0; c < kMaxC; ++c)
      for (int s = 0; s < ST_N; ++s) out->stats[c][s] = c < t.g.C ? t.stat(index, s, c) : 0;
  });
}

vt_status vt_tree_list_nodes(vt_tree* tree, int64_t* out, int32_t* fl, int64_t cap,
                             int64_t* n) {
  return guarded_on(tree->t.device, [&] {
    const Tree& t = tree->t;
    int64_t m = 0;
    for (int64_t i = 0; i < t.g.capacity; ++i)
      if (t.flags[i] & NF_EXISTS) {
        if (m < cap) {
          if (out) out[m] = i;
          if (fl) fl[m] = t.flags[i];
        }
        ++m;
      }
    *n = m;
  });
}

vt_status vt_tree_find_node(vt_tree* tree, const double point[3], int32_t target, int64_t* index) {
  return guarded_on(tree->t.device, [&] { *index = tree->t.find_node(point, target); });
}

vt_status vt_tree_read_brick(vt_tree* tree, int64_t index, void* out) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    VT_REQUIRE(index >= 0 && index < t.g.capacity && (t.flags[index] & NF_BRICK), VT_EINVAL,
               "node has no brick");
    t.flush();
    t.publish_halos();
    const int64_t bytes = t.g.brick_elems * t.g.sb;
    VT_CUDA(cudaMemcpyAsync(out, t.d_pool + (int64_t)t.slot[index] * bytes, bytes,
                            cudaMemcpyDeviceToHost, t.stream));
    VT_CUDA(cudaStreamSynchronize(t.stream));
  });
}

vt_status vt_tree_export(vt_tree* tree, int64_t n, const int64_t* indices, int32_t* stats,
                         void* bricks) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    t.flush();
    t.publish_halos();
    std::vector<int64_t> nodes(indices, indices + n);
    for (int64_t i : nodes)
      VT_REQUIRE(i >= 0 && i < t.g.capacity && (t.flags[i] & NF_EXISTS), VT_EINVAL,
                 "export of a node that does not exist");
    t.gather_stats(nodes);
    const int C = t.g.C;
    for (int64_t r = 0; r < n; ++r)
      for (int c = 0; c < C; ++c)
        for (int s = 0; s < ST_N; ++s) stats[(r * C + c) * ST_N + s] = t.stat(nodes[r], s, c);
    if (!bricks) return;
    std::vector<int32_t> slots;
    for (int64_t i : nodes)
      if (t.flags[i] & NF_BRICK) slots.push_back(t.slot[i]);
    const int64_t bb = t.g.brick_elems * t.g.sb;
    const int64_t batch = std::max<int64_t>(1, (256LL << 20) / bb);
    uint8_t* dbuf = nullptr;
    VT_CUDA(cudaMallocAsync(&dbuf, std::min<int64_t>(batch, std::max<size_t>(1, slots.size())) * bb,
                            t.stream));
    for (size_t o = 0; o < slots.size(); o += batch) {
      int m = (int)std::min<int64_t>(batch, slots.size() - o);
      std::vector<int32_t> part(slots.begin() + o, slots.begin() + o + m);
      int32_t* ds = upload(t, part);
      launch_gather_bricks(t, ds, m, dbuf);
      VT_CUDA(cudaMemcpyAsync((uint8_t*)bricks + o * bb, dbuf, m * bb, cudaMemcpyDeviceToHost,
                              t.stream));
      release(t, ds);
      VT_CUDA(cudaStreamSynchronize(t.stream));
    }
    release(t, dbuf);
    VT_CUDA(cudaStreamSynchronize(t.stream));
  });
}

vt_status vt_tree_checksum(vt_tree* tree, uint64_t* out) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    t.flush();
    t.publish_halos();
    std::vector<int64_t> nodes;
    std::vector<int32_t> slots;
    for (int64_t i = 0; i < t.g.capacity; ++i)
      if (t.flags[i] & NF_EXISTS) {
        nodes.push_back(i);
        if (t.flags[i] & NF_BRICK) slots.push_back(t.slot[i]);
      }
    std::vector<unsigned long long> bh(slots.size());
    if (!slots.empty()) {
      int32_t* ds = upload(t, slots);
      unsigned long long* dh = nullptr;
      VT_CUDA(cudaMallocAsync(&dh, slots.size() * sizeof(unsigned long long), t.stream));
      launch_brick_hash(t, ds, (int)slots.size(), dh);
      VT_CUDA(cudaMemcpyAsync(bh.data(), dh, bh.size() * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, t.stream));
      release(t, ds);
      release(t, dh);
    }
    t.gather_stats(nodes);
    // FNV-1a over (index, flags, stats, brick hash) in BFS order
    uint64_t h = 1469598103934665603ULL;
    auto eat = [&](uint64_t v) {
      for (int b = 0; b < 8; ++b) {
        h ^= (v >> (8 * b)) & 0xFF;
        h *= 1099511628211ULL;
      }
    };
    size_t bi = 0;
    for (int64_t i : nodes) {
      const uint8_t f = t.flags[i];
      eat((uint64_t)i);
      eat((uint64_t)(f & (NF_EXISTS | NF_CHILDREN | NF_INVOL | NF_BRICK)));
      for (int c = 0; c < t.g.C; ++c)
        for (int s2 = 0; s2 < ST_N; ++s2) eat((uint64_t)(uint32_t)t.stat(i, s2, c));
      if (f & NF_BRICK) eat(bh[bi++]);
    }
    eat((uint64_t)t.pruned);
    *out = h;
  });
}

vt_status vt_tree_export_nodes(vt_tree* tree, int64_t n, const int64_t* indices, int32_t* nflags,
                               int32_t* stats, void* bricks, int32_t bricks_mem_kind) {
  return guarded_on(tree->t.device, [&] {
    Tree& t = tree->t;
    t.flush();
    t.publish_halos();
    std::vector<int64_t> nodes(indices, indices + n);
    std::vector<int32_t> slots;
    for (int64_t r = 0; r < n; ++r) {
      const int64_t i = nodes[r];
      VT_REQUIRE(i >= 0 && i < t.g.capacity && (t.flags[i] & NF_EXISTS), VT_EINVAL,
                 "export of a node that does not exist");
      const uint8_t f = t.flags[i];
      if (nflags)
        nflags[r] = VT_NODE_EXISTS | ((f & NF_CHILDREN) ? VT_NODE_CHILDREN : 0) |
                    ((f & NF_INVOL) ? VT_NODE_IN_VOLUME : 0) | ((f & NF_BRICK) ? VT_NODE_BRICK : 0);
      if (f & NF_BRICK) slots.push_back(t.slot[i]);
    }
    if (stats) {
      t.gather_stats(nodes);
      const int C = t.g.C;
      for (int64_t r = 0; r < n; ++r)
        for (int c = 0; c < C; ++c)
          for (int s2 = 0; s2 < ST_N; ++s2) stats[(r * C + c) * ST_N + s2] = t.stat(nodes[r], s2, c);
    }
    if (!bricks || slots.empty()) return;
    const int64_t bb = t.g.brick_elems * t.g.sb;
    if (bricks_mem_kind == VT_MEM_DEVICE) {
      int32_t* ds = upload(t, slots);
      launch_gather_bricks(t, ds, (int)slots.size(), (uint8_t*)bricks);
      release(t, ds);
      VT_CUDA(cudaStreamSynchronize(t.stream));
      return;
    }
    const int64_t batch = std::max<int64_t>(1, (256LL << 20) / bb);
    uint8_t* dbuf = nullptr;
    VT_CUDA(cudaMallocAsync(&dbuf, std::min<int64_t>(batch, (int64_t)slots.size()) * bb, t.stream));
    for (size_t o = 0; o < slots.size(); o += batch) {
      const int m = (int)std::min<int64_t>(batch, slots.size() - o);
      std::vector<int32_t> part(slots.begin() + o, slots.begin() + o + m);
      int32_t* ds = upload(t, part);
      launch_gather_bricks(t, ds, m, dbuf);
      VT_CUDA(cudaMemcpyAsync((uint8_t*)bricks + o * bb, dbuf, m * bb, cudaMemcpyDeviceToHost,
                              t.stream));
      release(t, ds);
      VT_CUDA(cudaStreamSynchronize(t.stream));
    }
    release(t, dbuf);
    VT_CUDA(cudaStreamSynchronize(t.stream));
  });
}

vt_status vt_tree_merge(vt_tree* tree, int64_t n, const int64_t* indices, const int32_t* nflags,
                        const int32_t* stats, const void* bricks, int32_t bricks_mem_kind,
                        int64_t inserted_voxels) {
  return guarded_on(tree->t.device, [&] {
    tree->t.merge(n, indices, nflags, stats, bricks, bricks_mem_kind, inserted_voxels);
  });
}

vt_status vt_tree_import(vt_tree* tree, int64_t n, const int64_t* indices, const int32_t* nflags,
                         const int32_t* stats, const void* bricks, int32_t finished,
                         int32_t borders_filled, int64_t pruned_bricks) {
  return guarded_on(tree->t.device, [&] {
    ++tree->t.data_version;
    tree->t.touch_all();
    Tree& t = tree->t;
    VT_REQUIRE(t.node_count == 1 && t.brick_count == 0, VT_ESTATE, "import into a non-empty tree");
    const int C = t.g.C;
    std::vector<int64_t> nodes(indices, indices + n);
    std::vector<int32_t> st(n * ST_N * kMaxC, 0);
    std::vector<int32_t> slots;
    t.node_count = 0;
    for (int64_t r = 0; r < n; ++r) {
      int64_t i = nodes[r];
      VT_REQUIRE(i >= 0 && i < t.g.capacity, VT_EINVAL, "node index outside the tree");
      int f = nflags[r];
      uint8_t hf = NF_EXISTS;
      if (f & VT_NODE_CHILDREN) hf |= NF_CHILDREN;
      if (f & VT_NODE_IN_VOLUME) hf |= NF_INVOL;
      t.flags[i] = hf;
      t.slot[i] = -1;
      if (f & VT_NODE_BRICK) {
        t.flags[i] |= NF_BRICK;
        t.slot[i] = t.alloc_slot();
        slots.push_back(t.slot[i]);
        ++t.brick_count;
      }
      t.mark_struct(i);
      ++t.node_count;
      for (int c = 0; c < C; ++c)
        for (int s = 0; s < ST_N; ++s) {
          int v = stats[(r * C + c) * ST_N + s];
          st[(r * ST_N + s) * kMaxC + c] = v;
          t.h_stats[st_index(i, s, c)] = v;
        }
    }
    t.flush_structure();
    int64_t* dn = upload(t, nodes);
    int32_t* dst = upload(t, st);
    launch_set_stats(t, dn, (int)n, dst);
    release(t, dn);
    release(t, dst);
    const int64_t bb = t.g.brick_elems * t.g.sb;
    if (!slots.empty()) {
      uint8_t* dbuf = nullptr;
      VT_CUDA(cudaMallocAsync(&dbuf, slots.size() * bb, t.stream));
      VT_CUDA(cudaMemcpyAsync(dbuf, bricks, slots.size() * bb, cudaMemcpyHostToDevice, t.stream));
      int32_t* ds = upload(t, slots);
      launch_scatter_bricks(t, ds, (int)slots.size(), dbuf);
      release(t, ds);
      release(t, dbuf);
    }
    // plane partials for later incremental insertions
    std::vector<PlaneJob> planes;
    for (int64_t i : nodes)
      if (t.flags[i] & NF_BRICK) {
        int ce[3];
        t.node_in_extent(i, ce);
        if (ce[0] > 0 && ce[1] > 0 && ce[2] > 0) planes.push_back({t.slot[i], 0, ce[2], ce[0], ce[1]});
      }
    PlaneJob* dp = upload(t, planes);
    launch_plane(t, dp, (int)planes.size());
    release(t, dp);
    t.finished = finished != 0;
    t.borders = borders_filled != 0;
    t.pruned = pruned_bricks;
    VT_CUDA(cudaStreamSynchronize(t.stream));
  });
}

vt_status vt_halfsample(const int32_t* values, const int32_t shape[4], const int32_t ext[3],
                        const int32_t split[3], int32_t background, int32_t* out,
                        int32_t device) {
  return guarded([&] {
    VT_CUDA(cudaSetDevice(device));
    int mz = shape[0], my = shape[1], mx = shape[2], C = shape[3];
    int kx = split[0] ? 2 : 1, ky = split[1] ? 2 : 1, kz = split[2] ? 2 : 1;
    int64_t nin = (int64_t)mz * my * mx * C;
    int64_t nout = (int64_t)(mz / kz) * (my / ky) * (mx / kx) * C;
    int32_t *din = nullptr, *dout = nullptr;
    VT_CUDA(cudaMalloc(&din, std::max<int64_t>(1, nin) * 4));
    VT_CUDA(cudaMalloc(&dout, std::max<int64_t>(1, nout) * 4));
    VT_CUDA(cudaMemcpy(din, values, nin * 4, cudaMemcpyHostToDevice));
    if (nout) {
      k_halfsample<<<(unsigned)std::min<int64_t>((nout + 255) / 256, 4096), 256>>>(
          din, mz, my, mx, C, ext[0], ext[1], ext[2], kx, ky, kz, background, dout);
      VT_CUDA(cudaGetLastError());
    }
    VT_CUDA(cudaMemcpy(out, dout, nout * 4, cudaMemcpyDeviceToHost));
    cudaFree(din);
    cudaFree(dout);
  });
}

vt_status vt_synth(void* out, int32_t kind, const int32_t dims[3], int32_t C, int32_t sb,
                   uint32_t seed, int32_t z0, int32_t z1, void* stream) {
  return guarded([&] {
    VT_REQUIRE(sb == 1 || sb == 2, VT_EINVAL, "sample bytes must be 1 or 2");
    int64_t n = (int64_t)(z1 - z0) * dims[1] * dims[0];
    unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    if (n <= 0) return;
    if (sb == 1)
      k_synth<uint8_t><<<grid, 256, 0, (cudaStream_t)stream>>>(
          (uint8_t*)out, kind, dims[0], dims[1], dims[2], C, 255, seed, z0, z1);
    else
      k_synth<uint16_t><<<grid, 256, 0, (cudaStream_t)stream>>>(
          (uint16_t*)out, kind, dims[0], dims[1], dims[2], C, 65535, seed, z0, z1);
    VT_CUDA(cudaGetLastError());
  });
}

vt_status vt_last_kernel_ms(vt_tree* tree, double* render_ms, double* build_ms) {
  return guarded_on(tree->t.device, [&] {
    if (render_ms) *render_ms = tree->t.last_render_ms;
    if (build_ms) *build_ms = tree->t.last_build_ms;
  });
}

}  // extern "C"
