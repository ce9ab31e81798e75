// Host control plane of the incremental octree (octree.py:143-614) over the
// device pool.  The host owns the tree STRUCTURE (which nodes exist, which
// own bricks, pool slots, change events, prune decisions); all sample data
// and node statistics live in HBM and are computed by build_kernels.cu.
//
// One insertion = (a) a host walk that creates nodes / bricks and records
// dirty boxes, (b) stream-ordered kernels: structure mirror, child seeding,
// brick seeding, block scatter, then (c) per-level propagation:
// plane stats -> reduce (leaves), octant half-sample -> plane stats ->
// reduce (levels 1..N).  With tau == 0 (nothing is ever pruned, every seed is
// the background, every brick a pure function of the data) (c) is deferred
// and batched across insertions until something reads the tree.  With
// tau > 0 it runs per insertion, followed by a stats gather and the exact
// reference prune (octree.py:456-493).
#include <memory>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cstring>

#include "tree.cuh"

namespace vtx {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
const char* last_error() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------

static void build_geo(const vt_tree_desc& d, Geo& g) {
  int ns[3];
  int depth = 0;
  for (int a = 0; a < 3; ++a) {
    VT_REQUIRE(d.dims[a] > 0 && d.brick[a] > 0, VT_EINVAL, "dims and brick_dims must be positive");
    int n = 0;
    int64_t ext = d.brick[a];
    while (ext < d.dims[a]) {
      ext *= 2;
      ++n;
    }
    ns[a] = n;
    depth = std::max(depth, n);
  }
  VT_REQUIRE(depth <= kMaxDepth, VT_EINVAL,
             "tree needs " + std::to_string(depth + 1) +
                 " levels; child pointers address at most 9 (volume too large for this brick "
                 "resolution)");
  for (int a = 0; a < 3; ++a) {
    g.dims[a] = d.dims[a];
    g.brick[a] = d.brick[a];
    g.stored[a] = d.brick[a] + 2;
    g.virt[a] = ns[a] == 0 ? d.brick[a] : d.brick[a] << depth;
    g.split[a] = g.virt[a] > d.brick[a];
  }
  g.depth = depth;
  g.C = d.channels;
  g.sb = d.sample_bytes;
  g.bg = d.background;
  int64_t s = 0, w = 1;
  for (int i = 0; i < kMaxDepth + 2; ++i) {
    g.level_start[i] = s;
    s += w;
    w *= 8;
  }
  g.capacity = g.level_start[depth + 1];
  g.brick_elems = (int64_t)g.stored[0] * g.stored[1] * g.stored[2] * g.C;
}

namespace {
uint8_t* pinned_get(size_t& cap);

}  // namespace

Tree::Tree(const vt_tree_desc& d) {
  if (const char* e = std::getenv("VT_HOST_PROFILE")) prof.on = e[0] == '1';
  VT_REQUIRE(d.channels >= 1 && d.channels <= kMaxC, VT_EINVAL, "channels must be in [1, 4]");
  VT_REQUIRE(d.sample_bytes == 1 || d.sample_bytes == 2, VT_EINVAL, "unsupported sample format");
  for (int a = 0; a < 3; ++a)
    VT_REQUIRE(d.brick[a] >= 1 && (d.brick[a] == 1 || d.brick[a] % 2 == 0), VT_EINVAL,
               "brick dims must be even (or 1)");
  build_geo(d, g);
  tau = d.threshold;
  fmax = d.sample_bytes == 1 ? 255 : 65535;
  VT_REQUIRE(d.background >= 0 && d.background <= fmax, VT_EINVAL,
             "background_value outside the sample format range");
  device = d.device;
  VT_CUDA(cudaSetDevice(device));
  VT_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  own_stream = true;
  {
    cudaMemPool_t pool;
    VT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    VT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  const int64_t cap = g.capacity;
  flags.assign(cap, 0);
  slot.assign(cap, -1);
  struct_mark.assign(cap, 0);
  complete.assign(cap, 0);
  fused1.assign(cap, 0);
  pinv.assign(cap, 0);
  seed_of.assign(cap, -1);
  anc_mark.assign(cap, 0);
  {
    // staging ring up front: its first allocation syncs the stream
    size_t sc = (size_t)32 << 20;
    stage.h = pinned_get(sc);
    VT_CUDA(cudaMalloc(&stage.d, sc));
    stage.cap = sc;
  }
  // leaf BFS index = first index of the leaf depth + Morton interleave of the
  // split axes' brick coordinates (child_index, volume.py:252-254)
  for (int a = 0; a < 3; ++a) {
    const int n = (g.dims[a] + g.brick[a] - 1) / g.brick[a];
    morton[a].assign(n, 0);
    if (!g.split[a]) continue;
    for (int v = 0; v < n; ++v) {
      int64_t m = 0;
      for (int b = 0; b < g.depth; ++b)
        if ((v >> b) & 1) m |= (int64_t)1 << (3 * b + a);
      morton[a][v] = m;
    }
  }
  if (const char* e = std::getenv("VT_DENSE")) dense_enabled = e[0] != '0';
  if (const char* e = std::getenv("VT_PREFILL")) prefill_enabled = e[0] != '0';
  if (const char* e = std::getenv("VT_DEFER")) defer_enabled = e[0] != '0';
  h_stats.assign(cap * ST_N * kMaxC, 0);
  flags[0] = NF_EXISTS | NF_INVOL;
  for (int c = 0; c < g.C; ++c)
    for (int s2 = 0; s2 < ST_N; ++s2) h_stats[st_index(0, s2, c)] = g.bg;
  VT_CUDA(cudaMalloc(&d_flags, cap));
  VT_CUDA(cudaMalloc(&d_slot, cap * sizeof(int32_t)));
  VT_CUDA(cudaMalloc(&d_stats, cap * ST_N * kMaxC * sizeof(int32_t)));
  VT_CUDA(cudaMemset(d_flags, 0, cap));
  VT_CUDA(cudaMemset(d_slot, 0xFF, cap * sizeof(int32_t)));
  VT_CUDA(cudaMemcpy(d_flags, flags.data(), 1, cudaMemcpyHostToDevice));
  VT_CUDA(cudaMemcpy(d_stats, h_stats.data(), ST_N * kMaxC * sizeof(int32_t),
                     cudaMemcpyHostToDevice));
  dense_pending.box = Box{{0, 0, 0}, {g.brick[0], g.brick[1], g.brick[2]}};
  dense_pending.has_box = true;
  dense_pending.fresh = true;
  dense_pending.masked = true;
  dense_pending.dense = true;
  pend_nodes.assign(g.depth + 1, {});
  pend_pool.assign(g.depth + 1, {});
  pend_slot.assign(cap, -1);
  VT_CUDA(cudaEventCreate(&ev0));
  VT_CUDA(cudaEventCreate(&ev1));
  {
    // highest priority: its few CTAs are scheduled as leaf-kernel CTAs retire
    int lo = 0, hi = 0;
    VT_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    VT_CUDA(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, hi));
  }
  VT_CUDA(cudaEventCreateWithFlags(&ev_pre, cudaEventDisableTiming));
  VT_CUDA(cudaEventCreateWithFlags(&ev_aux, cudaEventDisableTiming));
  if (tau == 0 && dense_enabled) {
    // fused level-1 accumulators of the dense build, allocated up front
    VT_CUDA(cudaMalloc(&d_nsum, g.capacity * g.C * sizeof(unsigned long long)));
    VT_CUDA(cudaMalloc(&d_nmin, g.capacity * g.C * sizeof(int32_t)));
    VT_CUDA(cudaMalloc(&d_nmax, g.capacity * g.C * sizeof(int32_t)));
  }
  int64_t reserve = d.reserve_slots > 0 ? d.reserve_slots : 64;
  ensure_pool(reserve);
}

// process-wide cache of pinned staging blocks: page-locking costs
// milliseconds, so blocks outlive the trees that used them
namespace {
std::mutex g_pin_mu;
std::vector<std::pair<uint8_t*, size_t>> g_pin_free;

uint8_t* pinned_get(size_t& cap) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (size_t i = 0; i < g_pin_free.size(); ++i)
      if (g_pin_free[i].second >= cap) {
        uint8_t* p = g_pin_free[i].first;
        cap = g_pin_free[i].second;
        g_pin_free.erase(g_pin_free.begin() + i);
        return p;
      }
  }
  uint8_t* p = nullptr;
  VT_CUDA(cudaMallocHost(&p, cap));
  return p;
}

void pinned_put(uint8_t* p, size_t cap) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace_back(p, cap);
}
}  // namespace

void* Tree::stage_copy(const void* src, size_t bytes) const {
  const size_t need = (bytes + 255) & ~(size_t)255;
  // ring readers may sit on the tree stream and the side stream
  auto drain = [&] {
    VT_CUDA(cudaStreamSynchronize(stream));
    if (main_saved) VT_CUDA(cudaStreamSynchronize(main_saved));
    if (aux && aux != stream) VT_CUDA(cudaStreamSynchronize(aux));
  };
  if (need > stage.cap) {
    drain();
    pinned_put(stage.h, stage.cap);
    if (stage.d) cudaFree(stage.d);
    stage.h = nullptr;
    stage.d = nullptr;
    size_t cap = std::max<size_t>(need * 2, (size_t)8 << 20);
    stage.h = pinned_get(cap);
    VT_CUDA(cudaMalloc(&stage.d, cap));
    stage.cap = cap;
    stage.head = 0;
  } else if (stage.head + need > stage.cap) {
    // wrap: every earlier copy (and kernel reading the ring) must be done
    drain();
    stage.head = 0;
  }
  uint8_t* h = stage.h + stage.head;
  uint8_t* d = stage.d + stage.head;
  std::memcpy(h, src, bytes);
  VT_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream));
  stage.head += need;
  return d;
}

Tree::~Tree() {
  if (prof.on) {
    std::fprintf(stderr, "[vtx host profile ms]");
    for (int i = 0; i < HostProf::kN; ++i) std::fprintf(stderr, " %s=%.2f", HostProf::name(i), prof.t[i]);
    std::fprintf(stderr, "\n");
  }
  if (stream) cudaStreamSynchronize(stream);
  for (auto& e : prof.ev)
    if (e) cudaEventDestroy(e);
  pinned_put(stage.h, stage.cap);
  if (stage.d) cudaFree(stage.d);
  cudaFree(d_pool);
  cudaFree(d_bmax);
  cudaFree(d_flags);
  cudaFree(d_slot);
  cudaFree(d_stats);
  cudaFree(d_pmin);
  cudaFree(d_pmax);
  cudaFree(d_psum);
  cudaFree(d_nsum);
  cudaFree(d_acc);
  cudaFree(d_acc_il);
  cudaFree(d_nmin);
  cudaFree(d_nmax);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (ev_wait) cudaEventDestroy(ev_wait);
  if (ev_signal) cudaEventDestroy(ev_signal);
  if (ev_pre) cudaEventDestroy(ev_pre);
  if (ev_aux) cudaEventDestroy(ev_aux);
  if (aux) {
    cudaStreamSynchronize(aux);
    cudaStreamDestroy(aux);
  }
  if (own_stream && stream) cudaStreamDestroy(stream);
}

void Tree::ensure_pool(int64_t need) {
  if (need <= pool_slots) return;
  int64_t n = std::max<int64_t>(need, pool_slots * 2);
  const int64_t bb = g.brick_elems * g.sb;
  const int64_t pe = (int64_t)g.brick[2] * g.C;
  uint8_t* np = nullptr;
  int32_t *nmin = nullptr, *nmax = nullptr;
  unsigned long long* nsum = nullptr;
  VT_CUDA(cudaMalloc(&np, n * bb));
  VT_CUDA(cudaMalloc(&nmin, n * pe * sizeof(int32_t)));
  VT_CUDA(cudaMalloc(&nmax, n * pe * sizeof(int32_t)));
  VT_CUDA(cudaMalloc(&nsum, n * pe * sizeof(unsigned long long)));
  if (pool_slots) {
    VT_CUDA(cudaMemcpyAsync(np, d_pool, pool_slots * bb, cudaMemcpyDeviceToDevice, stream));
    VT_CUDA(cudaMemcpyAsync(nmin, d_pmin, pool_slots * pe * 4, cudaMemcpyDeviceToDevice, stream));
    VT_CUDA(cudaMemcpyAsync(nmax, d_pmax, pool_slots * pe * 4, cudaMemcpyDeviceToDevice, stream));
    VT_CUDA(cudaMemcpyAsync(nsum, d_psum, pool_slots * pe * 8, cudaMemcpyDeviceToDevice, stream));
    VT_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d_pool);
    cudaFree(d_pmin);
    cudaFree(d_pmax);
    cudaFree(d_psum);
  }
  d_pool = np;
  d_pmin = nmin;
  d_pmax = nmax;
  d_psum = nsum;
  pool_slots = n;
  slot_ver.resize(n, data_version);
  if (d_bmax) enable_bmax(bmax_nsb);  // grow the maxima table with the pool
}

// (re)size the brick-maxima table to the pool; new slots are "unknown"
// (0xFFFF: never skipped) until a kernel or a refresh computes them
void Tree::enable_bmax(int nsb) {
  if (d_bmax && bmax_cap >= pool_slots && nsb == bmax_nsb) return;
  const int64_t n = std::max<int64_t>(1, pool_slots);
  uint16_t* nb = nullptr;
  const size_t sub = (size_t)n * nsb * kMaxC, bytes = (sub + (size_t)n * kMaxC) * sizeof(uint16_t);
  VT_CUDA(cudaMalloc(&nb, bytes));
  VT_CUDA(cudaMemsetAsync(nb, 0xFF, bytes, stream));
  if (d_bmax && nsb == bmax_nsb) {
    VT_CUDA(cudaMemcpyAsync(nb, d_bmax, (size_t)bmax_cap * nsb * kMaxC * 2,
                            cudaMemcpyDeviceToDevice, stream));
    VT_CUDA(cudaMemcpyAsync(nb + sub, bmax_brick(), (size_t)bmax_cap * kMaxC * 2,
                            cudaMemcpyDeviceToDevice, stream));
    bmax_ver.resize(n, -1);
  } else {
    bmax_ver.assign(n, -1);
  }
  if (d_bmax) {
    VT_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d_bmax);
  }
  d_bmax = nb;
  bmax_cap = n;
  bmax_nsb = nsb;
}

// ---------------------------------------------------------------------------
// structure helpers
// ---------------------------------------------------------------------------

bool Tree::in_volume(int64_t idx) const {
  int lo[3];
  g.box_lo(idx, lo);
  int level = g.level_of(idx);
  for (int a = 0; a < 3; ++a)
    if (!(lo[a] < g.dims[a] && lo[a] + g.extent(a, level) > 0)) return false;
  return true;
}

void Tree::node_in_extent(int64_t idx, int c[3]) const {
  int lo[3];
  g.box_lo(idx, lo);
  g.in_extent(lo, g.level_of(idx), c);
}

void Tree::clear_seed_of() {
  for (int64_t c : seed_marked) seed_of[c] = -1;
  seed_marked.clear();
}

// ascending sort of node indices: LSD radix on 8-bit digits over the bits
// the maximum needs (two passes below 65,536 nodes) for large lists (a whole
// slab's leaves), std::sort otherwise
void sort_indices(std::vector<int64_t>& v) {
  if (v.size() < 2048) {
    std::sort(v.begin(), v.end());
    return;
  }
  int64_t mx = 0;
  for (int64_t x : v) mx = std::max(mx, x);
  int bits = 0;
  while (bits < 63 && (mx >> bits)) bits += 8;
  static thread_local std::vector<int64_t> tmp;
  tmp.resize(v.size());
  for (int sh = 0; sh < bits; sh += 8) {
    uint32_t cnt[257] = {0};
    for (int64_t x : v) ++cnt[((x >> sh) & 0xFF) + 1];
    for (int i = 0; i < 256; ++i) cnt[i + 1] += cnt[i];
    for (int64_t x : v) tmp[cnt[(x >> sh) & 0xFF]++] = x;
    v.swap(tmp);
  }
}

void Tree::mark_struct(int64_t idx) {
  if (struct_range) {
    struct_lo = std::min(struct_lo, idx);
    struct_hi = std::max(struct_hi, idx);
    return;
  }
  if (leaf_struct_by_kernel && idx >= g.level_start[g.depth] && (flags[idx] & NF_INVOL)) return;
  if (!struct_mark[idx]) {
    struct_mark[idx] = 1;
    struct_dirty.push_back(idx);
  }
}

int32_t Tree::alloc_slot() {
  // BrickStore.allocate: recycle the lowest freed slot, else open a new one
  // (paging.py:213-228)
  int32_t s;
  if (!free_slots.empty()) {
    s = free_slots.top();
    free_slots.pop();
  } else {
    VT_REQUIRE(cursor < INT32_MAX, VT_EOVERFLOW, "brick pool exhausted");
    s = (int32_t)cursor++;
    ensure_pool(cursor);
  }
  return s;
}

// ensure_children for a node on a leaf's descent path whose box follows
// from the leaf's grid coordinates (no index decoding); in fast_create mode
// (complete grid) every child is in volume and needs no seed job
void Tree::ensure_children_at(int64_t p, int lvl, const int gg[3]) {
  if (!fast_create) {
    ensure_children(p);
    return;
  }
  if (flags[p] & NF_CHILDREN) return;
  flags[p] |= NF_CHILDREN;
  mark_struct(p);
  (void)lvl;
  (void)gg;
  const int64_t c0 = 8 * p + 1;
  for (int k = 0; k < 8; ++k) {
    flags[c0 + k] = NF_EXISTS | NF_INVOL;
    slot[c0 + k] = -1;
  }
  mark_struct(c0);
  mark_struct(c0 + 7);
  node_count += 8;
  const size_t e0 = events.size();
  events.resize(e0 + 8);
  for (int k = 0; k < 8; ++k) events[e0 + k] = ev_pack(VT_EV_CREATED, c0 + k);
}

void Tree::ensure_children(int64_t p) {
  if (flags[p] & NF_CHILDREN) return;
  flags[p] |= NF_CHILDREN;
  mark_struct(p);
  const int64_t src = seed_of[p] >= 0 ? seed_of[p] : p;
  creates.push_back({p, src, create_skip_z0, create_skip_z1});
  int plo[3];
  g.box_lo(p, plo);
  const int clvl = g.level_of(p) - 1;
  for (int k = 0; k < 8; ++k) {
    if (!g.octant_real(k)) continue;
    int64_t c = 8 * p + 1 + k;
    bool inv = true;
    for (int a = 0; a < 3; ++a) {
      const int ext = g.extent(a, clvl);
      const int lo = plo[a] + (((k >> a) & 1) ? ext : 0);
      inv = inv && lo < g.dims[a] && lo + ext > 0;
    }
    flags[c] = NF_EXISTS | (inv ? NF_INVOL : 0);
    slot[c] = -1;
    mark_struct(c);
    if (seed_of[c] < 0) seed_marked.push_back(c);
    seed_of[c] = src;
    ++node_count;
    events.push_back(ev_pack(VT_EV_CREATED, c));
  }
}

bool Tree::ensure_brick(int64_t n, const int* cext, bool seed) {
  if (flags[n] & NF_BRICK) return false;
  int32_t s = alloc_slot();
  flags[n] |= NF_BRICK;
  slot[n] = s;
  mark_struct(n);
  ++brick_count;
  if (!seed) return true;
  SeedJob j{};
  j.node = n;
  j.slot = s;
  if (cext) {
    for (int a = 0; a < 3; ++a) j.cext[a] = cext[a];
  } else {
    node_in_extent(n, j.cext);
  }
  // no cover by default (set by the caller when it overwrites a region)
  seeds.push_back(j);
  return true;
}

void Tree::free_brick(int64_t n) {
  if (!(flags[n] & NF_BRICK)) return;
  free_slots.push(slot[n]);
  flags[n] &= ~NF_BRICK;
  slot[n] = -1;
  mark_struct(n);
  --brick_count;
  ++pruned;
}

void Tree::flush_structure() {
  if (struct_hi >= struct_lo) {
    // a range-mode insertion: one copy of the flag and slot ranges
    const int64_t lo = struct_lo, span = struct_hi - struct_lo + 1;
    struct_lo = INT64_MAX;
    struct_hi = -1;
    void* df = stage_copy(flags.data() + lo, span);
    VT_CUDA(cudaMemcpyAsync(d_flags + lo, df, span, cudaMemcpyDeviceToDevice, stream));
    void* ds = stage_copy(slot.data() + lo, span * sizeof(int32_t));
    VT_CUDA(cudaMemcpyAsync(d_slot + lo, ds, span * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            stream));
  }
  if (struct_dirty.empty()) return;
  int64_t lo = g.capacity, hi = -1;
  for (int64_t i : struct_dirty) {
    lo = std::min(lo, i);
    hi = std::max(hi, i);
  }
  const int64_t span = hi - lo + 1;
  if (span * 5 <= (int64_t)(struct_dirty.size() * sizeof(StructUpd) * 16)) {
    // dense dirty range (bulk / slab insertions): copy the flag and slot
    // ranges outright instead of per-node records
    for (int64_t i : struct_dirty) struct_mark[i] = 0;
    struct_dirty.clear();
    void* df = stage_copy(flags.data() + lo, span);
    VT_CUDA(cudaMemcpyAsync(d_flags + lo, df, span, cudaMemcpyDeviceToDevice, stream));
    void* ds = stage_copy(slot.data() + lo, span * sizeof(int32_t));
    VT_CUDA(cudaMemcpyAsync(d_slot + lo, ds, span * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                            stream));
    return;
  }
  std::vector<StructUpd> upd;
  upd.reserve(struct_dirty.size());
  for (int64_t i : struct_dirty) {
    upd.push_back({i, flags[i], slot[i]});
    struct_mark[i] = 0;
  }
  struct_dirty.clear();
  StructUpd* d = upload(*this, upd);
  launch_struct_update(*this, d, (int)upd.size());
  release(*this, d);
}

// ---------------------------------------------------------------------------
// insertion (octree.py:323-397)
// ---------------------------------------------------------------------------

static inline void box_union(Pending& p, const Box& b) {
  if (!p.has_box) {
    p.box = b;
    p.has_box = true;
    return;
  }
  for (int a = 0; a < 3; ++a) {
    p.box.lo[a] = std::min(p.box.lo[a], b.lo[a]);
    p.box.hi[a] = std::max(p.box.hi[a], b.hi[a]);
  }
}

void Tree::insert(int channel, const int origin[3], const int dims[3], const void* samples,
                  int mem_kind) {
  ProfScope ps(prof, 0);
  // validation exactly as octree.py:331-341 (channel -1 = all channels interleaved)
  VT_REQUIRE(channel == -1 || (channel >= 0 && channel < g.C), VT_EINVAL,
             "channel " + std::to_string(channel) + " out of range");
  for (int a = 0; a < 3; ++a) {
    VT_REQUIRE(dims[a] >= 0, VT_EINVAL, "block dims must be non-negative");
    VT_REQUIRE(origin[a] >= 0 && (int64_t)origin[a] + dims[a] <= g.dims[a], VT_EINVAL,
               "block [" + std::to_string(origin[0]) + "," + std::to_string(origin[1]) + "," +
                   std::to_string(origin[2]) + "] outside volume");
  }
  const int64_t nvox = (int64_t)dims[0] * dims[1] * dims[2];
  VT_CUDA(cudaSetDevice(device));
  const int nch = channel < 0 ? g.C : 1;
  if (prof.on) {
    for (auto& e : prof.ev)
      if (!e) VT_CUDA(cudaEventCreate(&e));
    VT_CUDA(cudaEventRecord(prof.ev[0], stream));
    prof.ev_armed = false;
  }
  if (nvox == 0) {
    // an empty block touches nothing: the reference still emits no events
    return;
  }
  const int64_t bytes = nvox * nch * g.sb;
  // stage the block on the device (stream ordered)
  const void* dsrc = samples;
  void* staged = nullptr;
  if (mem_kind == VT_MEM_HOST) {
    VT_CUDA(cudaMallocAsync(&staged, bytes, stream));
    VT_CUDA(cudaMemcpyAsync(staged, samples, bytes, cudaMemcpyHostToDevice, stream));
    dsrc = staged;
  }
  if (channel >= 0) {
    insert_staged(channel, origin, dims, dsrc, 1, 0, 1);
  } else if (tau > 0) {
    // exact sequential semantics: C successive single-channel insertions
    for (int c = 0; c < g.C; ++c) insert_staged(c, origin, dims, dsrc, g.C, c, 1);
  } else {
    // tau == 0: one fused pass; events as for C successive insertions
    insert_staged(-1, origin, dims, dsrc, g.C, 0, g.C);
  }
  if (staged) release(*this, staged);
  if (prof.on && prof.ev_armed) {
    // device-side split of this insertion (profiling only: synchronises)
    VT_CUDA(cudaEventRecord(prof.ev[3], stream));
    VT_CUDA(cudaEventSynchronize(prof.ev[3]));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, prof.ev[0], prof.ev[1]);
    cudaEventElapsedTime(&b, prof.ev[1], prof.ev[2]);
    cudaEventElapsedTime(&c, prof.ev[2], prof.ev[3]);
    prof.t[20] += a;
    prof.t[21] += b;
    prof.t[22] += c;
  }
  if (mem_kind == VT_MEM_HOST) {
    // a pinned source is read asynchronously: keep the borrow contract
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, samples) == cudaSuccess &&
        attr.type == cudaMemoryTypeHost)
      VT_CUDA(cudaStreamSynchronize(stream));
    else
      cudaGetLastError();
  }
}

// A block that spans the full x/y extent and whole brick layers in z, every
// channel at once, at threshold 0, over leaves that own no brick yet: its
// leaves end fully covered, so the dense kernels (dense_build.cu) can write
// their bricks and statistics outright.
bool Tree::dense_eligible(int channel, const int origin[3], const int dims[3], const void* dsrc,
                          int src_stride, int src_off) const {
  if (!dense_enabled || tau != 0) return false;
  if (!(channel < 0 || g.C == 1) || src_stride != g.C || src_off != 0) return false;
  if (g.sb == 2 && ((uintptr_t)dsrc & 3)) return false;
  if (origin[0] != 0 || origin[1] != 0 || dims[0] != g.dims[0] || dims[1] != g.dims[1])
    return false;
  const int* M = g.brick;
  const int z1 = origin[2] + dims[2];
  if (origin[2] % M[2] != 0 || (z1 % M[2] != 0 && z1 != g.dims[2])) return false;
  const int gz1 = (z1 - 1) / M[2];
  const int gx1 = (g.dims[0] - 1) / M[0], gy1 = (g.dims[1] - 1) / M[1];
  for (int gz = origin[2] / M[2]; gz <= gz1; ++gz)
    for (int gy = 0; gy <= gy1; ++gy)
      for (int gx = 0; gx <= gx1; ++gx) {
        if (flags[leaf_index(gx, gy, gz)] & NF_BRICK) return false;
      }
  return true;
}

namespace {
struct ParentCoord { int64_t idx; int px, py, pz; };
}  // namespace

void Tree::insert_staged(int channel, const int origin[3], const int dims[3], const void* dsrc,
                         int src_stride, int src_off, int reps, int64_t ev_reps) {
  const int64_t nvox = (int64_t)dims[0] * dims[1] * dims[2];
  if (ev_reps <= 0) ev_reps = reps;
  {
    ProfScope qd(prof, 18);
    if (try_defer(channel, origin, dims, dsrc, src_stride, src_off)) return;
  }
  const bool starting = defer_start;  // this insertion opens a deferred layer
  defer_start = false;
  ++data_version;
  ProfScope* qel = new ProfScope(prof, 23);
  const bool dense = dense_eligible(channel, origin, dims, dsrc, src_stride, src_off);
  delete qel;
  // per-thread scratch: a whole-volume job table is ~0.5 MB, and a fresh
  // allocation of it page-faults on first touch every insertion
  static thread_local std::vector<DenseJob> djobs;
  djobs.clear();
  creates.clear();
  seeds.clear();
  clear_seed_of();
  const int* M = g.brick;
  int g0[3], g1[3], gn[3];
  for (int a = 0; a < 3; ++a) {
    g0[a] = origin[a] / M[a];
    g1[a] = (origin[a] + dims[a] - 1) / M[a];
    gn[a] = g1[a] - g0[a] + 1;
  }
  const size_t nblock = (size_t)gn[0] * gn[1] * gn[2];
  // brick slot per block leaf (general path only)
  std::vector<int32_t> leaf_slots(dense ? 0 : nblock);
  static thread_local std::vector<std::vector<int64_t>> touched;  // scratch, as djobs
  // early path: the sorted level-1 parents (BFS order of the block's leaves)
  static thread_local std::vector<ParentCoord> early_par;
  early_par.clear();
  bool early_full = false;  // early launch over the complete leaf grid
  touched.resize(g.depth + 1);
  for (auto& v : touched) v.clear();
  touched[0].reserve(nblock);
  std::vector<int32_t> fused_slots;
  std::vector<int64_t> fused_nodes;
  // Dense early launch: with no recycled slots the reference's allocation
  // order is known up front — the block's leaves take cursor + (grid order),
  // then the fresh level-1 parents cursor + n_leaves + (BFS order) — so the
  // leaf kernel (with fused level-1 octants) is launched BEFORE the host walk
  // and the walk overlaps it; the walk re-derives every slot and checks.
  const bool early = dense && free_slots.empty() && !hold_dense;
  int launch_result = 0;
  if (early) {
    ProfScope q(prof, 7);
    ProfScope qe(prof, 12);
    const int64_t cur0 = cursor;
    const int64_t nleaves = (int64_t)gn[0] * gn[1] * gn[2];
    ProfScope* qdj = new ProfScope(prof, 26);
    djobs.resize(nleaves);
    {
      DenseJob* out = djobs.data();
      int64_t i = 0;
      for (int gz = g0[2]; gz <= g1[2]; ++gz) {
        const int64_t mz = g.level_start[g.depth] + morton[2][gz];
        for (int gy = g0[1]; gy <= g1[1]; ++gy) {
          const int64_t myz = mz + morton[1][gy];
          for (int gx = g0[0]; gx <= g1[0]; ++gx, ++i)
            out[i] = {myz + morton[0][gx], (int32_t)(cur0 + i), -1};
        }
      }
    }
    delete qdj;
    ProfScope* qpp = new ProfScope(prof, 24);
    // complete grid (every leaf of the tree in this block, no brick yet): the
    // block's parents are every level-1 node, in BFS order, so parent p takes
    // slot cur0 + n_leaves + (p - first level-1 index) — no sort
    const int64_t n1 = g.depth >= 1 ? g.level_start[g.depth] - g.level_start[g.depth - 1] : 0;
    bool complete_grid = g.depth >= 1 && g.split[0] && g.split[1] && g.split[2] &&
                         nleaves == ((int64_t)1 << (3 * g.depth)) && n1 * 8 == nleaves;
    for (int64_t p = 0; complete_grid && p < n1; ++p)
      if (flags[g.level_start[g.depth - 1] + p] & NF_BRICK) complete_grid = false;
    if (complete_grid) {
      early_full = true;
      const int64_t base1 = g.level_start[g.depth - 1];
      for (DenseJob& jd : djobs)
        jd.pad = (int32_t)(cur0 + nleaves + (((jd.node - 1) >> 3) - base1));
      fused_nodes.resize(n1);
      fused_slots.resize(n1);
      for (int64_t p = 0; p < n1; ++p) {
        fused_nodes[p] = base1 + p;
        fused_slots[p] = (int32_t)(cur0 + nleaves + p);
      }
    } else if (g.depth >= 1 && g.split[0] && g.split[1] && g.split[2]) {
      using P1 = ParentCoord;
      std::vector<int64_t> pidx;
      const int64_t base1 = g.level_start[g.depth - 1];
      for (int pz = g0[2] >> 1; pz <= g1[2] >> 1; ++pz)
        for (int py = 0; py <= g1[1] >> 1; ++py)
          for (int px = 0; px <= g1[0] >> 1; ++px)
            pidx.push_back(morton[0][px] + morton[1][py] + morton[2][pz]);
      sort_indices(pidx);
      std::vector<P1> par(pidx.size());
      for (size_t i = 0; i < pidx.size(); ++i) {
        // all three axes split: bit 3b + a of the Morton code is bit b of axis a
        int c[3] = {0, 0, 0};
        for (int b = 0; b < g.depth - 1; ++b)
          for (int a = 0; a < 3; ++a) c[a] |= (int)((pidx[i] >> (3 * b + a)) & 1) << b;
        par[i] = {base1 + pidx[i], c[0], c[1], c[2]};
      }
      early_par.assign(par.begin(), par.end());  // for the leaves' BFS order, after launch
      int64_t next = cur0 + nleaves;
      ProfScope qpd(prof, 27);
      for (const P1& q1 : par) {
        if (flags[q1.idx] & NF_BRICK) continue;  // existing brick: no new slot
        const int32_t ps = (int32_t)next++;
        bool ok = true;
        int64_t pos[8];
        for (int k = 0; k < 8 && ok; ++k) {
          const int gg[3] = {2 * q1.px + (k & 1), 2 * q1.py + ((k >> 1) & 1),
                             2 * q1.pz + ((k >> 2) & 1)};
          if (gg[0] > g1[0] || gg[1] > g1[1] || gg[2] < g0[2] || gg[2] > g1[2]) ok = false;
          pos[k] = ((int64_t)(gg[2] - g0[2]) * gn[1] + gg[1]) * gn[0] + gg[0];
        }
        if (!ok) continue;
        for (int k = 0; k < 8; ++k) djobs[pos[k]].pad = ps;
        fused_nodes.push_back(q1.idx);
        fused_slots.push_back(ps);
      }
    }
    delete qpp;
    ProfScope* qpa = new ProfScope(prof, 25);
    // every slot this insertion can allocate exists before the kernel runs:
    // the block's leaves plus every ancestor its leaves can touch
    int64_t nanc = 0;
    for (int l = 1; l <= g.depth; ++l) {
      int lo[3], hi[3];
      for (int a = 0; a < 3; ++a) {
        lo[a] = g.split[a] ? g0[a] >> l : 0;
        hi[a] = g.split[a] ? g1[a] >> l : 0;
      }
      const int64_t base = g.level_start[g.depth - l];
      for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
          for (int x = lo[0]; x <= hi[0]; ++x)
            if (!(flags[base + morton[0][x] + morton[1][y] + morton[2][z]] & NF_BRICK)) ++nanc;
    }
    delete qpa;
    {
      ProfScope qp(prof, 19);
      ensure_pool(cur0 + nleaves + nanc);
    }
    if (!fused_nodes.empty() && !d_nsum) {
      VT_CUDA(cudaMalloc(&d_nsum, g.capacity * g.C * sizeof(unsigned long long)));
      VT_CUDA(cudaMalloc(&d_nmin, g.capacity * g.C * sizeof(int32_t)));
      VT_CUDA(cudaMalloc(&d_nmax, g.capacity * g.C * sizeof(int32_t)));
    }
    {
      ProfScope qf(prof, 28);
      int64_t* dfn = upload(*this, fused_nodes);
      launch_init_fused(*this, dfn, (int)fused_nodes.size());
      release(*this, dfn);
    }
    DenseJob* dj;
    {
      ProfScope q2(prof, 29);
      dj = upload(*this, djobs);
    }
    const bool want = prefill_enabled && !borders;
    {
      ProfScope q3(prof, 11);
      if (prof.on) VT_CUDA(cudaEventRecord(prof.ev[1], stream));
      VT_CUDA(cudaEventRecord(ev_pre, stream));
      ProfScope qll(prof, 30);
      parent_shells_next = !fused_nodes.empty();
      launch_result = leaf_launch(dsrc, nvox * src_stride, origin[2], dims[2], want ? 1 : 0, dj,
                                  (int)djobs.size(), gn, g0[2]);
      parent_shells_next = false;
      if (prof.on) {
        VT_CUDA(cudaEventRecord(prof.ev[2], stream));
        prof.ev_armed = true;
      }
    }
    release(*this, dj);
    // chain creation below must not seed the statistics the kernel writes
    create_skip_z0 = g0[2];
    create_skip_z1 = g1[2];
  }
  if (dense) {
    // the events and dirty lists of a whole-layer block: created nodes, then
    // C reps of every touched node
    const size_t nl = nblock;
    events.reserve(events.size() + nl * 3 + 64);
    struct_dirty.reserve(struct_dirty.size() + nl * 2 + 64);
  }
  auto* walk_scope = new ProfScope(prof, 1);
  fast_create = struct_range = early_full;

  // leaves (octree.py:351-360): descend, create, ensure brick, dirty box
  auto* leaf_scope = new ProfScope(prof, 8);
  for (int gz = g0[2]; gz <= g1[2]; ++gz) {
    for (int gy = g0[1]; gy <= g1[1]; ++gy)
      for (int gx = g0[0]; gx <= g1[0]; ++gx) {
        int gg[3] = {gx, gy, gz};
        const int64_t idx = leaf_index(gx, gy, gz);
        if (!(flags[idx] & NF_EXISTS)) {
          ProfScope qc(prof, 31);
          // create the missing part of the chain, top down (creation order
          // and seeds exactly as the reference's descent)
          int64_t a = 0;
          for (int lvl = g.depth; lvl > 0; --lvl) {
            ensure_children_at(a, lvl, gg);
            int k = 0;
            for (int q = 0; q < 3; ++q)
              if (g.split[q] && ((gg[q] >> (lvl - 1)) & 1)) k |= 1 << q;
            a = 8 * a + 1 + k;
          }
        }
        int ce[3];
        for (int a = 0; a < 3; ++a) ce[a] = std::max(0, std::min(M[a], g.dims[a] - gg[a] * M[a]));
        bool fresh = ensure_brick(idx, ce, !dense);
        if (dense) {
          // structure only here; the dense kernel writes the whole stored
          // brick and its final statistics (pending entries after launch)
          if (early) {
            const int64_t i = ((int64_t)(gz - g0[2]) * gn[1] + (gy - g0[1])) * gn[0] + (gx - g0[0]);
            VT_REQUIRE(djobs[i].node == idx && djobs[i].slot == slot[idx], VT_ESTATE,
                       "dense build: leaf slot order diverged from the precomputed one");
          } else {
            djobs.push_back({idx, slot[idx], -1});
          }
          touched[0].push_back(idx);
          continue;
        }
        leaf_slots[((size_t)(gz - g0[2]) * gn[1] + (gy - g0[1])) * gn[0] + (gx - g0[0])] =
            slot[idx];
        Box b;
        for (int a = 0; a < 3; ++a) {
          int lo = gg[a] * M[a];
          b.lo[a] = fresh ? 0 : std::max(origin[a], lo) - lo;
          b.hi[a] = fresh ? M[a] : std::min(origin[a] + dims[a], lo + M[a]) - lo;
        }
        if (fresh && (channel < 0 || g.C == 1)) {
          // the scatter below writes every channel of block ∩ brick
          SeedJob& sj = seeds.back();
          for (int a = 0; a < 3; ++a) {
            int lo = gg[a] * M[a];
            sj.cov_lo[a] = std::max(origin[a], lo) - lo;
            sj.cov_hi[a] = std::min(origin[a] + dims[a], lo + M[a]) - lo;
          }
        }
        Pending& p = pend(0, idx);
        box_union(p, b);
        p.fresh |= fresh;
        p.dense = false;
        fused1[(idx - 1) >> 3] = 0;  // a fused parent octant would be stale
        if (g.brick[2] <= 128) {
          if (!p.masked) {
            // first touch since the last propagation: nothing owed yet
            p.masked = true;
            p.need[0] = p.need[1] = 0;
          }
          if (fresh) p.set_need_range(0, ce[2], true);
          if (pinv[idx]) {
            // partials never written by the dense kernel: recompute them all
            p.set_need_range(0, ce[2], true);
            pinv[idx] = 0;
          }
          const bool own = scatter_owns_stats(g, channel, origin, dims, gx, gy);
          const int z0 = std::max(origin[2], gz * M[2]) - gz * M[2];
          const int z1 = std::min(std::min(origin[2] + dims[2], (gz + 1) * M[2]) - gz * M[2], ce[2]);
          p.set_need_range(z0, z1, !own);
        }
        touched[0].push_back(idx);
      }
  }
  delete leaf_scope;
  auto* anc_scope = new ProfScope(prof, 9);
  // a dense block of one whole brick layer over the full x/y extent (slice
  // streams): its ancestors at level l are every level-l node of row z
  // g0z >> l, listed in closed form (Morton code = BFS offset in a level)
  const bool fullxy = dense && g.split[0] && g.split[1] && g.split[2] && origin[0] == 0 &&
                      origin[1] == 0 && dims[0] == g.dims[0] && dims[1] == g.dims[1] &&
                      g0[2] == g1[2];
  // ancestors (octree.py:363-387): ensure parent bricks, record freshness
  for (int lvl = 1; lvl <= g.depth; ++lvl) {
    std::vector<int64_t>& par = touched[lvl];
    ++anc_gen;
    {
      ProfScope qa(prof, 13);
      if (fullxy) {
        const int64_t base = g.level_start[g.depth - lvl];
        const int64_t mz = morton[2][g0[2] >> lvl];
        for (int y = 0; y <= (g1[1] >> lvl); ++y)
          for (int x = 0; x <= (g1[0] >> lvl); ++x) par.push_back(base + morton[0][x] + morton[1][y] + mz);
        sort_indices(par);
      } else {
        for (int64_t c : touched[lvl - 1]) {
          const int64_t q = (c - 1) >> 3;
          if (anc_mark[q] != anc_gen) {
            anc_mark[q] = anc_gen;
            par.push_back(q);
          }
        }
        std::sort(par.begin(), par.end());
      }
    }
    ProfScope qb(prof, 14);
    for (int64_t p : par) {
      bool fresh = ensure_brick(p);
      if (fresh) {
        // a fresh parent recomputes every real octant: its whole interior
        SeedJob& sj = seeds.back();
        for (int a = 0; a < 3; ++a) {
          sj.cov_lo[a] = 0;
          sj.cov_hi[a] = M[a];
        }
      }
      pend(lvl, p).fresh |= fresh;
    }
  }
  // dense: level-1 parents whose every octant is a leaf of this block get
  // their octants from the leaf kernel (fused half-sample)
  create_skip_z0 = 0;
  create_skip_z1 = -1;
  if (early) {
    for (size_t i = 0; i < fused_nodes.size(); ++i)
      VT_REQUIRE(slot[fused_nodes[i]] == fused_slots[i], VT_ESTATE,
                 "dense build: parent slot order diverged from the precomputed one");
    for (int64_t p : fused_nodes) fused1[p] = 1;
  }
  // (a held layer's parents are fused by launch_held, over both layers)
  if (dense && !early && !hold_dense && g.depth >= 1 && g.split[0] && g.split[1] && g.split[2]) {
    ProfScope qfs(prof, 33);
    for (int64_t p : touched[1]) {
      bool ok = true;
      int64_t pos[8];
      int plo[3];
      g.box_lo(p, plo);
      for (int k = 0; k < 8 && ok; ++k) {
        const int64_t c = 8 * p + 1 + k;
        if (!(flags[c] & NF_INVOL) || !(flags[c] & NF_BRICK)) {
          ok = false;
          break;
        }
        int gg[3];
        for (int a = 0; a < 3; ++a) gg[a] = plo[a] / M[a] + ((k >> a) & 1);
        if (gg[2] < g0[2] || gg[2] > g1[2]) ok = false;
        pos[k] = ((int64_t)(gg[2] - g0[2]) * gn[1] + gg[1]) * gn[0] + gg[0];
      }
      if (!ok) continue;
      for (int k = 0; k < 8; ++k) djobs[pos[k]].pad = slot[p];
      fused1[p] = 1;
      fused_slots.push_back(slot[p]);
      fused_nodes.push_back(p);
    }
  }
  {
    ProfScope qs(prof, 15);
    // early path: the block's leaves in BFS order are the children of the
    // sorted parents — no sort
    static thread_local std::vector<int64_t> sorted_leaves;
    sorted_leaves.clear();
    if (early_full) {
      // complete grid: the leaves are the whole last BFS level
      sorted_leaves.resize(touched[0].size());
      for (size_t i = 0; i < sorted_leaves.size(); ++i)
        sorted_leaves[i] = g.level_start[g.depth] + (int64_t)i;
    }
    for (const ParentCoord& q1 : early_par)
      for (int k = 0; k < 8; ++k) {
        const int cgx = 2 * q1.px + (k & 1), cgy = 2 * q1.py + ((k >> 1) & 1),
                  cgz = 2 * q1.pz + ((k >> 2) & 1);
        if (cgx >= g0[0] && cgx <= g1[0] && cgy >= g0[1] && cgy <= g1[1] && cgz >= g0[2] &&
            cgz <= g1[2])
          sorted_leaves.push_back(8 * q1.idx + 1 + k);
      }
    if (fullxy && early_par.empty() && g.depth >= 1) {
      // the layer's leaves in BFS order: the in-volume children of the
      // sorted level-1 parents on this layer's side of the z split
      const int zb = g0[2] & 1;
      for (int64_t p : touched[1])
        for (int k = zb << 2; k < (zb << 2) + 4; ++k) {
          const int64_t c = 8 * p + 1 + k;
          if ((flags[c] & (NF_EXISTS | NF_INVOL)) == (NF_EXISTS | NF_INVOL)) sorted_leaves.push_back(c);
        }
    }
    if (!sorted_leaves.empty() && sorted_leaves.size() == touched[0].size())
      touched[0].swap(sorted_leaves);  // the same set, already ordered
    else
      sort_indices(touched[0]);
  }
  has_pending = true;
  {
    ProfScope qt(prof, 34);
    for (const auto& lv : touched)
      for (int64_t n : lv)
        if (flags[n] & NF_BRICK) touch_slot(slot[n]);
  }
  delete anc_scope;
  delete walk_scope;
  ProfScope enq_scope(prof, 2);

  // device pre-work for this insertion; behind an early dense launch it goes
  // to the side stream (ordered after everything before the leaf kernel) so
  // it runs alongside the leaf kernel rather than after it
  struct SideJoin {
    Tree& t;
    bool on;
    ~SideJoin() {  // back to the tree stream, which waits for the side work
      if (!on) return;
      t.stream = t.main_saved;
      t.main_saved = nullptr;
      cudaEventRecord(t.ev_aux, t.aux);
      cudaStreamWaitEvent(t.stream, t.ev_aux, 0);
    }
  };
  static const bool side_on = [] {
    const char* e = std::getenv("VT_SIDE_STREAM");
    return !(e && e[0] == '0');
  }();
  const bool side = side_on && early && (launch_result & kLeafTma) && aux;
  if (side) {
    VT_CUDA(cudaStreamWaitEvent(aux, ev_pre, 0));
    main_saved = stream;
    stream = aux;
  }
  std::unique_ptr<SideJoin> side_join(new SideJoin{*this, side});
  { ProfScope q(prof, 5); flush_structure(); }
  fast_create = struct_range = false;
  CreateJob* dc;
  SeedJob* ds;
  {
    ProfScope q(prof, 6);
    dc = upload(*this, creates);
    launch_create(*this, dc, (int)creates.size());
    if (starting) {
      // leaf seeds are held (the dense kernel writes whole leaf bricks, a
      // materialisation launches them); ancestor shells go out now
      dl.seeds.clear();
      std::vector<SeedJob> now;
      for (const SeedJob& sj : seeds) (g.level_of(sj.node) == 0 ? dl.seeds : now).push_back(sj);
      seeds.swap(now);
    }
    // fresh ancestors of an early launch or a held pair: their interior is
    // rewritten whole by propagation and fill_borders overwrites every shell
    // voxel, so the background shell is owed (publish_halos writes it for an
    // earlier reader) instead of written
    if ((early || hold_dense) && prefill_enabled && !borders) {
      size_t w = 0;
      for (const SeedJob& sj : seeds) {
        bool full = g.level_of(sj.node) > 0;
        for (int a = 0; a < 3; ++a)
          full = full && sj.cov_lo[a] == 0 && sj.cov_hi[a] == M[a];
        if (full) owed_shells.push_back(sj.slot);
        else seeds[w++] = sj;
      }
      seeds.resize(w);
    }
    ds = upload(*this, seeds);
    launch_seed(*this, ds, (int)seeds.size());
  }
  side_join.reset();
  int32_t* dlp = nullptr;
  if (dense && hold_dense) {
    // the even layer of a pair: its leaves wait for the odd layer's walk
    if (!held.active) {
      held.active = true;
      held.djobs.clear();
      held.z0 = origin[2];
      held.nz = 0;
      held.gz0 = g0[2];
    }
    held.djobs.insert(held.djobs.end(), djobs.begin(), djobs.end());
    held.nz += dims[2];
    held.gz1 = g1[2];
  } else if (dense) {
    ProfScope q(prof, 7);
    int lr = launch_result;
    if (!early) {
      // recycled slots: launch after the walk, with the walk's slots
      if (!fused_nodes.empty() && !d_nsum) {
        VT_CUDA(cudaMalloc(&d_nsum, g.capacity * g.C * sizeof(unsigned long long)));
        VT_CUDA(cudaMalloc(&d_nmin, g.capacity * g.C * sizeof(int32_t)));
        VT_CUDA(cudaMalloc(&d_nmax, g.capacity * g.C * sizeof(int32_t)));
      }
      int64_t* dfn = upload(*this, fused_nodes);
      launch_init_fused(*this, dfn, (int)fused_nodes.size());
      release(*this, dfn);
      DenseJob* dj = upload(*this, djobs);
      const bool want = prefill_enabled && !borders;
      lr = leaf_launch(dsrc, nvox * src_stride, origin[2], dims[2], want ? 1 : 0, dj,
                       (int)djobs.size(), gn, g0[2]);
      release(*this, dj);
    }
    dense_after_launch(lr, djobs, fused_nodes, origin[2], origin[2] + dims[2], g0[2], g1[2],
                       &touched[0]);
    if (lr & kLeafParentShells) mark_parent_shells(fused_nodes, true);
  } else if (starting) {
    // open the deferred layer: slots and events are final, data waits
    ProfScope q(prof, 7);
    dl.active = true;
    dl.gz = g0[2];
    dl.z0 = g0[2] * M[2];
    dl.nz = std::min(M[2], g.dims[2] - dl.z0);
    dl.got.assign((size_t)dl.nz * g.C, 0);
    dl.remaining = dl.nz * g.C;
    dl.order.clear();
    dl.leaf_slots = leaf_slots;
    dl.djobs.clear();
    dl.seeds.clear();  // the leaf kernel writes whole bricks: no seeds owed
    dl.prefilled = false;
    for (int gy = g0[1]; gy <= g1[1]; ++gy)
      for (int gx = g0[0]; gx <= g1[0]; ++gx) {
        const int64_t idx = leaf_index(gx, gy, g0[2]);
        dl.djobs.push_back({idx, slot[idx], -1});
      }
    if (!d_acc)
      VT_CUDA(cudaMalloc(&d_acc, (size_t)M[2] * g.dims[1] * g.dims[0] * g.C * g.sb));
    defer_copy(channel, origin, dims, dsrc);
  } else {
    prefill_valid = false;
    ProfScope q(prof, 7);
    dlp = upload(*this, leaf_slots);
    launch_scatter(*this, dsrc, channel, src_stride, src_off, origin, dims, g0, gn, dlp);
  }
  release(*this, dc);
  release(*this, ds);
  release(*this, dlp);
  inserted += nvox * reps;
  if (early && tau == 0 && origin[0] == 0 && origin[1] == 0 && origin[2] == 0 &&
      dims[0] == g.dims[0] && dims[1] == g.dims[1] && dims[2] == g.dims[2]) {
    // the whole volume in one dense insertion: no later block of a batch can
    // share these parents, so the pyramid is queued now, right behind the
    // leaf kernel, instead of at the next flush (the host work overlaps the
    // leaf kernel; the result is the one flush would compute)
    propagate();
    if (halo_prefill && prefill_valid && owed_lo.empty() && owed_hi.empty() && !borders &&
        complete[0]) {
      // and the shells of every level > 0 brick, as fill_borders' fast path
      // would write them (leaf shells came prefilled from the leaf kernel)
      std::vector<BorderJob> bj;
      for (int64_t i = 0; i < g.capacity; ++i)
        if ((flags[i] & NF_EXISTS) && (flags[i] & NF_BRICK) && g.level_of(i) > 0)
          bj.push_back({i, slot[i], skipx(i) ? 1 : 0});
      BorderJob* d = upload(*this, bj);
      launch_borders(*this, d, (int)bj.size());
      release(*this, d);
      upper_borders = true;
      owed_shells.clear();
    }
  }

  std::vector<char> dmark;
  std::vector<int64_t> deleted;
  if (tau > 0) {
    propagate();
    std::vector<int64_t> all;
    for (auto& v : touched) all.insert(all.end(), v.begin(), v.end());
    { ProfScope q(prof, 37); gather_stats(all); }
    { ProfScope q(prof, 38); prune(touched, dmark, deleted); }
    { ProfScope q(prof, 39); flush_structure(); }
  }
  // NODE_UPDATED for every touched, non-deleted node, sorted (octree.py:393-395)
  // every level's list is sorted and unique and higher levels hold smaller
  // BFS indices, so root-first concatenation is the sorted union
  ProfScope qu(prof, 17);
  static thread_local std::vector<int64_t> upd;
  upd.clear();
  for (int lvl = g.depth; lvl >= 0; --lvl) upd.insert(upd.end(), touched[lvl].begin(), touched[lvl].end());
  events.reserve(events.size() + upd.size());
  const size_t ev0 = events.size();
  for (int64_t i : upd)
    if (flags[i] & NF_EXISTS) events.push_back(ev_pack(VT_EV_UPDATED, i));
  if (ev_reps > 1) {
    // the later blocks' lists: the same UPDATED list, expanded when taken
    push_replay(std::make_shared<std::vector<uint64_t>>(events.begin() + ev0, events.end()),
                ev_reps - 1);
  }
  if (starting) {
    dl.upd = upd;  // every later block of the layer touches the same nodes
    dl_upd_ev.reset();
    if (dl.remaining == 0) finish_layer();
  }
}

void Tree::dense_after_launch(int lr, const std::vector<DenseJob>& djobs,
                              const std::vector<int64_t>& fused_nodes, int z0, int z1, int gz0,
                              int gz1, const std::vector<int64_t>* sorted_leaves,
                              bool pend_leaves) {
  const int* M = g.brick;
  const bool prefilled = lr & kLeafPrefilled;
  if (!(lr & kLeafTma)) {
    for (int64_t p : fused_nodes) fused1[p] = 0;  // the fallback kernels do not fuse
  } else {
    for (const DenseJob& jd : djobs) pinv[jd.node] = 1;
    for (int64_t p : fused_nodes) pinv[p] = 1;
  }
  // host bookkeeping overlaps the device work: pending entries of leaves
  // whose statistics the kernel writes outright (djobs are in (gz, gy, gx)
  // order; propagate sorts its lists)
  ProfScope qd(prof, 16);
  if (pend_leaves) {
    pend_nodes[0].reserve(pend_nodes[0].size() + djobs.size());
    if (sorted_leaves)
      for (int64_t n : *sorted_leaves) pend_dense(n);  // BFS order: propagate needs no sort
    else
      for (const DenseJob& jd : djobs) pend_dense(jd.node);
  }
  for (const DenseJob& jd : djobs) complete[jd.node] = 1;
  if (lr & kLeafBmax) leaves_bmax_valid(djobs);
  ++dense_leaf_inserts;
  if (prefilled) {
    ProfScope qo(prof, 36);
    // z-shell planes whose block plane lies outside this insertion are owed
    // to the z-neighbour's leaf; one whose neighbour is already built (a
    // slice stream's previous layer, or this launch for an earlier owed
    // entry) is copied right away — the plane fill_borders' fast path would
    // copy, logically background until then like every prefilled shell
    halo_prefill = true;
    const int mz = M[2];
    std::vector<int32_t> pj;
    auto built = [&](int64_t nb) { return (flags[nb] & NF_BRICK) && complete[nb]; };
    const bool eager = prefill_valid;
    if (eager) {
      for (auto* v : {&owed_lo, &owed_hi}) {
        const bool lo = v == &owed_lo;
        size_t w = 0;
        for (const Owed& o : *v) {
          if (built(o.nb))
            pj.insert(pj.end(), {slot[o.leaf], lo ? 0 : mz + 1, slot[o.nb], lo ? mz : 1});
          else
            (*v)[w++] = o;
        }
        v->resize(w);
      }
    }
    const int gx1 = (g.dims[0] - 1) / M[0], gy1 = (g.dims[1] - 1) / M[1];
    for (int gz = gz0; gz <= gz1; ++gz) {
      const int lo = gz * M[2] - 1, hi = (gz + 1) * M[2];
      const bool olo = lo >= 0 && lo < z0, ohi = hi < g.dims[2] && hi >= z1;
      if (!olo && !ohi) continue;
      for (int gy = 0; gy <= gy1; ++gy)
        for (int gx = 0; gx <= gx1; ++gx) {
          const int64_t idx = leaf_index(gx, gy, gz);
          if (!(flags[idx] & NF_BRICK) || !complete[idx]) continue;
          if (olo) {
            const int64_t nb = leaf_index(gx, gy, gz - 1);
            if (eager && built(nb)) pj.insert(pj.end(), {slot[idx], 0, slot[nb], mz});
            else owed_lo.push_back({idx, nb});
          }
          if (ohi) {
            const int64_t nb = leaf_index(gx, gy, gz + 1);
            if (eager && built(nb)) pj.insert(pj.end(), {slot[idx], mz + 1, slot[nb], 1});
            else owed_hi.push_back({idx, nb});
          }
        }
    }
    if (!pj.empty()) {
      int32_t* dp = upload(*this, pj);
      launch_plane_copy(*this, dp, (int)(pj.size() / 4));
      release(*this, dp);
    }
  } else {
    prefill_valid = false;
  }
}

bool Tree::parent_interior(int64_t p, bool interleaved) const {
  const int* M = g.brick;
  int lo[3];
  g.box_lo(p, lo);
  const int px = lo[0] / (2 * M[0]), py = lo[1] / (2 * M[1]);
  if (!(px >= 1 && py >= 1 && (px + 1) * 2 * M[0] + 2 <= g.dims[0] &&
        (py + 1) * 2 * M[1] + 2 <= g.dims[1]))
    return false;
  if (!interleaved) return true;
  // k_dense_leaf_tma: (Mx + 3) * C + xoff <= staged row, for both child columns
  const int brow = ((M[0] + 2) * g.C + 14) / 8 * 8;
  for (int gx = 2 * px; gx <= 2 * px + 1; ++gx) {
    const int x0c = (gx * M[0] - 1) * g.C;
    const int xoff = ((x0c % 8) + 8) % 8;
    if (xoff < g.C || (M[0] + 3) * g.C + xoff > brow) return false;
  }
  return true;
}

void Tree::mark_parent_shells(const std::vector<int64_t>& nodes, bool interleaved) {
  // tracked even when prefill is no longer valid: publish_halos resets every
  // tracked shell for a reader
  if (pshell.empty()) pshell.assign(g.capacity, 0);
  for (int64_t p : nodes)
    if (parent_interior(p, interleaved)) pshell[p] |= 1;
}

// the held even layer and the odd layer after it: one leaf launch over both,
// level-1 parents whose eight children are all in the pair fused
void Tree::launch_held() {
  if (!held.active) return;
  ProfScope qh(prof, 35);
  held.active = false;
  const int* M = g.brick;
  const int gnx = (g.dims[0] - 1) / M[0] + 1, gny = (g.dims[1] - 1) / M[1] + 1;
  const int nl = held.gz1 - held.gz0 + 1;
  std::vector<DenseJob>& dj = held.djobs;
  VT_REQUIRE((int64_t)dj.size() == (int64_t)gnx * gny * nl, VT_ESTATE,
             "held dense layers: leaf count mismatch");
  std::vector<int64_t> fused_nodes;
  std::vector<int32_t> fused_slots;
  std::vector<int64_t> shell_nodes;  // interior fused parents (x/y shells by the kernel)
  if (nl == 2 && (held.gz0 & 1) == 0 && g.depth >= 1 && g.split[0] && g.split[1] && g.split[2]) {
    for (int gy = 0; gy + 1 < gny; gy += 2)
      for (int gx = 0; gx + 1 < gnx; gx += 2) {
        const int64_t c0 = dj[(size_t)gy * gnx + gx].node;
        const int64_t p = (c0 - 1) >> 3;
        if (!(flags[p] & NF_BRICK)) continue;
        bool ok = true;
        int64_t pos[8];
        for (int k = 0; k < 8 && ok; ++k) {
          const int x = gx + (k & 1), y = gy + ((k >> 1) & 1), z = (k >> 2) & 1;
          pos[k] = ((int64_t)z * gny + y) * gnx + x;
          const int64_t c = dj[pos[k]].node;
          ok = c == 8 * p + 1 + k && (flags[c] & NF_INVOL) && (flags[c] & NF_BRICK);
        }
        if (!ok) continue;
        for (int k = 0; k < 8; ++k) dj[pos[k]].pad = slot[p];
        fused_nodes.push_back(p);
        fused1[p] = 1;
        // the kernel's interior rule (k_dense_leaf_tma_planar `pxy`)
        const int px = gx >> 1, py = gy >> 1;
        if (px >= 1 && py >= 1 && (px + 1) * 2 * M[0] + 2 <= g.dims[0] &&
            (py + 1) * 2 * M[1] + 2 <= g.dims[1])
          shell_nodes.push_back(p);
      }
  }
  if (!fused_nodes.empty() && !d_nsum) {
    VT_CUDA(cudaMalloc(&d_nsum, g.capacity * g.C * sizeof(unsigned long long)));
    VT_CUDA(cudaMalloc(&d_nmin, g.capacity * g.C * sizeof(int32_t)));
    VT_CUDA(cudaMalloc(&d_nmax, g.capacity * g.C * sizeof(int32_t)));
  }
  int64_t* dfn = upload(*this, fused_nodes);
  launch_init_fused(*this, dfn, (int)fused_nodes.size());
  release(*this, dfn);
  DenseJob* d = upload(*this, dj);
  const bool want = prefill_enabled && !borders;
  const int gn[3] = {gnx, gny, nl};
  const int64_t nvox = (int64_t)g.dims[0] * g.dims[1] * held.nz;
  int lr;
  if (leaf_struct_by_kernel) {
    // the walks left the leaves' device flags / slots to this kernel
    lr = launch_dense_leaf_planar(*this, planar.base, planar.zstride, planar.cstride, held.z0,
                                  held.nz, want ? 1 : 0, d, (int)dj.size(), gn, held.gz0, true,
                                  !shell_nodes.empty());
    if (lr < 0) {
      // no tensor-map encoder after all: the records the walks skipped
      std::vector<StructUpd> upd;
      upd.reserve(dj.size());
      for (const DenseJob& jd : dj) upd.push_back({jd.node, flags[jd.node], slot[jd.node]});
      StructUpd* du = upload(*this, upd);
      launch_struct_update(*this, du, (int)upd.size());
      release(*this, du);
      lr = leaf_launch(planar.base, nvox * g.C, held.z0, held.nz, want ? 1 : 0, d,
                       (int)dj.size(), gn, held.gz0);
    }
  } else {
    lr = leaf_launch(planar.base, nvox * g.C, held.z0, held.nz, want ? 1 : 0, d, (int)dj.size(),
                     gn, held.gz0);
  }
  release(*this, d);
  // No pending entries for the pair's leaves: their statistics are final
  // and every level-1 parent over them is fresh (all octants) or dense
  // (recomputed whole from complete children), so propagate never needs
  // them as dirty children; a later general touch of a leaf opens its own
  // entry (and pinv makes it recompute every plane partial).
  bool parents_fresh = true;
  for (int64_t i = 0; i < (int64_t)dj.size() && parents_fresh; ++i) {
    const int64_t p = (dj[i].node - 1) >> 3;
    const Pending* pp = pend_find(p, 1);
    parents_fresh = pp && pp->fresh;
  }
  dense_after_launch(lr, dj, fused_nodes, held.z0, held.z0 + held.nz, held.gz0, held.gz1,
                     nullptr, !parents_fresh);
  if (lr & kLeafParentShells) mark_parent_shells(shell_nodes, false);
  dj.clear();
}

// ---------------------------------------------------------------------------
// deferred brick layers of slice streams (see Tree::DeferredLayer)
// ---------------------------------------------------------------------------

bool Tree::try_defer(int channel, const int origin[3], const int dims[3], const void* dsrc,
                     int src_stride, int src_off) {
  defer_start = false;
  const int* M = g.brick;
  const int64_t nvox = (int64_t)dims[0] * dims[1] * dims[2];
  const bool shape = defer_enabled && dense_enabled && tau == 0 && channel >= 0 && g.C > 1 && src_stride == 1 &&
                     src_off == 0 && nvox > 0 && origin[0] == 0 && origin[1] == 0 &&
                     dims[0] == g.dims[0] && dims[1] == g.dims[1] &&
                     origin[2] / M[2] == (origin[2] + dims[2] - 1) / M[2];
  const int layer = origin[2] / M[2];
  if (dl.active) {
    bool cont = shape && layer == dl.gz;
    for (int z = origin[2]; cont && z < origin[2] + dims[2]; ++z)
      cont = !dl.got[(size_t)(z - dl.z0) * g.C + channel];
    if (cont) {
      ++data_version;
      defer_copy(channel, origin, dims, dsrc);
      // this block's events: the layer's UPDATED list once more (replayed
      // lazily: a 2048^2 slice of 32^3 bricks updates ~5.5k nodes)
      if (!dl_upd_ev) {
        dl_upd_ev = std::make_shared<std::vector<uint64_t>>();
        dl_upd_ev->reserve(dl.upd.size());
        for (int64_t i : dl.upd) dl_upd_ev->push_back(ev_pack(VT_EV_UPDATED, i));
      }
      push_replay(dl_upd_ev, 1);
      inserted += nvox;
      if (dl.remaining == 0) finish_layer();
      return true;
    }
    materialize_layer(true);
  }
  if (!shape) return false;
  // open a layer only over brick-less leaves (its leaf bricks are fresh)
  const int gx1 = (g.dims[0] - 1) / M[0], gy1 = (g.dims[1] - 1) / M[1];
  for (int gy = 0; gy <= gy1; ++gy)
    for (int gx = 0; gx <= gx1; ++gx)
      if (flags[leaf_index(gx, gy, layer)] & NF_BRICK) return false;
  defer_start = true;
  return false;  // the caller runs the walk in opening mode
}

// the block's planes into the planar layer buffer [C][Mz][Y][X]
void Tree::defer_copy(int channel, const int origin[3], const int dims[3], const void* dsrc) {
  const int64_t plane = (int64_t)g.dims[0] * g.dims[1] * g.sb;
  uint8_t* dst = d_acc + ((size_t)channel * g.brick[2] + (origin[2] - dl.z0)) * plane;
  VT_CUDA(cudaMemcpyAsync(dst, dsrc, plane * dims[2], cudaMemcpyDeviceToDevice, stream));
  for (int z = origin[2]; z < origin[2] + dims[2]; ++z) dl.got[(size_t)(z - dl.z0) * g.C + channel] = 1;
  dl.remaining -= dims[2];
  dl.dirty = true;
  dl.order.push_back({origin[2], dims[2], channel});
}

// the dense leaf kernel over the layer buffer; `partial`: planes not received
// yet hold the leaves' seed value (the background at threshold 0: every
// fresh leaf brick is seeded with its AVG = the background, octree.py:225-241)
void Tree::run_layer(bool partial) {
  const int* M = g.brick;
  const int64_t plane = (int64_t)g.dims[0] * g.dims[1];
  if (partial) {
    std::vector<int32_t> miss;  // planes not received yet hold the background
    for (int zi = 0; zi < dl.nz; ++zi)
      for (int c = 0; c < g.C; ++c)
        if (!dl.got[(size_t)zi * g.C + c]) miss.push_back(c * M[2] + zi);
    launch_fill_planes(*this, d_acc, plane, miss.data(), (int)miss.size());
  }
  const int gn[3] = {(g.dims[0] - 1) / M[0] + 1, (g.dims[1] - 1) / M[1] + 1, 1};
  DenseJob* dj = upload(*this, dl.djobs);
  const bool want = prefill_enabled && !borders;
  PlanarSrc saved = planar;
  planar = {true, d_acc, plane * g.sb, (int64_t)M[2] * plane * g.sb};
  const int lr = leaf_launch(nullptr, 0, dl.z0, dl.nz, want ? 1 : 0, dj, (int)dl.djobs.size(), gn,
                             dl.gz);
  planar = saved;
  release(*this, dj);
  for (const DenseJob& jd : dl.djobs) {
    pend_dense(jd.node);
    complete[jd.node] = 1;
    if (lr & kLeafTma) pinv[jd.node] = 1;
  }
  // the layer's ancestors are owed a recompute: pending since the opening
  // walk, or again when a reader's flush already consumed that entry
  ++data_version;
  if (lr & kLeafBmax) leaves_bmax_valid(dl.djobs);
  for (int64_t p : dl.upd) {
    const int lvl = g.level_of(p);
    if (lvl > 0) pend(lvl, p);
    if (flags[p] & NF_BRICK) touch_slot(slot[p]);
  }
  has_pending = true;
  dl.prefilled = (lr & kLeafPrefilled) != 0;
  if (dl.prefilled) halo_prefill = true;
  else prefill_valid = false;
  dl.dirty = false;
}

void Tree::close_layer() {
  if (dl.prefilled) {
    // z-shell planes of the neighbouring layers are owed to fill_borders
    const int lo = dl.z0 - 1, hi = dl.z0 + g.brick[2];
    const int gnx = (g.dims[0] - 1) / g.brick[0] + 1;
    for (size_t k = 0; k < dl.djobs.size(); ++k) {  // (gy, gx) order
      const int gx = (int)(k % gnx), gy = (int)(k / gnx);
      if (lo >= 0) owed_lo.push_back({dl.djobs[k].node, leaf_index(gx, gy, dl.gz - 1)});
      if (hi < g.dims[2]) owed_hi.push_back({dl.djobs[k].node, leaf_index(gx, gy, dl.gz + 1)});
    }
  }
  ++deferred_layers;
  ++dense_leaf_inserts;
  dl.active = false;
  dl.seeds.clear();
}

// the layer is complete: one dense leaf kernel over the layer buffer
void Tree::finish_layer() {
  run_layer(false);
  close_layer();
}

// a reader needs the tree now: the leaves as the blocks received so far
// leave them (the same bytes the general path's held seeds + one scatter per
// block produce); the layer stays open for its remaining blocks unless
// `close` (a non-follower insertion arrives)
void Tree::materialize_layer(bool close) {
  if (!dl.active) return;
  if (dl.dirty) run_layer(true);
  if (close) close_layer();
}

// dense leaf launch from the current source: the planar block of a layer
// group / deferred layer (4-D TMA; 8-bit or unaligned planar sources are
// interleaved into a scratch block first), else the interleaved block
int Tree::leaf_launch(const void* dsrc, int64_t nsrc, int oz, int dz, int prefill,
                      const DenseJob* dj, int n, const int gn[3], int g0z) {
  if (!planar.active) return launch_dense_leaf(*this, dsrc, nsrc, oz, prefill, dj, n, gn, g0z);
  const int r = launch_dense_leaf_planar(*this, planar.base, planar.zstride, planar.cstride, oz, dz,
                                         prefill, dj, n, gn, g0z);
  if (r >= 0) return r;
  const int64_t need = (int64_t)dz * g.dims[1] * g.dims[0] * g.C * g.sb;
  if (need > d_acc_il_bytes) {
    if (d_acc_il) VT_CUDA(cudaFreeAsync(d_acc_il, stream));
    VT_CUDA(cudaMallocAsync(&d_acc_il, need, stream));
    d_acc_il_bytes = need;
  }
  launch_planar_to_interleaved(*this, planar.base, planar.zstride, planar.cstride, dz, d_acc_il);
  return launch_dense_leaf(*this, d_acc_il, need / g.sb, oz, prefill, dj, n, gn, g0z);
}

// ---------------------------------------------------------------------------
// batched insertion (vt_tree_insert_many)
// ---------------------------------------------------------------------------

// Blocks [i, i + len) form a complete brick layer group when, at threshold
// 0 with the dense path on and no deferred layer open, each is one channel's
// full-x/y block inside one brick layer over brick-less leaves and together
// they cover every (z, channel) of the layer exactly once.  Returns len, or
// 0 when block i starts no such group.
int64_t Tree::layer_group(int64_t i, int64_t n, const vt_block* blocks, int mem_kind) {
  const int* M = g.brick;
  if (!dense_enabled || tau != 0 || dl.active) return 0;
  auto fits = [&](const vt_block& b, int layer) {
    if (b.channel < 0 || b.channel >= g.C || !b.samples) return false;
    if (b.origin[0] != 0 || b.origin[1] != 0 || b.dims[0] != g.dims[0] || b.dims[1] != g.dims[1])
      return false;
    if (b.dims[2] <= 0 || b.origin[2] < 0 || (int64_t)b.origin[2] + b.dims[2] > g.dims[2]) return false;
    if (b.origin[2] / M[2] != (b.origin[2] + b.dims[2] - 1) / M[2]) return false;
    return layer < 0 || b.origin[2] / M[2] == layer;
  };
  if (!fits(blocks[i], -1)) return 0;
  const int layer = blocks[i].origin[2] / M[2];
  const int z0 = layer * M[2], nz = std::min(M[2], g.dims[2] - z0);
  const int gx1 = (g.dims[0] - 1) / M[0], gy1 = (g.dims[1] - 1) / M[1];
  for (int gy = 0; gy <= gy1; ++gy)
    for (int gx = 0; gx <= gx1; ++gx)
      if (flags[leaf_index(gx, gy, layer)] & NF_BRICK) return 0;
  std::vector<uint8_t> got((size_t)nz * g.C, 0);
  int64_t need = (int64_t)nz * g.C, j = i;
  while (need > 0 && j < n && fits(blocks[j], layer)) {
    const vt_block& b = blocks[j];
    bool fresh = true;
    for (int z = b.origin[2]; z < b.origin[2] + b.dims[2]; ++z)
      fresh = fresh && !got[(size_t)(z - z0) * g.C + b.channel];
    if (!fresh) break;
    for (int z = b.origin[2]; z < b.origin[2] + b.dims[2]; ++z) got[(size_t)(z - z0) * g.C + b.channel] = 1;
    need -= b.dims[2];
    ++j;
  }
  (void)mem_kind;
  return need == 0 ? j - i : 0;
}

// where a complete layer group's samples are: in place (the blocks sit at
// an affine (z, channel) stride) or gathered into the planar layer buffer
bool Tree::group_source(int64_t i, int64_t len, const vt_block* blocks, int mem_kind, bool gather,
                        PlanarSrc& src) {
  const int* M = g.brick;
  const int64_t plane = (int64_t)g.dims[0] * g.dims[1] * g.sb;
  const int layer = blocks[i].origin[2] / M[2];
  const int z0 = layer * M[2], nz = std::min(M[2], g.dims[2] - z0);
  if (mem_kind == VT_MEM_DEVICE) {
    auto at = [&](const vt_block& b, int z) {
      return (const uint8_t*)b.samples + (int64_t)(z - b.origin[2]) * plane;
    };
    const uint8_t *p00 = nullptr, *p10 = nullptr, *p01 = nullptr;
    for (int64_t k = i; k < i + len; ++k) {
      const vt_block& b = blocks[k];
      for (int z = b.origin[2]; z < b.origin[2] + b.dims[2]; ++z) {
        if (z == z0 && b.channel == 0) p00 = at(b, z);
        if (z == z0 + 1 && b.channel == 0) p10 = at(b, z);
        if (z == z0 && b.channel == 1) p01 = at(b, z);
      }
    }
    const int64_t zs = nz > 1 ? (int64_t)(p10 - p00) : plane;
    const int64_t cs = g.C > 1 ? (int64_t)(p01 - p00) : (int64_t)nz * plane;
    bool affine = zs > 0 && cs > 0;
    for (int64_t k = i; k < i + len && affine; ++k) {
      const vt_block& b = blocks[k];
      for (int z = b.origin[2]; z < b.origin[2] + b.dims[2] && affine; ++z)
        affine = at(b, z) == p00 + (int64_t)(z - z0) * zs + (int64_t)b.channel * cs;
    }
    if (affine && planar_leaf_ok(*this, p00, zs, cs)) {
      src = {true, p00, zs, cs};
      return true;
    }
  }
  if (!gather) return false;
  if (!d_acc) VT_CUDA(cudaMalloc(&d_acc, (size_t)M[2] * g.dims[1] * g.dims[0] * g.C * g.sb));
  for (int64_t k = i; k < i + len; ++k) {
    const vt_block& b = blocks[k];
    uint8_t* dst = d_acc + ((size_t)b.channel * M[2] + (b.origin[2] - z0)) * plane;
    VT_CUDA(cudaMemcpyAsync(dst, b.samples, plane * b.dims[2],
                            mem_kind == VT_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyHostToDevice,
                            stream));
  }
  src = {true, d_acc, plane, (int64_t)M[2] * plane};
  return false;
}

void Tree::insert_many(int64_t n, const vt_block* blocks, int mem_kind) {
  VT_CUDA(cudaSetDevice(device));
  if (prof.on)
    for (auto& e : prof.ev)
      if (!e) VT_CUDA(cudaEventCreate(&e));
  const int* M = g.brick;
  const int nlayers = (g.dims[2] - 1) / M[2] + 1;
  static const bool pairs_on = [] {
    const char* e = std::getenv("VT_LAYER_PAIRS");
    return !(e && e[0] == '0');
  }();
  int64_t i = 0;
  while (i < n) {
    const int64_t len = layer_group(i, n, blocks, mem_kind);
    if (len == 0) {
      const vt_block& b = blocks[i];
      VT_REQUIRE(b.channel >= 0, VT_EINVAL, "channel " + std::to_string(b.channel) + " out of range");
      insert(b.channel, b.origin, b.dims, b.samples, mem_kind);
      ++i;
      continue;
    }
    // one dense insertion per layer: the first block's walk and events,
    // then the same UPDATED list for each later block
    const int layer = blocks[i].origin[2] / M[2];
    PlanarSrc a{};
    const bool in_place = group_source(i, len, blocks, mem_kind, false, a);
    // an even layer read in place with its odd layer right behind it (also
    // in place, the same strides, contiguous in z): build the pair at once
    int64_t len2 = 0;
    PlanarSrc b{};
    if (pairs_on && in_place && (layer & 1) == 0 && layer + 1 < nlayers && i + len < n) {
      // the odd layer's leaves must be brick-less too: layer_group checks
      len2 = layer_group(i + len, n, blocks, mem_kind);
      const int nza = M[2];
      if (len2 > 0 && blocks[i + len].origin[2] / M[2] == layer + 1 &&
          group_source(i + len, len2, blocks, mem_kind, false, b) && b.zstride == a.zstride &&
          b.cstride == a.cstride && b.base == a.base + (int64_t)nza * a.zstride &&
          planar_leaf_ok(*this, a.base, a.zstride, a.cstride)) {
      } else {
        len2 = 0;
      }
    }
    if (!in_place) {
      group_source(i, len, blocks, mem_kind, true, a);
    } else {
      ++zero_copy_layers;
    }
    const int z0 = layer * M[2], nz = std::min(M[2], g.dims[2] - z0);
    const int o[3] = {0, 0, z0}, d[3] = {g.dims[0], g.dims[1], nz};
    planar = a;
    if (len2 == 0) {
      try {
        insert_staged(-1, o, d, a.base, g.C, 0, g.C, len);
      } catch (...) {
        planar = PlanarSrc{};
        throw;
      }
      planar = PlanarSrc{};
      ++layer_groups;
      i += len;
      continue;
    }
    // the pair: walk both (their events in order), then one leaf launch
    const int z1 = z0 + M[2], nz1 = std::min(M[2], g.dims[2] - z1);
    const int o1[3] = {0, 0, z1}, d1[3] = {g.dims[0], g.dims[1], nz1};
    hold_dense = true;
    leaf_struct_by_kernel = true;
    try {
      insert_staged(-1, o, d, a.base, g.C, 0, g.C, len);
      insert_staged(-1, o1, d1, b.base, g.C, 0, g.C, len2);
    } catch (...) {
      hold_dense = false;
      launch_held();  // whatever was walked must be built
      leaf_struct_by_kernel = false;
      planar = PlanarSrc{};
      throw;
    }
    hold_dense = false;
    launch_held();
    leaf_struct_by_kernel = false;
    planar = PlanarSrc{};
    layer_groups += 2;
    zero_copy_layers += 1;
    ++layer_pairs;
    i += len + len2;
  }
}

// ---------------------------------------------------------------------------
// propagation of dirty boxes up the tree
// ---------------------------------------------------------------------------

bool Tree::dense_parent(int64_t p) const {
  if (!dense_enabled || tau != 0) return false;
  if (!(flags[p] & NF_BRICK) || !(flags[p] & NF_CHILDREN)) return false;
  for (int k = 0; k < 8; ++k) {
    if (!g.octant_real(k)) continue;
    const int64_t c = 8 * p + 1 + k;
    if (!(flags[c] & NF_INVOL)) continue;
    if (!(flags[c] & NF_EXISTS) || !(flags[c] & NF_BRICK) || !complete[c]) return false;
  }
  return true;
}

void Tree::propagate() {
  if (!has_pending) return;
  ProfScope ps(prof, 4);
  VT_CUDA(cudaEventRecord(ev0, stream));
  const int* M = g.brick;
  for (int lvl = 0; lvl <= g.depth; ++lvl) {
    std::vector<int64_t>& nodes = pend_nodes[lvl];
    if (nodes.empty()) continue;
    if (!std::is_sorted(nodes.begin(), nodes.end())) sort_indices(nodes);
    std::vector<OctJob> oct;
    std::vector<int64_t> dense_nodes, fused_done;
    if (lvl > 0) {
      // dirty children are sorted: those of parent p are a contiguous run
      const std::vector<int64_t>& kids = pend_nodes[lvl - 1];
      size_t ci = 0;
      for (int64_t p : nodes) {
        Pending& pp = *pend_find(p, lvl);
        if (lvl == 1 && fused1[p] && dense_parent(p)) {
          // octants and accumulators written by the leaf kernel: only the
          // AVG and subtree extrema are owed (k_finish_fused)
          fused1[p] = 0;
          pp.box = Box{{0, 0, 0}, {M[0], M[1], M[2]}};
          pp.has_box = true;
          pp.dense = true;
          complete[p] = 1;
          fused_done.push_back(p);
          continue;
        }
        fused1[p] = 0;
        if (dense_parent(p)) {
          pinv[p] = 0;  // the dense level kernel writes every plane partial
          // every in-volume child complete: recompute the whole interior and
          // the statistics in one dense pass (dense_build.cu)
          dense_nodes.push_back(p);
          pp.box = Box{{0, 0, 0}, {M[0], M[1], M[2]}};
          pp.has_box = true;
          pp.dense = true;
          complete[p] = 1;
          continue;
        }
        complete[p] = 0;
        if (pinv[p]) {
          // a general-path parent over unmaintained partials: every plane
          pinv[p] = 0;
          pp.box = Box{{0, 0, 0}, {M[0], M[1], M[2]}};
          pp.has_box = true;
        }
        auto emit = [&](int64_t c, const Box* cb) {
          OctJob j{};
          j.pslot = slot[p];
          j.cslot = (flags[c] & NF_BRICK) ? slot[c] : -1;
          j.child = c;
          j.k = (int)((c - 1) & 7);
          node_in_extent(c, j.cext);
          Box pb;
          for (int a = 0; a < 3; ++a) {
            int kk = g.split[a] ? 2 : 1;
            int off = (((j.k >> a) & 1) && g.split[a]) ? M[a] / 2 : 0;
            if (cb) {
              j.r0[a] = cb->lo[a] / kk;
              j.r1[a] = (cb->hi[a] + kk - 1) / kk;
            } else {
              j.r0[a] = 0;
              j.r1[a] = M[a] / kk;
            }
            pb.lo[a] = off + j.r0[a];
            pb.hi[a] = off + j.r1[a];
          }
          if (j.r1[0] > j.r0[0] && j.r1[1] > j.r0[1] && j.r1[2] > j.r0[2]) {
            oct.push_back(j);
            box_union(pp, pb);
          }
        };
        while (ci < kids.size() && ((kids[ci] - 1) >> 3) < p) ++ci;
        if (pp.fresh) {
          // fresh parent brick: every real octant (octree.py:375-377)
          for (int k = 0; k < 8; ++k) {
            if (!g.octant_real(k)) continue;
            emit(8 * p + 1 + k, nullptr);
          }
          pp.box = Box{{0, 0, 0}, {M[0], M[1], M[2]}};
          pp.has_box = true;
        } else {
          for (size_t q = ci; q < kids.size() && ((kids[q] - 1) >> 3) == p; ++q) {
            const Pending& cp = *pend_find(kids[q], lvl - 1);
            if (cp.has_box) emit(kids[q], &cp.box);
          }
        }
      }
      ProfScope ql(prof, 11);
      OctJob* d = upload(*this, oct);
      launch_octant(*this, d, (int)oct.size());
      release(*this, d);
      int64_t* dfd = upload(*this, fused_done);
      launch_finish_fused(*this, dfd, (int)fused_done.size());
      release(*this, dfd);
      // nodes whose 8 children are full in-volume bricks take the
      // shared-memory kernel; the rest (volume edges) the general one
      std::vector<int64_t> dfull, dpart;
      if (level_smem_ok(*this)) {
        for (int64_t q : dense_nodes) {
          bool full = true;
          for (int k = 0; k < 8 && full; ++k) {
            const int64_t ch = 8 * q + 1 + k;
            if ((flags[ch] & (NF_EXISTS | NF_BRICK)) != (NF_EXISTS | NF_BRICK)) {
              full = false;
              break;
            }
            int ce[3];
            node_in_extent(ch, ce);
            full = ce[0] == M[0] && ce[1] == M[1] && ce[2] == M[2];
          }
          (full ? dfull : dpart).push_back(q);
        }
      } else {
        dpart = dense_nodes;
      }
      const int zsplit = dense_level_split(*this, (int)dense_nodes.size());
      int64_t* dd = upload(*this, dfull);
      launch_dense_level(*this, dd, (int)dfull.size(), zsplit, true);
      release(*this, dd);
      dd = upload(*this, dpart);
      launch_dense_level(*this, dd, (int)dpart.size(), zsplit, false);
      release(*this, dd);
      if (zsplit > 1)
        for (int64_t q : dense_nodes) {
          // plane partials written, statistics owed to the reduce below
          Pending& pq = *pend_find(q, lvl);
          pq.dense = false;
          pq.fused = true;
        }
      dense_level_nodes += (int64_t)dense_nodes.size();
    }
    // stats of this level's dirty nodes
    std::vector<PlaneJob> planes;
    std::vector<ReduceJob> reds;
    planes.reserve(nodes.size());
    reds.reserve(nodes.size());
    for (int64_t n : nodes) {
      const Pending& p = *pend_find(n, lvl);
      if (p.dense) continue;  // statistics written by the dense kernel
      ReduceJob r{};
      r.node = n;
      r.slot = slot[n];
      node_in_extent(n, r.cext);
      r.leafish = (lvl == 0 || !(flags[n] & NF_CHILDREN)) ? 1 : 0;
      if (p.has_box && r.cext[0] > 0 && r.cext[1] > 0 && !p.fused) {
        if (lvl == 0 && p.masked) {
          // runs of planes whose stats the scatter did not compute
          if (p.need[0] | p.need[1]) {
            int z = 0;
            while (z < r.cext[2]) {
              if (!p.needs(z)) {
                ++z;
                continue;
              }
              int e = z;
              while (e < r.cext[2] && p.needs(e)) ++e;
              planes.push_back({r.slot, z, e, r.cext[0], r.cext[1]});
              z = e;
            }
          }
        } else {
          int z1 = std::min(p.box.hi[2], r.cext[2]);
          if (z1 > p.box.lo[2]) planes.push_back({r.slot, p.box.lo[2], z1, r.cext[0], r.cext[1]});
        }
      }
      reds.push_back(r);
    }
    ProfScope ql(prof, 11);
    PlaneJob* dp = upload(*this, planes);
    launch_plane(*this, dp, (int)planes.size());
    ReduceJob* dr = upload(*this, reds);
    launch_reduce(*this, dr, (int)reds.size());
    release(*this, dp);
    release(*this, dr);
  }
  for (int lvl = 0; lvl <= g.depth; ++lvl) {
    for (int64_t i : pend_nodes[lvl]) pend_slot[i] = -1;
    pend_nodes[lvl].clear();
    pend_pool[lvl].clear();
  }
  has_pending = false;
  VT_CUDA(cudaEventRecord(ev1, stream));
}

void Tree::flush() {
  VT_CUDA(cudaSetDevice(device));
  materialize_layer(false);
  flush_structure();
  propagate();
}

void Tree::sync() {
  flush();
  VT_CUDA(cudaStreamSynchronize(stream));
  float ms = 0;
  if (cudaEventElapsedTime(&ms, ev0, ev1) == cudaSuccess) last_build_ms = ms;
  else cudaGetLastError();  // events never recorded (nothing ran): not an error
}

void Tree::gather_stats(const std::vector<int64_t>& nodes) {
  if (nodes.empty()) return;
  const size_t row = ST_N * kMaxC;
  int64_t* dn = upload(*this, nodes);
  int32_t* dout = nullptr;
  VT_CUDA(cudaMallocAsync(&dout, nodes.size() * row * sizeof(int32_t), stream));
  launch_gather_stats(*this, dn, (int)nodes.size(), dout);
  std::vector<int32_t> host(nodes.size() * row);
  VT_CUDA(cudaMemcpyAsync(host.data(), dout, host.size() * sizeof(int32_t),
                          cudaMemcpyDeviceToHost, stream));
  release(*this, dn);
  release(*this, dout);
  VT_CUDA(cudaStreamSynchronize(stream));
  for (size_t i = 0; i < nodes.size(); ++i)
    std::memcpy(&h_stats[nodes[i] * row], &host[i * row], row * sizeof(int32_t));
}

// ---------------------------------------------------------------------------
// pruning (octree.py:446-493), on the gathered statistics
// ---------------------------------------------------------------------------

void Tree::delete_below(int64_t p, std::vector<char>& mark, std::vector<int64_t>& deleted) {
  for (int k = 0; k < 8; ++k) {
    if (!g.octant_real(k)) continue;
    int64_t c = 8 * p + 1 + k;
    if (!(flags[c] & NF_EXISTS)) continue;
    if (flags[c] & NF_CHILDREN) delete_below(c, mark, deleted);
    free_brick(c);
    --node_count;
    flags[c] = 0;
    slot[c] = -1;
    mark_struct(c);
    deleted.push_back(c);
    events.push_back(ev_pack(VT_EV_DELETED, c));
  }
  flags[p] &= ~NF_CHILDREN;
  mark_struct(p);
}

void Tree::prune(std::vector<std::vector<int64_t>>& touched, std::vector<char>& mark,
                 std::vector<int64_t>& deleted) {
  auto homog = [&](int64_t n, int lo_stat, int hi_stat) {
    for (int c = 0; c < g.C; ++c)
      if (!((double)(stat(n, hi_stat, c) - stat(n, lo_stat, c)) < tau)) return false;
    return true;
  };
  // pass 1: bricks (ascending level, index)
  for (int lvl = 0; lvl <= g.depth; ++lvl)
    for (int64_t n : touched[lvl]) {
      if (n == 0 || !(flags[n] & NF_BRICK)) continue;
      if (homog(n, ST_MIN, ST_MAX)) free_brick(n);
    }
  // pass 2: homogeneous subtrees
  for (int lvl = 1; lvl <= g.depth; ++lvl)
    for (int64_t n : touched[lvl]) {
      if (n == 0 || !(flags[n] & NF_EXISTS) || !(flags[n] & NF_CHILDREN)) continue;
      bool sub_h = !(flags[n] & NF_INVOL) || homog(n, ST_SUBMIN, ST_SUBMAX);
      if (sub_h) delete_below(n, mark, deleted);
    }
  // root: collapse only when the whole tree is homogeneous
  if (homog(0, ST_SUBMIN, ST_SUBMAX) && ((flags[0] & NF_CHILDREN) || (flags[0] & NF_BRICK))) {
    if (flags[0] & NF_CHILDREN) delete_below(0, mark, deleted);
    free_brick(0);
  }
}

// ---------------------------------------------------------------------------
// borders (octree.py:540-614)
// ---------------------------------------------------------------------------

void Tree::fill_borders() {
  ProfScope pf(prof, 3);
  flush();
  ++data_version;
  touch_all();
  std::vector<BorderJob> jobs;
  static thread_local std::vector<int64_t> bricks;  // scratch: every brick, BFS order
  bricks.resize(g.capacity);  // an upper bound; the scratch keeps its pages
  {
    size_t nb = 0;
    for (int64_t i = 0; i < g.capacity; ++i)
      if ((flags[i] & (NF_EXISTS | NF_BRICK)) == (NF_EXISTS | NF_BRICK)) bricks[nb++] = i;
    bricks.resize(nb);
  }
  // Fast path: every in-volume leaf complete and every leaf shell prefilled
  // by the dense build (dense_build.cu) with nothing mutated since.  Then
  // each leaf shell already holds its fill_borders value except owed z-shell
  // planes, which equal the z-neighbour's adjacent stored plane (shell
  // included — the neighbour's x/y shell is the same volume voxels).
  const bool fast = halo_prefill && prefill_valid && !borders && complete[0];
  if (fast) {
    ++fast_borders;
    std::vector<int32_t> pj;
    const int mz = g.brick[2];
    pj.reserve(4 * (owed_lo.size() + owed_hi.size()));
    auto add = [&](const Owed& o, int dz_) {
      VT_REQUIRE((flags[o.nb] & NF_BRICK), VT_ESTATE, "fill_borders: neighbour brick missing");
      pj.insert(pj.end(), {slot[o.leaf], dz_ < 0 ? 0 : mz + 1, slot[o.nb], dz_ < 0 ? mz : 1});
    };
    for (const Owed& o : owed_lo) add(o, -1);
    for (const Owed& o : owed_hi) add(o, +1);
    int32_t* dp = upload(*this, pj);
    launch_plane_copy(*this, dp, (int)(pj.size() / 4));
    release(*this, dp);
    if (!upper_borders)
      for (int64_t i : bricks)
        if (g.level_of(i) > 0) jobs.push_back({i, slot[i], skipx(i) ? 1 : 0});
  } else {
    for (int64_t i : bricks) jobs.push_back({i, slot[i]});
  }
  BorderJob* d = upload(*this, jobs);
  launch_borders(*this, d, (int)jobs.size());
  release(*this, d);
  {
    const size_t e0 = events.size();
    events.resize(e0 + bricks.size());
    uint64_t* ev = events.data() + e0;
    for (size_t k = 0; k < bricks.size(); ++k) ev[k] = ev_pack(VT_EV_UPDATED, bricks[k]);
  }
  borders = true;
  halo_prefill = false;
  if (!pshell.empty()) std::fill(pshell.begin(), pshell.end(), 0);
  owed_shells.clear();  // every level > 0 brick's shell was just written
  upper_borders = false;
  owed_lo.clear();
  owed_hi.clear();
}

// Prefilled leaf shells are the reference's background until fill_borders:
// any reader of pool shells first resets them (then fill_borders takes the
// general path).
void Tree::publish_halos() {
  const bool ps = !pshell.empty();
  if ((!halo_prefill && owed_shells.empty() && !upper_borders && !ps) || borders) return;
  flush();
  std::vector<int32_t> sl;
  if (halo_prefill || upper_borders || ps)
    for (int64_t i = 0; i < g.capacity; ++i)
      if ((flags[i] & NF_EXISTS) && (flags[i] & NF_BRICK) &&
          (g.level_of(i) == 0 ? halo_prefill : (upper_borders || (ps && pshell[i]))))
        sl.push_back(slot[i]);
  if (ps) pshell.clear();
  upper_borders = false;
  sl.insert(sl.end(), owed_shells.begin(), owed_shells.end());
  owed_shells.clear();
  int32_t* d = upload(*this, sl);
  launch_clear_shells(*this, d, (int)sl.size());
  release(*this, d);
  ++data_version;
  touch_all();
  halo_prefill = false;
  prefill_valid = false;
  owed_lo.clear();
  owed_hi.clear();
}

// ---------------------------------------------------------------------------
// z-slab sharded build: merge node records of complete subtrees
// ---------------------------------------------------------------------------

void Tree::merge(int64_t n, const int64_t* idx, const int32_t* nflags, const int32_t* stats_in,
                 const void* bricks, int mem_kind, int64_t inserted_voxels) {
  publish_halos();
  prefill_valid = false;
  flush();
  ++data_version;
  touch_all();
  const int C = g.C;
  std::vector<int64_t> order(n);
  for (int64_t r = 0; r < n; ++r) order[r] = r;
  // parents before children (BFS order)
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return idx[a] < idx[b]; });
  creates.clear();
  seeds.clear();
  clear_seed_of();
  std::vector<int64_t> rec_nodes;
  std::vector<int32_t> rec_stats;
  std::vector<int32_t> brick_slots;
  std::vector<int64_t> brick_src;  // record row of each incoming brick
  std::vector<int64_t> brick_row(n, -1);
  int64_t nb = 0;
  for (int64_t r = 0; r < n; ++r)
    if (nflags[r] & VT_NODE_BRICK) brick_row[r] = nb++;
  int top = -1;  // highest level among the records
  for (int64_t q = 0; q < n; ++q) {
    const int64_t r = order[q];
    const int64_t i = idx[r];
    VT_REQUIRE(i > 0 && i < g.capacity, VT_EINVAL, "merge: node index outside the tree");
    const int lvl = g.level_of(i);
    top = std::max(top, lvl);
    // the ancestor chain exists exactly as an insertion walk would leave it
    {
      std::vector<int64_t> chain;
      for (int64_t a = (i - 1) >> 3; ; a = (a - 1) >> 3) {
        chain.push_back(a);
        if (a == 0) break;
      }
      for (auto it = chain.rbegin(); it != chain.rend(); ++it) ensure_children(*it);
    }
    VT_REQUIRE(flags[i] & NF_EXISTS, VT_EINVAL, "merge: record is not a real octant");
    // the record replaces the placeholder that stood here (a brick-less,
    // childless sibling created by an insertion walk elsewhere)
    const int f = nflags[r];
    VT_REQUIRE(!(flags[i] & NF_CHILDREN) || (f & VT_NODE_CHILDREN), VT_EINVAL,
               "merge: record would drop an existing subtree");
    if (f & VT_NODE_CHILDREN) ensure_children(i);  // children records follow
    const bool want_brick = f & VT_NODE_BRICK;
    if (want_brick && !(flags[i] & NF_BRICK)) {
      const int32_t s = alloc_slot();
      flags[i] |= NF_BRICK;
      slot[i] = s;
      ++brick_count;
    } else if (!want_brick && (flags[i] & NF_BRICK)) {
      free_slots.push(slot[i]);
      flags[i] &= ~NF_BRICK;
      slot[i] = -1;
      --brick_count;
    }
    mark_struct(i);
    if (want_brick) {
      brick_slots.push_back(slot[i]);
      brick_src.push_back(brick_row[r]);
    }
    rec_nodes.push_back(i);
    complete[i] = 0;
    pinv[i] = 0;  // merge recomputes every plane of incoming bricks
    for (int s2 = 0; s2 < ST_N; ++s2)
      for (int c = 0; c < kMaxC; ++c) {
        const int v = c < C ? stats_in[(r * C + c) * ST_N + s2] : 0;
        rec_stats.push_back(v);
        h_stats[st_index(i, s2, c)] = v;
      }
  }
  // ancestors above the merged subtrees: bricks, then a fresh recompute of
  // every real octant, level by level (octree.py:372-387 with fresh parents)
  std::vector<int64_t> anc;
  for (int64_t i : rec_nodes)
    for (int64_t a = (i - 1) >> 3; ; a = (a - 1) >> 3) {
      if (g.level_of(a) > top) anc.push_back(a);
      if (a == 0) break;
    }
  std::sort(anc.begin(), anc.end());
  anc.erase(std::unique(anc.begin(), anc.end()), anc.end());
  for (int64_t a : anc) {
    if (ensure_brick(a)) {
      SeedJob& sj = seeds.back();
      for (int d = 0; d < 3; ++d) {
        sj.cov_lo[d] = 0;
        sj.cov_hi[d] = g.brick[d];
      }
    }
    Pending& p = pend(g.level_of(a), a);
    p.fresh = true;
    has_pending = true;
  }
  flush_structure();
  CreateJob* dc = upload(*this, creates);
  launch_create(*this, dc, (int)creates.size());
  release(*this, dc);
  SeedJob* ds = upload(*this, seeds);
  launch_seed(*this, ds, (int)seeds.size());
  release(*this, ds);
  // record stats + bricks
  if (!rec_nodes.empty()) {
    int64_t* dn = upload(*this, rec_nodes);
    int32_t* dst = upload(*this, rec_stats);
    launch_set_stats(*this, dn, (int)rec_nodes.size(), dst);
    release(*this, dn);
    release(*this, dst);
  }
  if (!brick_slots.empty()) {
    const int64_t bb = g.brick_elems * g.sb;
    const uint8_t* src = static_cast<const uint8_t*>(bricks);
    uint8_t* staged = nullptr;
    if (mem_kind == VT_MEM_HOST) {
      VT_CUDA(cudaMallocAsync(&staged, nb * bb, stream));
      VT_CUDA(cudaMemcpyAsync(staged, bricks, nb * bb, cudaMemcpyHostToDevice, stream));
      src = staged;
    }
    // incoming bricks are in record order; scatter row brick_src[j] -> slot
    std::vector<int32_t> slots_by_row(nb, -1);
    for (size_t j = 0; j < brick_slots.size(); ++j) slots_by_row[brick_src[j]] = brick_slots[j];
    int32_t* dsl = upload(*this, slots_by_row);
    launch_scatter_bricks(*this, dsl, (int)nb, src);
    release(*this, dsl);
    if (staged) release(*this, staged);
    std::vector<PlaneJob> planes;
    for (int64_t i : rec_nodes)
      if (flags[i] & NF_BRICK) {
        int ce[3];
        node_in_extent(i, ce);
        if (ce[0] > 0 && ce[1] > 0 && ce[2] > 0) planes.push_back({slot[i], 0, ce[2], ce[0], ce[1]});
      }
    PlaneJob* dp = upload(*this, planes);
    launch_plane(*this, dp, (int)planes.size());
    release(*this, dp);
    if (mem_kind == VT_MEM_HOST) VT_CUDA(cudaStreamSynchronize(stream));
  }
  inserted += inserted_voxels;
  propagate();
}

int64_t Tree::find_node(const double pt[3], int target) const {
  int64_t idx = 0;
  int lvl = g.depth;
  int lo[3] = {0, 0, 0};
  while (lvl > target && (flags[idx] & NF_CHILDREN)) {
    int k = 0;
    for (int a = 0; a < 3; ++a) {
      int half = g.extent(a, lvl - 1);
      if (g.split[a] && pt[a] >= lo[a] + half) {
        k |= 1 << a;
        lo[a] += half;
      }
    }
    idx = 8 * idx + 1 + k;
    --lvl;
  }
  return idx;
}

}  // namespace vtx
