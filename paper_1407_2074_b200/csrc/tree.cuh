// Host-side octree control plane (structure, slots, events, pruning) over a
// device-resident brick pool and node-stat arrays.  Replaces voxtree's
// Octree (octree.py:143-614) + BrickStore (paging.py) for the hot path.
#pragma once

#include <algorithm>
#include <climits>
#include <array>
#include <atomic>
#include <chrono>
#include <deque>
#include <memory>
#include <queue>
#include <unordered_map>
#include <vector>

#include "vtx_common.cuh"

namespace vtx {

struct Box {
  int lo[3], hi[3];  // brick-interior voxel coords, [lo, hi)
};

struct Pending {
  Box box;
  bool has_box = false;
  bool fresh = false;
  // statistics already final (written by a dense-build kernel): no plane /
  // reduce work owed.  Any later general-path touch clears it.
  bool dense = false;
  // level-1 octants and plane partials written by the leaf kernel (fused)
  bool fused = false;
  // leaves: planes whose partial stats are still owed (bit z); planes whose
  // stats the scatter computed in-kernel are cleared (requires Mz <= 128)
  bool masked = false;
  uint64_t need[2] = {0, 0};
  void set_need(int z, bool v) {
    uint64_t bit = 1ULL << (z & 63);
    if (v) need[z >> 6] |= bit;
    else need[z >> 6] &= ~bit;
  }
  // planes [z0, z1) at once
  void set_need_range(int z0, int z1, bool v) {
    for (int w = 0; w < 2; ++w) {
      const int lo = std::max(z0, w * 64), hi = std::min(z1, w * 64 + 64);
      if (lo >= hi) continue;
      const int n = hi - lo;
      const uint64_t m = (n == 64 ? ~0ULL : ((1ULL << n) - 1)) << (lo - w * 64);
      if (v) need[w] |= m;
      else need[w] &= ~m;
    }
  }
  bool needs(int z) const { return (need[z >> 6] >> (z & 63)) & 1; }
};

// optional host-side phase timing (env VT_HOST_PROFILE=1), printed when the
// tree is destroyed
struct HostProf {
  bool on = false;
  static constexpr int kN = 40;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // insert entry, leaf launch, leaf end, insert end
  bool ev_armed = false;
  double t[kN] = {0};
  static const char* name(int i) {
    static const char* n[kN] = {"insert", "walk", "enqueue", "fill_borders", "propagate", "flush_struct",
                                "seed", "scatter", "leaves", "ancestors", "prop_build", "prop_launch",
                                "early_pre", "anc_collect", "anc_brick", "sort_leaves",
                                "dense_book", "updated_ev", "defer", "pool",
                                "gpu_entry_to_leaf", "gpu_leaf", "gpu_leaf_to_end",
                                "eligible", "pre_parents", "pre_anc", "pre_djobs",
                                "pre_pads", "pre_fused_up", "pre_djob_up", "pre_leaf_launch",
                                "chain", "leaf_brick", "fused_scan", "touch", "held", "owed",
                                "tau_gather", "tau_prune", "tau_flush"};
    return n[i];
  }
};
struct ProfScope {
  HostProf& p;
  int i;
  std::chrono::steady_clock::time_point t0;
  ProfScope(HostProf& p_, int i_) : p(p_), i(i_) {
    if (p.on) t0 = std::chrono::steady_clock::now();
  }
  ~ProfScope() {
    if (p.on)
      p.t[i] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                    .count();
  }
};

struct Tree {
  HostProf prof;
  Geo g{};
  double tau = 0;
  int fmax = 255;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  // -- host structure (authoritative) --
  std::vector<uint8_t> flags;
  std::vector<int32_t> slot;
  int64_t node_count = 1, brick_count = 0, pruned = 0, inserted = 0;
  bool finished = false, borders = false;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_slots;
  int64_t cursor = 0;
  int64_t data_version = 0;  // bumped by every pool mutation
  // data_version of each pool slot's last write (every slot changed at
  // all_ver or later): renderers refresh derived per-brick data (brick
  // maxima) for the changed slots only
  std::vector<int64_t> slot_ver;
  int64_t all_ver = 0;
  void touch_slot(int32_t s) {
    if (s >= 0 && (size_t)s < slot_ver.size()) slot_ver[s] = data_version;
  }
  void touch_all() { all_ver = data_version; }
  // Brick maxima for the renderer's exact empty-space skip (render.cu):
  // [bmax_cap][bmax_nsb][kMaxC] sub-brick maxima, then [bmax_cap][kMaxC]
  // whole-brick maxima, per channel, over every stored voxel a trilinear
  // corner can touch.  Allocated by the first zero-copy mirror; the dense
  // leaf kernels write a leaf's brick maxima as they build it (its
  // sub-brick maxima become "unknown", 0xFFFF), so a live stream's refresh
  // re-reads only the bricks written by other kernels.  bmax_ver[s]: the
  // data_version at which slot s's maxima were last made valid.
  uint16_t* d_bmax = nullptr;
  int64_t bmax_cap = 0;
  int bmax_nsb = 0;
  std::vector<int64_t> bmax_ver;
  uint16_t* bmax_brick() const {
    return d_bmax ? d_bmax + bmax_cap * bmax_nsb * kMaxC : nullptr;
  }
  void enable_bmax(int nsb);
  void leaves_bmax_valid(const std::vector<DenseJob>& djobs) {
    for (const DenseJob& jd : djobs)
      if (jd.slot >= 0 && (size_t)jd.slot < bmax_ver.size()) bmax_ver[jd.slot] = data_version;
  }
  // tau == 0 dense build (dense_build.cu): complete[n] = every in-volume leaf
  // under n was fully covered by one dense insertion, so n's brick is a pure
  // function of the data; VT_DENSE=0 disables the path (A/B testing)
  bool dense_enabled = true;
  std::vector<uint8_t> complete;
  std::vector<uint8_t> fused1;  // level-1 parent whose octants the leaf kernel wrote
  // per-plane partial statistics not maintained (TMA dense leaves, fused
  // parents): a later general-path touch recomputes every plane first
  std::vector<uint8_t> pinv;
  // [capacity][C] fused-parent accumulators (lazy)
  unsigned long long* d_nsum = nullptr;
  int32_t *d_nmin = nullptr, *d_nmax = nullptr;
  int32_t create_skip_z0 = 0, create_skip_z1 = -1;  // CreateJob skip range (dense)
  std::vector<int64_t> morton[3];
  // shells of dense leaves written with their fill_borders values at
  // insertion (dense_build.cu).  While !borders they are logically the
  // background: every reader of pool shells calls publish_halos() first.
  bool prefill_enabled = true;   // env VT_PREFILL=0 / a device mirror turns it off
  bool halo_prefill = false;     // some leaf shells hold prefilled values
  bool prefill_valid = true;     // no general-path mutation since (fast fill_borders)
  // leaves whose z-shell plane awaits a neighbour: (leaf, z-neighbour leaf)
  struct Owed { int64_t leaf, nb; };
  std::vector<Owed> owed_lo, owed_hi;
  // fresh level >= 1 bricks of an early dense launch whose background shell
  // is not written at insertion: fill_borders overwrites every shell voxel
  // of those bricks anyway, and publish_halos() writes the background first
  // if anything reads the pool before it
  std::vector<int32_t> owed_shells;
  // level > 0 shells already hold their fill_borders values (computed right
  // after a whole-volume dense insertion, overlapping its host epilogue);
  // logically background until fill_borders, as halo_prefill
  bool upper_borders = false;
  void publish_halos();

  // Threshold-0 slice streams (ingest_stream's VSTR order: per z, one
  // single-channel full-x/y block per channel).  The first block of a fresh
  // brick layer runs the ordinary host walk (structure, slots, events) with
  // its leaf seeds and scatter held back; later blocks of that layer only
  // append the same UPDATED events and land in a device layer buffer; a
  // complete layer is built by the dense leaf kernel.  Any reader (flush)
  // first materialises a partial layer through the general path: the held
  // seeds and one scatter per received block, in arrival order — exactly
  // the device work the general path would have done.
  struct DeferredLayer {
    bool active = false;
    int gz = 0, z0 = 0, nz = 0, remaining = 0;
    std::vector<uint8_t> got;                // [nz][C] blocks received
    std::vector<SeedJob> seeds;              // held leaf seeds
    std::vector<int32_t> leaf_slots;         // (gy, gx) order
    std::vector<DenseJob> djobs;             // (gy, gx) order
    std::vector<std::array<int, 3>> order;   // (z, dz, channel) in arrival order
    std::vector<int64_t> upd;                // one block's UPDATED list
    bool dirty = false;                      // blocks received since the last leaf launch
    bool prefilled = false;                  // the last leaf launch prefilled shells
  } dl;
  bool defer_enabled = true;    // env VT_DEFER=0 turns it off
  bool defer_start = false;     // set by try_defer: this insertion opens a layer
  uint8_t* d_acc = nullptr;     // [C][Mz][Y][X] planar layer buffer (lazy)
  uint8_t* d_acc_il = nullptr;  // interleaved scratch for the non-TMA leaf kernels (lazy)
  int64_t d_acc_il_bytes = 0;
  int64_t deferred_layers = 0, layer_groups = 0, zero_copy_layers = 0;
  bool try_defer(int channel, const int origin[3], const int dims[3], const void* dsrc,
                 int src_stride, int src_off);
  void defer_copy(int channel, const int origin[3], const int dims[3], const void* dsrc);
  // a reader needs the tree: launch the leaf kernel over the received planes
  // (missing ones are the background seeds); `close` ends the layer (a
  // non-follower insertion arrives)
  void materialize_layer(bool close = false);
  void run_layer(bool partial);
  void close_layer();
  void finish_layer();
  // planar source of the current dense insertion (insert_many layer groups):
  // sample (x, y, z, c) at base + c*cstride + (z - oz)*zstride + (y*X + x)*sb
  struct PlanarSrc {
    bool active = false;
    const uint8_t* base = nullptr;
    int64_t zstride = 0, cstride = 0;
  } planar;
  // dense leaf launch from the current source (planar if set, else the
  // interleaved block at dsrc)
  int leaf_launch(const void* dsrc, int64_t nsrc, int oz, int dz, int prefill, const DenseJob* dj,
                  int n, const int gn[3], int g0z);
  // Layer pairs (insert_many): the even brick layer's walk holds its leaf
  // launch; the odd layer's walk adds its leaves and one leaf kernel builds
  // both layers, writing every level-1 parent's octants on the fly (fused
  // half-sample, as a two-layer block) instead of re-reading the leaves in
  // propagate.  Events are the per-layer walks' events.
  struct HeldDense {
    bool active = false;
    std::vector<DenseJob> djobs;  // (gz, gy, gx) order
    int z0 = 0, nz = 0, gz0 = 0, gz1 = 0;
  } held;
  bool hold_dense = false;
  // while a pair is walked: in-volume leaves get no per-node structure
  // record — the pair's leaf kernel writes their device flags and slots
  bool leaf_struct_by_kernel = false;
  // level-1 parents whose x-face shell rows a leaf kernel already wrote with
  // their fill_borders values (bit 1): k_borders skips those two segments;
  // logically background until fill_borders like every prefilled shell
  std::vector<uint8_t> pshell;
  bool parent_shells_next = false;  // the next interleaved TMA leaf launch writes them
  // interior fused level-1 parents (the leaf kernels' `pxy` rule; `xoff_ok`:
  // the interleaved kernel's staged row also reaches two voxels past the brick)
  bool parent_interior(int64_t p, bool interleaved) const;
  // after a leaf launch that wrote the x-face shells of `nodes`' interior
  // parents: mark them
  void mark_parent_shells(const std::vector<int64_t>& nodes, bool interleaved);
  bool skipx(int64_t i) const { return !pshell.empty() && (pshell[i] & 1); }
  void launch_held();
  // bookkeeping after a dense leaf launch over leaves `djobs` of the block
  // z in [z0, z1), layers [gz0, gz1]
  void dense_after_launch(int lr, const std::vector<DenseJob>& djobs,
                          const std::vector<int64_t>& fused_nodes, int z0, int z1, int gz0,
                          int gz1, const std::vector<int64_t>* sorted_leaves,
                          bool pend_leaves = true);
  // B200 batched insertion: same tree and queued events as n successive
  // insert() calls; whole brick layers of single-channel full-x/y blocks
  // become one dense insertion
  void insert_many(int64_t n, const vt_block* blocks, int mem_kind);
  int64_t layer_group(int64_t i, int64_t n, const vt_block* blocks, int mem_kind);
  bool group_source(int64_t i, int64_t len, const vt_block* blocks, int mem_kind, bool gather,
                    PlanarSrc& src);
  int64_t layer_pairs = 0;
  int64_t leaf_index(int gx, int gy, int gz) const {
    return g.level_start[g.depth] + morton[0][gx] + morton[1][gy] + morton[2][gz];
  }
  int64_t dense_leaf_inserts = 0, dense_level_nodes = 0, fast_borders = 0;

  // -- device state --
  uint8_t* d_pool = nullptr;  // [pool_slots][Sz][Sy][Sx][C] samples
  int64_t pool_slots = 0;
  uint8_t* d_flags = nullptr;
  int32_t* d_slot = nullptr;
  int32_t* d_stats = nullptr;  // [capacity][5][4]
  int32_t* d_pmin = nullptr;   // [pool_slots][Mz][C] plane partials
  int32_t* d_pmax = nullptr;
  unsigned long long* d_psum = nullptr;

  // -- host stat cache (valid for nodes gathered since last device change) --
  std::vector<int32_t> h_stats;

  // -- events (octree.py:41-50) --
  // packed (kind << 56 | node index): 8 bytes per event, a whole-volume
  // insertion emits ~4 per node
  std::vector<uint64_t> events;
  // Change events are queued in order as sealed chunks, then the open tail
  // `events`.  A chunk is a shared list repeated `reps` times: the UPDATED
  // list every later block of a brick layer repeats (a 2048^2 slice of 32^3
  // bricks updates ~5.5k nodes, a cfg3 stream ~16M events) is stored once
  // and expanded only when the events are taken.
  struct EvChunk {
    std::shared_ptr<std::vector<uint64_t>> list;
    int64_t reps = 1;
    int64_t done = 0;  // expanded elements already taken
    int64_t left() const { return (int64_t)list->size() * reps - done; }
  };
  std::deque<EvChunk> ev_q;
  void seal_events() {
    if (events.empty()) return;
    ev_q.push_back({std::make_shared<std::vector<uint64_t>>(std::move(events)), 1, 0});
    events.clear();
  }
  void push_replay(const std::shared_ptr<std::vector<uint64_t>>& l, int64_t reps) {
    if (reps <= 0 || !l || l->empty()) return;
    if (events.empty() && !ev_q.empty() && ev_q.back().list == l && ev_q.back().done == 0) {
      ev_q.back().reps += reps;
      return;
    }
    seal_events();
    ev_q.push_back({l, reps, 0});
  }
  int64_t event_total() const {
    int64_t n = (int64_t)events.size();
    for (const EvChunk& c : ev_q) n += c.left();
    return n;
  }
  // move up to cap events out, oldest first; returns how many
  int64_t take_events(int32_t* kinds, int64_t* indices, int64_t cap) {
    int64_t m = 0;
    while (m < cap && !ev_q.empty()) {
      EvChunk& c = ev_q.front();
      const int64_t L = (int64_t)c.list->size();
      while (m < cap && c.left() > 0) {
        const int64_t j = c.done % L;
        const int64_t n = std::min(cap - m, L - j);
        const uint64_t* src = c.list->data() + j;
        for (int64_t k = 0; k < n; ++k) {
          kinds[m + k] = ev_kind(src[k]);
          indices[m + k] = ev_index(src[k]);
        }
        c.done += n;
        m += n;
      }
      if (c.left() == 0) ev_q.pop_front();
    }
    if (m < cap && !events.empty()) {
      const int64_t n = std::min<int64_t>(cap - m, (int64_t)events.size());
      for (int64_t k = 0; k < n; ++k) {
        kinds[m + k] = ev_kind(events[k]);
        indices[m + k] = ev_index(events[k]);
      }
      if (n == (int64_t)events.size()) events.clear();
      else events.erase(events.begin(), events.begin() + n);
      m += n;
    }
    return m;
  }
  // take every queued event without expanding replayed lists: returns the
  // event count, appends the NODE_DELETED indices (in order) to `deleted`
  int64_t discard_events(std::vector<int64_t>& deleted) {
    int64_t m = 0;
    for (EvChunk& c : ev_q) {
      const int64_t L = (int64_t)c.list->size(), left = c.left();
      m += left;
      bool any = false;  // replayed lists are UPDATED runs: usually no deletions
      for (int64_t k = 0; k < L && !any; ++k) any = ev_kind((*c.list)[k]) == VT_EV_DELETED;
      if (!any) continue;
      for (int64_t k = 0; k < left; ++k) {
        const uint64_t e = (*c.list)[(c.done + k) % L];
        if (ev_kind(e) == VT_EV_DELETED) deleted.push_back(ev_index(e));
      }
    }
    ev_q.clear();
    for (uint64_t e : events)
      if (ev_kind(e) == VT_EV_DELETED) deleted.push_back(ev_index(e));
    m += (int64_t)events.size();
    events.clear();
    return m;
  }
  // copy queued events [from, from + n) (oldest = 0) without taking them
  void copy_events(int64_t from, int64_t n, int32_t* kinds, int64_t* indices) const {
    int64_t pos = 0, m = 0;
    auto emit = [&](uint64_t e) {
      kinds[m] = ev_kind(e);
      indices[m] = ev_index(e);
      ++m;
    };
    for (const EvChunk& c : ev_q) {
      const int64_t len = c.left();
      if (pos + len > from && m < n) {
        const int64_t L = (int64_t)c.list->size();
        for (int64_t k = std::max<int64_t>(0, from - pos); k < len && m < n; ++k)
          emit((*c.list)[(c.done + k) % L]);
      }
      pos += len;
    }
    for (int64_t k = std::max<int64_t>(0, from - pos); k < (int64_t)events.size() && m < n; ++k)
      emit(events[k]);
  }
  std::shared_ptr<std::vector<uint64_t>> dl_upd_ev;  // a deferred layer's UPDATED events
  static uint64_t ev_pack(int32_t kind, int64_t idx) {
    return ((uint64_t)(uint32_t)kind << 56) | (uint64_t)idx;
  }
  static int32_t ev_kind(uint64_t e) { return (int32_t)(e >> 56); }
  static int64_t ev_index(uint64_t e) { return (int64_t)(e & ((1ULL << 56) - 1)); }

  // -- deferred propagation (tau == 0 batches; tau > 0 per insertion) --
  // dirty nodes per level: pend_nodes[lvl] lists them, pend_slot[node]
  // indexes pend_pool[lvl] (-1 = clean); flat arrays, no hashing
  std::vector<std::vector<int64_t>> pend_nodes;
  std::vector<std::vector<Pending>> pend_pool;
  std::vector<int32_t> pend_slot;
  bool has_pending = false;
  // Leaves a dense kernel wrote share one pending state (full box, fresh,
  // statistics final): pend_slot = -2, no per-leaf entry unless a general
  // insertion touches the leaf before the next propagation.
  Pending dense_pending;
  void pend_dense(int64_t idx) {  // level 0
    int32_t& k = pend_slot[idx];
    if (k == -1) {
      k = -2;
      pend_nodes[0].push_back(idx);
    } else if (k >= 0) {
      pend_pool[0][k] = dense_pending;
    }
  }
  Pending& pend(int lvl, int64_t idx) {
    int32_t& k = pend_slot[idx];
    if (k < 0) {
      const bool was_dense = k == -2;
      k = (int32_t)pend_pool[lvl].size();
      pend_pool[lvl].push_back(was_dense ? dense_pending : Pending{});
      if (!was_dense) pend_nodes[lvl].push_back(idx);
    }
    return pend_pool[lvl][k];
  }
  Pending* pend_find(int64_t idx, int lvl) {
    const int32_t k = pend_slot[idx];
    return k >= 0 ? &pend_pool[lvl][k] : (k == -2 ? &dense_pending : nullptr);
  }

  // complete-grid whole-volume insertion (every node in volume, every
  // created node's statistics rewritten by the dense kernels before anything
  // reads them): ensure_children skips the CreateJob / seed bookkeeping, and
  // structure records are one dirty index range
  bool fast_create = false;
  bool struct_range = false;
  int64_t struct_lo = INT64_MAX, struct_hi = -1;
  void ensure_children_at(int64_t p, int lvl, const int gg[3]);
  // -- per-insertion device work lists --
  std::vector<int64_t> struct_dirty;
  std::vector<uint8_t> struct_mark;
  std::vector<CreateJob> creates;
  std::vector<SeedJob> seeds;
  // node created this insertion -> its seed source (flat, reset per insertion)
  std::vector<int64_t> seed_of, seed_marked;
  void clear_seed_of();
  std::vector<uint32_t> anc_mark;  // ancestor dedupe, generation stamped
  uint32_t anc_gen = 0;

  // pinned host -> device staging ring for job lists (no implicit syncs of
  // pageable copies; wraps only after the stream has drained the old data)
  struct Staging {
    uint8_t* h = nullptr;
    uint8_t* d = nullptr;
    size_t cap = 0, head = 0;
  };
  mutable Staging stage;
  void* stage_copy(const void* src, size_t bytes) const;
  bool is_staged(const void* p) const {
    return stage.d && p >= (const void*)stage.d && p < (const void*)(stage.d + stage.cap);
  }

  // timing of the last build flush (CUDA events)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // side stream for the small structure kernels of an early dense launch
  // (flags/slots, chain creation, ancestor shells): they overlap the leaf
  // kernel instead of queueing behind it; the main stream joins right after
  cudaStream_t aux = nullptr;
  cudaStream_t main_saved = nullptr;  // the tree stream while `stream` is aux
  cudaEvent_t ev_pre = nullptr, ev_aux = nullptr;
  cudaEvent_t ev_wait = nullptr;    // cross-stream ordering (vt_tree_wait_stream)
  cudaEvent_t ev_signal = nullptr;  // (vt_tree_signal_stream)
  double last_build_ms = 0, last_render_ms = 0;

  Tree(const vt_tree_desc& d);
  ~Tree();

  // structure helpers
  bool in_volume(int64_t idx) const;
  void mark_struct(int64_t idx);
  int32_t alloc_slot();
  void ensure_pool(int64_t slots_needed);
  void ensure_children(int64_t p);
  bool ensure_brick(int64_t n, const int* cext = nullptr, bool seed = true);
  void node_in_extent(int64_t idx, int c[3]) const;

  // insertion / propagation
  void insert(int channel, const int origin[3], const int dims[3], const void* samples,
              int mem_kind);
  bool dense_eligible(int channel, const int origin[3], const int dims[3], const void* dsrc,
                      int src_stride, int src_off) const;
  void insert_staged(int channel, const int origin[3], const int dims[3], const void* dsrc,
                     int src_stride, int src_off, int reps, int64_t ev_reps = 0);
  void flush_structure();
  void propagate();
  bool dense_parent(int64_t p) const;
  void flush();  // propagate pending + structure
  void sync();
  void gather_stats(const std::vector<int64_t>& nodes);
  void prune(std::vector<std::vector<int64_t>>& touched, std::vector<char>& deleted_mark,
             std::vector<int64_t>& deleted);
  void delete_below(int64_t p, std::vector<char>& mark, std::vector<int64_t>& deleted);
  void free_brick(int64_t n);
  void fill_borders();
  int64_t find_node(const double pt[3], int target) const;
  // z-slab sharded build: splice complete subtrees built elsewhere into this
  // tree, then recompute every ancestor level from its children
  void merge(int64_t n, const int64_t* idx, const int32_t* nflags, const int32_t* stats,
             const void* bricks, int mem_kind, int64_t inserted_voxels);

  int32_t stat(int64_t node, int s, int c) const { return h_stats[st_index(node, s, c)]; }
};

void sort_indices(std::vector<int64_t>& v);

// launch helpers implemented in build_kernels.cu
void launch_struct_update(const Tree& t, const StructUpd* d_upd, int n);
void launch_create(const Tree& t, const CreateJob* d_jobs, int n);
void launch_seed(const Tree& t, const SeedJob* d_jobs, int n);
void launch_scatter(const Tree& t, const void* src, int channel, int src_stride, int src_off,
                    const int origin[3],
                    const int dims[3], const int g0[3], const int gn[3], const int32_t* d_leaf_slots);
// the scatter computes a leaf plane's partial stats itself iff this holds
bool scatter_owns_stats(const Geo& g, int channel, const int origin[3], const int dims[3], int gx,
                        int gy);
void launch_octant(const Tree& t, const OctJob* d_jobs, int n);
// dense_build.cu
// returns kLeafPrefilled (shells prefilled) | kLeafTma (TMA kernel: fused
// parent octants of jobs with pad >= 0 written too)
// kLeafBmax: brick maxima written; kLeafParentShells: the x/y shells of the
// interior fused level-1 parents written (held pairs)
constexpr int kLeafPrefilled = 1, kLeafTma = 2, kLeafBmax = 4, kLeafParentShells = 8;
int launch_dense_leaf(const Tree& t, const void* src, int64_t nsrc, int oz, int prefill,
                      const DenseJob* jobs, int n, const int gn[3], int g0z);
// planar (c, z, y, x) source through a 4-D TMA tensor map; -1 = unsupported
// here (8-bit samples, unaligned strides, oversized bricks)
bool planar_leaf_ok(const Tree& t, const void* base, int64_t zstride, int64_t cstride);
int launch_dense_leaf_planar(const Tree& t, const void* base, int64_t zstride, int64_t cstride,
                             int oz, int64_t dz, int prefill, const DenseJob* jobs, int n,
                             const int gn[3], int g0z, bool write_struct = false,
                             bool parent_shells = false);
void launch_planar_to_interleaved(const Tree& t, const void* base, int64_t zstride,
                                  int64_t cstride, int dz, void* dst);
void launch_fill_bg(const Tree& t, void* dst, int64_t n);
// background into n planes of `plane` samples at base + idx[k] * plane
constexpr int kMaxFillPlanes = 128;
void launch_fill_planes(const Tree& t, void* base, int64_t plane, const int32_t* idx, int n);
// fused level-1 parents: accumulators before / statistics after the leaf kernel
void launch_init_fused(const Tree& t, const int64_t* d_nodes, int n);
// channel `c` of an n-voxel single-channel block into an interleaved buffer
void launch_interleave(const Tree& t, const void* src, int64_t n, int c, void* dst);
void launch_finish_fused(const Tree& t, const int64_t* d_nodes, int n);
// z-shell plane copies between leaf bricks: dst plane <- src plane
void launch_plane_copy(const Tree& t, const int32_t* d_jobs, int n);
// every shell voxel of the given bricks <- background
void launch_clear_shells(const Tree& t, const int32_t* d_slots, int n);
// smem: every node has 8 full in-volume bricked children (the shared-memory
// kernel, when level_smem_ok); else the general dense level kernel
void launch_dense_level(const Tree& t, const int64_t* nodes, int n, int zsplit, bool smem = false);
bool level_smem_ok(const Tree& t);
// CTAs per parent for a dense level of n parents (> 1: statistics by k_reduce)
int dense_level_split(const Tree& t, int n);
void launch_plane(const Tree& t, const PlaneJob* d_jobs, int n);
void launch_reduce(const Tree& t, const ReduceJob* d_jobs, int n);
void launch_borders(const Tree& t, const BorderJob* d_jobs, int n);
void launch_gather_stats(const Tree& t, const int64_t* d_nodes, int n, int32_t* d_out);
void launch_gather_bricks(const Tree& t, const int32_t* d_slots, int n, uint8_t* d_out);
void launch_scatter_bricks(const Tree& t, const int32_t* d_slots, int n, const uint8_t* d_in);
void launch_pool_fill(const Tree& t, int64_t first_slot, int64_t n_slots);
void launch_brick_hash(const Tree& t, const int32_t* d_slots, int n, unsigned long long* d_out);
// stats rows [n][ST_N][kMaxC] -> node stats
void launch_set_stats(const Tree& t, const int64_t* d_nodes, int n, const int32_t* d_rows);

// device scratch: stream-ordered allocation of a host vector's copy
template <class T>
T* upload(const Tree& t, const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  return static_cast<T*>(t.stage_copy(v.data(), v.size() * sizeof(T)));
}
// frees stream-ordered allocations; staging-ring pointers are recycled by the ring
inline void release(const Tree& t, void* p) {
  if (p && !t.is_staged(p)) VT_CUDA(cudaFreeAsync(p, t.stream));
}

}  // namespace vtx

// the opaque ABI handle (include/vtx.h)
// Reference counted: a mirror (and its ray sessions) keep the tree alive, so
// Python finalizers may run in any order (GC of reference cycles).
struct vt_tree {
  vtx::Tree t;
  std::atomic<int> refs{1};
  explicit vt_tree(const vt_tree_desc& d) : t(d) {}
};
inline void vt_tree_retain(vt_tree* t) { t->refs.fetch_add(1); }
inline void vt_tree_release(vt_tree* t) {
  if (t && t->refs.fetch_sub(1) == 1) delete t;
}
