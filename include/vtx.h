/*
 * vtx.h — C ABI of libvtx.so, the B200-native (sm_100a) octree build +
 * octree ray-casting engine.  Plain pointers and sizes only; no torch types.
 *
 * Each entry point replaces one piece of the reference package `voxtree`
 * (pure Python, /root/reference/pkg/src/voxtree).  The reference interface
 * each function stands in for is cited as file:line.  INTEGRATION.md shows
 * the ctypes binding a voxtree maintainer would add.
 *
 * Conventions
 *  - every function returns vt_status; 0 = OK.  On error a thread-local
 *    message is available from vt_last_error().  Status -> reference
 *    exception: VT_EINVAL -> ValueError, VT_EOVERFLOW -> OverflowError,
 *    VT_EIO -> StoreIOError, VT_ECUDA / VT_ENOMEM / VT_ESTATE -> RuntimeError.
 *  - input sample buffers are borrowed for the duration of the call; outputs
 *    are caller owned; handles are library owned.
 *  - a tree is single-writer (the Python shim holds a lock mirroring
 *    Octree.lock, octree.py:153).
 *  - all device work is ordered on the stream set with vt_tree_set_stream
 *    (default: a stream owned by the tree).
 */
#ifndef VTX_H
#define VTX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t vt_status;
#define VT_OK 0
#define VT_EINVAL 1
#define VT_EOVERFLOW 2
#define VT_ENOMEM 3
#define VT_ECUDA 4
#define VT_ESTATE 5
#define VT_EIO 6

#define VT_MEM_HOST 0   /* pageable or pinned host memory            */
#define VT_MEM_DEVICE 1 /* device pointer, stream-ordered on the tree stream */

#define VT_EV_CREATED 1 /* octree.py:41-45 ChangeKind */
#define VT_EV_DELETED 2
#define VT_EV_UPDATED 3

#define VT_NODE_EXISTS 1
#define VT_NODE_CHILDREN 2
#define VT_NODE_IN_VOLUME 4
#define VT_NODE_BRICK 8

typedef struct vt_tree vt_tree;
typedef struct vt_mirror vt_mirror;
typedef struct vt_rays vt_rays;

/* VolumeDescriptor (volume.py:35-99) + BrickPoolConfig (volume.py:102-152),
 * already validated by the host shim; threshold already resolved
 * (BrickPoolConfig.resolve_threshold, volume.py:136-139). */
typedef struct {
  int32_t dims[3];       /* x, y, z voxels                           */
  int32_t channels;      /* 1..4                                     */
  int32_t sample_bytes;  /* 1 = uint8, 2 = uint16                    */
  int32_t background;    /* background_value                         */
  int32_t brick[3];      /* brick_dims M (x, y, z), even or 1        */
  double threshold;      /* homogeneity threshold tau (strict <)     */
  int64_t reserve_slots; /* initial device pool slots (0 = auto)     */
  int32_t device;        /* CUDA ordinal                             */
} vt_tree_desc;

typedef struct {
  int64_t node_count;      /* Octree.node_count                        */
  int64_t brick_count;     /* Octree.brick_count (octree.py:530-532)    */
  int64_t pruned_bricks;   /* Octree.pruned_bricks                      */
  int64_t inserted_voxels; /* Octree.inserted_voxels                    */
  int64_t capacity;        /* TreeGeometry.node_capacity                */
  int64_t pool_slots;      /* allocated device pool slots               */
  int32_t depth;           /* TreeGeometry.depth                        */
  int32_t virtual_dims[3]; /* TreeGeometry.virtual                      */
  int32_t finished;        /* construction_finished                     */
  int32_t borders_filled;  /* borders_filled                            */
} vt_tree_info;

/* per-node record, stats are [channel][avg, smin, smax, sub_min, sub_max]
 * (OctreeNode, octree.py:102-127; sub_* are 0 when not in volume) */
typedef struct {
  int32_t flags; /* VT_NODE_* */
  int32_t level;
  int32_t box_lo[3];
  int32_t slot; /* device pool slot, -1 when brickless */
  int32_t stats[4][5];
} vt_node;

const char* vt_last_error(void);
int32_t vt_abi_version(void);

/* ---- construction: replaces Octree (octree.py:143-614) ----------------- */

/* Octree.create / Octree.__init__ (octree.py:146-176) */
vt_status vt_tree_create(const vt_tree_desc* desc, vt_tree** out);
vt_status vt_tree_destroy(vt_tree* tree);
/* order all device work on a caller stream (cudaStream_t as void*) */
vt_status vt_tree_set_stream(vt_tree* tree, void* stream);

/* order the tree's device work after everything already queued on
 * `stream` (e.g. the producer of a device-resident block), without a host
 * synchronisation */
vt_status vt_tree_wait_stream(vt_tree* tree, void* stream);
/* the converse: make `stream` wait for everything queued on the tree so far
 * (a caller-owned device block may then be freed or reused in stream order) */
vt_status vt_tree_signal_stream(vt_tree* tree, void* stream);
/* Octree.insert_block (octree.py:323-397): one channel, values (dz,dy,dx)
 * x-fastest.  Errors exactly as octree.py:331-341 (VT_EINVAL). */
/* B200 extension: vt_tree_insert (channel -1 = vt_tree_insert_channels) in
 * one call with the caller-stream ordering of a device block (wait on
 * caller_stream before reading it, make caller_stream wait for the reads;
 * a null caller_stream is the legacy default stream)
 * and a copy of THIS insertion's change events when they fit in `cap` (they
 * stay queued for vt_tree_take_events, as insert_block's returned list stays
 * in Octree._events, octree.py:393-395); *n_events = how many it emitted
 * (more than cap: none copied — vt_tree_copy_events(event_count - n, n)) */
vt_status vt_tree_insert_ev(vt_tree* tree, int32_t channel, const int32_t origin[3],
                            const int32_t dims[3], const void* samples, int32_t mem_kind,
                            void* caller_stream, int32_t* kinds, int64_t* indices, int64_t cap,
                            int64_t* n_events);
vt_status vt_tree_insert(vt_tree* tree, int32_t channel, const int32_t origin[3],
                         const int32_t dims[3], const void* samples, int32_t mem_kind);
/* fused multi-channel variant: values (dz,dy,dx,C) channel-interleaved; the
 * same result and events as C successive vt_tree_insert calls, channel 0..C-1 */
vt_status vt_tree_insert_channels(vt_tree* tree, const int32_t origin[3],
                                  const int32_t dims[3], const void* samples,
                                  int32_t mem_kind);
/* B200 extension: a batch of insertions in one call — the same tree and the
 * same queued change events (drained with vt_tree_take_events) as n
 * successive vt_tree_insert calls in order; what ingest_stream's frame loop
 * (ingest.py:306-358) does per VSTR frame.  All blocks share `mem_kind` and
 * are borrowed for the duration of the call (device blocks: ordered after
 * caller_stream, which waits for the reads).  At threshold 0, consecutive
 * single-channel blocks spanning the full x/y extent that cover every
 * (z, channel) of one brick layer exactly once become one dense insertion
 * (a device layer whose blocks sit at an affine stride, e.g. slices of a
 * planar (C, Z, Y, X) volume, is read in place through a 4-D TMA tensor
 * map).  An invalid block raises after the blocks before it are inserted,
 * as the loop would. */
typedef struct {
  int32_t channel;   /* 0..C-1 */
  int32_t origin[3]; /* x, y, z */
  int32_t dims[3];   /* x, y, z extent of values (dz, dy, dx), x-fastest */
  int32_t pad;
  const void* samples;
} vt_block;
vt_status vt_tree_insert_many(vt_tree* tree, int64_t n, const vt_block* blocks, int32_t mem_kind,
                              void* caller_stream);
/* move pending change events out (Octree.drain_events, octree.py:180-183);
 * *n returns the number written (<= cap); call again while *more != 0 */
vt_status vt_tree_take_events(vt_tree* tree, int32_t* kinds, int64_t* indices, int64_t cap,
                              int64_t* n, int32_t* more);
/* B200 extension: copy queued events [from, from + n) (0 = oldest) without
 * taking them (vt_tree_insert_ev reports an insertion's events this way
 * when they exceed its buffer) */
vt_status vt_tree_copy_events(vt_tree* tree, int64_t from, int64_t n, int32_t* kinds,
                              int64_t* indices);
/* number of pending change events (size the take_events buffers) */
vt_status vt_tree_event_count(vt_tree* tree, int64_t* n);
/* Octree.finalize / fill_borders (octree.py:536-614) */
vt_status vt_tree_finalize(vt_tree* tree);
vt_status vt_tree_fill_borders(vt_tree* tree);
/* complete all deferred device work and wait for it */
vt_status vt_tree_sync(vt_tree* tree);
/* B200 extension: enqueue every deferred device update (an open slice
 * layer's received planes, pending pyramid propagation) on the tree stream
 * without waiting for it — what any reader does first (octree.py:323-397
 * leaves the tree complete after every insert_block). */
vt_status vt_tree_flush(vt_tree* tree);
vt_status vt_tree_info_get(vt_tree* tree, vt_tree_info* out);
/* B200 extension: threshold-0 dense build (dense_build.cu).  A fused
 * all-channel block spanning the full x/y extent and whole brick layers over
 * brick-less leaves (ingest_bulk's z-slabs, ingest.py:182-224) writes its
 * leaf bricks and statistics outright, and parents whose in-volume children
 * are all complete are recomputed in one pass; results, events and slots are
 * identical to the general path.  Enabled by default (env VT_DENSE=0 or
 * enabled = 0 turns it off); counts = dense leaf insertions / dense parents /
 * fill_borders calls that only had to patch owed z-shells of prefilled
 * leaves (env VT_PREFILL=0 disables shell prefill). */
vt_status vt_tree_set_dense(vt_tree* tree, int32_t enabled);
vt_status vt_tree_dense_counts(vt_tree* tree, int64_t* leaf_inserts, int64_t* level_nodes,
                               int64_t* fast_borders);
/* B200 extension: brick layers built as one dense insertion by
 * vt_tree_insert_many (of which read in place), and deferred layers of
 * per-block slice streams (diagnostics for tests and the bench) */
vt_status vt_tree_stream_counts(vt_tree* tree, int64_t* layer_groups, int64_t* zero_copy_layers,
                                int64_t* deferred_layers);
/* B200 extension: leaf shells the dense build prefilled with their
 * fill_borders values are the reference's background until fill_borders
 * (octree.py:234-237); every pool reader publishes them first — call this
 * before reading the pool through a zero-copy alias */
vt_status vt_tree_publish_halos(vt_tree* tree);
/* Octree.node_by_index (octree.py:515-528): *exists = 0 when absent */
vt_status vt_tree_node(vt_tree* tree, int64_t index, vt_node* out, int32_t* exists);
/* Octree.iter_nodes order (BFS == ascending index, octree.py:507-513);
 * flags (VT_NODE_*) optional; *n = total count even when > cap */
vt_status vt_tree_list_nodes(vt_tree* tree, int64_t* out, int32_t* flags, int64_t cap,
                             int64_t* n);
/* Octree.find_node (octree.py:497-505): point in level-0 virtual voxels */
vt_status vt_tree_find_node(vt_tree* tree, const double point[3], int32_t target_level,
                            int64_t* index);
/* brick payload copy (BrickStore.read_brick, paging.py:398-403) */
vt_status vt_tree_read_brick(vt_tree* tree, int64_t index, void* out);
/* bulk export for save_octree (serialize.py:61-125): stats for n nodes
 * (n * C * 5 int32, layout as vt_node.stats) and the bricks of the bricked
 * ones among them, concatenated in the given order */
vt_status vt_tree_export(vt_tree* tree, int64_t n, const int64_t* indices, int32_t* stats,
                         void* bricks);
/* load_octree (serialize.py:128-206): rebuild a tree from node records */
vt_status vt_tree_import(vt_tree* tree, int64_t n, const int64_t* indices,
                         const int32_t* flags, const int32_t* stats, const void* bricks,
                         int32_t finished, int32_t borders_filled, int64_t pruned_bricks);

/* 64-bit digest of the whole tree computed on the device: structure, node
 * statistics and a position-dependent hash of every brick, in BFS order.
 * Equal trees give equal digests: the size-independent stand-in for the
 * VXOC/VXBP sha256 at sizes where serialising tens of GB is impractical. */
vt_status vt_tree_checksum(vt_tree* tree, uint64_t* out);

/* z-slab sharded build (no reference counterpart).  Export the
 * records of the given nodes: VT_NODE_* flags, stats as vt_tree_export, and
 * the bricks of the bricked ones in the given order into host or device
 * memory (bricks_mem_kind). */
vt_status vt_tree_export_nodes(vt_tree* tree, int64_t n, const int64_t* indices, int32_t* flags,
                               int32_t* stats, void* bricks, int32_t bricks_mem_kind);
/* Splice complete subtrees (records as exported above, parents before
 * children not required) into this tree: ancestor chains are created as an
 * insertion walk would create them, every ancestor above the records is
 * given a brick and recomputed from all of its children.  With tau == 0 the
 * result is byte-identical to inserting the subtrees' data here. */
vt_status vt_tree_merge(vt_tree* tree, int64_t n, const int64_t* indices, const int32_t* flags,
                        const int32_t* stats, const void* bricks, int32_t bricks_mem_kind,
                        int64_t inserted_voxels);

/* halfsample_block (octree.py:58-92) as a standalone device op on host
 * buffers: values (mz,my,mx,C) int32 -> out (mz/kz,my/ky,mx/kx,C) int32 */
vt_status vt_halfsample(const int32_t* values, const int32_t shape[4],
                        const int32_t in_extent[3], const int32_t split[3], int32_t background,
                        int32_t* out, int32_t device);

/* ---- device mirror: replaces DeviceState (device.py:124-386) ------------ */

/* slot_count < 0: zero-copy mirror whose brick buffer IS the tree pool
 * (every brick resident, slot = pool slot).  Otherwise a bounded brick
 * buffer of slot_count slots, nothing resident (device.py:134-164). */
vt_status vt_mirror_create(vt_tree* tree, int64_t slot_count, vt_mirror** out);
vt_status vt_mirror_destroy(vt_mirror* m);
/* device pointers + sizes of node_buffer (u64[capacity]), flag_buffer
 * (u8[capacity]) and brick_buffer ([slots, bz, by, bx, C]) */
/* B200 extension: brick-maxima refreshes of a zero-copy mirror done
 * incrementally (only pool slots written since the last refresh) and the
 * slot count of the last refresh */
vt_status vt_mirror_bmax_stats(vt_mirror* m, int64_t* incremental, int64_t* last_slots);
vt_status vt_mirror_buffers(vt_mirror* m, void** node_buffer, void** flag_buffer,
                            void** brick_buffer, int64_t* capacity, int64_t* slots);
/* residency edits: slot >= 0 copies the node's pool brick into brick_buffer
 * [slot] (upload, device.py:341) and marks it resident; slot < 0 drops it */
vt_status vt_mirror_set_resident(vt_mirror* m, int64_t n, const int64_t* nodes,
                                 const int32_t* slots, int32_t copy);
/* rewrite every node entry from the tree + residency (device.py:168-203) */
vt_status vt_mirror_repack(vt_mirror* m);
/* B200 extension for zero-copy mirrors: DeviceState.apply_events(
 * octree.drain_events()) without moving the events to the host — every
 * queued change event is taken inside the library, NODE_DELETED flags are
 * cleared (device.py:214-220), node entries re-packed and brick maxima of
 * the changed slots refreshed.  Returns the events consumed and deletions. */
vt_status vt_mirror_apply_queued(vt_mirror* m, int64_t* n_events, int64_t* n_deleted);
/* flag buffer transfer; clear != 0 zeroes it after reading (device.py:250-252) */
vt_status vt_mirror_read_flags(vt_mirror* m, uint8_t* out, int32_t clear);

/* ---- rendering: replaces OutOfCoreRenderer (render/raycast.py:53-339) ---- */

#define VT_MAX_TF_POINTS 16

typedef struct {
  /* Camera (render/camera.py:17-61).  The host shim computes the basis
   * exactly as Camera.basis()/rays()/pixel_footprint_scale() do (numpy), so
   * transcendental and BLAS-dependent values are bit-identical. */
  double position[3];
  double fwd[3], right[3], up[3]; /* Camera.basis() */
  double tan_half;                /* np.tan(fov_y / 2)  */
  double aspect;                  /* width / height     */
  double footprint_scale;         /* pixel_footprint_scale() */
  int32_t width, height;
  /* RenderSettings (render/settings.py:44-68) */
  int32_t mode_mip;          /* 0 dvr, 1 mip */
  double step;               /* resolved sampling step */
  double corr_exp;           /* opacity_exponent */
  double et_limit;           /* early_termination_alpha; >= 1 or <0 disables */
  double lod_scale;          /* 2.0 ** lod_bias, computed on the host */
  /* TransferFunction per channel (render/transfer.py), sorted points */
  int32_t tf_count[4];
  double tf_x[4][VT_MAX_TF_POINTS];
  double tf_rgba[4][VT_MAX_TF_POINTS][4];
  /* ClipSet (render/settings.py:15-41) */
  int32_t n_clips;
  double clip_normal[3][3];
  double clip_offset[3];
  /* VolumeDescriptor.spacing and per-channel affine transforms */
  double spacing[3];
  int32_t has_transforms;
  double transforms[4][12]; /* row-major 3x4 */
  /* sample reconstruction precision of vt_render_fullframe/tile/strips:
   * 0 FP64 (default; trilinear as fused-multiply-add lerps, matches the
   * reference to ~1e-15), 1 FP32 trilinear + transfer functions with FP64 ray
   * accumulation (within the 1/255 tolerance) */
  int32_t precision;
  /* exact empty-space skipping: 0 library default (bricks), 1 off,
   * 2 whole bricks, 3 bricks + sub-bricks.  Never changes images or
   * counters, only how many samples are reconstructed. */
  int32_t empty_skip;
} vt_scene;

typedef struct {
  int64_t samples, tf_lookups, avg_fallbacks, coarse_fallbacks, bricks_requested,
      bricks_used_marks; /* RenderCounters, render/core.py:20-31 */
  /* not a reference counter: of `samples`, those the exact empty-space skip
   * accounted without computing them (transfer-function alpha provably 0) */
  int64_t samples_skipped;
} vt_counters;

/* RayBatch + CompositeState on the device (render/core.py:75-97, 100-107);
 * tile = {x0,y0,x1,y1} or NULL (raycast.py:304-318) */
vt_status vt_rays_create(vt_mirror* m, const vt_scene* scene, const int32_t* tile,
                         vt_rays** out);
vt_status vt_rays_destroy(vt_rays* r);
/* one march pass (render/core.py:162-187); strategy 0 fullframe, 1 refinement.
 * counters are ADDED to *cnt; *suspended = rays left suspended */
vt_status vt_rays_march(vt_rays* r, int32_t strategy, vt_counters* cnt, int64_t* suspended);
/* finalize_image (render/core.py:137-155) -> host float64 (H,W,4) */
vt_status vt_rays_image(vt_rays* r, double* out_host, vt_counters* cnt);
/* per-ray k / n_steps / suspended (RefinementSession.rays) to host */
vt_status vt_rays_state(vt_rays* r, int64_t* k, int64_t* n_steps, uint8_t* suspended);

/* fused full-frame pass (render_fullframe, raycast.py:282-290): ray setup,
 * march and finalize in one kernel, no per-ray state.  out_kind 0: float64
 * (H,W,4); 1: float32; 2: RGBA8 (image_to_rgba8, core.py:158-159).
 * out is a DEVICE pointer when out_on_device, else host. */
vt_status vt_render_fullframe(vt_mirror* m, const vt_scene* scene, void* out,
                              int32_t out_kind, int32_t out_on_device, vt_counters* cnt);
/* the same, rows [row0,row1) x cols [col0,col1) only (sort-first tile) */
vt_status vt_render_tile(vt_mirror* m, const vt_scene* scene, const int32_t rect[4], void* out,
                         int32_t out_kind, int32_t out_on_device, vt_counters* cnt);

/* sort-first strip partition (multi-GPU): render the rows of
 * strips part, part + n_parts, part + 2 n_parts, ... (strip_rows rows each,
 * full width) into a compact (vt_strip_part_rows(H, strip_rows, n_parts), W, 4)
 * buffer; rows past the frame are zero.  Interleaving balances the per-GPU
 * sample load; n_parts == 1 equals vt_render_fullframe. */
vt_status vt_render_strips(vt_mirror* m, const vt_scene* scene, int32_t strip_rows,
                           int32_t n_parts, int32_t part, void* out, int32_t out_kind,
                           int32_t out_on_device, vt_counters* cnt);
int32_t vt_strip_part_rows(int32_t height, int32_t strip_rows, int32_t n_parts);

/* synthetic volumes (oracle/voxtree_oracle.py synth_*): device fill of
 * z in [z0,z1) as (z,y,x,C) interleaved samples; kind 0 uniform, 1 spim */
vt_status vt_synth(void* out_device, int32_t kind, const int32_t dims[3], int32_t channels,
                   int32_t sample_bytes, uint32_t seed, int32_t z0, int32_t z1, void* stream);

/* last-launch profiling: device milliseconds of the most recent render /
 * build kernels measured with CUDA events on the tree stream */
vt_status vt_last_kernel_ms(vt_tree* tree, double* render_ms, double* build_ms);

#ifdef __cplusplus
}
#endif
#endif
