/*
 * linevox_b200.h -- C ABI of liblinevox_b200.so, the B200 (sm_100a) drop-in for
 * the hot path of the `linevox` reference (arXiv 1801.01155):
 *   voxelize -> LoD -> ray-cast (+ density-grid AO / soft shadows).
 *
 * Conventions
 *   - every entry point returns int: 0 = ok, nonzero = LVX_E_* (never throws);
 *     lvx_last_error() gives a thread-local message for the last failure;
 *   - every `*_d` / device pointer is CALLER-OWNED device memory (e.g. the
 *     data_ptr() of a torch CUDA tensor).  The library never allocates device
 *     memory behind the caller's back; scratch space is passed in explicitly;
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it and
 *     the call returns without synchronising unless stated otherwise;
 *   - plain C types only: no torch / C++ types cross this boundary.
 *
 * Each declaration cites the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/linevox/).
 */
#ifndef LINEVOX_B200_H
#define LINEVOX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LVX_OK 0
#define LVX_E_INVALID 1   /* bad argument */
#define LVX_E_CUDA 2      /* CUDA runtime error (see lvx_last_error) */
#define LVX_E_NO_DEVICE 3 /* no sm_100-class device visible */
#define LVX_E_RANGE 4     /* size exceeds a documented limit */

#define LVX_ABI_VERSION 2

/* mode codes: _kernels.py:43-55 */
#define LVX_OPACITY_CONSTANT 0
#define LVX_OPACITY_TRANSFER 1
#define LVX_OPACITY_DISTANCE 2
#define LVX_SHADOW_NONE 0
#define LVX_SHADOW_HARD 1     /* geometry shadow rays (needs the neighbour grids) */
#define LVX_SHADOW_REPLINES 2 /* representative-line shadow rays (needs lvx_lod.rep) */
#define LVX_SHADOW_CONE 3
#define LVX_AO_NONE 0
#define LVX_AO_HEMISPHERE 1 /* geometry hemisphere rays (needs the neighbour grids + lattice) */
#define LVX_AO_DENSITY 2
#define LVX_AO_PRECOMPUTED 3

/* caps that are part of the reference's observable behaviour (_kernels.py:36-38) */
#define LVX_MAX_WINDOW_HITS 1024
#define LVX_MAX_SEEN 256
#define LVX_MAX_LEVELS 24

int lvx_abi_version(void);
const char *lvx_last_error(void);
/* 0 when a compute-capability 10.x device is current; LVX_E_NO_DEVICE otherwise. */
int lvx_device_check(void);

/* ------------------------------------------------------------------------- */
/* Voxelizer: replaces _plane_events/_clip_batch/_faces_and_bins/             */
/* build_voxel_model/_pack_all (voxelizer.py:174-263, 358-394, 397-488).      */
/*                                                                           */
/* Input batch layout (what voxelizer.py:419-425 concatenates per chunk):     */
/*   pts_d   f64 [P,3]  vertices of all curves, curve after curve             */
/*   attrs_d f64 [P]    per-vertex attribute                                  */
/*   curve_off_d i64 [n_curves+1]  first vertex of each curve, last = P       */
/* The parallel unit is the polyline EDGE (vertex i -> i+1).                  */
/* ------------------------------------------------------------------------- */

/* first_d u8[P]: 1 at the first vertex of every curve (the reference's
 * `point_curve[1:] == point_curve[:-1]` test, voxelizer.py:216). */
int lvx_mark_curve_starts(const int64_t *curve_off_d, int64_t n_curves, int64_t n_points,
                          uint8_t *first_d, void *stream);

/* Prefix sums over the per-voxel chord counts: cursor_d = exclusive scan of the raw counts
 * (start of every voxel's group), offsets_d / counts_d = the model's headers (counts capped at
 * 255, voxelizer.py:442-466), totals_d[0] = chords, totals_d[1] = segments kept. */
size_t lvx_scan_scratch_bytes(int64_t n);
int lvx_voxel_scan(const uint32_t *vox_cnt_d, int64_t n_voxels, uint32_t *cursor_d,
                   uint32_t *offsets_d, uint8_t *counts_d, uint64_t *totals_d,
                   void *scratch_d, void *stream);

/* Raw chord slots written by the clipper (SoA, coalesced):
 *   raw_key_d u64  (edge index << 16) | kept-chord ordinal inside the edge -- strictly
 *                  increasing in (curve, chord order)
 *   raw_q_d   u64  face_in | bin_in<<3 | face_out<<19 | bin_out<<22 | attr<<38
 *   raw_lin_d u32  voxel linear index, 0xFFFFFFFF for a slot without a chord
 * edge_kept_d u16[P] (nullable): kept chords ending in each edge (for seg_order). */
/* Single-pass clipper: the vertices are read from HBM once (voxelizer.py:174-263, 358-380,
 * 419-449: _plane_events, _clip_batch, _faces_and_bins and the chunk loop of build_voxel_model).
 *   lvx_voxelize_bound  number of plane crossings = upper bound of the chord count; sizes raw_*
 *   lvx_voxelize_clip   clip + emit: one slot per crossing in raw_*[0, *n_slots); raw_lin of a
 *                       slot whose chord was dropped is 0xFFFFFFFF; per-voxel chord counts are
 *                       added into vox_cnt_d (caller zeroes it); err_d: 1 = an endpoint off
 *                       every face (voxelizer.py:366-368), 2 = capacity too small
 * followed by lvx_voxel_scan -> lvx_raw_regroup -> lvx_voxelize_compact. */
int lvx_voxelize_bound(const double *pts_d, const uint8_t *first_d, int64_t n_points,
                       uint64_t *total_d, void *stream);
int lvx_voxelize_clip(const double *pts_d, const double *attrs_d, const uint8_t *first_d,
                      int64_t n_points, const int32_t dims[3], int32_t n_bins, uint64_t capacity,
                      uint32_t *vox_cnt_d, uint64_t *raw_key_d, uint64_t *raw_q_d,
                      uint32_t *raw_lin_d, uint64_t *n_slots_d, uint16_t *edge_kept_d, int32_t *err_d,
                      void *stream);

typedef struct {
    float ax, ay, az;
    uint32_t meta; /* attr | lid << 8 */
    float bx, by, bz;
    float half_len; /* >= |b-a|/2 (rounded up): radius of the segment's bounding sphere */
} lvx_seg_record;

/* One chord grouped by voxel (32 bytes = one memory sector, so the scatter that groups
 * them writes whole sectors). */
typedef struct {
    uint64_t key; /* global edge index << 16 | ordinal of the chord on its edge */
    uint64_t q;   /* face_in 3 | bin_in 16 | face_out 3 | bin_out 16 | attr 8 */
    uint32_t lin; /* voxel */
    uint32_t _pad[3];
} lvx_raw_record;

/* Scatter raw slots (any order; 0xFFFFFFFF voxels skipped) into per-voxel groups through the
 * cursors from lvx_voxel_scan, which end up at the END of every voxel's range. */
int lvx_raw_regroup(const uint64_t *in_key_d, const uint64_t *in_q_d, const uint32_t *in_lin_d,
                    int64_t n_slots, uint32_t *cursor_d, lvx_raw_record *grouped_d, void *stream);

/* Order every voxel's group by key (= the reference's stable argsort by voxel,
 * voxelizer.py:435-438), keep the first 255, lid = rank % 32, decode bin centres, pack
 * (voxelizer.py:439-488, 383-394).  Optional outputs may be NULL.
 * Alignment: grouped_d (lvx_raw_regroup, lvx_voxelize_compact) and seg_rec_d (lvx_voxelize_compact,
 * lvx_decode_packed, lvx_build_seg_records) are accessed with 256-bit loads / stores and must be
 * 32-byte aligned; the calls return LVX_E_INVALID otherwise. */
int lvx_voxelize_compact(const lvx_raw_record *grouped_d, int64_t n_raw, const uint32_t *vox_cnt_d,
                         const uint32_t *cursor_end_d, const uint32_t *offsets_d,
                         const int32_t dims[3], int32_t n_bins, uint8_t *packed_d, float *seg_a_d,
                         float *seg_b_d, uint8_t *seg_attr_d, uint8_t *seg_lid_d,
                         int32_t *seg_voxel_d, uint8_t *seg_face_in_d, uint16_t *seg_bin_in_d,
                         uint8_t *seg_face_out_d, uint16_t *seg_bin_out_d, uint64_t *seg_key_d,
                         lvx_seg_record *seg_rec_d, void *stream);

/* Device-side decode of the packed records (model_io.py:151-179
 * _decode_records + _bin_centers, the expansion load_vxl does on the host): render records
 * and, optionally, the reference's per-segment caches straight from (counts, offsets, packed).
 * err_d = 1 when a record carries a face id > 5 (model_io.py:277-278).  Outputs may be NULL. */
int lvx_decode_packed(const uint8_t *packed_d, const uint8_t *counts_d, const uint32_t *offsets_d,
                      const int32_t dims[3], int32_t n_bins, float *seg_a_d, float *seg_b_d,
                      uint8_t *seg_attr_d, uint8_t *seg_lid_d, int32_t *seg_voxel_d,
                      uint8_t *seg_face_in_d, uint16_t *seg_bin_in_d, uint8_t *seg_face_out_d,
                      uint16_t *seg_bin_out_d, lvx_seg_record *seg_rec_d, int32_t *err_d, void *stream);

int lvx_scan_u16(const uint16_t *in_d, int64_t n, uint32_t *out_d, void *scratch_d,
                 void *stream);

/* seg_curve / seg_order (voxelizer.py:254-262, 486-487) from provenance keys. */
int lvx_provenance(const uint64_t *seg_key_d, int64_t n_seg, const uint32_t *edge_base_d,
                   const int64_t *curve_off_d, int64_t n_curves, int32_t *seg_curve_d,
                   int32_t *seg_order_d, void *stream);

/* Rebuild the 32-byte render records from the reference-layout caches (used when
 * a model arrives from host arrays, e.g. a decoded .vxl). */
int lvx_build_seg_records(const float *seg_a_d, const float *seg_b_d,
                          const uint8_t *seg_attr_d, const uint8_t *seg_lid_d, int64_t n_seg,
                          lvx_seg_record *seg_rec_d, void *stream);

/* ------------------------------------------------------------------------- */
/* LoD: compute_density_level0 (lod.py:82-94), _coarsen/build_octree          */
/* (lod.py:97-119), _occupancy_dilated (raycast.py:351-366).                  */
/* ------------------------------------------------------------------------- */

int lvx_density_l0(const uint8_t *counts_d, const uint32_t *offsets_d,
                   const lvx_seg_record *seg_rec_d, const float *table_d, int64_t n_voxels,
                   float *level0_d, void *stream);

/* The same sums from the encoded records (voxelizer.py:79-89) instead of the render records: the
 * endpoints are reconstructed like the voxelizer does (model_io.py:169-179), the result is
 * bit-identical, the kernel reads 5 instead of 32 bytes per segment at N = 32.  packed_d 8-byte
 * aligned and readable up to the next multiple of 8 bytes. */
int lvx_density_l0_packed(const uint8_t *counts_d, const uint32_t *offsets_d, const uint8_t *packed_d,
                          const int32_t dims[3], int32_t n_bins, const float *table_d, float *level0_d, void *stream);

/* The same for a grouping that is not the model's headers: uncapped u32 counts / offsets over records
 * gathered into voxel order.  compute_density_level0 (lod.py:82-94) bins by `seg_voxel`, so a
 * hand-assembled model whose seg_voxel disagrees with its headers (the reference's tests build
 * such models, tests/test_lod.py:14-37) is binned the same way: stable sort by voxel, then this. */
int lvx_density_l0_u32(const uint32_t *counts_d, const uint32_t *offsets_d, const lvx_seg_record *seg_rec_d,
                       const float *table_d, int64_t n_voxels, float *level0_d, void *stream);

/* Host helper: level offsets/dims of the flat octree buffer (_octree_args,
 * raycast.py:369-388).  off[n_levels+1], ldims[n_levels*3] as (dx,dy,dz). */
int lvx_octree_layout(const int32_t dims[3], int64_t *off, int64_t *ldims, int32_t *n_levels);

/* Fills levels 1.. of flat_d (level 0 already at offset 0) with the 2x2x2 means. */
int lvx_build_octree(float *flat_d, const int32_t dims[3], void *stream);

int lvx_occupancy_dilate(const uint8_t *counts_d, const int32_t dims[3], uint8_t *occ_d,
                         void *stream);

/* Per cell of the grid padded by one voxel, over the cell's in-grid 27-neighbourhood:
 *   nsum_d  u16[(rz+2)(ry+2)(rx+2)]  sum of counts.  nsum > 0 is the dilated occupancy
 *           of _occupancy_dilated (raycast.py:351-366); the value is the number of
 *           candidate segments the reference's neighbour gather visits for a window in
 *           that cell (_kernels.py:811-821), i.e. what `intersection_tests` adds per window;
 *   nmask_d u32[same] (nullable)  bit (dz+1)*9+(dy+1)*3+(dx+1) set when that neighbour
 *           holds segments; bit order == the reference's gather order;
 *   ncell_d u64[same] (nullable)  nmask | (u64)nsum << 32: both in ONE 8-byte load per DDA window
 *           (the wavefront engine's walk reads these).
 * The frame kernel reads these instead of 27 voxel headers per window. */
int lvx_neighbor_sums(const uint8_t *counts_d, const int32_t dims[3], uint16_t *nsum_d,
                      uint32_t *nmask_d, uint64_t *ncell_d, void *stream);

/* ------------------------------------------------------------------------- */
/* Ray-caster: render_rows + stream_hit + dda_collect + tube/sphere + sort     */
/* (_kernels.py:76-341, 625-923) and the density-grid secondary rays           */
/* (cone_blocking :386-422, ao_density_point :592-605, trilinear :346-383).    */
/* ------------------------------------------------------------------------- */

typedef struct {
    double o[3], r[3], u[3], f[3]; /* position, right, up, forward: _camera_args raycast.py:335-341 */
    double tan_half, aspect;
    int32_t width, height;
} lvx_camera;

typedef struct {
    int32_t rx, ry, rz;
    int32_t n_bins;            /* bin resolution of packed_d (only read when the frame renders from packed_d) */
    const uint8_t *counts_d;
    const uint32_t *offsets_d;
    const lvx_seg_record *seg_rec_d;
    const float *table_d;      /* f32[256,4] */
    const uint16_t *nsum_d;    /* from lvx_neighbor_sums (all three needed in neighbour mode) */
    const uint32_t *nmask_d;
    const uint64_t *ncell_d;
    const uint8_t *packed_d;   /* the encoded records (voxelizer.py:79-89); NULL unless the frame is to be
                                * rendered straight from them (lvx_render_wf) */
} lvx_model;

typedef struct {
    double tube_r, base_alpha, tau;
    double ka, kd, ks, shininess;
    double light[3];
    double bg[4];
    int32_t opacity_mode, neighbor, joints, headlight;
    int32_t shadow_mode, ao_mode, ao_n_rays, _pad;
    double ao_radius;
} lvx_params;

/* One level of the representative-line field (lod.py:61-79 RepLevel + _rep_args,
 * raycast.py:391-402): one optional line per voxel of the grid coarsened `level` times. */
typedef struct {
    const uint8_t *valid_d; /* u8[V_level] */
    const float *a_d;       /* f32[V_level,3] grid units */
    const float *b_d;
    const float *w_d;       /* f32[V_level] summed member length */
    int32_t dims[3];        /* ceil(grid / 2^level) */
    int32_t _pad;
    double size;            /* 2^level */
} lvx_replines;

typedef struct {
    const float *oct_flat_d;           /* flat octree (nullable when unused) */
    int64_t oct_off[LVX_MAX_LEVELS + 1];
    int64_t oct_dims[LVX_MAX_LEVELS * 3];
    int32_t n_levels, _pad;
    const float *ao_flat_d;            /* baked AO field f32[V] (nullable) */
    const double *ao_dirs_d;           /* f64[ao_n_rays,3] hemisphere lattice (nullable) */
    lvx_replines rep;                  /* level used by shadow_mode = LVX_SHADOW_REPLINES (valid_d nullable) */
} lvx_lod;

/* Screen partition for multi-GPU: the image is cut into tile_w x tile_h pixel
 * tiles numbered row-major; this call renders tiles tile_first, tile_first +
 * tile_step, ...  With compact != 0 the output is the rank's tiles back to back
 * ([n_my_tiles, tile_h, tile_w, 4] f32, the NCCL send buffer); otherwise pixels
 * are written in place into the full (H, W, 4) image. */
typedef struct {
    int32_t tile_w, tile_h, tile_first, tile_step, compact, _pad;
} lvx_tiling;

/* img_d f32, row_stats_d i64[H,3] (steps, tests, overflow; caller zeroes it),
 * hitbuf_d: per-thread hit scratch, lvx_render_scratch_bytes() bytes.
 * Every pixel of the image is written exactly once and never read, so img_d may also be
 * pinned host memory mapped into the device's address space (cudaHostAlloc under unified
 * addressing): the image then reaches the host while the frame is still being computed.
 * lvx_render_wf recognises such a pointer (cudaPointerGetAttributes) and lets a copy engine lay
 * the pixels of the rays that miss the grid (a constant) from a second stream of its own, joined
 * inside the call. */
size_t lvx_render_scratch_bytes(const lvx_camera *cam, const lvx_tiling *tiling);
int lvx_render(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
               const lvx_lod *lod, const lvx_tiling *tiling, float *img_d,
               int64_t *row_stats_d, void *scratch_d, void *stream);

/* Measurement aid (bench.py roofline): the same frame, additionally setting bit v of
 * voxel_bits_d (u32[ceil(V/32)], caller-zeroed) for every voxel whose header the
 * reference's gather would read (`counts[lin]`, _kernels.py:817-820): the window's
 * voxel and, in neighbour mode, its 26 in-grid neighbours, for every non-skipped
 * window up to early termination.  Distinct voxels / their segments give the
 * unique-bytes-touched figure of SURVEY.md 8(d). */
/* Wavefront frame path (csrc/lvx_wavefront.cu): the same frame as lvx_render -- same image,
 * same row_stats -- computed by streaming kernels over device queues (init / walk /
 * candidates / exact / composite, iterated until every ray is finished) instead of one
 * monolithic kernel.  Replaces the same reference call, _kernels.render_rows
 * (_kernels.py:735-923, called from raycast.py:498-510).  `scratch_d` is caller-owned,
 * 256-byte aligned, at least lvx_render_wf_scratch_bytes(cam, tiling, scale) bytes;
 * `scale` >= 1 enlarges the queues.  Returns LVX_E_RANGE when a queue overflowed (the
 * image is then undefined): call again with a larger scale.  Synchronises the stream. */
size_t lvx_render_wf_scratch_bytes(const lvx_camera *cam, const lvx_tiling *tiling, double scale);
int lvx_render_wf(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                  const lvx_lod *lod, const lvx_tiling *tiling, float *img_d,
                  int64_t *row_stats_d, void *scratch_d, size_t scratch_bytes, double scale,
                  void *stream);

/* Kernel launches (and walk/composite iterations) of this thread's last lvx_render_wf call. */
int lvx_render_wf_last_launches(int *iterations);

int lvx_render_footprint(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                         const lvx_lod *lod, const lvx_tiling *tiling, float *img_d,
                         int64_t *row_stats_d, uint32_t *voxel_bits_d, void *stream);

/* Scatter compact tiles (any rank's send buffer) into the full image. */
int lvx_untile(const float *tiles_d, const lvx_tiling *tiling, int32_t width, int32_t height,
               float *img_d, void *stream);

/* Multi-GPU frame assembly on the gathering rank (no reference counterpart: the reference is
 * single-process, raycast.py:468-521 writes rows in place): the compact tile buffers of all
 * `world` ranks, rank r's at recv_d + r * rank_stride_floats (tile k of the frame is tile
 * k / world of rank k % world, tiles of tile_w x tile_h RGBA float32 pixels), are scattered
 * into the (height, width, 4) image with ONE launch.  Pointers 16-byte aligned. */
int lvx_untile_all(const float *recv_d, int64_t rank_stride_floats, int32_t world, int32_t tile_w,
                   int32_t tile_h, int32_t width, int32_t height, float *img_d, void *stream);

/* ------------------------------------------------------------------------- */
/* AO bake: precompute_ao_kernel (_kernels.py:608-620) + the clip/cast of      */
/* precompute_voxel_ao (illumination.py:193-214).                              */
/* ------------------------------------------------------------------------- */

/* Host: Fibonacci lattice (fibonacci_dir, _kernels.py:541-552) with libm cos/sin. */
int lvx_fibonacci_dirs(int32_t n, int32_t hemisphere, double jitter, double *out_host);

int lvx_ao_bake(const uint8_t *counts_d, const int32_t dims[3], int32_t n_rays,
                double radius, double step, const double *dirs_d, const float *level0_d,
                float *ao_d, void *stream);

/* ------------------------------------------------------------------------- */
/* Point probes (the Python-level reference ops used by the parity tests):     */
/* traverse_voxels raycast.py:170-181, intersect_ray_tube/sphere :184-213,     */
/* cone_soft_shadow / ao_density_rays / sample_ao illumination.py:142-225.     */
/* ------------------------------------------------------------------------- */

/* windows of one ray: out_vox_d i64[cap,3], out_t_d f64[cap,2], n_d i64[1] */
int lvx_probe_dda(const double o[3], const double d[3], const int32_t dims[3], int32_t pad,
                  int64_t cap, int64_t *out_vox_d, double *out_t_d, int64_t *n_d, void *stream);
/* n queries; rays_d f64[n,6] (o,d); a_d,b_d f32[n,3] (f32_axis=1: the frame-kernel
 * specialisation) or f64[n,3] (f32_axis=0); out_d f64[n,6] = hit,t_in,t_out,normal */
int lvx_probe_tube(const double *rays_d, const void *a_d, const void *b_d, double radius,
                   int32_t f32_axis, int64_t n, double *out_d, void *stream);
int lvx_probe_sphere(const double *rays_d, const double *c_d, double radius, int64_t n,
                     double *out_d, void *stream);
int lvx_probe_trilinear(const float *flat_d, int64_t off, const int64_t ldims[3], double scale,
                        const double *pts_d, int64_t n, double *out_d, void *stream);
int lvx_probe_cone(const lvx_lod *lod, const double *pts_d, const double light[3],
                   double eps, int64_t n, double *out_d, void *stream);
int lvx_probe_ao_density(const lvx_lod *lod, const double *pts_d, const double *normals_d,
                         int32_t n_rays, double radius, double step, const double *dirs_d,
                         int64_t n, double *out_d, void *stream);

/* Representative lines.
 * lvx_rep_level: one level of build_rep_lines (lod.py:224-284): every parent voxel averages
 * its members -- level 1: the segments of its 2x2x2 child voxels (counts/offsets/seg_rec of
 * the model, c_valid/c_a/c_b/c_w NULL); level >= 2: the representatives of the level below
 * (seg_rec NULL) -- with the flip rule and face-bin snap of representative_line (:141-169)
 * and, if `adjacency`, the three passes of _adjacency_snap (:176-221).  child_dims is the
 * grid of the level below; outputs cover ceil(child_dims / 2).
 * lvx_probe_replines: _kernels.replines_ray_blocked (_kernels.py:498-538), the kernel behind
 * illumination.replines_shadow (illumination.py:115-139); out[i] = 1 when blocked. */
int lvx_rep_level(const int32_t child_dims[3], const uint8_t *c_counts_d, const uint32_t *c_offsets_d,
                  const lvx_seg_record *seg_rec_d, const uint8_t *c_valid_d, const float *c_a_d,
                  const float *c_b_d, const float *c_w_d, int32_t level, int32_t n_bins,
                  int32_t adjacency, uint8_t *valid_d, float *rep_a_d, float *rep_b_d, float *rep_w_d,
                  void *stream);
int lvx_probe_replines(const lvx_replines *rep, const double *rays_d, const double *max_t_d,
                       double radius_base, int64_t n, int32_t *out_d, void *stream);

/* Brute-force reference renderer: _kernels.oracle_rows (_kernels.py:926-1082)
 * behind metrics.brute_force_render (metrics.py:58-107) -- every primitive against every pixel,
 * hits ordered globally, the shared compositing rules; no DDA, windows or ownership.
 *   lvx_brute_count   hit_count_d[y*W+x] = hits of the pixel (uncapped)
 *   lvx_brute_render  hit_off_d = exclusive scan of min(hit_count, 8192) (caller); the hit buffers
 *                     hold sum(min(hit_count, 8192)) entries; seg_lin_d[i] = home voxel of segment
 *                     i; row_stats as lvx_render with voxel_steps 0 and the definitional test count */
int lvx_brute_count(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                    int64_t n_seg, uint32_t *hit_count_d, void *stream);
int lvx_brute_render(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                     const lvx_lod *lod, int64_t n_seg, const uint32_t *seg_lin_d,
                     uint32_t *hit_count_d, const int64_t *hit_off_d, double *hit_t_d,
                     uint64_t *hit_key_d, double *hit_scale_d, double *hit_alpha_d, float *hit_c_d,
                     float *img_d, int64_t *row_stats_d, void *stream);

/* Geometry secondary rays as point probes.
 * lvx_probe_blocked: _kernels.geometry_ray_blocked (_kernels.py:450-495), the kernel behind
 * illumination.hard_shadow (illumination.py:96-112): rays f64[n,6] = origin + unit direction,
 * out[i] = 1 if a tube (or joint sphere) is entered at 1e-9 < t_in < max_t[i].
 * lvx_probe_ao_hemisphere: _kernels.ao_hemisphere_point (_kernels.py:572-589), behind
 * illumination.ao_hemisphere_geometry (illumination.py:158-173), jitter 0; dirs_d is the
 * hemisphere lattice of lvx_fibonacci_dirs(n_rays, 1, 0).  The model needs counts, offsets,
 * seg_rec and nmask. */
int lvx_probe_blocked(const lvx_model *model, const double *rays_d, const double *max_t_d,
                      double radius, int32_t joints, int64_t n, int32_t *out_d, void *stream);
int lvx_probe_ao_hemisphere(const lvx_model *model, const double *pts_d, const double *normals_d,
                            int32_t n_rays, double radius, const double *dirs_d, double tube_r,
                            int64_t n, double *out_d, void *stream);

/* ------------------------------------------------------------------------- */
/* Probes behind the remaining Python-level reference ops (tests re-pointed at   */
/* this package call them through the same names as the reference's).            */
/* ------------------------------------------------------------------------- */

/* _clip_batch (voxelizer.py:213-263) with its float64 outputs, as used by the reference op
 * clip_curve_to_voxels (voxelizer.py:273-287): every kept chord's voxel (i64[.,3]), entry and
 * exit point (f64[.,3]), entry / exit attribute (f64[.,2]) and its key (edge index << 16 |
 * ordinal on the edge).  Chords are appended in arbitrary order; sorting by key gives the
 * reference's order.  *n_d = number of chords found (may exceed `capacity`: call again). */
int lvx_probe_clip(const double *pts_d, const double *attrs_d, const uint8_t *first_d, int64_t n_points,
                   const int32_t dims[3], uint64_t capacity, int64_t *vox_d, double *p_in_d, double *p_out_d,
                   double *attr_d, uint64_t *key_d, uint64_t *n_d, void *stream);

/* shade_scalar (_kernels.py:316-329) for n rows of (normal, light, view) = f64[n,9]; the op behind
 * shade_local (raycast.py:286-294). */
int lvx_probe_shade(const double *nlv_d, double ka, double kd, double ks, double shininess, int64_t n,
                    double *out_d, void *stream);

/* representative_line (lod.py:141-169) for one explicit member list: starts/ends f64[m,3] in the
 * given order, voxel cube (origin, size), bin resolution.  out_d f64[7] = a, b, weight;
 * scratch_d f64[m]. */
int lvx_probe_rep_line(const double *starts_d, const double *ends_d, int64_t m, const double origin[3],
                       double size, int32_t n_bins, double *scratch_d, double *out_d, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LINEVOX_B200_H */
