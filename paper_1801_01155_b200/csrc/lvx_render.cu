// Ray-caster for sm_100a: one thread per pixel in warp-coherent 8x4 pixel tiles,
// incremental 3D-DDA, exact float64 tube / joint-sphere tests, ordered insertion of
// the owned hits, front-to-back compositing with the reference's de-duplication
// rules and early ray termination.
//
//   render_rows   _kernels.py:735-923     stream_hit   _kernels.py:650-730
//   dda_collect   _kernels.py:164-256     _hit_before  _kernels.py:261-270
//   _seen_check_and_mark / _sphere_seen   _kernels.py:625-647
//
// The reference visits, for every non-empty window of a ray, all segments of the
// window's 27-voxel neighbourhood and runs three float64 intersection tests on each
// (~700 tests per ray on the bench scene).  A hit only counts for a window if its
// entry parameter t_in falls inside the window ("ownership").  This kernel produces
// the same composited sequence and the same counters with far less work:
//
//  * `intersection_tests` is a sum of candidate counts, so it is read from the
//    neighbour-sum grid (one u16 per window, lvx_neighbor_sums) instead of counted;
//  * a hit owned by a window has its entry point on the ray piece inside the window's
//    voxel and within tube_radius of its segment, which lies in its home voxel: only
//    neighbour voxels within tube_radius of the ray piece's bounding box can own
//    anything (sub-box cull, a subset of the 27 in the same scan order);
//  * per candidate, a float32 bounding-sphere test in window-local coordinates
//    (conservative: margins orders of magnitude above float32 rounding) rejects
//    segments that cannot be hit inside this window; survivors are queued and then
//    run through the exact float64 tests in a second, warp-converged phase;
//  * a hit is buffered as (t_in, voxel, segment, lid/kind/ordinal) only; t_out and
//    the normal are recomputed (bit-identically) for hits that are composited.  A
//    window with more owned hits than the buffer holds is finished by extra gather
//    passes that continue after the last composited key, so the composited sequence
//    is the reference's total order (t_in, home voxel, lid, kind, gather order).
#include <math_constants.h>

#include "lvx_geom.cuh"
#include "lvx_shade.cuh"

namespace {

// tuning knobs (overridable with -D for experiments)
#ifndef LVX_HIT_FLUSH
#define LVX_HIT_FLUSH 20
#endif
#ifndef LVX_SHADE_BATCH
#define LVX_SHADE_BATCH 4
#endif
#ifndef LVX_SLOTS
#define LVX_SLOTS 8
#endif
#ifndef LVX_MIN_BLOCKS
#define LVX_MIN_BLOCKS 3
#endif
#ifndef LVX_WALK_STEPS
#define LVX_WALK_STEPS 8
#endif
constexpr int kHitCap = 32;                 // sorted per-thread hit buffer (entries)
constexpr int kHitFlush = LVX_HIT_FLUSH;    // a lane with this many buffered hits asks for a composite
constexpr int kSlots = LVX_SLOTS;           // windows a lane may open between two composites (<= 16)
constexpr int kShadeBatch = LVX_SHADE_BATCH;  // hits per ray and round in the pooled shading stage
constexpr int kWalkSteps = LVX_WALK_STEPS;  // DDA steps a lane may take per round looking for a window
constexpr int kItemCap = 1024;              // voxel items per round and block (>= 27)
#ifndef LVX_WPB
#define LVX_WPB 4
#endif
#ifndef LVX_CAND
#define LVX_CAND 2
#endif
constexpr int kWarpsPerBlock = LVX_WPB;
constexpr int kCand = LVX_CAND;             // candidates per thread and chunk of the pre-reject stage
constexpr double kCullMargin = 1e-4;   // sub-box cull slack (float64 path, rounding ~1e-12)
constexpr float kRejectMargin = 2e-3f; // bounding-sphere slack (float32 path, rounding ~1e-5)

struct RenderArgs {
    lvx_camera cam;
    lvx_params p;
    int rx, ry, rz;
    const u8 *counts;
    const u32 *offsets;
    const lvx_seg_record *rec;
    const float *table;
    const u16 *nsum;
    const u32 *nmask;
    LvxOctree oc;
    const float *ao_flat;
    const double *ao_dirs;
    LvxRepLevel rep;          // representative-line level of shadow_mode = replines
    double rep_radius_base;   // tube_radius * 2^level (raycast.py:425)
    lvx_tiling tl;
    int tiles_x, n_my_tiles;
    float *img;
    unsigned long long *row_stats;
    u32 *footprint;  // instrumentation pass only: bitmap of voxels whose header the reference reads
};

// hit meta word: lid 5 bits | kind3 2 (0 tube, 1 sphere A, 2 sphere B) | gather ordinal 10 | slot 4
__device__ __forceinline__ u32 meta_lid(u32 m) { return m & 31u; }
__device__ __forceinline__ u32 meta_kind3(u32 m) { return (m >> 5) & 3u; }
__device__ __forceinline__ u32 meta_ord(u32 m) { return (m >> 7) & 1023u; }
__device__ __forceinline__ u32 meta_slot(u32 m) { return m >> 17; }

// _hit_before (_kernels.py:261-270) extended by the gather ordinal, which is what a
// stable insertion sort resolves remaining ties with.
__device__ __forceinline__ bool key_before(double ta, u32 la, u32 ma, double tb, u32 lb, u32 mb) {
    if (ta != tb) return ta < tb;
    if (la != lb) return la < lb;
    const u32 lida = meta_lid(ma), lidb = meta_lid(mb);
    if (lida != lidb) return lida < lidb;
    const u32 ka = meta_kind3(ma) ? 1u : 0u, kb = meta_kind3(mb) ? 1u : 0u;
    if (ka != kb) return ka < kb;
    return meta_ord(ma) < meta_ord(mb);
}

struct PixelState {
    double acc[4];
    int n_seen, n_sph;
    // 64-bit Bloom filters over the keys of the two tables below: a clear bit proves the key
    // was never inserted, so the linear search (the reference's, :625-647) can be skipped
    unsigned long long seen_bloom, sph_bloom;
    u32 seen_key[LVX_MAX_SEEN];
    u32 seen_mask[LVX_MAX_SEEN];
    float sph[LVX_MAX_SEEN][3];
};

// stream_hit, _kernels.py:650-730, split in two.  Everything that does not depend on the
// pixel's running state -- shadow term, AO term, alpha, Blinn scale (:673-718) -- is
// `shade_hit`, which any lane of the warp can evaluate for any ray's hit; the
// de-duplication rules and the front-to-back accumulation (:666-670, :719-730) are
// `accumulate_hit`, run by the ray's own lane in hit order.  The arithmetic and its
// order are the reference's, so the result is bit-identical to the fused form.
// Returns the accumulated alpha.
__device__ __forceinline__ double accumulate_hit(PixelState &S, const RenderArgs &A, double scale,
                                                 double alpha, u32 lin, u32 lid, u32 attr,
                                                 bool is_sphere, float cx, float cy, float cz) {
    unsigned long long sph_bit = 0;
    if (is_sphere) {
        const u32 hsh = (__float_as_uint(cx) * 0x9E3779B1u) ^ (__float_as_uint(cy) * 0x85EBCA77u) ^
                        (__float_as_uint(cz) * 0xC2B2AE3Du);
        sph_bit = 1ull << (hsh >> 26);
        if (S.sph_bloom & sph_bit) {
            for (int i = S.n_sph - 1; i >= 0; --i)  // the most recent centres are the likely repeats
                if (S.sph[i][0] == cx && S.sph[i][1] == cy && S.sph[i][2] == cz) return S.acc[3];
        }
    }
    {
        const u32 bit = 1u << lid;
        const unsigned long long kb = 1ull << ((lin * 0x9E3779B1u) >> 26);
        bool found = false;
        if (S.seen_bloom & kb) {
            for (int i = S.n_seen - 1; i >= 0; --i) {
                if (S.seen_key[i] == lin) {
                    if (S.seen_mask[i] & bit) return S.acc[3];
                    S.seen_mask[i] |= bit;
                    found = true;
                    break;
                }
            }
        }
        if (!found && S.n_seen < LVX_MAX_SEEN) {
            S.seen_key[S.n_seen] = lin;
            S.seen_mask[S.n_seen] = bit;
            S.n_seen += 1;
            S.seen_bloom |= kb;
        }
    }
    const float4 col = __ldg(reinterpret_cast<const float4 *>(A.table) + attr);
    const double trans = 1.0 - S.acc[3];
    const double w = trans * alpha;
    S.acc[0] += w * scale * (double)col.x;
    S.acc[1] += w * scale * (double)col.y;
    S.acc[2] += w * scale * (double)col.z;
    S.acc[3] += w;
    if (is_sphere && S.n_sph < LVX_MAX_SEEN) {
        S.sph[S.n_sph][0] = cx;
        S.sph[S.n_sph][1] = cy;
        S.sph[S.n_sph][2] = cz;
        S.n_sph += 1;
        S.sph_bloom |= sph_bit;
    }
    return S.acc[3];
}

// Conservative float32 test in window-local coordinates: can a primitive whose points
// all lie within `reach` of centre c be entered by the ray inside this window?
//   q0    ray point at the window start, d unit direction, tlen window length
// The entry point lies on the ray piece [0, tlen] and within `reach` of c.
__device__ __forceinline__ bool may_enter(float cx, float cy, float cz, float q0x, float q0y,
                                          float q0z, float dx, float dy, float dz, float tlen,
                                          float reach) {
    const float wx = cx - q0x, wy = cy - q0y, wz = cz - q0z;
    const float tc = wx * dx + wy * dy + wz * dz;
    const float d2 = (wx * wx + wy * wy + wz * wz) - tc * tc;
    return d2 <= reach * reach && tc >= -reach && tc <= tlen + reach;
}

// Instrumentation (lvx_render_footprint): set the bits of the voxels whose headers the
// reference's gather reads for a window at packed voxel `pv` (own voxel, or the in-grid
// 27-neighbourhood in neighbour mode).
__device__ void mark_footprint(const RenderArgs &A, u32 pv, bool neighbor) {
    const int wx = (int)(pv & 1023u) - 1, wy = (int)((pv >> 10) & 1023u) - 1, wz = (int)(pv >> 20) - 1;
    const int r = neighbor ? 1 : 0;
    for (int nz_ = max(wz - r, 0); nz_ <= min(wz + r, A.rz - 1); ++nz_)
        for (int ny_ = max(wy - r, 0); ny_ <= min(wy + r, A.ry - 1); ++ny_)
            for (int nx_ = max(wx - r, 0); nx_ <= min(wx + r, A.rx - 1); ++nx_) {
                const u32 l = (u32)(nx_ + A.rx * (ny_ + A.ry * nz_));
                atomicOr(&A.footprint[l >> 5], 1u << (l & 31u));
            }
}

// The rays of a thread block (kWarpsPerBlock 8x4 pixel tiles, one ray per thread) are
// processed in bulk-synchronous ROUNDS.  Rays are bound to threads only where per-ray state
// is needed (the DDA walk, the sorted hit buffer, the running colour); every gather-type
// stage is pooled in shared memory and dealt out evenly over all threads of the block, so
// the few rays that cross crowded voxels do not serialise their warp, threads whose own ray
// is finished keep working for the others, and all warps of the block run the same stage at
// the same time (the kernel is far larger than the instruction cache):
//
//  W  "walk": every thread that may open a window steps its DDA (at most kWalkSteps steps)
//     until it finds a window whose culled neighbourhood holds segments; it opens a slot
//     and publishes the window (cell, local ray start, length, [t0,t1)) in shared memory.
//  V  "voxels": the occupied neighbour voxels of all open windows are listed (thread-major,
//     the reference's z,y,x scan order inside a window); threads read the voxel headers
//     item-parallel and a prefix sum of the counts enumerates the candidates.
//  C  "candidates": kThreads candidates at a time, one per thread whichever ray they belong
//     to: record load + conservative float32 pre-reject against the owner's window.
//     Survivors are appended (order-preserving) to a ring in shared memory.
//  E  "exact": whenever kThreads survivors are queued, one exact float64 test set per
//     thread, including the ownership test t0 <= t_in < t1 of the owner's window; each
//     owner then takes its owned hits in candidate order (gather ordinals, sorted insertion
//     into its private hit buffer).
//  S  "composite": when some thread has enough hits buffered (or nobody can walk on), every
//     thread composites its buffered hits in order; shading is pooled like the exact tests.
//
// Every window opened in a round is completely scanned by the end of that round, so the
// buffered hits always belong to complete windows.  A ray may have scanned a few windows
// past the one in which it terminates; that is invisible in the output: the counters are
// snapshotted per window (w_tests / w_over) and the snapshot of the terminating hit's
// window is what gets reported, exactly the reference's count.
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr int kChunk = kThreads * kCand;    // candidates per pre-reject chunk
constexpr int kSurvNeed = kThreads + kChunk;  // fewer than kThreads queued + one chunk of survivors
constexpr int kSurvCap = kSurvNeed <= 256 ? 256 : (kSurvNeed <= 512 ? 512 : (kSurvNeed <= 1024 ? 1024 : 2048));
static_assert(kThreads < 255, "owner ids travel in 8 bits and 255 is the idle mark");
static_assert(kSurvCap >= kSurvNeed, "survivor ring too small");

struct BlockPool {
    double dir[kThreads][3];       // ray directions (the origin is shared)
    double wt[kThreads][2];        // open window of each thread: parameter range [t0, t1)
    union {
        struct {                       // stages V, C, E
            double res[kThreads][3];   // exact batch: t_in of tube / sphere A / sphere B
            u32 it_lin[kItemCap];      // voxel items: linear index, first record, candidate prefix
            u32 it_base[kItemCap];
            u32 it_cstart[kItemCap + 1];
            u32 sv_seg[kSurvCap];      // survivor ring
            u32 sv_lin[kSurvCap];
            u16 it_key[kItemCap];      // owner thread << 5 | neighbour bit
            u16 sv_meta[kSurvCap];     // primitive mask 3 | owner << 8
            u16 sv_hit[kSurvCap];      // exact stage's result: owned-hit mask 3 | lid << 3 | owner << 8
            u8 o_first[kThreads], o_last[kThreads];
        } g;
        struct {                       // stage S
            double res[kThreads * kShadeBatch][2];  // scale, alpha
            u32 seg[kThreads * kShadeBatch];
            u16 meta[kThreads * kShadeBatch];       // kind | owner thread << 3
        } s;
    };
    float fdir[kThreads][3];       // float32 copies for the pre-reject
    float wq0[kThreads][3];        // open window: ray point at t0, window-local
    float wtlen[kThreads];
    int wcell[kThreads][3];
    int wsum[2][kWarpsPerBlock];   // per-warp partial sums of the block scans (double-buffered)
    int total_v;
};

// Exclusive prefix sum over the block's threads (one barrier).  `scratch` must not be the
// buffer used by the previous call.
__device__ __forceinline__ int block_scan_excl(int v, int *scratch, int lane, int warp, int &total) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) scratch[warp] = inc;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarpsPerBlock; ++w) {
        const int t = scratch[w];
        if (w < warp) base += t;
        tot += t;
    }
    total = tot;
    return base + inc - v;
}

// Developer instrumentation (-DLVX_STAGE_CLOCKS): thread 0 of every block accumulates the
// cycles between stage boundaries and a few work counters into lvx_stage_clk.
#ifdef LVX_STAGE_CLOCKS
__device__ unsigned long long lvx_stage_clk[32];
#define LVX_CLK(k)                                         \
    do {                                                   \
        if (tid == 0) {                                    \
            const long long now_ = clock64();              \
            s_clk[k] += (unsigned long long)(now_ - clk_last); \
            clk_last = now_;                               \
        }                                                  \
    } while (0)
#define LVX_CNT(k, v)                                      \
    do {                                                   \
        if (tid == 0) s_clk[k] += (unsigned long long)(v); \
    } while (0)
#else
#define LVX_CLK(k) do {} while (0)
#define LVX_CNT(k, v) do {} while (0)
#endif

// GEOM: the frame uses geometry secondary rays (hard shadows / hemisphere AO); kept out of
// the common instantiation, whose register budget is tight
template <bool FOOTPRINT, bool GEOM>
__global__ void __launch_bounds__(kThreads, LVX_MIN_BLOCKS)
render_kernel(const RenderArgs A) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const i64 gw = (i64)blockIdx.x * kWarpsPerBlock + warp;
    const int wpt_x = A.tl.tile_w >> 3, wpt_y = A.tl.tile_h >> 2;
    const int warps_per_tile = wpt_x * wpt_y;
    const i64 k = gw / warps_per_tile;  // index into this rank's tile list
    const int wi = (int)(gw % warps_per_tile);
    const bool tile_ok = k < A.n_my_tiles;
    const i64 tile = (i64)A.tl.tile_first + k * A.tl.tile_step;
    const int tx = (int)(tile % A.tiles_x), ty = (int)(tile / A.tiles_x);
    const int lx = (wi % wpt_x) * 8 + (lane & 7), ly = (wi / wpt_x) * 4 + (lane >> 3);
    const int x = tx * A.tl.tile_w + lx, y = ty * A.tl.tile_h + ly;
    const int W = A.cam.width, H = A.cam.height;
    const bool active = tile_ok && x < W && y < H;

    unsigned long long steps = 0, tests = 0, overflow = 0;
    const lvx_params &p = A.p;
    // primary ray, _kernels.py:769-776
    const double ndc_x = (((double)x + 0.5) / (double)W * 2.0 - 1.0) * A.cam.tan_half * A.cam.aspect;
    const double ndc_y = (1.0 - ((double)y + 0.5) / (double)H * 2.0) * A.cam.tan_half;
    double ddx = A.cam.f[0] + ndc_x * A.cam.r[0] + ndc_y * A.cam.u[0];
    double ddy = A.cam.f[1] + ndc_x * A.cam.r[1] + ndc_y * A.cam.u[1];
    double ddz = A.cam.f[2] + ndc_x * A.cam.r[2] + ndc_y * A.cam.u[2];
    const double dn = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx = ddx / dn;
    ddy = ddy / dn;
    ddz = ddz / dn;
    const double ox = A.cam.o[0], oy = A.cam.o[1], oz = A.cam.o[2];
    const int rx = A.rx, ry = A.ry, rz = A.rz;
    const bool neighbor = p.neighbor != 0, joints = p.joints != 0;
    const double tube_r = p.tube_r;
    const u32 tmul = joints ? 3u : 1u;
    const float reach_pt = (float)tube_r + kRejectMargin;  // joint sphere about an endpoint
    const double cull = tube_r + kCullMargin;

    __shared__ BlockPool P;
    P.dir[tid][0] = ddx;
    P.dir[tid][1] = ddy;
    P.dir[tid][2] = ddz;
    P.fdir[tid][0] = (float)ddx;
    P.fdir[tid][1] = (float)ddy;
    P.fdir[tid][2] = (float)ddz;
    P.g.o_first[tid] = 255;
    if (tid == 0) P.total_v = 0;
    int par = 0;   // which scratch buffer the next block scan uses

    PixelState S;
    S.acc[0] = S.acc[1] = S.acc[2] = S.acc[3] = 0.0;
    S.n_seen = 0;
    S.n_sph = 0;
    S.seen_bloom = 0;
    S.sph_bloom = 0;
    // sorted hit buffer: the hits of the windows scanned since the last composite
    double h_t[kHitCap];
    u32 h_lin[kHitCap], h_seg[kHitCap], h_meta[kHitCap];  // meta: lid 5 | kind3 2 | ordinal 10 | slot 4
    // windows opened since the last composite ("slots")
    unsigned long long w_tests[kSlots];  // intersection_tests up to and including the window
    u32 w_over[kSlots];                  // window_overflow of the window
    u32 w_vox[FOOTPRINT ? kSlots : 1];   // instrumentation: packed window voxel (+1 per axis)

    LvxDda dda;
    dda.alive = false;
    if (active) dda.init(ox, oy, oz, ddx, ddy, ddz, rx, ry, rz, neighbor ? 1 : 0);
    bool alive = active && dda.alive;  // the walk has windows left
    bool done = false;                 // early ray termination reached

    bool has_win = false;              // an open window waits to be scanned this round
    u32 m = 0, cw_mask = 0;            // its occupied sub-box bits: still to list / all
    int cur_slot = 0;
    int nh = 0, nw = 0;
    int win_start = 0;                 // first hit of the window being scanned
    u32 ord = 0;                       // gather ordinal of its next owned hit
    bool spilled = false;
    bool have_last = false;            // continuation key of a window that overflowed the buffer
    double last_t = 0.0;
    u32 last_lin = 0, last_meta = 0;
    unsigned long long over_committed = 0;

#ifdef LVX_STAGE_CLOCKS
    __shared__ unsigned long long s_clk[32];
    if (tid < 32) s_clk[tid] = 0;
    __syncthreads();
    long long clk_last = clock64();
#endif
    bool pending = false;  // (block-uniform) some thread's window did not fit into the last round
    for (;;) {
        LVX_CLK(8);
        LVX_CNT(10, 1);
        // ================= W: walk to the next window worth scanning ================================
        if (!pending) {
#pragma unroll 1
            for (int it = 0; it < kWalkSteps; ++it) {
                const bool want = alive && !done && !has_win &&
                                  !(nh >= kHitFlush || nw >= kSlots || spilled);
                if (!__any_sync(FULL, want)) break;
                if (!want) continue;
                int wx, wy, wz;
                double t0, t1;
                if (!dda.next(wx, wy, wz, t0, t1)) {
                    alive = false;
                    continue;
                }
                steps += 1;  // the reference counts every window of the full walk (:785-786)
                have_last = false;
                u32 nm, n;
                if (neighbor) {
                    const i64 pc = ((i64)(wz + 1) * (ry + 2) + (wy + 1)) * (rx + 2) + (wx + 1);
                    nm = __ldg(A.nmask + pc);
                    n = nm ? (u32)__ldg(A.nsum + pc) : 0u;
                } else {
                    n = __ldg(A.counts + (wx + (i64)rx * (wy + (i64)ry * wz)));
                    nm = n ? (1u << 13) : 0u;
                }
                if (nm == 0) continue;  // the reference's cheap skip (:793-799)
                tests += (unsigned long long)n * tmul;  // :833,855 summed over the window's gather
                // neighbour voxels that can own a hit of this window: within tube_r of the bounding
                // box of the ray piece inside the window's voxel
                const double p0x = ox + t0 * ddx, p0y = oy + t0 * ddy, p0z = oz + t0 * ddz;
                if (neighbor) {
                    const double p1x = ox + t1 * ddx, p1y = oy + t1 * ddy, p1z = oz + t1 * ddz;
                    u32 bx_ = 0x2492492u, by_ = 0x0E07038u, bz_ = 0x003FE00u;  // centre column/row/slab
                    if (fmin(p0x, p1x) - cull < (double)wx) bx_ |= 0x1249249u;
                    if (fmax(p0x, p1x) + cull > (double)(wx + 1)) bx_ |= 0x4924924u;
                    if (fmin(p0y, p1y) - cull < (double)wy) by_ |= 0x01C0E07u;
                    if (fmax(p0y, p1y) + cull > (double)(wy + 1)) by_ |= 0x70381C0u;
                    if (fmin(p0z, p1z) - cull < (double)wz) bz_ |= 0x00001FFu;
                    if (fmax(p0z, p1z) + cull > (double)(wz + 1)) bz_ |= 0x7FC0000u;
                    nm &= bx_ & by_ & bz_;
                }
                if (nm == 0 && !FOOTPRINT) continue;
                // open a slot for the window
                cur_slot = nw++;
                w_tests[cur_slot] = tests;
                w_over[cur_slot] = 0;
                if (FOOTPRINT) w_vox[cur_slot] = (u32)(wx + 1) | ((u32)(wy + 1) << 10) | ((u32)(wz + 1) << 20);
                if (nm == 0) continue;  // (only possible in the instrumented build)
                P.wcell[tid][0] = wx;
                P.wcell[tid][1] = wy;
                P.wcell[tid][2] = wz;
                P.wq0[tid][0] = (float)(p0x - (double)wx);  // window-local float32 frame
                P.wq0[tid][1] = (float)(p0y - (double)wy);
                P.wq0[tid][2] = (float)(p0z - (double)wz);
                P.wtlen[tid] = (float)(t1 - t0);
                P.wt[tid][0] = t0;
                P.wt[tid][1] = t1;
                cw_mask = m = nm;
                has_win = true;
                ord = 0;
                win_start = nh;
            }
        }

        // ================= V: list the voxels of the open windows, read their headers ================
        LVX_CLK(0);
        {
            const int nv = has_win ? __popc(m) : 0;
            int total_all;
            const int voff = block_scan_excl(nv, P.wsum[par], lane, warp, total_all);
            par ^= 1;
            if (total_all > 0) {
                // threads are admitted in thread order while their voxels fit (the first always does)
                const bool admitted = has_win && voff + nv <= kItemCap;
                if (admitted) {
                    int kk = voff;
                    for (u32 mm = m; mm; mm &= mm - 1, ++kk)
                        P.g.it_key[kk] = (u16)(((u32)tid << 5) | (u32)(__ffs((int)mm) - 1));
                    atomicMax(&P.total_v, voff + nv);
                    has_win = false;
                }
                pending = __syncthreads_or(has_win) != 0;
                const int total_v = P.total_v;
                // headers: each warp takes a contiguous slice of the items
                const int q = (total_v + kWarpsPerBlock - 1) / kWarpsPerBlock;
                const int s0 = warp * q, s1 = min(total_v, s0 + q);
                u32 run = 0;
                for (int i0 = s0; i0 < s1; i0 += 32) {
                    const int i = i0 + lane;
                    u32 cnt = 0;
                    if (i < s1) {
                        const u32 key = P.g.it_key[i];
                        const int owner = (int)(key >> 5), b = (int)(key & 31u);
                        const int bz_ = b / 9, by_ = (b - 9 * bz_) / 3, bx_ = b - 9 * bz_ - 3 * by_;
                        const u32 lin = (u32)((P.wcell[owner][0] + bx_ - 1) +
                                              rx * ((P.wcell[owner][1] + by_ - 1) + ry * (P.wcell[owner][2] + bz_ - 1)));
                        cnt = __ldg(A.counts + lin);
                        P.g.it_lin[i] = lin;
                        P.g.it_base[i] = __ldg(A.offsets + lin);
                    }
                    u32 inc = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const u32 t = __shfl_up_sync(FULL, inc, o);
                        if (lane >= o) inc += t;
                    }
                    if (i < s1) P.g.it_cstart[i] = run + inc - cnt;
                    run += __shfl_sync(FULL, inc, 31);
                }
                if (lane == 0) P.wsum[par][warp] = (int)run;
                __syncthreads();
                int total_c = 0;
                {
                    u32 base = 0;
#pragma unroll
                    for (int w = 0; w < kWarpsPerBlock; ++w) {
                        const int t = P.wsum[par][w];
                        if (w < warp) base += (u32)t;
                        total_c += t;
                    }
                    par ^= 1;
                    for (int i = s0 + lane; i < s1; i += 32) P.g.it_cstart[i] += base;
                    if (tid == 0) {
                        P.g.it_cstart[total_v] = (u32)total_c;
                        P.total_v = 0;  // for the next round
                    }
                }
                __syncthreads();

                LVX_CLK(1);
                LVX_CNT(14, total_v);
                LVX_CNT(15, total_c);
                // ============= C + E: pre-reject kChunk candidates at a time, exact tests in batches ====
                int sv_head = 0, nsv = 0;  // survivor ring (block-uniform)
                int g0 = 0;                // first candidate of the next chunk
                for (;;) {
                    if (nsv < kThreads && g0 < total_c) {
                        // ---- C: kCand consecutive candidates per thread; all record loads are issued
                        // before the first test so their latencies overlap
                        const int gf = g0 + tid * kCand;
                        int item = 0;
                        if (gf < total_c) {
                            // the item of candidate gf: the last one starting at or before gf
                            int lo = 0, hi = total_v;  // it_cstart[lo] <= gf < it_cstart[hi]
                            while (hi - lo > 1) {
                                const int mid = (lo + hi) >> 1;
                                if (P.g.it_cstart[mid] <= (u32)gf) lo = mid;
                                else hi = mid;
                            }
                            item = lo;
                        }
                        u32 mask[kCand], seg[kCand];
                        int itm[kCand];
                        float4 ra[kCand], rb[kCand];
#pragma unroll
                        for (int j = 0; j < kCand; ++j) {
                            const int g = gf + j;
                            mask[j] = 0;
                            seg[j] = 0;
                            itm[j] = item;
                            if (g < total_c) {
                                while ((u32)g >= P.g.it_cstart[item + 1]) ++item;
                                itm[j] = item;
                                seg[j] = P.g.it_base[item] + ((u32)g - P.g.it_cstart[item]);
                                ra[j] = __ldg(reinterpret_cast<const float4 *>(A.rec + seg[j]));
                                rb[j] = __ldg(reinterpret_cast<const float4 *>(A.rec + seg[j]) + 1);
                            }
                        }
                        int nmine = 0;
#pragma unroll
                        for (int j = 0; j < kCand; ++j) {
                            if (gf + j < total_c) {
                                const int owner = (int)(P.g.it_key[itm[j]] >> 5);
                                const float fwx = (float)P.wcell[owner][0], fwy = (float)P.wcell[owner][1],
                                            fwz = (float)P.wcell[owner][2];
                                const float q0x = P.wq0[owner][0], q0y = P.wq0[owner][1], q0z = P.wq0[owner][2];
                                const float fdx = P.fdir[owner][0], fdy = P.fdir[owner][1], fdz = P.fdir[owner][2];
                                const float tlen = P.wtlen[owner];
                                const float ax = ra[j].x - fwx, ay = ra[j].y - fwy, az = ra[j].z - fwz;
                                const float bx = rb[j].x - fwx, by = rb[j].y - fwy, bz = rb[j].z - fwz;
                                u32 mk = 0;
                                // the tube AND both joint spheres lie inside the segment's bounding sphere
                                if (may_enter(0.5f * (ax + bx), 0.5f * (ay + by), 0.5f * (az + bz), q0x, q0y, q0z, fdx,
                                              fdy, fdz, tlen, rb[j].w + reach_pt)) {
                                    // the tube's entry point lies on the ray within tube_r of the segment's
                                    // axis line, so the two lines pass within tube_r of each other:
                                    // |w . (d x u)| <= reach |d x u|  (absolute slack >> float32 rounding)
                                    const float ux = bx - ax, uy = by - ay, uz = bz - az;
                                    const float nx = fdy * uz - fdz * uy, ny = fdz * ux - fdx * uz, nz = fdx * uy - fdy * ux;
                                    const float wn = (ax - q0x) * nx + (ay - q0y) * ny + (az - q0z) * nz;
                                    if (wn * wn <= reach_pt * reach_pt * (nx * nx + ny * ny + nz * nz) + 1e-6f) mk = 1u;
                                    if (joints) {
                                        if (may_enter(ax, ay, az, q0x, q0y, q0z, fdx, fdy, fdz, tlen, reach_pt)) mk |= 2u;
                                        if (may_enter(bx, by, bz, q0x, q0y, q0z, fdx, fdy, fdz, tlen, reach_pt)) mk |= 4u;
                                    }
                                }
                                mask[j] = mk;
                                nmine += mk != 0;
                            }
                        }
                        // order-preserving append: thread-major, then candidate order
                        int tot;
                        int pos = sv_head + nsv + block_scan_excl(nmine, P.wsum[par], lane, warp, tot);
                        par ^= 1;
#pragma unroll
                        for (int j = 0; j < kCand; ++j) {
                            if (mask[j]) {
                                const int e = pos++ & (kSurvCap - 1);
                                const u32 key = P.g.it_key[itm[j]];
                                P.g.sv_seg[e] = seg[j];
                                P.g.sv_lin[e] = P.g.it_lin[itm[j]];
                                P.g.sv_meta[e] = (u16)(mask[j] | ((key >> 5) << 8));
                            }
                        }
                        nsv += tot;
                        g0 += kChunk;
                        LVX_CLK(2);
                        LVX_CNT(11, 1);
                        LVX_CNT(16, tot);
                        continue;
                    }
                    if (nsv == 0) break;
                    __syncthreads();
                    // ---- E: exact float64 tests + ownership, one survivor per thread ---------------------
                    const int nb = min(nsv, kThreads);
                    if (tid < nb) {
                        const int e = (sv_head + tid) & (kSurvCap - 1);
                        const u32 i = P.g.sv_seg[e], im = P.g.sv_meta[e];
                        const int owner = (int)(im >> 8);
                        // survivors are queued in thread-major owner order: every owner's share is contiguous
                        if (tid == 0 || (int)(P.g.sv_meta[(e - 1) & (kSurvCap - 1)] >> 8) != owner) P.g.o_first[owner] = (u8)tid;
                        if (tid == nb - 1 || (int)(P.g.sv_meta[(e + 1) & (kSurvCap - 1)] >> 8) != owner) P.g.o_last[owner] = (u8)tid;
                        const double rdx = P.dir[owner][0], rdy = P.dir[owner][1], rdz = P.dir[owner][2];
                        const double t0 = P.wt[owner][0], t1 = P.wt[owner][1];
                        const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + i));
                        const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + i) + 1);
                        u32 hits = 0;  // hits the owner's window OWNS: t0 <= t_in < t1 (:838, :858, :878)
                        LvxHit h;
                        if ((im & 1u) && lvx_tube_f32axis(ox, oy, oz, rdx, rdy, rdz, ra.x, ra.y, ra.z, rb.x, rb.y, rb.z,
                                                          tube_r, h) && t0 <= h.t_in && h.t_in < t1) {
                            hits |= 1u;
                            P.g.res[tid][0] = h.t_in;
                        }
                        if ((im & 2u) && lvx_sphere<false>(ox, oy, oz, rdx, rdy, rdz, (double)ra.x, (double)ra.y,
                                                           (double)ra.z, tube_r, h) && t0 <= h.t_in && h.t_in < t1) {
                            hits |= 2u;
                            P.g.res[tid][1] = h.t_in;
                        }
                        if ((im & 4u) && lvx_sphere<false>(ox, oy, oz, rdx, rdy, rdz, (double)rb.x, (double)rb.y,
                                                           (double)rb.z, tube_r, h) && t0 <= h.t_in && h.t_in < t1) {
                            hits |= 4u;
                            P.g.res[tid][2] = h.t_in;
                        }
                        // (a separate array: the neighbours read sv_meta's owner bits at the same time)
                        P.g.sv_hit[e] = (u16)(hits | (((__float_as_uint(ra.w) >> 8) & 31u) << 3) | (im & 0xFF00u));
                    }
                    __syncthreads();
                    LVX_CLK(3);
                    LVX_CNT(12, 1);
                    // ---- each owner takes its owned hits in candidate order ------------------------------
                    // (one hit per thread and iteration, so the insertions of different rays run side by side)
                    {
                        const int first = P.g.o_first[tid];
                        const int last = first == 255 ? -1 : (int)P.g.o_last[tid];
                        int j = first == 255 ? 0 : first;
                        u32 hbits = 0, om = 0;
                        int e = 0, eb = 0;  // ring slot / batch position of the survivor being taken
                        for (;;) {
                            while (hbits == 0 && j <= last) {
                                eb = j;
                                e = (sv_head + j) & (kSurvCap - 1);
                                om = P.g.sv_hit[e];
                                hbits = om & 7u;
                                ++j;
                            }
                            if (!__any_sync(FULL, hbits != 0)) break;
                            if (hbits == 0) continue;
                            const u32 kind3 = (u32)(__ffs((int)hbits) - 1);
                            hbits &= hbits - 1;
                            const double t_in = P.g.res[eb][kind3];
                            const u32 my_ord = ord++;
                            if (my_ord >= (u32)LVX_MAX_WINDOW_HITS) {
                                // the reference drops hits past its 1024-entry window buffer
                                if (!have_last) w_over[cur_slot] += 1;
                                continue;
                            }
                            const u32 qlin = P.g.sv_lin[e];
                            const u32 meta = ((om >> 3) & 31u) | (kind3 << 5) | (my_ord << 7) | ((u32)cur_slot << 17);
                            if (have_last && !key_before(last_t, last_lin, last_meta, t_in, qlin, meta))
                                continue;  // composited in an earlier pass over this window
                            int pos;
                            if (nh < kHitCap && !spilled) {
                                pos = nh++;
                            } else {
                                // keep the smallest keys of this window and redo the rest in another pass.
                                // Once a hit has been dropped nothing larger than the buffer's last key may
                                // be accepted, or the pass order would break.
                                spilled = true;
                                if (!key_before(t_in, qlin, meta, h_t[nh - 1], h_lin[nh - 1], h_meta[nh - 1])) continue;
                                pos = nh - 1;
                            }
                            while (pos > win_start &&
                                   key_before(t_in, qlin, meta, h_t[pos - 1], h_lin[pos - 1], h_meta[pos - 1])) {
                                h_t[pos] = h_t[pos - 1];
                                h_lin[pos] = h_lin[pos - 1];
                                h_seg[pos] = h_seg[pos - 1];
                                h_meta[pos] = h_meta[pos - 1];
                                --pos;
                            }
                            h_t[pos] = t_in;
                            h_lin[pos] = qlin;
                            h_seg[pos] = P.g.sv_seg[e];
                            h_meta[pos] = meta;
                        }
                    }
                    P.g.o_first[tid] = 255;
                    sv_head = (sv_head + nb) & (kSurvCap - 1);
                    nsv -= nb;
                    __syncthreads();
                    LVX_CLK(4);
                }
                // threads that did not fit this round keep their window and go first in the next one
                if (pending) continue;
            }
        }

        // ================= S: composite, _kernels.py:898-914 ============================================
        const bool walker = alive && !done;
        const bool blocked = walker && (nh >= kHitFlush || nw >= kSlots || spilled);
        const bool any_blocked = __syncthreads_or(blocked) != 0;
        const bool any_walker = __syncthreads_or(walker) != 0;
        LVX_CLK(9);
        if (any_blocked || !any_walker) {
            LVX_CNT(17, 1);
            const int n_comp = nh;  // every buffered hit belongs to a completely scanned window
            // Up to kShadeBatch hits per ray and round are listed in shared memory, every thread
            // recomputes one hit (t_out, normal) and its state-free shading terms, then each ray's
            // own thread applies them in order.
            int q = 0;
            bool comp = !done && n_comp > 0;
            for (;;) {
                const int nb = comp ? min(kShadeBatch, n_comp - q) : 0;
                int total;
                const int off = block_scan_excl(nb, P.wsum[par], lane, warp, total);
                par ^= 1;
                if (total == 0) break;
                for (int j = 0; j < nb; ++j) {
                    P.s.seg[off + j] = h_seg[q + j];
                    P.s.meta[off + j] = (u16)(meta_kind3(h_meta[q + j]) | ((u32)tid << 3));
                }
                __syncthreads();
                for (int idx = tid; idx < total; idx += kThreads) {
                    const u32 i = P.s.seg[idx], im = P.s.meta[idx];
                    const int owner = (int)(im >> 3);
                    const u32 kind3 = im & 3u;
                    const double rdx = P.dir[owner][0], rdy = P.dir[owner][1], rdz = P.dir[owner][2];
                    const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + i));
                    const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + i) + 1);
                    LvxHit h;
                    if (kind3 == 0) {
                        lvx_tube_f32axis(ox, oy, oz, rdx, rdy, rdz, ra.x, ra.y, ra.z, rb.x, rb.y, rb.z, tube_r, h);
                    } else {
                        const float cx = kind3 == 1 ? ra.x : rb.x, cy = kind3 == 1 ? ra.y : rb.y,
                                    cz = kind3 == 1 ? ra.z : rb.z;
                        lvx_sphere<true>(ox, oy, oz, rdx, rdy, rdz, (double)cx, (double)cy, (double)cz, tube_r, h);
                    }
                    double scale, alpha;
                    lvx_shade_hit<GEOM>(A, ox, oy, oz, rdx, rdy, rdz, h, __float_as_uint(ra.w) & 0xFFu, scale, alpha);
                    P.s.res[idx][0] = scale;
                    P.s.res[idx][1] = alpha;
                }
                __syncthreads();
                LVX_CLK(5);
                LVX_CNT(13, 1);
                LVX_CNT(18, total);
                for (int j = 0; j < nb; ++j) {
                    const u32 i = h_seg[q], meta = h_meta[q];
                    const u32 kind3 = meta_kind3(meta);
                    const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + i));
                    float cx = 0.0f, cy = 0.0f, cz = 0.0f;
                    if (kind3 == 1) {
                        cx = ra.x;
                        cy = ra.y;
                        cz = ra.z;
                    } else if (kind3 == 2) {
                        const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + i) + 1);
                        cx = rb.x;
                        cy = rb.y;
                        cz = rb.z;
                    }
                    const double a_now = accumulate_hit(S, A, P.s.res[off + j][0], P.s.res[off + j][1], h_lin[q],
                                                        meta_lid(meta), __float_as_uint(ra.w) & 0xFFu,
                                                        kind3 != 0, cx, cy, cz);
                    if (a_now >= p.tau) {
                        // terminated inside window `slot`: report the counters as of that window
                        const int slot = (int)meta_slot(meta);
                        done = true;
                        comp = false;
                        tests = w_tests[slot];
                        overflow = over_committed;
                        for (int jj = 0; jj <= slot; ++jj) overflow += w_over[jj];
                        if (FOOTPRINT)
                            for (int jj = 0; jj <= slot; ++jj) mark_footprint(A, w_vox[jj], neighbor);
                        break;
                    }
                    if (++q >= n_comp) comp = false;
                }
                LVX_CLK(6);
                // (the next listing is fenced from these reads by the barrier inside block_scan_excl)
            }
            // the pools of stages V/C/E overlay the shading pool: restore their idle state
            P.g.o_first[tid] = 255;
            if (!done) {
                // commit the composited windows
                for (int j = 0; j < nw; ++j) over_committed += w_over[j];
                if (FOOTPRINT)
                    for (int j = 0; j < nw; ++j) mark_footprint(A, w_vox[j], neighbor);
                if (spilled) {
                    // the buffer held only the smallest keys of the last window: scan it again
                    // (its row in P.w* is still in place), continuing after the last composited key
                    have_last = true;
                    last_t = h_t[nh - 1];
                    last_lin = h_lin[nh - 1];
                    last_meta = h_meta[nh - 1] & 0x1FFFFu;  // slot bits are not part of the order
                    w_tests[0] = w_tests[cur_slot];
                    w_over[0] = 0;  // its overflow was committed above; later passes do not recount
                    if (FOOTPRINT) w_vox[0] = w_vox[cur_slot];
                    cur_slot = 0;
                    nw = 1;
                    m = cw_mask;
                    has_win = true;
                    ord = 0;
                    win_start = 0;
                    spilled = false;
                } else {
                    nw = 0;
                }
                nh = 0;
            }
            // a window re-opened after a spill is scanned before anybody walks on
            pending = __syncthreads_or(has_win) != 0;
            LVX_CLK(6);
            if (!any_walker && !pending) break;
        }
    }
    if (!done) overflow = over_committed;
    LVX_CLK(6);

    // tail: a terminated ray still reports the window count of its full walk
    for (;;) {
        const bool go = alive;
        if (!__any_sync(FULL, go)) break;
        if (go) {
            int wx, wy, wz;
            double t0, t1;
            if (dda.next(wx, wy, wz, t0, t1)) steps += 1;
            else alive = false;
        }
    }

    LVX_CLK(7);
#ifdef LVX_STAGE_CLOCKS
    if (tid == 0) {
        s_clk[19] += 1;
        for (int q = 0; q < 32; ++q)
            if (s_clk[q]) atomicAdd(&lvx_stage_clk[q], s_clk[q]);
    }
#endif
    if (active) {
        // _kernels.py:916-920
        const double a = S.acc[3];
        float4 outp;
        outp.x = (float)(S.acc[0] + (1.0 - a) * p.bg[3] * p.bg[0]);
        outp.y = (float)(S.acc[1] + (1.0 - a) * p.bg[3] * p.bg[1]);
        outp.z = (float)(S.acc[2] + (1.0 - a) * p.bg[3] * p.bg[2]);
        outp.w = (float)(a + (1.0 - a) * p.bg[3]);
        i64 o;
        if (A.tl.compact) o = ((k * A.tl.tile_h + ly) * (i64)A.tl.tile_w + lx);
        else o = (i64)y * W + x;
        reinterpret_cast<float4 *>(A.img)[o] = outp;
    }

    // per-row counters: reduce over the 8 lanes that share an image row
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        steps += __shfl_xor_sync(FULL, steps, o);
        tests += __shfl_xor_sync(FULL, tests, o);
        overflow += __shfl_xor_sync(FULL, overflow, o);
    }
    if ((lane & 7) == 0 && tile_ok && y < H) {
        if (steps) atomicAdd(A.row_stats + 3 * (i64)y, steps);
        if (tests) atomicAdd(A.row_stats + 3 * (i64)y + 1, tests);
        if (overflow) atomicAdd(A.row_stats + 3 * (i64)y + 2, overflow);
    }
}

__global__ void __launch_bounds__(256)
untile_kernel(const float4 *__restrict__ tiles, lvx_tiling tl, int tiles_x, i64 n_tiles_mine, int W,
              int H, float4 *__restrict__ img) {
    const i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const i64 per_tile = (i64)tl.tile_w * tl.tile_h;
    if (idx >= n_tiles_mine * per_tile) return;
    const i64 k = idx / per_tile;
    const int r = (int)(idx % per_tile), lx = r % tl.tile_w, ly = r / tl.tile_w;
    const i64 tile = (i64)tl.tile_first + k * tl.tile_step;
    const int x = (int)(tile % tiles_x) * tl.tile_w + lx, y = (int)(tile / tiles_x) * tl.tile_h + ly;
    if (x < W && y < H) img[(i64)y * W + x] = tiles[idx];
}

// All ranks' compact tile buffers (rank r's tiles start at recv + r * rank_stride float4s;
// tile k of the frame is tile k / world of rank k % world) -> the full image, one thread per
// output pixel: coalesced stores, one launch whatever the number of ranks.
__global__ void __launch_bounds__(256)
untile_all_kernel(const float4 *__restrict__ recv, i64 rank_stride, int world, int tile_w, int tile_h,
                  int tiles_x, int W, int H, float4 *__restrict__ img) {
    const i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (i64)W * H) return;
    const int x = (int)(idx % W), y = (int)(idx / W);
    const i64 tile = (i64)(y / tile_h) * tiles_x + x / tile_w;
    const i64 k = tile / world;
    const int r = (int)(tile % world);
    const i64 src = (k * tile_h + (y % tile_h)) * tile_w + (x % tile_w);
    img[idx] = recv[(i64)r * rank_stride + src];
}

int check_tiling(const lvx_tiling *t) {
    LVX_REQUIRE(t && t->tile_w >= 8 && t->tile_h >= 4 && (t->tile_w % 8) == 0 &&
                    (t->tile_h % 4) == 0 && t->tile_step >= 1 && t->tile_first >= 0 &&
                    t->tile_first < t->tile_step,
                "tiling: tile_w %% 8 == 0, tile_h %% 4 == 0, 0 <= tile_first < tile_step required");
    return LVX_OK;
}

i64 my_tile_count(const lvx_tiling *t, int W, int H, int *tiles_x_out) {
    const i64 tiles_x = lvx_ceil_div(W, t->tile_w), tiles_y = lvx_ceil_div(H, t->tile_h);
    const i64 total = tiles_x * tiles_y;
    if (tiles_x_out) *tiles_x_out = (int)tiles_x;
    if (t->tile_first >= total) return 0;
    return (total - t->tile_first + t->tile_step - 1) / t->tile_step;
}

void fill_octree(LvxOctree &oc, const lvx_lod *lod) {
    memset(&oc, 0, sizeof(oc));
    if (!lod) return;
    oc.flat = lod->oct_flat_d;
    oc.n_levels = lod->n_levels;
    for (int l = 0; l <= lod->n_levels && l <= LVX_MAX_LEVELS; ++l) oc.off[l] = lod->oct_off[l];
    for (int l = 0; l < lod->n_levels * 3 && l < LVX_MAX_LEVELS * 3; ++l)
        oc.dims[l] = (int)lod->oct_dims[l];
}

}  // namespace

extern "C" {

size_t lvx_render_scratch_bytes(const lvx_camera *, const lvx_tiling *) {
    // the per-thread hit buffer and de-duplication tables live in local memory;
    // no caller-provided scratch is needed in this ABI version
    return 0;
}

static int render_impl(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                       const lvx_lod *lod, const lvx_tiling *tiling, float *img_d,
                       int64_t *row_stats_d, uint32_t *footprint_d, void *stream) {
    LVX_REQUIRE(cam && model && params && img_d && row_stats_d, "null argument");
    LVX_REQUIRE(cam->width >= 1 && cam->height >= 1, "image dims must be >= 1");
    if (int rc = check_tiling(tiling)) return rc;
    LVX_REQUIRE(model->rx >= 1 && model->ry >= 1 && model->rz >= 1 && model->counts_d &&
                    model->offsets_d && model->table_d,
                "bad model");
    LVX_REQUIRE((i64)model->rx * model->ry * model->rz < ((i64)1 << 31), "grid too large to render");
    LVX_REQUIRE(!params->neighbor || (model->nsum_d && model->nmask_d),
                "neighbour mode needs the neighbour grids (lvx_neighbor_sums)");
    LVX_REQUIRE(params->opacity_mode >= 0 && params->opacity_mode <= 2, "bad opacity mode");
    LVX_REQUIRE(params->shadow_mode >= LVX_SHADOW_NONE && params->shadow_mode <= LVX_SHADOW_CONE, "bad shadow_mode %d",
                params->shadow_mode);
    LVX_REQUIRE(params->shadow_mode != LVX_SHADOW_REPLINES ||
                    (lod && lod->rep.valid_d && lod->rep.a_d && lod->rep.b_d && lod->rep.w_d && lod->rep.size >= 2.0),
                "replines shadows need a representative-line level (lvx_lod.rep)");
    LVX_REQUIRE(params->ao_mode >= LVX_AO_NONE && params->ao_mode <= LVX_AO_PRECOMPUTED, "bad ao_mode %d",
                params->ao_mode);
    LVX_REQUIRE((params->shadow_mode != LVX_SHADOW_HARD && params->ao_mode != LVX_AO_HEMISPHERE) || model->nmask_d,
                "geometry secondary rays (hard shadows, hemisphere AO) need the neighbour grids (lvx_neighbor_sums)");
    const bool need_oct = params->shadow_mode == LVX_SHADOW_CONE || params->ao_mode == LVX_AO_DENSITY;
    LVX_REQUIRE(!need_oct || (lod && lod->oct_flat_d && lod->n_levels >= 1 &&
                              lod->n_levels <= LVX_MAX_LEVELS),
                "cone shadows / density-rays AO need a density octree");
    LVX_REQUIRE(params->ao_mode != LVX_AO_PRECOMPUTED || (lod && lod->ao_flat_d),
                "precomputed AO requested but no AO field given");
    LVX_REQUIRE((params->ao_mode != LVX_AO_DENSITY && params->ao_mode != LVX_AO_HEMISPHERE) ||
                    (lod && lod->ao_dirs_d && params->ao_n_rays >= 1),
                "density-rays / hemisphere AO need the direction lattice");

    RenderArgs A;
    memset(&A, 0, sizeof(A));
    A.cam = *cam;
    A.p = *params;
    A.rx = model->rx;
    A.ry = model->ry;
    A.rz = model->rz;
    A.counts = model->counts_d;
    A.offsets = model->offsets_d;
    A.rec = model->seg_rec_d;
    A.table = model->table_d;
    A.nsum = model->nsum_d;
    A.nmask = model->nmask_d;
    fill_octree(A.oc, lod);
    A.ao_flat = lod ? lod->ao_flat_d : nullptr;
    A.ao_dirs = lod ? lod->ao_dirs_d : nullptr;
    if (lod && lod->rep.valid_d) {
        A.rep = LvxRepLevel{lod->rep.valid_d, lod->rep.a_d, lod->rep.b_d, lod->rep.w_d, lod->rep.dims[0], lod->rep.dims[1],
                            lod->rep.dims[2], lod->rep.size};
        A.rep_radius_base = params->tube_r * lod->rep.size;
    }
    A.tl = *tiling;
    A.n_my_tiles = (int)my_tile_count(tiling, cam->width, cam->height, &A.tiles_x);
    A.img = img_d;
    A.row_stats = reinterpret_cast<unsigned long long *>(row_stats_d);
    if (A.n_my_tiles == 0) return LVX_OK;
    const i64 warps = (i64)A.n_my_tiles * (tiling->tile_w / 8) * (tiling->tile_h / 4);
    const i64 blocks = lvx_ceil_div(warps, kWarpsPerBlock);
    A.footprint = footprint_d;
    const bool geom = params->shadow_mode == LVX_SHADOW_HARD || params->shadow_mode == LVX_SHADOW_REPLINES ||
                      params->ao_mode == LVX_AO_HEMISPHERE;
    if (footprint_d && geom)
        render_kernel<true, true><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(A);
    else if (footprint_d)
        render_kernel<true, false><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(A);
    else if (geom)
        render_kernel<false, true><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(A);
    else
        render_kernel<false, false><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, (cudaStream_t)stream>>>(A);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_render(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
               const lvx_lod *lod, const lvx_tiling *tiling, float *img_d, int64_t *row_stats_d,
               void *scratch_d, void *stream) {
    (void)scratch_d;
    return render_impl(cam, model, params, lod, tiling, img_d, row_stats_d, nullptr, stream);
}

int lvx_render_footprint(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                         const lvx_lod *lod, const lvx_tiling *tiling, float *img_d,
                         int64_t *row_stats_d, uint32_t *voxel_bits_d, void *stream) {
    LVX_REQUIRE(voxel_bits_d, "null footprint bitmap");
    LVX_REQUIRE(model && model->rx <= 1022 && model->ry <= 1022 && model->rz <= 1022,
                "footprint instrumentation supports grids up to 1022 per axis");
    return render_impl(cam, model, params, lod, tiling, img_d, row_stats_d, voxel_bits_d, stream);
}

#ifdef LVX_STAGE_CLOCKS
// developer builds only: read and reset the stage counters
int lvx_debug_stage_clocks(unsigned long long *out32) {
    unsigned long long zero[32] = {0};
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out32, lvx_stage_clk, sizeof(zero));
    cudaMemcpyToSymbol(lvx_stage_clk, zero, sizeof(zero));
    return 0;
}
#endif

int lvx_untile(const float *tiles_d, const lvx_tiling *tiling, int32_t width, int32_t height,
               float *img_d, void *stream) {
    LVX_REQUIRE(tiles_d && img_d && width >= 1 && height >= 1, "bad arguments");
    if (int rc = check_tiling(tiling)) return rc;
    int tiles_x = 0;
    const i64 n = my_tile_count(tiling, width, height, &tiles_x);
    if (n == 0) return LVX_OK;
    const i64 px = n * tiling->tile_w * tiling->tile_h;
    untile_kernel<<<(unsigned)lvx_ceil_div(px, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4 *>(tiles_d), *tiling, tiles_x, n, width, height,
        reinterpret_cast<float4 *>(img_d));
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_untile_all(const float *recv_d, int64_t rank_stride_floats, int32_t world, int32_t tile_w,
                   int32_t tile_h, int32_t width, int32_t height, float *img_d, void *stream) {
    LVX_REQUIRE(recv_d && img_d && width >= 1 && height >= 1 && world >= 1, "bad arguments");
    LVX_REQUIRE(tile_w >= 8 && tile_h >= 4 && (tile_w % 8) == 0 && (tile_h % 4) == 0,
                "tiling: tile_w %% 8 == 0, tile_h %% 4 == 0 required");
    LVX_REQUIRE(rank_stride_floats >= 0 && (rank_stride_floats % 4) == 0 && ((uintptr_t)recv_d & 15) == 0 &&
                    ((uintptr_t)img_d & 15) == 0,
                "tile buffers must be 16-byte aligned and a whole number of pixels apart");
    const i64 tiles_x = lvx_ceil_div(width, tile_w), tiles_y = lvx_ceil_div(height, tile_h);
    const i64 per_rank = lvx_ceil_div(tiles_x * tiles_y, world) * tile_w * tile_h;
    LVX_REQUIRE(world == 1 || rank_stride_floats / 4 >= per_rank, "rank stride %lld floats is smaller than a rank's tiles",
                (long long)rank_stride_floats);
    const i64 px = (i64)width * height;
    untile_all_kernel<<<(unsigned)lvx_ceil_div(px, 256), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4 *>(recv_d), rank_stride_floats / 4, world, tile_w, tile_h, (int)tiles_x, width,
        height, reinterpret_cast<float4 *>(img_d));
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
