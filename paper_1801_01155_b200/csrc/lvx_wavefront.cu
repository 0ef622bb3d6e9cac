// Wavefront ray-caster for sm_100a: the frame is computed by a short sequence of
// streaming kernels over device-resident queues instead of one monolithic kernel.
//
//   render_rows   _kernels.py:735-923     stream_hit   _kernels.py:650-730
//   dda_collect   _kernels.py:164-256     _hit_before  _kernels.py:261-270
//   _seen_check_and_mark / _sphere_seen   _kernels.py:625-647
//
// Why: the per-ray work of the reference is a chain of dependent, data-dependent steps
// (walk -> gather 27 voxels -> intersect -> sort -> composite -> maybe terminate).  Bound
// to one thread (or one block) per ray that chain is latency-bound at low occupancy: the
// float64 tests need ~170 registers, the rays of a warp diverge, and the tile kernel
// (lvx_render.cu) spends most of its cycles at block barriers.  Here every link of the
// chain is its own kernel over ALL live rays, with its own register budget, full
// occupancy; the links talk through queues in device memory.  That decoupling is not free: the
// queues and the per-ray state move ~13 GB per C3 frame through L2/HBM (ncu, profiles/) against
// 0.16 GB of model bytes the algorithm touches -- ~1.5 TB/s, a fifth of the HBM peak -- and the
// frame is bound by load latency and lane divergence of the ray-parallel links, not by bandwidth:
//
//   init       one thread per pixel: primary ray, slab clip, full-walk window count
//              (`voxel_steps`), background for rays that miss; live rays are listed.
//   walk       one thread per live ray: advance the DDA by a budget of non-empty windows,
//              cull the 27-neighbourhood to the voxels that can own a hit, write one
//              window record per window and one item (window, neighbour) per voxel.
//   candidates one thread per item: voxel header, conservative float32 pre-reject of
//              every segment against the window; survivors are queued.
//   exact      one thread per survivor: exact float64 tube / joint-sphere tests, the
//              ownership test t0 <= t_in < t1, state-free shading of the owned hits
//              (AO / cone shadow / Blinn / alpha); hits go to a pool and are linked into
//              their ray's list.
//   composite  one thread per live ray: order the ray's hits by the reference's key
//              (t_in, home voxel, lid, kind, gather order), apply the de-duplication
//              rules, blend front to back, terminate at tau; finished rays write their
//              pixel and counters, the others are listed for the next iteration.
//
// The composited sequence, the image and the three counters are the reference's:
//  * gather order inside a window is (voxel z,y,x scan, segment, tube/A/B), which is the
//    order of (segment index, primitive) because records are stored in voxel scan order;
//    so the total order is a function of the hit alone and no ordinal has to be carried;
//  * `intersection_tests` is cumulative per window (neighbour-sum grid) and a terminated
//    ray reports the value of the window that owns its last composited hit;
//  * the 1024-hits-per-window cap (`window_overflow`) can only bite in windows whose
//    candidate count exceeds 1024/3; those are flagged and handled by an exact slow path.
#include <cooperative_groups.h>
#include <math_constants.h>
#include <stdlib.h>

#include "lvx_geom.cuh"
#include "lvx_shade.cuh"

namespace cg = cooperative_groups;

namespace {

// Programmatic dependent launch: every kernel of the frame is launched with the stream-serialisation
// attribute, so its launch is set up while the previous kernel of the chain drains; the first
// statement of every kernel waits for that kernel's completion and memory flush.  The ~74 launches of a frame are all dependent
// and short -- in a multi-GPU share they last 10-100 us each -- so the launch gaps are worth hiding.
#define WF_PDL_ENTER() asm volatile("griddepcontrol.wait;" ::: "memory")
// (letting the dependents in EARLY -- griddepcontrol.launch_dependents at the top of every kernel -- was
// measured and dropped: their waiting blocks take the place of the running kernel's later waves, C3
// 7.42 -> 7.79 ms; in the one-block bookkeeping kernels alone it changes nothing)

template <typename... KArgs, typename... Args>
cudaError_t wf_launch(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

constexpr int kNQ = 64;            // sub-queues per queue (spreads the allocation atomics)
constexpr int kInline = 16;        // de-duplication table entries kept inline per ray
constexpr int kThreadsWf = 256;
constexpr int kSortCap = 48;       // hits per ray and iteration sorted in local memory
constexpr u32 kNil = 0xFFFFFFFFu;
constexpr double kCullMarginWf = 1e-4;
constexpr float kRejectMarginWf = 2e-3f;
// the ray point of an item in the frame of its voxel lies in [-1, 2]: 13 fraction bits (step 1.2e-4);
// the pre-reject is conservative, its reach grows by the rounding (<= 1.06e-4 as a distance)
constexpr float kItemQScale = 8192.0f;
constexpr float kItemQSlack = 1.5e-4f;
__device__ __forceinline__ u32 item_q16(float v) {
    const float s = fminf(fmaxf(v * kItemQScale, -32768.0f), 32767.0f);
    return (u32)(unsigned short)(short)__float2int_rn(s);
}
__device__ __forceinline__ float item_unq16(u32 h) { return (float)(short)(unsigned short)(h & 0xFFFFu) * (1.0f / kItemQScale); }

// one record per window that can own hits (per-ray stride layout: ray place * wn + k)
struct __align__(16) WfWindow {
    double t1;                 // end of the window's parameter range
    unsigned long long tests;  // intersection_tests up to and including this window | big << 63
};
static_assert(sizeof(WfWindow) == 16, "window record is 16 bytes");
constexpr unsigned long long kBigBit = 1ull << 63;

// One hit = ONE 32-byte sector, written whole (no read-modify-write of a partly written sector on
// its way to DRAM) and read whole.  The sphere centre of a joint hit lives in a 16-byte side record
// that only joint hits write and only the de-duplication of joint hits reads.
struct __align__(32) WfHit {
    double t_in;
    // the rest of the reference's order (home voxel, lid, kind, then gather order) and the
    // hit's small fields as one integer:
    //   lin << 24 | lid << 19 | (kind != tube) << 18 | index in voxel << 10 | kind3 << 8 | attr
    // bit 63: dropped by the window cap (slow path only)
    unsigned long long key2;
    double scale, alpha;
};
static_assert(sizeof(WfHit) == 32, "hit record is one sector");
constexpr unsigned long long kDroppedBit = 1ull << 63;
constexpr u32 kJointRef = 0x80000000u;  // flag on a sorted hit reference: the hit is a joint sphere
__device__ __forceinline__ u32 hit_lin(unsigned long long k) { return (u32)(k >> 24) & 0x7FFFFFFFu; }
__device__ __forceinline__ u32 hit_lid(unsigned long long k) { return (u32)(k >> 19) & 31u; }
__device__ __forceinline__ u32 hit_kind3(unsigned long long k) { return (u32)(k >> 8) & 3u; }
__device__ __forceinline__ u32 hit_attr(unsigned long long k) { return (u32)k & 0xFFu; }
// gather order inside a window: (voxel scan order, index in voxel, primitive)
__device__ __forceinline__ unsigned long long hit_gather(unsigned long long k) {
    k &= ~kDroppedBit;
    return ((k >> 24) << 10) | (((k >> 10) & 255ull) << 2) | ((k >> 8) & 3ull);
}

#ifndef LVX_WF_HITSLOTS
#define LVX_WF_HITSLOTS 24
#endif
constexpr int kHitSlots = LVX_WF_HITSLOTS;  // hits per ray and iteration stored ray-parallel (the rest is listed)

// what an exact test needs of its ray, by place: one 32-byte sector, two hops from the queue
// entry (entry -> item_place -> here) instead of three (-> live -> the ray's state record)
struct __align__(32) WfRayDir {
    double dx, dy, dz, t_lo;
};

struct __align__(16) WfEntry {
    u32 seg;    // segment (| sphere B << 31 in the sphere queue)
    u32 place;  // the ray's position in the live list (saves the exact kernels a dependent load)
    u32 lin;    // home voxel of the segment
    u32 aux;    // neighbour mode: index of the segment in its voxel; own-voxel mode: the item (its window range)
};
static_assert(sizeof(WfEntry) == 16, "survivor entry is one 16-byte access");

// per-ray state, one record per pixel slot (read and written with 16-byte accesses)
struct __align__(16) WfRayWalk {   // owned by the walk
    double dir[3];
    double t_cur, t_exit, tmax_x, tmax_y, tmax_z;
    int ix, iy, iz;
    u32 flags;                     // bit 0 walk alive, bit 1 big window seen this iteration
    unsigned long long tests;      // intersection_tests of the windows walked so far
    u32 nwin, pad;                 // windows recorded this iteration
};
static_assert(sizeof(WfRayWalk) == 96, "walk state is 96 bytes");

struct __align__(32) WfRayPix {    // owned by the compositor: two sectors, read and written whole
    double acc[4];
    unsigned long long seen_bloom, sph_bloom;
    unsigned long long over;
    u16 n_seen, n_sph;
    u32 ovf;
};
static_assert(sizeof(WfRayPix) == 64, "pixel state is 64 bytes");

// control block in device memory
// windows a ray may record in the first iteration (doubling per iteration after that); also
// what the window arrays are sized for.  Swept with the spread / tail rules in place: 8 -> 12 is
// worth 0.05-0.15 ms on C2, C3 and the 1M-line scene.
#ifndef LVX_WF_WINFIRST
#define LVX_WF_WINFIRST 12
#endif
constexpr int kWinFirst = LVX_WF_WINFIRST;

struct WfCtl {
    u32 n_live[2];
    u32 item_cnt[kNQ], tube_cnt[kNQ], sph_cnt[kNQ], hit_cnt[kNQ];
    u32 pool_cnt;
    u32 err;   // bit 0 items / candidates, 1 survivors, 2 listed hits, 3 table pool
    u32 wn;    // windows per ray of the current iteration
    u32 budget;  // candidate budget per ray of the current iteration (neighbour-sum units)
    u32 live0;   // rays alive after the first iteration (what "few rays left" is measured against)
    u32 done_it;  // the iteration count the frame needed (set once, when the live list first comes up empty)
#ifdef LVX_WF_STATS
    unsigned long long dbg[8];  // developer counters: owned hits, composited, suppressed, rays with hits, terminated
#endif
};
#ifdef LVX_WF_STATS
#define WF_STAT(k, v) atomicAdd(&A.ctl->dbg[k], (unsigned long long)(v))
#else
#define WF_STAT(k, v)
#endif

struct WfArgs {
    lvx_camera cam;
    lvx_params p;
    int rx, ry, rz;
    const u8 *counts;
    const u32 *offsets;
    const lvx_seg_record *rec;
    LvxPacked pk;  // the encoded records (frames rendered straight from them: rec may then be null)
    const float *table;
    const u16 *nsum;
    const u32 *nmask;
    const unsigned long long *ncell;  // nmask | nsum << 32 per padded cell (one load per window)
    LvxOctree oc;
    const float *ao_flat;
    const double *ao_dirs;
    LvxRepLevel rep;          // representative-line level of shadow_mode = replines
    double rep_radius_base;   // tube_radius * 2^level (raycast.py:425)
    lvx_tiling tl;
    int tiles_x, n_my_tiles;
    int skip_miss;  // the pixels of rays that miss the grid are written by a copy engine (host image), not by wf_init
    float *img;
    unsigned long long *row_stats;
    // scratch
    u32 R;          // ray slots (threads of init)
    WfCtl *ctl;
    WfRayWalk *rw;  // [R]
    WfRayPix *rp;   // [R]
    uint2 *rpix;    // [R] constants of the ray: x | y << 16, offset of its pixel in the output
    u32 *head;      // [R] overflow hit list
    // de-duplication tables, contiguous per ray: a search walks ONE ray's sectors back to front
    uint2 *tab_seen;           // [R][kInline] (home voxel, lid mask)
    float4 *tab_sph;           // [R][kInline] joint-sphere centres
    uint2 *pool_seen;          // [pool_cap][LVX_MAX_SEEN - kInline]
    float4 *pool_sph;          // [pool_cap][LVX_MAX_SEEN - kInline]
    u32 pool_cap;
    u32 *live[2];
    WfWindow *win;
    u32 cap_win;
    // one 16-byte record per (ray, voxel) item: ray place in the live list, home voxel, and the ray
    // point near the voxel relative to the voxel's corner as 3 x int16 fixed point (kItemQScale)
    uint4 *item;
    double2 *item_t;             // own-voxel mode: parameter range of the item's window
    u32 capq_item;
    float4 *fdir;                // [R] float32 ray direction by place (one sector per item in the pre-reject)
    double *span;                // [2][R] parameter range walked this iteration, by place
    WfRayDir *rdir;              // [R] float64 direction + start of the walked range, by place (exact kernels)
    WfEntry *tube, *sph;
    u32 capq_surv;
    WfHit *hit;       // overflow pool (linked lists through hit_next)
    float4 *hit_c;    // [capq_hit * kNQ] sphere centres of the pool's joint hits
    u32 *hit_next;    // [capq_hit * kNQ]
    u32 capq_hit;
    WfHit *hit_slot;  // [kHitSlots][R], indexed by the ray's position in the live list
    float4 *slot_c;   // [kHitSlots][R] sphere centres of the joint hits
    u32 *hcnt;        // hits of the ray this iteration, by place
    u32 *win_over;  // [cap_win] overflow of a window (slow path only)
    int wn_sched, cand_budget, grow_from, grow_bits, wn_shift_max, tail_rays, tail_bits, tail_mode, tail_from;
    u32 ray_threads;  // threads of a walk / composite launch
};

// Rays per warp in the ray-parallel kernels (walk, composite).  Lanes of a warp run their rays
// in lock step, so a warp is as slow as the union of its rays' paths; once the live list is
// shorter than the launch, the rays are spread over more warps: ray i is worked on by thread
// i << spread (the other lanes only take part in the warp-cooperative steps).
#ifndef LVX_WF_SPREAD_MAX
#define LVX_WF_SPREAD_MAX 5
#endif
__device__ __forceinline__ u32 wf_spread(u32 n_live, u32 threads) {
    u32 ls = 0;
    while (ls < (u32)LVX_WF_SPREAD_MAX && ((unsigned long long)n_live << (ls + 1)) <= threads) ++ls;
    return ls;
}

// sub-queue of the warp that works on flat index f (warp-uniform: f is lane + a multiple of 32)
__device__ __forceinline__ int warp_queue(u32 f) { return (int)((f >> 5) & (kNQ - 1)); }

// Allocate `n` consecutive entries of sub-queue q for this thread alone.  Returns the global
// index or kNil when the queue is full.
__device__ __forceinline__ u32 queue_alloc(u32 *cnt, int q, u32 capq, u32 n, u32 *err, u32 err_bit) {
    const u32 base = atomicAdd(&cnt[q], n);
    if (base + n > capq) {
        atomicOr(err, err_bit);
        return kNil;
    }
    return (u32)q * capq + base;
}

// Allocate a + b entries (a, b in {0, 1}) for every lane that is converged here; one atomic
// per warp.  `q` must be warp-uniform.  Returns the index of the lane's first entry or kNil.
__device__ __forceinline__ u32 queue_alloc_bits(u32 *cnt, int q, u32 capq, bool a, bool b, u32 *err, u32 err_bit) {
    const unsigned mask = __activemask();
    const unsigned ba = __ballot_sync(mask, a), bb = __ballot_sync(mask, b);
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    const u32 total = (u32)(__popc(ba) + __popc(bb)), pre = (u32)(__popc(ba & lt) + __popc(bb & lt));
    const int leader = __ffs((int)mask) - 1;
    u32 base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(&cnt[q], total);
    base = __shfl_sync(mask, base, leader);
    const u32 n = (a ? 1u : 0u) + (b ? 1u : 0u);
    if (base + pre + n > capq) {
        atomicOr(err, err_bit);
        return kNil;
    }
    return (u32)q * capq + base + pre;
}

// Flat index over the filled parts of the kNQ sub-queues -> global entry index.
struct QueueView {
    u32 pre[kNQ + 1];
};
__device__ __forceinline__ void queue_view_load(QueueView &v, const u32 *cnt, u32 capq, u32 err) {
    // (called by all threads of the block; v lives in shared memory.  The first warp scans the kNQ
    // counters, two per lane: one memory round trip instead of a serial loop at the top of every block)
    static_assert(kNQ == 64, "two counters per lane of one warp");
    if (threadIdx.x < 32) {
        const int lane = (int)threadIdx.x;
        u32 c0 = cnt[2 * lane], c1 = cnt[2 * lane + 1];
        c0 = c0 < capq ? c0 : capq;
        c1 = c1 < capq ? c1 : capq;
        u32 inc = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += t;
        }
        const u32 ex = inc - (c0 + c1);
        v.pre[2 * lane] = ex;
        v.pre[2 * lane + 1] = ex + c0;
        // an overflowed queue holds unwritten entries: the frame is void (the host retries
        // with larger queues), nothing downstream may touch it
        if (lane == 31) v.pre[kNQ] = err ? 0u : inc;
    }
    __syncthreads();
}
// Global entry index of the 32 consecutive flat indices f0 + lane of a converged warp (f0 a multiple
// of 32): the sub-queue of f0 is the number of boundaries at or below it -- two ballots instead of a
// six-step binary search per lane -- and a lane steps on only when the warp's range runs into the
// next sub-queue.  (Lanes past the end of the queue get an index they must not use.)
__device__ __forceinline__ u32 queue_view_index_warp(const QueueView &v, u32 f0, int lane, u32 capq) {
    const unsigned b1 = __ballot_sync(0xFFFFFFFFu, v.pre[lane + 1] <= f0);                 // boundaries 1 .. 32
    const unsigned b2 = __ballot_sync(0xFFFFFFFFu, lane < 31 && v.pre[lane + 33] <= f0);   // 33 .. 63
    u32 lo = (u32)(__popc(b1) + __popc(b2));
    const u32 f = f0 + (u32)lane;
    while (lo + 1 < (u32)kNQ && v.pre[lo + 1] <= f) ++lo;
    return lo * capq + (f - v.pre[lo]);
}

__device__ __forceinline__ void ray_dir(const lvx_camera &cam, int x, int y, double &ddx, double &ddy,
                                        double &ddz) {
    // primary ray, _kernels.py:769-776
    const int W = cam.width, H = cam.height;
    const double ndc_x = (((double)x + 0.5) / (double)W * 2.0 - 1.0) * cam.tan_half * cam.aspect;
    const double ndc_y = (1.0 - ((double)y + 0.5) / (double)H * 2.0) * cam.tan_half;
    ddx = cam.f[0] + ndc_x * cam.r[0] + ndc_y * cam.u[0];
    ddy = cam.f[1] + ndc_x * cam.r[1] + ndc_y * cam.u[1];
    ddz = cam.f[2] + ndc_x * cam.r[2] + ndc_y * cam.u[2];
    const double dn = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx = ddx / dn;
    ddy = ddy / dn;
    ddz = ddz / dn;
}

__device__ __forceinline__ void write_pixel(const WfArgs &A, u32 o, double a0, double a1, double a2,
                                            double a) {
    // _kernels.py:916-920
    const lvx_params &p = A.p;
    float4 outp;
    outp.x = (float)(a0 + (1.0 - a) * p.bg[3] * p.bg[0]);
    outp.y = (float)(a1 + (1.0 - a) * p.bg[3] * p.bg[1]);
    outp.z = (float)(a2 + (1.0 - a) * p.bg[3] * p.bg[2]);
    outp.w = (float)(a + (1.0 - a) * p.bg[3]);
    reinterpret_cast<float4 *>(A.img)[o] = outp;
}

// The pixel of a ray that misses the grid, repeated n times: the source of the copy-engine transfers
// that lay the background of a HOST image (see lvx_render_wf).
__global__ void __launch_bounds__(256) wf_bgfill_kernel(const WfArgs A, float4 *__restrict__ buf, u32 n) {
    const lvx_params &p = A.p;
    float4 outp;  // write_pixel with nothing accumulated (_kernels.py:916-920)
    outp.x = (float)(0.0 + (1.0 - 0.0) * p.bg[3] * p.bg[0]);
    outp.y = (float)(0.0 + (1.0 - 0.0) * p.bg[3] * p.bg[1]);
    outp.z = (float)(0.0 + (1.0 - 0.0) * p.bg[3] * p.bg[2]);
    outp.w = (float)(0.0 + (1.0 - 0.0) * p.bg[3]);
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = outp;
}

__device__ __forceinline__ void dda_store(WfRayWalk &r, const LvxDda &d) {
    r.t_cur = d.t_cur;
    r.t_exit = d.t_exit;
    r.tmax_x = d.tmax_x;
    r.tmax_y = d.tmax_y;
    r.tmax_z = d.tmax_z;
    r.ix = d.ix;
    r.iy = d.iy;
    r.iz = d.iz;
}

// Rebuild the walker from its stored progress (the constants are functions of the ray).
__device__ __forceinline__ void dda_load(const WfArgs &A, const WfRayWalk &r, int pad, LvxDda &d) {
    const double dx = r.dir[0], dy = r.dir[1], dz = r.dir[2];
    d.t_cur = r.t_cur;
    d.t_exit = r.t_exit;
    d.tmax_x = r.tmax_x;
    d.tmax_y = r.tmax_y;
    d.tmax_z = r.tmax_z;
    d.ix = r.ix;
    d.iy = r.iy;
    d.iz = r.iz;
    d.step_x = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
    d.step_y = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
    d.step_z = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
    const double big = CUDART_INF;
    d.tdel_x = d.step_x != 0 ? fabs(1.0 / dx) : big;
    d.tdel_y = d.step_y != 0 ? fabs(1.0 / dy) : big;
    d.tdel_z = d.step_z != 0 ? fabs(1.0 / dz) : big;
    d.ilo = -pad;
    d.ihx = A.rx + pad - 1;
    d.ihy = A.ry + pad - 1;
    d.ihz = A.rz + pad - 1;
    d.alive = true;
}

// ---------------------------------------------------------------------------------------
// init: one thread per pixel (8x4 tiles per warp, the tile kernel's mapping)
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreadsWf) wf_init_kernel(const WfArgs A) {
    WF_PDL_ENTER();
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int wpt_x = A.tl.tile_w >> 3, wpt_y = A.tl.tile_h >> 2;
    const int warps_per_tile = wpt_x * wpt_y;
    const i64 k = gw / warps_per_tile;
    const int wi = (int)(gw % warps_per_tile);
    const bool tile_ok = k < A.n_my_tiles;
    const i64 tile = (i64)A.tl.tile_first + k * A.tl.tile_step;
    const int tx = (int)(tile % A.tiles_x), ty = (int)(tile / A.tiles_x);
    const int lx = (wi % wpt_x) * 8 + (lane & 7), ly = (wi / wpt_x) * 4 + (lane >> 3);
    const int x = tx * A.tl.tile_w + lx, y = ty * A.tl.tile_h + ly;
    const int W = A.cam.width, H = A.cam.height;
    const bool active = tile_ok && x < W && y < H;
    const u32 slot = (u32)(gw * 32 + lane);

    unsigned long long steps = 0;
    bool live = false;
    // hit counters and overflow-list heads are indexed by PLACE (position in the live list of
    // the iteration): every possible place starts empty, composite re-empties what it reads
    if (tile_ok) {
        A.head[slot] = kNil;
        A.hcnt[slot] = 0;
    }
    if (active) {
        double ddx, ddy, ddz;
        ray_dir(A.cam, x, y, ddx, ddy, ddz);
        const int pad = A.p.neighbor != 0 ? 1 : 0;
        LvxDda dda;
        dda.init(A.cam.o[0], A.cam.o[1], A.cam.o[2], ddx, ddy, ddz, A.rx, A.ry, A.rz, pad);
        i64 o;
        if (A.tl.compact) o = ((k * A.tl.tile_h + ly) * (i64)A.tl.tile_w + lx);
        else o = (i64)y * W + x;
        if (dda.alive) {
            // the reference collects the whole walk up front (:785-786): voxel_steps does not
            // depend on where compositing stops
            LvxDda full = dda;
            int wx, wy, wz;
            double t0, t1;
            while (full.next(wx, wy, wz, t0, t1)) steps += 1;
            WfRayWalk rw;
            rw.dir[0] = ddx;
            rw.dir[1] = ddy;
            rw.dir[2] = ddz;
            dda_store(rw, dda);
            rw.flags = 1;
            rw.tests = 0;
            rw.nwin = 0;
            rw.pad = 0;
            A.rw[slot] = rw;
            WfRayPix rp;
            rp.acc[0] = rp.acc[1] = rp.acc[2] = rp.acc[3] = 0.0;
            rp.seen_bloom = rp.sph_bloom = 0;
            rp.over = 0;
            rp.n_seen = rp.n_sph = 0;
            rp.ovf = kNil;
            A.rp[slot] = rp;
            A.rpix[slot] = make_uint2((u32)x | ((u32)y << 16), (u32)o);
            live = true;
        } else if (!A.skip_miss) {
            write_pixel(A, (u32)o, 0.0, 0.0, 0.0, 0.0);
        }
    }
    // list the live rays (warp order keeps neighbouring pixels together)
    const unsigned lb = __ballot_sync(FULL, live);
    if (lb) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&A.ctl->n_live[0], (u32)__popc(lb));
        base = __shfl_sync(FULL, base, 0);
        if (live) A.live[0][base + __popc(lb & ((1u << lane) - 1u))] = slot;
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) steps += __shfl_xor_sync(FULL, steps, o);
    if ((lane & 7) == 0 && tile_ok && y < H && steps) atomicAdd(A.row_stats + 3 * (i64)y, steps);
}

// ---------------------------------------------------------------------------------------
// walk: one thread per live ray
// ---------------------------------------------------------------------------------------

// The windows that bring fresh voxels are staged per warp in shared memory and expanded to
// items when the warp is converged again (end of the rays' batches): one global atomic and
// one scan per warp instead of an allocation round trip inside the walk (neighbour mode).
constexpr int kWalkStage = 176;
#ifndef LVX_WF_FLUSH_SCAN
#define LVX_WF_FLUSH_SCAN 1
#endif
struct __align__(16) WalkRec {
    u32 place, fresh;
    unsigned long long cell;  // (x + 1) | (y + 1) << 20 | (z + 1) << 40
    float qx, qy, qz, pad;    // ray point at the window start, window-local
};
static_assert(sizeof(WalkRec) == 32, "staged window record is 32 bytes");
struct WalkStage {
    WalkRec rec[kThreadsWf / 32][kWalkStage];
    u16 pre[kThreadsWf / 32][kWalkStage];  // items before record r (exclusive prefix of popc(fresh))
    u32 n[kThreadsWf / 32];
};
// own-voxel mode: the parameter range of the staged window (its one item is owned by that window alone)
struct WalkStageT {
    double2 t[kThreadsWf / 32][kWalkStage];
};

// all 32 lanes of the warp.  The staged windows are expanded to items so that CONSECUTIVE LANES
// WRITE CONSECUTIVE ITEMS: every store instruction fills whole sectors (a lane that wrote the
// items of "its" window one after the other touched a different sector per lane and store).
__device__ __forceinline__ void walk_flush(const WfArgs &A, WalkStage &S, const WalkStageT *ST, int warp, int lane,
                                           int q) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __syncwarp();
    const u32 n = min(S.n[warp], (u32)kWalkStage);
    if (n) {
        u32 total = 0;
        for (u32 r0 = 0; r0 < n; r0 += 32) {
            const u32 r = r0 + (u32)lane;
            const u32 v = r < n ? (u32)__popc(S.rec[warp][r].fresh) : 0u;
            u32 inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(FULL, inc, o);
                if (lane >= o) inc += t;
            }
            if (r < n) S.pre[warp][r] = (u16)(total + inc - v);
            total += __shfl_sync(FULL, inc, 31);
        }
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&A.ctl->item_cnt[q], total);
        base = __shfl_sync(FULL, base, 0);
        __syncwarp();
        if (base + total > A.capq_item) {
            if (lane == 0) atomicOr(&A.ctl->err, 1u);
        } else {
            const u32 out0 = (u32)q * A.capq_item + base;
#if LVX_WF_FLUSH_SCAN
            // Items are expanded 32 at a time; the record that holds item j is found from the START FLAGS
            // of the records in the batch (one warp reduction + a population count) instead of a binary
            // search over the prefix array per item -- those eight dependent shared-memory loads were a
            // fifth of this kernel's stall samples (profiles/r2_wavefront_hot_lines.txt, before).
            u32 r_lo = 0;  // first record with items at or after the batch start (warp-uniform)
            for (u32 b0 = 0; b0 < total; b0 += 32) {
                // records whose first item lies in [b0, b0 + 32): at most 32 of them, starting at r_lo
                const u32 r = r_lo + (u32)lane;
                const u32 pr = r < n ? (u32)S.pre[warp][r] : 0xFFFFFFFFu;
                const bool in_batch = pr >= b0 && pr < b0 + 32u;  // (pr < b0 only for r_lo itself, handled below)
                const unsigned starts = __reduce_or_sync(FULL, in_batch ? 1u << (pr - b0) : 0u);
                const u32 j = b0 + (u32)lane;
                // item j belongs to the last record that starts at or before it: r_lo - 1 if none in the batch does
                const u32 ahead = (u32)__popc(starts & (0xFFFFFFFFu >> (31 - lane)));
                const u32 lo = r_lo + ahead - 1u;
                r_lo += (u32)__popc(starts);
                if (j >= total) continue;
#else
            for (u32 j = (u32)lane; j < total; j += 32) {
                // the record that holds item j: the last r with pre[r] <= j
                u32 lo = 0, hi = n;
                while (hi - lo > 1) {
                    const u32 mid = (lo + hi) >> 1;
                    if ((u32)S.pre[warp][mid] <= j) lo = mid;
                    else hi = mid;
                }
#endif
                const WalkRec w = S.rec[warp][lo];
                u32 mm = w.fresh;
                for (u32 k = j - (u32)S.pre[warp][lo]; k; --k) mm &= mm - 1;  // its k-th fresh voxel
                const int b = __ffs((int)mm) - 1;
                const int wx = (int)(w.cell & 0xFFFFFu) - 1, wy = (int)((w.cell >> 20) & 0xFFFFFu) - 1,
                          wz = (int)(w.cell >> 40) - 1;
                const int bz_ = b / 9, by_ = (b - 9 * bz_) / 3, bx_ = b - 9 * bz_ - 3 * by_;
                // (voxel-local frame for the conservative pre-reject)
                // {place, x | y << 16, z | qx << 16, qy | qz << 16}: the voxel's coordinates rather than its
                // linear index (the pre-reject wants both; two multiplies there instead of two divisions)
                A.item[out0 + j] = make_uint4(
                    w.place, (u32)(wx + bx_ - 1) | ((u32)(wy + by_ - 1) << 16),
                    (u32)(wz + bz_ - 1) | (item_q16(w.qx - (float)(bx_ - 1)) << 16),
                    item_q16(w.qy - (float)(by_ - 1)) | (item_q16(w.qz - (float)(bz_ - 1)) << 16));
                // own-voxel mode: only the window of the voxel itself gathers it (:797-799)
                if (ST) A.item_t[out0 + j] = ST->t[warp][lo];
            }
        }
    }
    __syncwarp();
    if (lane == 0) S.n[warp] = 0;
    __syncwarp();
}

// (3 blocks/SM: with 4 the lock-step walk spills its DDA state; same-box A/B 9.34 -> 8.94 ms)
#ifndef LVX_WF_WALK_MINB
#define LVX_WF_WALK_MINB 3
#endif
__global__ void __launch_bounds__(kThreadsWf, LVX_WF_WALK_MINB) wf_walk_kernel(const WfArgs A, int par) {
    WF_PDL_ENTER();
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const u32 n_live = A.ctl->err ? 0u : A.ctl->n_live[par];
    const u32 wn = A.ctl->wn;
    const u32 budget = A.ctl->budget;
    const lvx_params &p = A.p;
    const bool neighbor = p.neighbor != 0;
    const int rx = A.rx, ry = A.ry;
    const u32 tmul = p.joints != 0 ? 3u : 1u;
    const double cull = p.tube_r + kCullMarginWf;
    const double ox = A.cam.o[0], oy = A.cam.o[1], oz = A.cam.o[2];
    const size_t R = A.R;
    extern __shared__ __align__(16) unsigned char wf_walk_smem[];
    WalkStage &S = *reinterpret_cast<WalkStage *>(wf_walk_smem);
    // (the window ranges are staged only in own-voxel mode: the launch sizes the shared memory)
    WalkStageT *ST = neighbor ? nullptr : reinterpret_cast<WalkStageT *>(wf_walk_smem + sizeof(WalkStage));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) S.n[warp] = 0;
    __syncwarp();
    // (the loop bound is warp-uniform: the stage is flushed by the whole warp)
    const u32 spread = wf_spread(n_live, gridDim.x * blockDim.x);
    for (u32 g0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); (g0 >> spread) < n_live; g0 += gridDim.x * blockDim.x) {
        const u32 i = (g0 + (u32)lane) >> spread;
        const int q = warp_queue(g0);
        const bool mine = (((u32)lane) & ((1u << spread) - 1u)) == 0 && i < n_live;
        u32 slot = 0;
        WfRayWalk rw;
        LvxDda dda;
        double ddx = 0.0, ddy = 0.0, ddz = 0.0, span0 = 0.0;
        unsigned long long tests = 0;
        if (mine) {
            slot = A.live[par][i];
            rw = A.rw[slot];
            ddx = rw.dir[0];
            ddy = rw.dir[1];
            ddz = rw.dir[2];
            dda_load(A, rw, neighbor ? 1 : 0, dda);
            tests = rw.tests;
            span0 = dda.t_cur;
        }
        u32 kw = 0, csum = 0;
        bool big_any = false;
        // voxels already listed in this iteration, as a 27-neighbourhood mask around the
        // previous cell: a voxel is tested once per iteration however many windows see it
        u32 listed = 0;
        int px = 0, py = 0, pz = 0;
        // The rays of the warp advance in lock step, one DDA window per round: the loads of a
        // round are issued together, and between rounds the warp is converged, so the stage of
        // fresh windows is flushed (one global atomic, coalesced stores) BEFORE it can overflow
        // -- no allocation round trip ever sits inside a ray's walk.
        // (measured and dropped: requesting the NEXT window's neighbour cell one round ahead -- the walker
        // already stands on it after next() -- changes nothing; a round is bound by its chain of
        // dependent float64 instructions, not by that load)
        bool go = mine;
        for (;;) {
            go = go && kw < wn && csum < budget;
            if (!__any_sync(FULL, go)) break;
            if (go) {
                int wx, wy, wz;
                double t0, t1;
                if (!dda.next(wx, wy, wz, t0, t1)) {
                    go = false;
                } else {
                    if (listed) {
                        const int dx = wx - px, dy = wy - py, dz = wz - pz;
                        listed = (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1)
                                     ? 0u
                                     : lvx_shift_mask27(listed, dx, dy, dz);
                    }
                    px = wx;
                    py = wy;
                    pz = wz;
                    u32 nm, n;
                    if (neighbor) {
                        // one 8-byte cell: occupancy bits of the 27-neighbourhood | its segment count << 32
                        const i64 pc = ((i64)(wz + 1) * (ry + 2) + (wy + 1)) * (rx + 2) + (wx + 1);
                        const unsigned long long cell = __ldg(A.ncell + pc);
                        nm = (u32)cell;
                        n = (u32)(cell >> 32);
                    } else {
                        n = __ldg(A.counts + (wx + (i64)rx * (wy + (i64)ry * wz)));
                        nm = n ? (1u << 13) : 0u;
                    }
                    if (nm != 0) {  // (else: the reference's cheap skip, :793-799)
                        tests += (unsigned long long)n * tmul;  // :833,855 summed over the window's gather
                        const double p0x = ox + t0 * ddx, p0y = oy + t0 * ddy, p0z = oz + t0 * ddz;
                        if (neighbor) {
                            // neighbour voxels that can own a hit of this window: within tube_r of the
                            // bounding box of the ray piece inside the window's voxel
                            const double p1x = ox + t1 * ddx, p1y = oy + t1 * ddy, p1z = oz + t1 * ddz;
                            u32 bx_ = 0x2492492u, by_ = 0x0E07038u, bz_ = 0x003FE00u;
                            if (fmin(p0x, p1x) - cull < (double)wx) bx_ |= 0x1249249u;
                            if (fmax(p0x, p1x) + cull > (double)(wx + 1)) bx_ |= 0x4924924u;
                            if (fmin(p0y, p1y) - cull < (double)wy) by_ |= 0x01C0E07u;
                            if (fmax(p0y, p1y) + cull > (double)(wy + 1)) by_ |= 0x70381C0u;
                            if (fmin(p0z, p1z) - cull < (double)wz) bz_ |= 0x00001FFu;
                            if (fmax(p0z, p1z) + cull > (double)(wz + 1)) bz_ |= 0x7FC0000u;
                            nm &= bx_ & by_ & bz_;
                        }
                        csum += n;
                        if (nm != 0) {
                            const bool big = n * tmul > (u32)LVX_MAX_WINDOW_HITS;
                            big_any |= big;
                            WfWindow w;
                            w.t1 = t1;
                            w.tests = tests | (big ? kBigBit : 0ull);
                            A.win[i * wn + kw] = w;
                            if (big) A.win_over[i * wn + kw] = 0;
                            kw += 1;
                            const u32 fresh = nm & ~listed;
                            listed |= nm;
                            if (fresh != 0) {
                                const u32 pos = atomicAdd(&S.n[warp], 1u);  // (< kWalkStage: flushed below)
                                WalkRec wr;
                                wr.place = i;
                                wr.fresh = fresh;
                                wr.cell = (unsigned long long)(u32)(wx + 1) | ((unsigned long long)(u32)(wy + 1) << 20) |
                                          ((unsigned long long)(u32)(wz + 1) << 40);
                                wr.qx = (float)(p0x - (double)wx);
                                wr.qy = (float)(p0y - (double)wy);
                                wr.qz = (float)(p0z - (double)wz);
                                wr.pad = 0.0f;
                                S.rec[warp][pos] = wr;
                                if (ST) ST->t[warp][pos] = make_double2(t0, t1);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            // every round adds at most one record per lane
            if (S.n[warp] + 32u > (u32)kWalkStage) walk_flush(A, S, ST, warp, lane, q);
        }
        if (mine) {
            dda_store(rw, dda);
            rw.tests = tests;
            rw.nwin = kw;
            rw.flags = (dda.alive ? 1u : 0u) | (big_any ? 2u : 0u);
            A.rw[slot] = rw;
            A.fdir[i] = make_float4((float)ddx, (float)ddy, (float)ddz, 0.0f);
            A.span[i] = span0;
            A.span[R + i] = dda.t_cur;
            WfRayDir rd;
            rd.dx = ddx;
            rd.dy = ddy;
            rd.dz = ddz;
            rd.t_lo = span0;
            A.rdir[i] = rd;
        }
        walk_flush(A, S, ST, warp, lane, q);
    }
}

// Conservative float32 test: can a primitive whose points all lie within `reach` of
// centre c be touched by the ray (q0, unit d)?  (distance of c to the ray's line)
__device__ __forceinline__ bool wf_near_line(float cx, float cy, float cz, float q0x, float q0y, float q0z,
                                             float dx, float dy, float dz, float reach) {
    const float wx = cx - q0x, wy = cy - q0y, wz = cz - q0z;
    const float tc = wx * dx + wy * dy + wz * dz;
    const float d2 = (wx * wx + wy * wy + wz * wz) - tc * tc;
    return d2 <= reach * reach;
}

// ---------------------------------------------------------------------------------------
// candidates: one thread per (ray, voxel) item: conservative float32 pre-reject of the
// voxel's segments against the ray
// ---------------------------------------------------------------------------------------
// what the pre-reject needs of one item
struct CandItem {
    u32 it, cnt, base, place, lin;
    u32 aux0, aux_step;  // WfEntry::aux of segment seg = aux0 + (seg - base) * aux_step
    float q0x, q0y, q0z, fdx, fdy, fdz, fhx, fhy, fhz;
};

// Survivors are staged per warp in shared memory (positions from ballots and one shared-
// memory atomic per converged subset) and flushed to the global queues at warp-converged
// points with one global atomic and coalesced stores: the round trip of a global atomic is
// off the inner loop.  Entries that do not fit the stage go to the global queue directly.
constexpr int kStageTube = 96, kStageSph = 192;
struct CandStage {
    WfEntry tube[kThreadsWf / 32][kStageTube];
    WfEntry sph[kThreadsWf / 32][kStageSph];
    u32 n_tube[kThreadsWf / 32], n_sph[kThreadsWf / 32];
};

// all 32 lanes of the warp
__device__ __forceinline__ void cand_flush(const WfArgs &A, CandStage &S, int warp, int lane, int q) {
    __syncwarp();
    const u32 nt = min(S.n_tube[warp], (u32)kStageTube), ns = min(S.n_sph[warp], (u32)kStageSph);
    if (nt) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&A.ctl->tube_cnt[q], nt);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (base + nt > A.capq_surv) {
            if (lane == 0) atomicOr(&A.ctl->err, 2u);
        } else {
            for (u32 k = lane; k < nt; k += 32) A.tube[(u32)q * A.capq_surv + base + k] = S.tube[warp][k];
        }
    }
    if (ns) {
        u32 base = 0;
        if (lane == 0) base = atomicAdd(&A.ctl->sph_cnt[q], ns);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (base + ns > A.capq_surv) {
            if (lane == 0) atomicOr(&A.ctl->err, 2u);
        } else {
            for (u32 k = lane; k < ns; k += 32) A.sph[(u32)q * A.capq_surv + base + k] = S.sph[warp][k];
        }
    }
    __syncwarp();
    if (lane == 0) {
        S.n_tube[warp] = 0;
        S.n_sph[warp] = 0;
    }
    __syncwarp();
}

// (ax..bz: the segment's endpoints in the frame of its voxel; half_len: bounding-sphere radius)
__device__ __forceinline__ void cand_segment(const WfArgs &A, CandStage &S, int warp, const CandItem &I, u32 seg,
                                             float ax, float ay, float az, float bx, float by, float bz, float half_len,
                                             bool joints, float reach_pt, int q) {
    u32 mk = 0;
    // the tube AND both joint spheres lie inside the segment's bounding sphere
    if (wf_near_line(0.5f * (ax + bx), 0.5f * (ay + by), 0.5f * (az + bz), I.q0x, I.q0y, I.q0z, I.fdx, I.fdy, I.fdz,
                     half_len + reach_pt)) {
        // the tube's entry point lies on the ray within tube_r of the segment's axis line:
        // |w . (d x u)| <= reach |d x u|  (absolute slack >> float32 rounding)
        const float ux = bx - ax, uy = by - ay, uz = bz - az;
        const float nx = I.fdy * uz - I.fdz * uy, ny = I.fdz * ux - I.fdx * uz, nz = I.fdx * uy - I.fdy * ux;
        const float wn = (ax - I.q0x) * nx + (ay - I.q0y) * ny + (az - I.q0z) * nz;
        if (wn * wn <= reach_pt * reach_pt * (nx * nx + ny * ny + nz * nz) + 1e-6f) mk = 1u;
        if (joints) {
            if (wf_near_line(ax, ay, az, I.q0x, I.q0y, I.q0z, I.fdx, I.fdy, I.fdz, reach_pt)) mk |= 2u;
            if (wf_near_line(bx, by, bz, I.q0x, I.q0y, I.q0z, I.fdx, I.fdy, I.fdz, reach_pt)) mk |= 4u;
        }
    }
    const unsigned act = __activemask();
    if (!__any_sync(act, mk != 0)) return;  // (the usual case: one vote instead of three ballots)
    const unsigned bt = __ballot_sync(act, (mk & 1u) != 0);
    const unsigned ba = __ballot_sync(act, (mk & 2u) != 0), bb = __ballot_sync(act, (mk & 4u) != 0);
    if ((bt | ba | bb) == 0) return;
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    const int leader = __ffs((int)act) - 1;
    u32 t0 = 0, s0 = 0;
    if ((int)(threadIdx.x & 31) == leader) {
        if (bt) t0 = atomicAdd(&S.n_tube[warp], (u32)__popc(bt));
        if (ba | bb) s0 = atomicAdd(&S.n_sph[warp], (u32)(__popc(ba) + __popc(bb)));
    }
    t0 = __shfl_sync(act, t0, leader);
    s0 = __shfl_sync(act, s0, leader);
    if (mk & 1u) {
        const u32 pos = t0 + (u32)__popc(bt & lt);
        const WfEntry c = {seg, I.place, I.lin, I.aux0 + (seg - I.base) * I.aux_step};
        if (pos < (u32)kStageTube) {
            S.tube[warp][pos] = c;
        } else {
            const u32 e = queue_alloc(A.ctl->tube_cnt, q, A.capq_surv, 1u, &A.ctl->err, 2u);
            if (e != kNil) A.tube[e] = c;
        }
    }
    if (mk & 6u) {
        u32 pos = s0 + (u32)(__popc(ba & lt) + __popc(bb & lt));
        WfEntry c = {seg, I.place, I.lin, I.aux0 + (seg - I.base) * I.aux_step};
        if (mk & 2u) {
            if (pos < (u32)kStageSph) {
                S.sph[warp][pos] = c;
            } else {
                const u32 e = queue_alloc(A.ctl->sph_cnt, q, A.capq_surv, 1u, &A.ctl->err, 2u);
                if (e != kNil) A.sph[e] = c;
            }
            ++pos;
        }
        if (mk & 4u) {
            c.seg |= 0x80000000u;
            if (pos < (u32)kStageSph) {
                S.sph[warp][pos] = c;
            } else {
                const u32 e = queue_alloc(A.ctl->sph_cnt, q, A.capq_surv, 1u, &A.ctl->err, 2u);
                if (e != kNil) A.sph[e] = c;
            }
        }
    }
}

#ifndef LVX_WF_CAND_MINB
#define LVX_WF_CAND_MINB 4
#endif
// segment `seg` of an item: endpoints in the voxel's frame, from the render record or the encoded one
template <bool PACKED>
__device__ __forceinline__ void cand_fetch(const WfArgs &A, const CandItem &I, u32 seg, float a[3], float b[3],
                                           float &half_len) {
    if (PACKED) {
        const LvxPackedFields f = lvx_packed_fields(A.pk, lvx_packed_word(A.pk, seg));
        lvx_packed_local(f.face_in, f.bin_in, A.pk, a);
        lvx_packed_local(f.face_out, f.bin_out, A.pk, b);
        half_len = lvx_half_len(a[0], a[1], a[2], b[0], b[1], b[2]);
    } else {
        const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + seg));
        const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + seg) + 1);
        a[0] = ra.x - I.fhx;
        a[1] = ra.y - I.fhy;
        a[2] = ra.z - I.fhz;
        b[0] = rb.x - I.fhx;
        b[1] = rb.y - I.fhy;
        b[2] = rb.z - I.fhz;
        half_len = rb.w;
    }
}

template <bool PACKED>
__global__ void __launch_bounds__(kThreadsWf, LVX_WF_CAND_MINB) wf_cand_kernel(const WfArgs A) {
    WF_PDL_ENTER();
    __shared__ QueueView V;
    __shared__ CandStage S;
    queue_view_load(V, A.ctl->item_cnt, A.capq_item, A.ctl->err);
    const u32 total = V.pre[kNQ];
    const bool joints = A.p.joints != 0;
    const bool nbr = A.p.neighbor != 0;
    const float reach_pt = (float)A.p.tube_r + kRejectMarginWf + kItemQSlack;
    const u32 stride = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        S.n_tube[warp] = 0;
        S.n_sph[warp] = 0;
    }
    __syncwarp();
    int q = 0;
    // two items per thread and round (the loop bound is warp-uniform: the stage is flushed
    // by the whole warp)
    for (u32 f0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); f0 < total; f0 += 2 * stride) {
        q = warp_queue(f0);
        if (S.n_tube[warp] > (u32)kStageTube / 2 || S.n_sph[warp] > (u32)kStageSph / 2) cand_flush(A, S, warp, lane, q);
        const u32 f = f0 + (u32)lane;
        CandItem I[2];
        u32 lin[2], place[2], hx[2], hy[2], hz[2];
        float4 q0[2];
        bool have[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const u32 fk = f + (u32)k * stride;
            have[k] = fk < total;
            const u32 it_w = queue_view_index_warp(V, f0 + (u32)k * stride, lane, A.capq_item);
            I[k].it = have[k] ? it_w : 0u;
            // (a lane past the end of the queue reads item 0, which may be stale: its fields are not used
            // as addresses)
            uint4 itm = A.item[I[k].it];
            if (!have[k]) itm = make_uint4(0u, 0u, 0u, 0u);
            place[k] = itm.x;
            I[k].place = place[k];
            // voxel coordinates (16 bits each) and the ray point in the voxel's frame (wf_item)
            hx[k] = itm.y & 0xFFFFu;
            hy[k] = itm.y >> 16;
            hz[k] = itm.z & 0xFFFFu;
            lin[k] = hx[k] + (u32)A.rx * (hy[k] + (u32)A.ry * hz[k]);
            q0[k] = make_float4(item_unq16(itm.z >> 16), item_unq16(itm.w), item_unq16(itm.w >> 16), 0.0f);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float4 fd = A.fdir[place[k]];
            I[k].fdx = fd.x;
            I[k].fdy = fd.y;
            I[k].fdz = fd.z;
            I[k].cnt = have[k] ? __ldg(A.counts + lin[k]) : 0u;
            I[k].base = __ldg(A.offsets + lin[k]);
            I[k].lin = lin[k];
            // neighbour mode: the segment's index in its voxel; own-voxel mode: the item
            I[k].aux0 = nbr ? 0u : I[k].it;
            I[k].aux_step = nbr ? 1u : 0u;
        }
        float ea[2][3], eb[2][3], hl[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            I[k].fhx = (float)hx[k];
            I[k].fhy = (float)hy[k];
            I[k].fhz = (float)hz[k];
            I[k].q0x = q0[k].x;
            I[k].q0y = q0[k].y;
            I[k].q0z = q0[k].z;
            // (a listed voxel holds at least one record)
            cand_fetch<PACKED>(A, I[k], I[k].base, ea[k], eb[k], hl[k]);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (I[k].cnt == 0) continue;
            cand_segment(A, S, warp, I[k], I[k].base, ea[k][0], ea[k][1], ea[k][2], eb[k][0], eb[k][1], eb[k][2], hl[k],
                         joints, reach_pt, q);
            for (u32 sg = 1; sg < I[k].cnt; ++sg) {
                const u32 seg = I[k].base + sg;
                float a3[3], b3[3], h1;
                cand_fetch<PACKED>(A, I[k], seg, a3, b3, h1);
                cand_segment(A, S, warp, I[k], seg, a3[0], a3[1], a3[2], b3[0], b3[1], b3[2], h1, joints, reach_pt, q);
            }
        }
        __syncwarp();
    }
    cand_flush(A, S, warp, lane, q);
}

// one 256-bit store / load per hit record (st/ld.global.v4.b64: whole-sector accesses)
__device__ __forceinline__ void wf_store_hit(WfHit *p, const WfHit &h) {
    lvx_st256(p, (u64)__double_as_longlong(h.t_in), h.key2, (u64)__double_as_longlong(h.scale),
              (u64)__double_as_longlong(h.alpha));
}
__device__ __forceinline__ WfHit wf_load_hit(const WfHit *p) {
    u64 a, b, c, d;
    lvx_ld256(p, a, b, c, d);
    WfHit h;
    h.t_in = __longlong_as_double((long long)a);
    h.key2 = b;
    h.scale = __longlong_as_double((long long)c);
    h.alpha = __longlong_as_double((long long)d);
    return h;
}

// ---------------------------------------------------------------------------------------
// exact: one thread per surviving primitive (KIND 0: tubes, 1: joint spheres)
// ---------------------------------------------------------------------------------------
#ifndef LVX_WF_EXACT_MINB
#define LVX_WF_EXACT_MINB 4
#endif
#ifndef LVX_WF_EXACT_THREADS
#define LVX_WF_EXACT_THREADS 256
#endif
constexpr int kThreadsExact = LVX_WF_EXACT_THREADS;
template <int KIND, bool GEOM, bool PACKED>
__device__ __forceinline__ void wf_exact_body(const WfArgs &A, int par, QueueView &V, u32 block, u32 n_blocks) {
    queue_view_load(V, KIND == 0 ? A.ctl->tube_cnt : A.ctl->sph_cnt, A.capq_surv, A.ctl->err);
    const u32 total = V.pre[kNQ];
    const double ox = A.cam.o[0], oy = A.cam.o[1], oz = A.cam.o[2];
    const double tube_r = A.p.tube_r;
    const size_t R = A.R;
    const WfEntry *queue = KIND == 0 ? A.tube : A.sph;
    const bool neighbor = A.p.neighbor != 0;
    // (the loop bound is warp-uniform: the queue index is found by the converged warp)
    for (u32 f0 = block * blockDim.x + (threadIdx.x & ~31u); f0 < total; f0 += n_blocks * blockDim.x) {
        __syncwarp();
        const u32 f = f0 + (threadIdx.x & 31u);
        const u32 qi = queue_view_index_warp(V, f0, (int)(threadIdx.x & 31u), A.capq_surv);
        if (f >= total) continue;
        const int q = warp_queue(f);
        const WfEntry c = queue[qi];
        const u32 seg = c.seg & 0x7FFFFFFFu;
        const u32 place = c.place;
        const WfRayDir rd = A.rdir[place];
        // (the end of the walked range / the item's window are requested NOW, with the ray record: loaded
        // where they are used they cost a second memory round trip after the intersection test)
        double own_lo = 0.0, own_hi = 0.0;
        if (neighbor) {
            own_hi = A.span[R + place];
        } else {
            const double2 tr = A.item_t[c.aux];
            own_lo = tr.x;
            own_hi = tr.y;
        }
        const double rdx = rd.dx, rdy = rd.dy, rdz = rd.dz;
        // the segment's endpoints as the reference's float32 arrays hold them, + attr | lid << 8
        float pa[3], pb[3];
        u32 rmeta;
        if (PACKED) {
            const LvxPackedFields f = lvx_packed_fields(A.pk, lvx_packed_word(A.pk, seg));
            const u32 plane = (u32)A.rx * (u32)A.ry;
            const u32 vz = c.lin / plane, vy = (c.lin - vz * plane) / (u32)A.rx, vx = c.lin - vz * plane - vy * (u32)A.rx;
            if (KIND == 0 || !(c.seg & 0x80000000u))
                lvx_packed_point(f.face_in, f.bin_in, A.pk, (int)vx, (int)vy, (int)vz, pa);
            if (KIND == 0 || (c.seg & 0x80000000u))
                lvx_packed_point(f.face_out, f.bin_out, A.pk, (int)vx, (int)vy, (int)vz, pb);
            rmeta = f.attr | (f.lid << 8);
        } else {
            const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + seg));
            pa[0] = ra.x;
            pa[1] = ra.y;
            pa[2] = ra.z;
            rmeta = __float_as_uint(ra.w);
            if (KIND == 0 || (c.seg & 0x80000000u)) {
                const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + seg) + 1);
                pb[0] = rb.x;
                pb[1] = rb.y;
                pb[2] = rb.z;
            }
        }
        LvxHit h;
        bool hit;
        u32 kind3;
        float ccx = 0.0f, ccy = 0.0f, ccz = 0.0f;
        if (KIND == 0) {
            hit = lvx_tube_f32axis(ox, oy, oz, rdx, rdy, rdz, pa[0], pa[1], pa[2], pb[0], pb[1], pb[2], tube_r, h);
            kind3 = 0;
        } else {
            const bool end_b = (c.seg & 0x80000000u) != 0;
            kind3 = end_b ? 2 : 1;
            ccx = end_b ? pb[0] : pa[0];
            ccy = end_b ? pb[1] : pa[1];
            ccz = end_b ? pb[2] : pa[2];
            hit = lvx_sphere<true>(ox, oy, oz, rdx, rdy, rdz, (double)ccx, (double)ccy, (double)ccz, tube_r, h);
        }
        // ownership (:838, :858, :878): a hit belongs to the window whose range holds its entry
        // parameter; the windows tile the walked range, so every hit entered inside the range
        // walked this iteration is owned by exactly one of this iteration's windows
        if (!hit) continue;
        if (neighbor) own_lo = rd.t_lo;
        if (!(own_lo <= h.t_in && h.t_in < own_hi)) continue;
        const u32 attr = rmeta & 0xFFu, lid = (rmeta >> 8) & 31u;
        double scale, alpha;
        lvx_shade_hit<GEOM>(A, ox, oy, oz, rdx, rdy, rdz, h, attr, scale, alpha);
        const u32 lin = c.lin;
        const u32 rank = neighbor ? c.aux : seg - __ldg(A.offsets + lin);  // index in the voxel's list
        WfHit rec;
        rec.t_in = h.t_in;
        rec.key2 = ((unsigned long long)lin << 24) | ((unsigned long long)lid << 19) | (kind3 ? 1ull << 18 : 0ull) |
                   ((unsigned long long)(rank & 255u) << 10) | ((unsigned long long)kind3 << 8) | attr;
        rec.scale = scale;
        rec.alpha = alpha;
        const u32 j = atomicAdd(&A.hcnt[place], 1u);
        if (j < (u32)kHitSlots) {
            wf_store_hit(A.hit_slot + ((size_t)j * R + place), rec);
            if (KIND != 0) A.slot_c[(size_t)j * R + place] = make_float4(ccx, ccy, ccz, 0.0f);
        } else {
            const u32 e = queue_alloc_bits(A.ctl->hit_cnt, q, A.capq_hit, true, false, &A.ctl->err, 4u);
            if (e == kNil) continue;
            A.hit_next[e] = atomicExch(&A.head[place], e);
            wf_store_hit(A.hit + e, rec);
            if (KIND != 0) A.hit_c[e] = make_float4(ccx, ccy, ccz, 0.0f);
        }
    }
}

// Tubes and joint spheres in ONE launch: the blocks of the grid are divided between the two queues in
// proportion to their lengths (a sphere entry weighs 5/4 of a tube entry: more of them are hits and
// get shaded), so neither half waits for the other and the frame has one launch, one ramp-up and one
// drain less per iteration.
template <bool GEOM, bool PACKED>
__global__ void __launch_bounds__(kThreadsExact, LVX_WF_EXACT_MINB) wf_exact_kernel(const WfArgs A, int par) {
    WF_PDL_ENTER();
    __shared__ QueueView V;
    __shared__ u32 s_split;
    if (threadIdx.x < 32) {
        unsigned long long t = 0, sp = 0;
        if (A.p.joints != 0) sp = (unsigned long long)A.ctl->sph_cnt[threadIdx.x] + A.ctl->sph_cnt[threadIdx.x + 32];
        t = (unsigned long long)A.ctl->tube_cnt[threadIdx.x] + A.ctl->tube_cnt[threadIdx.x + 32];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
            sp += __shfl_xor_sync(0xFFFFFFFFu, sp, o);
        }
        if (threadIdx.x == 0) {
            const unsigned long long ws = sp * 5ull, wt = t * 4ull;
            u32 nt = gridDim.x;  // blocks on the tube queue
            if (sp != 0) {
                nt = t == 0 ? 0u : (u32)((wt * gridDim.x + (ws + wt) / 2) / (ws + wt));
                if (t != 0 && nt == 0) nt = 1;
                if (nt >= gridDim.x && gridDim.x > 1) nt = gridDim.x - 1;
            }
            s_split = nt;
        }
    }
    __syncthreads();
    const u32 nt = s_split;
    if (blockIdx.x < nt) wf_exact_body<0, GEOM, PACKED>(A, par, V, blockIdx.x, nt);
    else wf_exact_body<1, GEOM, PACKED>(A, par, V, blockIdx.x - nt, gridDim.x - nt);
}

// ---------------------------------------------------------------------------------------
// composite: one thread per live ray
// ---------------------------------------------------------------------------------------

// total order of the reference: _hit_before (_kernels.py:261-270) = (t_in, home voxel, lid,
// kind), remaining ties in gather order = (index in voxel, primitive): (t_in, key2)
__device__ __forceinline__ bool wf_before(double ta, unsigned long long ka, double tb, unsigned long long kb) {
    return ta < tb || (ta == tb && (ka >> 8) < (kb >> 8));
}

struct WfTables {
    const WfArgs &A;
    u32 slot;
    u32 ovf;
    __device__ __forceinline__ uint2 *seen(u32 i) const {
        return i < (u32)kInline ? A.tab_seen + (size_t)slot * kInline + i
                                : A.pool_seen + (size_t)ovf * (LVX_MAX_SEEN - kInline) + (i - kInline);
    }
    __device__ __forceinline__ float4 *sph(u32 i) const {
        return i < (u32)kInline ? A.tab_sph + (size_t)slot * kInline + i
                                : A.pool_sph + (size_t)ovf * (LVX_MAX_SEEN - kInline) + (i - kInline);
    }
};

#ifndef LVX_WF_COMP_PIPE
#define LVX_WF_COMP_PIPE 1
#endif
struct WfPixel {
    double acc[4];
    u32 n_seen, n_sph;
    unsigned long long seen_bloom, sph_bloom;
};

// de-duplication + front-to-back accumulation of stream_hit (_kernels.py:666-670, 719-730).
// Returns false when the pool of overflow tables is exhausted (reported through ctl->err).
__device__ __forceinline__ void wf_accumulate(const WfArgs &A, WfTables &T, WfPixel &S, double scale,
                                              double alpha, u32 lin, u32 lid, u32 attr, bool is_sphere,
                                              float cx, float cy, float cz) {
    unsigned long long sph_bit = 0;
    if (is_sphere) {
        const u32 hsh = (__float_as_uint(cx) * 0x9E3779B1u) ^ (__float_as_uint(cy) * 0x85EBCA77u) ^
                        (__float_as_uint(cz) * 0xC2B2AE3Du);
        sph_bit = 1ull << (hsh >> 26);
        if (S.sph_bloom & sph_bit) {
            for (int i = (int)S.n_sph - 1; i >= 0; --i) {
                const float4 c = *T.sph(i);
                if (c.x == cx && c.y == cy && c.z == cz) return;
            }
        }
    }
    const bool need_pool = (S.n_seen == (u32)kInline || (is_sphere && S.n_sph == (u32)kInline)) && T.ovf == kNil;
    if (need_pool) {
        const u32 blk = atomicAdd(&A.ctl->pool_cnt, 1u);
        if (blk >= A.pool_cap) {
            atomicOr(&A.ctl->err, 8u);
            return;
        }
        T.ovf = blk;
    }
    {
        const u32 bit = 1u << lid;
        const unsigned long long kb = 1ull << ((lin * 0x9E3779B1u) >> 26);
        bool found = false;
        // (measured and dropped: keeping the entry touched last in registers -- the three primitives of
        // a segment ask for the same one -- costs more in register pressure than the loads it saves)
        if (S.seen_bloom & kb) {
            for (int i = (int)S.n_seen - 1; i >= 0; --i) {
                uint2 *ep = T.seen(i);
                const uint2 e = *ep;
                if (e.x == lin) {
                    if (e.y & bit) return;
                    ep->y = e.y | bit;
                    found = true;
                    break;
                }
            }
        }
        if (!found && S.n_seen < (u32)LVX_MAX_SEEN) {
            *T.seen(S.n_seen) = make_uint2(lin, bit);
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
    if (is_sphere && S.n_sph < (u32)LVX_MAX_SEEN) {
        *T.sph(S.n_sph) = make_float4(cx, cy, cz, 0.0f);
        S.n_sph += 1;
        S.sph_bloom |= sph_bit;
    }
}

// The hits of one ray and iteration: the first kHitSlots sit ray-parallel in hit_slot
// ([j][place in the live list]: neighbouring threads read neighbouring records), the
// rest hangs in a linked list.  A reference is j for the former, kHitSlots + pool index
// for the latter.
struct WfRayHits {
    const WfArgs &A;
    u32 place, nslot, head;
    __device__ __forceinline__ WfHit *at(u32 ref) const {
        return ref < (u32)kHitSlots ? A.hit_slot + (size_t)ref * A.R + place : A.hit + (ref - kHitSlots);
    }
    __device__ __forceinline__ float4 centre(u32 ref) const {
        return ref < (u32)kHitSlots ? A.slot_c[(size_t)ref * A.R + place] : A.hit_c[ref - kHitSlots];
    }
    // iteration: ref = first(); while (ref != kNil) { ...; ref = next(ref); }
    __device__ __forceinline__ u32 first() const {
        return nslot ? 0u : (head == kNil ? kNil : head + kHitSlots);
    }
    __device__ __forceinline__ u32 next(u32 ref) const {
        if (ref < (u32)kHitSlots) {
            if (ref + 1 < nslot) return ref + 1;
            return head == kNil ? kNil : head + kHitSlots;
        }
        const u32 e = A.hit_next[ref - kHitSlots];
        return e == kNil ? kNil : e + kHitSlots;
    }
};

// Index (within the ray's windows of this iteration) of the window that owns parameter t:
// the first one whose range ends after t.
// (8-way search: the seven probes of a round are independent loads, so 128 windows take three
// memory round trips instead of seven)
__device__ __forceinline__ u32 wf_find_window(const WfWindow *w, u32 nw, double t) {
    u32 lo = 0, hi = nw;  // answer in [lo, hi); "answer >= p" <=> w[p - 1].t1 <= t (ends are monotonic)
    while (hi - lo > 8) {
        const u32 step = (hi - lo) >> 3;
        u32 c = 0;
#pragma unroll
        for (u32 j = 1; j < 8; ++j) c += w[lo + j * step - 1].t1 <= t ? 1u : 0u;
        if (c < 7) hi = lo + (c + 1) * step;
        lo += c * step;
    }
    u32 c = 0;
#pragma unroll
    for (u32 j = 1; j < 8; ++j)
        if (lo + j < hi) c += w[lo + j - 1].t1 <= t ? 1u : 0u;
    return lo + c;
}

// Slow path for rays that crossed a window with more than 1024/3 candidates: the reference
// keeps the first 1024 owned hits of a window in gather order and counts the rest in
// window_overflow (_kernels.py:852-853).  Gather order is (segment, primitive).
__device__ void wf_apply_window_cap(const WfArgs &A, const WfRayHits &H, const WfWindow *w, u32 nw, u32 w0) {
    for (u32 a = H.first(); a != kNil; a = H.next(a)) {
        WfHit *ha = H.at(a);
        const u32 k = wf_find_window(w, nw, ha->t_in);
        if (!(w[k].tests & kBigBit)) continue;
        const unsigned long long ga = hit_gather(ha->key2);
        u32 rank = 0;
        for (u32 b = H.first(); b != kNil; b = H.next(b)) {
            const WfHit *hb = H.at(b);
            if (wf_find_window(w, nw, hb->t_in) != k) continue;
            if (hit_gather(hb->key2) < ga) rank += 1;
        }
        if (rank >= (u32)LVX_MAX_WINDOW_HITS) {
            ha->key2 |= kDroppedBit;
            A.win_over[w0 + k] += 1;
        }
    }
}

__device__ __forceinline__ bool wf_composite_hit(const WfArgs &A, WfTables &T, WfPixel &S, const WfHit &h,
                                                 const float4 c, double tau) {
    WF_STAT(1, 1);
    wf_accumulate(A, T, S, h.scale, h.alpha, hit_lin(h.key2), hit_lid(h.key2), hit_attr(h.key2),
                  hit_kind3(h.key2) != 0, c.x, c.y, c.z);
    return S.acc[3] >= tau;
}
__device__ __forceinline__ bool wf_composite_one(const WfArgs &A, WfTables &T, WfPixel &S, const WfRayHits &H,
                                                 u32 ref, double tau, double &t_in) {
    const WfHit h = wf_load_hit(H.at(ref));
    t_in = h.t_in;
    float4 c = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (hit_kind3(h.key2) != 0) c = H.centre(ref);
    return wf_composite_hit(A, T, S, h, c, tau);
}

#ifndef LVX_WF_LIGHT
#define LVX_WF_LIGHT 8
#endif
constexpr int kLight = LVX_WF_LIGHT;  // up to this many hits a ray orders by itself; more are ranked by its warp
static_assert(kLight <= kHitSlots && kHitSlots <= 127 && kHitSlots <= kSortCap, "a light ray's hits are all in slots, and a slot index fits 8 bits");

struct SortStage {
    double t[kThreadsWf / 32][kSortCap];
    unsigned long long k[kThreadsWf / 32][kSortCap];
    u32 ref[kThreadsWf / 32][kSortCap], out[kThreadsWf / 32][kSortCap];
    u32 n[kThreadsWf / 32];
};

#ifndef LVX_WF_COMP_MINB
#define LVX_WF_COMP_MINB 4
#endif
__global__ void __launch_bounds__(kThreadsWf, LVX_WF_COMP_MINB) wf_composite_kernel(const WfArgs A, int par) {
    WF_PDL_ENTER();
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ SortStage Q;
    // sort buffers of the rays with few hits, one column per thread ([entry][thread]: conflict-free).
    // In shared memory because thread-local arrays indexed at run time live in local memory, and
    // the insertion sort's stores were a third of this kernel's L2 write traffic.
    __shared__ double L_t[kLight][kThreadsWf];
    __shared__ unsigned long long L_k[kLight][kThreadsWf];  // key2 with the hit's slot in its low 8 bits
    __shared__ unsigned char O8[kHitSlots][kThreadsWf];      // order of a heavier ray's slots (| 0x80: joint sphere)
    const int tid = threadIdx.x;
    const u32 n_live = A.ctl->err ? 0u : A.ctl->n_live[par];
    const u32 wn = A.ctl->wn;
    const size_t R = A.R;
    const double tau = A.p.tau;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // (the loop bound is warp-uniform: rays with many hits are ordered by the whole warp)
    const u32 spread = wf_spread(n_live, gridDim.x * blockDim.x);
    for (u32 g0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); (g0 >> spread) < n_live; g0 += gridDim.x * blockDim.x) {
        const u32 i = (g0 + (u32)lane) >> spread;
        const bool valid = (((u32)lane) & ((1u << spread) - 1u)) == 0 && i < n_live;
        u32 slot = 0, nhit = 0, fl = 1;
        if (valid) {
            slot = A.live[par][i];
            nhit = A.hcnt[i];
            fl = A.rw[slot].flags;
        }
        bool finished = valid && !(fl & 1);  // the walk is over: this was the last batch
        bool terminated = false;
        unsigned long long tests = 0, over = 0;
        const bool big = (fl & 2) != 0;
        const u32 w0 = i * wn;
        u32 nw = 0;
        const WfWindow *wins = A.win + w0;
        WfRayHits H = {A, i, nhit < (u32)kHitSlots ? nhit : (u32)kHitSlots, kNil};
        if (nhit) {
            WF_STAT(0, nhit);
            WF_STAT(3, 1);
            // the hit records sit in kHitSlots different planes: fetch them all at once, the
            // ordering loop below then reads them from cache one after the other
#pragma unroll
            for (int j = 0; j < kHitSlots; ++j)
                if ((u32)j < nhit) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.hit_slot + (size_t)j * R + i));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.rp + slot));
            A.hcnt[i] = 0;
            if (nhit > (u32)kHitSlots) {
                H.head = A.head[i];
                A.head[i] = kNil;
            }
            nw = A.rw[slot].nwin;
            if (big) wf_apply_window_cap(A, H, wins, nw, w0);
        }
        // ---- order the hits: (t_in, key2) ---------------------------------------------------
        u32 order[kSortCap];
        int n = 0;
        const bool light = nhit <= (u32)kLight;
        // more than a light ray's hits, all of them in slots, none dropped: ranked by the warp into O8
        const bool in_slots = !light && nhit <= (u32)kHitSlots && !big;
        if (nhit && light) {
            // few hits (all of them in slots: kLight <= kHitSlots): insertion sort by the ray's own thread
            for (u32 ref = H.first(); ref != kNil; ref = H.next(ref)) {
                const WfHit *hp = H.at(ref);
                if (big && (hp->key2 & kDroppedBit)) continue;  // dropped by the window cap
                const double2 v = *reinterpret_cast<const double2 *>(hp);
                const double t = v.x;
                // (the low 8 bits -- attr -- are not part of the order: they carry the slot here)
                const unsigned long long k2 = ((unsigned long long)__double_as_longlong(v.y) & ~0xFFull) | ref;
                int pos = n++;
                while (pos > 0 && wf_before(t, k2, L_t[pos - 1][tid], L_k[pos - 1][tid])) {
                    L_t[pos][tid] = L_t[pos - 1][tid];
                    L_k[pos][tid] = L_k[pos - 1][tid];
                    --pos;
                }
                L_t[pos][tid] = t;
                L_k[pos][tid] = k2;
            }
        }
        __syncwarp();
        // many hits: the warp ranks them together, one such ray at a time
        unsigned hm = __ballot_sync(FULL, nhit > (u32)kLight && nhit <= (u32)kSortCap);
        while (hm) {
            const int L = __ffs((int)hm) - 1;
            hm &= hm - 1;
            const u32 placeL = __shfl_sync(FULL, i, L);
            const u32 nhL = __shfl_sync(FULL, nhit, L);
            if (__shfl_sync(FULL, (int)in_slots, L)) {
                // the usual heavy ray: every hit sits in a slot and none is dropped, so hit j IS slot j --
                // nothing is listed by the ray's own lane, the ranks go straight into the ray's
                // byte column (no copy into its local array either)
                // (t_in >= 0, and + 0.0 makes a -0.0 a +0.0: the order of the doubles is the order of their
                // bit patterns, so (t_in, key >> 8) is ONE 128-bit unsigned comparison -- no FP64-pipe
                // compares in the m x m loop)
                for (u32 j = lane; j < nhL; j += 32) {
                    const double2 v = *reinterpret_cast<const double2 *>(A.hit_slot + (size_t)j * R + placeL);
                    Q.t[warp][j] = v.x + 0.0;
                    Q.k[warp][j] = (unsigned long long)__double_as_longlong(v.y) >> 8;
                }
                __syncwarp();
                for (u32 j = lane; j < nhL; j += 32) {
                    const unsigned __int128 mine = ((unsigned __int128)(unsigned long long)__double_as_longlong(Q.t[warp][j]) << 64) |
                                                   Q.k[warp][j];
                    u32 rank = 0;
                    for (u32 q = 0; q < nhL; ++q) {
                        const unsigned __int128 other =
                            ((unsigned __int128)(unsigned long long)__double_as_longlong(Q.t[warp][q]) << 64) | Q.k[warp][q];
                        rank += other < mine ? 1u : 0u;
                    }
                    // (keys are unique: a permutation; bit 18 of the key -- joint sphere -- is bit 10 here)
                    O8[rank][(warp << 5) + L] = (unsigned char)(j | (((Q.k[warp][j] >> 10) & 1ull) ? 0x80u : 0u));
                }
                if (lane == L) n = (int)nhL;
                __syncwarp();
                continue;
            }
            if (lane == L) {
                u32 m = 0;
                for (u32 ref = H.first(); ref != kNil; ref = H.next(ref)) {
                    if (big && (H.at(ref)->key2 & kDroppedBit)) continue;
                    Q.ref[warp][m++] = ref;
                }
                Q.n[warp] = m;
            }
            __syncwarp();
            const u32 m = Q.n[warp];
            for (u32 j = lane; j < m; j += 32) {
                const u32 ref = Q.ref[warp][j];
                const WfHit *hp = ref < (u32)kHitSlots ? A.hit_slot + (size_t)ref * R + placeL : A.hit + (ref - kHitSlots);
                const double2 v = *reinterpret_cast<const double2 *>(hp);
                Q.t[warp][j] = v.x;
                Q.k[warp][j] = (unsigned long long)__double_as_longlong(v.y);
            }
            __syncwarp();
            for (u32 j = lane; j < m; j += 32) {
                const double t = Q.t[warp][j];
                const unsigned long long k2 = Q.k[warp][j];
                u32 rank = 0;
                for (u32 q = 0; q < m; ++q) rank += wf_before(Q.t[warp][q], Q.k[warp][q], t, k2) ? 1u : 0u;
                // (keys are unique: a permutation)
                Q.out[warp][rank] = Q.ref[warp][j] | (((k2 >> 18) & 1ull) ? kJointRef : 0u);
            }
            __syncwarp();
            if (lane == L) {
                for (u32 j = 0; j < m; ++j) order[j] = Q.out[warp][j];
                n = (int)m;
            }
            __syncwarp();
        }
        // reference (slot or pool entry, | kJointRef for a joint sphere) of the j-th hit in order
        auto sorted_ref = [&](int j) -> u32 {
            if (in_slots) {
                const u32 b = O8[j][tid];
                return (b & 0x7Fu) | ((b & 0x80u) ? kJointRef : 0u);
            }
            if (!light) return order[j];
            const unsigned long long k2 = L_k[j][tid];
            return (u32)(k2 & 0xFFull) | (((k2 >> 18) & 1ull) ? kJointRef : 0u);
        };
        // ---- composite ----------------------------------------------------------------------
        WfRayPix rp;
        if (nhit) {
            WfPixel S;
            rp = A.rp[slot];
            S.acc[0] = rp.acc[0];
            S.acc[1] = rp.acc[1];
            S.acc[2] = rp.acc[2];
            S.acc[3] = rp.acc[3];
            S.n_seen = rp.n_seen;
            S.n_sph = rp.n_sph;
            S.seen_bloom = rp.seen_bloom;
            S.sph_bloom = rp.sph_bloom;
            WfTables T = {A, slot, rp.ovf};
            double term_t = 0.0;
            if (nhit <= (u32)kSortCap) {
#if LVX_WF_COMP_PIPE
                // the record (and joint centre) of hit j + 1 is in flight while hit j is composited
                WfHit hc;
                float4 cc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (n > 0) {
                    const u32 r0 = sorted_ref(0);
                    hc = wf_load_hit(H.at(r0 & ~kJointRef));
                    if (r0 & kJointRef) cc = H.centre(r0 & ~kJointRef);
                }
                for (int j = 0; j < n; ++j) {
                    WfHit hn = hc;
                    float4 cn = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    if (j + 1 < n) {
                        const u32 r1 = sorted_ref(j + 1);
                        hn = wf_load_hit(H.at(r1 & ~kJointRef));
                        if (r1 & kJointRef) cn = H.centre(r1 & ~kJointRef);
                    }
                    if (wf_composite_hit(A, T, S, hc, cc, tau)) {
                        terminated = true;
                        term_t = hc.t_in;
                        break;
                    }
                    hc = hn;
                    cc = cn;
                }
#else
                for (int j = 0; j < n; ++j) {
                    double t_hit;
                    if (wf_composite_one(A, T, S, H, sorted_ref(j) & ~kJointRef, tau, t_hit)) {
                        terminated = true;
                        term_t = t_hit;
                        break;
                    }
                }
#endif
            } else {
                // more hits than the buffers hold: selection instead of sorting --
                // repeatedly take the smallest key after the last composited one
                bool have_last = false;
                double lt = 0.0;
                unsigned long long lk = 0;
                for (;;) {
                    u32 best = kNil;
                    double bt = 0.0;
                    unsigned long long bk = 0;
                    for (u32 ref = H.first(); ref != kNil; ref = H.next(ref)) {
                        const WfHit *hp = H.at(ref);
                        if (hp->key2 & kDroppedBit) continue;
                        const double t = hp->t_in;
                        const unsigned long long k2 = hp->key2;
                        if (have_last && !wf_before(lt, lk, t, k2)) continue;
                        if (best == kNil || wf_before(t, k2, bt, bk)) {
                            best = ref;
                            bt = t;
                            bk = k2;
                        }
                    }
                    if (best == kNil) break;
                    double t_hit;
                    if (wf_composite_one(A, T, S, H, best, tau, t_hit)) {
                        terminated = true;
                        term_t = t_hit;
                        break;
                    }
                    have_last = true;
                    lt = bt;
                    lk = bk;
                }
            }
            rp.acc[0] = S.acc[0];
            rp.acc[1] = S.acc[1];
            rp.acc[2] = S.acc[2];
            rp.acc[3] = S.acc[3];
            rp.n_seen = (u16)S.n_seen;
            rp.n_sph = (u16)S.n_sph;
            rp.seen_bloom = S.seen_bloom;
            rp.sph_bloom = S.sph_bloom;
            rp.ovf = T.ovf;
            const u32 term_k = terminated ? wf_find_window(wins, nw, term_t) : 0u;
            if (big) {
                // window_overflow of the windows gathered up to (and including) the last one used
                unsigned long long ov = 0;
                for (u32 k = 0; k < nw; ++k) {
                    if (wins[k].tests & kBigBit) ov += A.win_over[w0 + k];
                    if (terminated && k == term_k) break;
                }
                rp.over += ov;
            }
            if (terminated) {
                tests = wins[term_k].tests & ~kBigBit;
                finished = true;
                WF_STAT(4, 1);
                WF_STAT(5, S.n_seen);
                WF_STAT(6, S.n_sph);
            }
            if (!finished) A.rp[slot] = rp;
        } else if (finished) {
            rp = A.rp[slot];
        }
        if (finished) {
            if (!terminated) tests = A.rw[slot].tests;
            over = rp.over;
            const uint2 px = A.rpix[slot];
            write_pixel(A, px.y, rp.acc[0], rp.acc[1], rp.acc[2], rp.acc[3]);
            const u32 y = px.x >> 16;
            if (tests) atomicAdd(A.row_stats + 3 * (i64)y + 1, tests);
            if (over) atomicAdd(A.row_stats + 3 * (i64)y + 2, over);
        } else if (valid) {
            const unsigned mask = __activemask();
            const int leader = __ffs((int)mask) - 1;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(&A.ctl->n_live[par ^ 1], (u32)__popc(mask));
            base = __shfl_sync(mask, base, leader);
            A.live[par ^ 1][base + __popc(mask & ((1u << lane) - 1u))] = slot;
        }
        __syncwarp();
    }
}

// between iterations: clear the queues, retire the consumed live list, set the next budget
__global__ void wf_next_kernel(const WfArgs A, int par, int it_next) {
    WF_PDL_ENTER();
    const int t = threadIdx.x;
    if (t < kNQ) {
        A.ctl->item_cnt[t] = 0;
        A.ctl->tube_cnt[t] = 0;
        A.ctl->sph_cnt[t] = 0;
        A.ctl->hit_cnt[t] = 0;
    }
    if (t == 0) {
        A.ctl->n_live[par] = 0;
        const u32 live = A.ctl->n_live[par ^ 1];
        if (live == 0 && A.ctl->done_it == 0) A.ctl->done_it = (u32)it_next;
        u32 wn = (u32)A.wn_sched << (it_next < A.wn_shift_max ? it_next : A.wn_shift_max);
        const u32 fit = live ? A.cap_win / live : A.cap_win;
        if (wn > fit) wn = fit;
        if (wn < 1) wn = 1;
        A.ctl->wn = wn;
        // later iterations hold few rays, all with low hit rates: let them run further
        {
            const int g = it_next - A.grow_from;
            int sh = g < 0 ? 0 : g * A.grow_bits;
            // the last few thousand rays: finish them in few iterations (their over-scan is noise)
            if (live < (u32)A.tail_rays) sh += A.tail_bits;
            // once the rays are spread over the warps (wf_spread) a ray no longer waits for
            // the others of its warp: a larger budget then only saves iterations
            // (only the tail of a frame: rays that have survived tail_from iterations, once
            // fewer than 1/16 of the frame's rays are left -- those rarely terminate and collect
            // few hits, so walking further ahead of the compositing is not wasted; in a small or
            // very transparent frame every ray is spread and long-lived, and a larger budget
            // only pushes rays onto the many-hits paths of the composite kernel)
            if (it_next == 1) A.ctl->live0 = live;
            const bool tail = it_next >= A.tail_from && (unsigned long long)live * 16u <= A.ctl->live0;
            const u32 ls = tail ? wf_spread(live, A.ray_threads) : 0u;
            if (A.tail_mode == 1) sh += (ls >= 3 ? 1 : 0) + (ls >= 5 ? 1 : 0);
            else if (A.tail_mode == 2) sh += (ls >= 2 ? 1 : 0) + (ls >= 4 ? 1 : 0);
            else if (A.tail_mode == 3) sh += (ls >= 3 ? 1 : 0) + (ls >= 5 ? 2 : 0);
            else if (A.tail_mode == 4) sh += (ls >= 1 ? 1 : 0) + (ls >= 5 ? 1 : 0);
            A.ctl->budget = (u32)A.cand_budget << (sh < 12 ? sh : 12);
        }
    }
}

__global__ void wf_begin_kernel(const WfArgs A) {
    WF_PDL_ENTER();
    const int t = threadIdx.x;
    if (t < kNQ) {
        A.ctl->item_cnt[t] = 0;
        A.ctl->tube_cnt[t] = 0;
        A.ctl->sph_cnt[t] = 0;
        A.ctl->hit_cnt[t] = 0;
    }
    if (t == 0) {
        A.ctl->n_live[0] = 0;
        A.ctl->n_live[1] = 0;
        A.ctl->pool_cnt = 0;
        A.ctl->err = 0;
        A.ctl->done_it = 0;
#ifdef LVX_WF_STATS
        for (int k = 0; k < 8; ++k) A.ctl->dbg[k] = 0;
#endif
        // (the window records of iteration 0 must fit whatever LVX_WF_WN asks for)
        const u32 fit = A.R ? (u32)(A.cap_win / A.R) : A.cap_win;
        A.ctl->wn = (u32)A.wn_sched < fit ? (u32)A.wn_sched : (fit ? fit : 1u);
        A.ctl->budget = (u32)A.cand_budget;
    }
}

// scratch layout ------------------------------------------------------------------------
struct WfLayout {
    size_t total;
    size_t ctl, rw, rp, rpix, head, tab_seen, tab_sph, pool_seen, pool_sph, live0, live1, win,
        win_over, item, item_t, fdir, span, rdir, tube, sph, hit, hit_c, hit_next, hit_slot,
        slot_c, hcnt, bgfill;
    u32 R, pool_cap, cap_win, capq_item, capq_surv, capq_hit;
};

constexpr size_t kBgChunk = (size_t)8 << 20;  // background pattern the copy engine repeats over a host image

size_t take(size_t &cur, size_t bytes) {
    const size_t at = (cur + 255) & ~(size_t)255;
    cur = at + bytes;
    return at;
}

WfLayout wf_layout(i64 R, double scale) {
    WfLayout L;
    memset(&L, 0, sizeof(L));
    L.R = (u32)R;
    const double f = scale < 1.0 / 64.0 ? 1.0 / 64.0 : scale;  // (< 1 only to exercise the overflow path)
    L.pool_cap = (u32)(R / 16 * f) + 1024;
    L.cap_win = (u32)fmin(4.0e9, (double)R * (double)kWinFirst);  // every ray may record kWinFirst windows in iteration 0
    L.capq_item = (u32)fmin(4.0e9 / kNQ, ((double)R * 24.0 * f + 65536.0) / kNQ);
    L.capq_surv = (u32)fmin(4.0e9 / kNQ, ((double)R * 10.0 * f + 65536.0) / kNQ);
    L.capq_hit = (u32)fmin(2.0e9 / kNQ, ((double)R * 2.0 * f + 65536.0) / kNQ);  // (references keep bit 31 free)
    size_t c = 0;
    const size_t r = (size_t)R, po = (size_t)L.pool_cap * (LVX_MAX_SEEN - kInline);
    L.ctl = take(c, sizeof(WfCtl));
    L.rw = take(c, r * sizeof(WfRayWalk));
    L.rp = take(c, r * sizeof(WfRayPix));
    L.head = take(c, r * 4);
    L.rpix = take(c, r * 8);
    L.tab_seen = take(c, r * 8 * kInline);
    L.tab_sph = take(c, r * 16 * kInline);
    L.pool_seen = take(c, po * 8);
    L.pool_sph = take(c, po * 16);
    L.live0 = take(c, r * 4);
    L.live1 = take(c, r * 4);
    L.win = take(c, (size_t)L.cap_win * sizeof(WfWindow));
    L.win_over = take(c, (size_t)L.cap_win * 4);
    L.item = take(c, (size_t)L.capq_item * kNQ * 16);
    L.item_t = take(c, (size_t)L.capq_item * kNQ * 16);
    L.fdir = take(c, r * 16);
    L.span = take(c, r * 16);
    L.rdir = take(c, r * sizeof(WfRayDir));
    L.tube = take(c, (size_t)L.capq_surv * kNQ * sizeof(WfEntry));
    L.sph = take(c, (size_t)L.capq_surv * kNQ * sizeof(WfEntry));
    L.hit = take(c, (size_t)L.capq_hit * kNQ * sizeof(WfHit));
    L.hit_c = take(c, (size_t)L.capq_hit * kNQ * 16);
    L.hit_next = take(c, (size_t)L.capq_hit * kNQ * 4);
    L.hit_slot = take(c, r * kHitSlots * sizeof(WfHit));
    L.slot_c = take(c, r * kHitSlots * 16);
    L.hcnt = take(c, r * 4);
    L.bgfill = take(c, kBgChunk);
    L.total = take(c, 0);
    return L;
}

i64 wf_ray_slots(const lvx_camera *cam, const lvx_tiling *t) {
    const i64 tiles_x = lvx_ceil_div(cam->width, t->tile_w), tiles_y = lvx_ceil_div(cam->height, t->tile_h);
    const i64 total = tiles_x * tiles_y;
    i64 mine = 0;
    if (t->tile_first < total) mine = (total - t->tile_first + t->tile_step - 1) / t->tile_step;
    return mine * t->tile_w * t->tile_h;
}

int wf_check_tiling(const lvx_tiling *t) {
    LVX_REQUIRE(t && t->tile_w >= 8 && t->tile_h >= 4 && (t->tile_w % 8) == 0 && (t->tile_h % 4) == 0 &&
                    t->tile_step >= 1 && t->tile_first >= 0 && t->tile_first < t->tile_step,
                "tiling: tile_w %% 8 == 0, tile_h %% 4 == 0, 0 <= tile_first < tile_step required");
    return LVX_OK;
}

// Schedule constants of the engine.  The environment is consulted once per process (developer
// sweeps), never per frame.
struct WfTuning {
    int wn_sched = kWinFirst;
    int cand_budget = 192;
    int grow_from = 24;  // (growing earlier does not pay: the late iterations are cheap, over-scanning is not)
    int grow_bits = 1;
    int tail_rays = 0, tail_bits = 4, tail_mode = 1, tail_from = 6;
    int wn_shift_max = 4;
    int rays_mult = 0;  // 0: by the number of ray slots
    bool debug = false;
    bool pdl = true;  // programmatic dependent launch of the frame's kernels (LVX_WF_PDL=0: plain launches)
    bool bg_copy = true;  // background of a host image by the copy engine (LVX_WF_BGCOPY=0: by wf_init)
    bool adaptive_burst = true;  // first burst sized by the previous frame's iteration count (LVX_WF_ADAPT=0: always six)
};

int env_int(const char *name, int dflt, bool positive_only = false) {
    const char *e = getenv(name);
    if (!e) return dflt;
    const int v = atoi(e);
    return positive_only && v <= 0 ? dflt : v;
}

const WfTuning &wf_tuning() {
    static const WfTuning T = [] {
        WfTuning t;
        t.tail_mode = env_int("LVX_WF_TAIL_MODE", t.tail_mode);
        t.tail_from = env_int("LVX_WF_TAIL_FROM", t.tail_from);
        t.tail_rays = env_int("LVX_WF_TAIL_RAYS", t.tail_rays);
        t.tail_bits = env_int("LVX_WF_TAIL_BITS", t.tail_bits);
        t.grow_bits = env_int("LVX_WF_GROW_BITS", t.grow_bits);
        t.wn_shift_max = env_int("LVX_WF_WN_SHIFT", t.wn_shift_max);
        t.cand_budget = env_int("LVX_WF_BUDGET", t.cand_budget, true);
        t.grow_from = env_int("LVX_WF_GROW", t.grow_from);
        t.wn_sched = env_int("LVX_WF_WN", t.wn_sched, true);
        t.rays_mult = env_int("LVX_WF_GRID_RAYS", t.rays_mult, true);
        t.debug = getenv("LVX_WF_DEBUG") != nullptr;
        t.pdl = env_int("LVX_WF_PDL", 1) != 0;
        t.adaptive_burst = env_int("LVX_WF_ADAPT", 1) != 0;
        t.bg_copy = env_int("LVX_WF_BGCOPY", 1) != 0;
        return t;
    }();
    return T;
}

// a second stream of the calling thread on the current device, for the copy-engine transfers that run
// next to a frame (created once)
struct WfSide {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
WfSide *wf_side() {
    static thread_local WfSide sides[16];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    WfSide &s = sides[dev];
    if (s.device != dev) {
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
        s.device = dev;
    }
    return &s;
}

// is p pinned host memory (mapped into the device's address space)?
bool wf_is_host_pointer(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

}  // namespace

static thread_local int g_last_launches = 0, g_last_iterations = 0;
static thread_local int g_needed_iterations = 0;  // of this thread's previous frame (sizes the next frame's first burst)

extern "C" {

int lvx_render_wf_last_launches(int *iterations) {
    if (iterations) *iterations = g_last_iterations;
    return g_last_launches;
}

size_t lvx_render_wf_scratch_bytes(const lvx_camera *cam, const lvx_tiling *tiling, double scale) {
    if (!cam || !tiling || tiling->tile_w < 8 || tiling->tile_h < 4 || tiling->tile_step < 1) return 0;
    const i64 R = wf_ray_slots(cam, tiling);
    return wf_layout(R > 0 ? R : 32, scale).total;
}

int lvx_render_wf(const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
                  const lvx_lod *lod, const lvx_tiling *tiling, float *img_d, int64_t *row_stats_d,
                  void *scratch_d, size_t scratch_bytes, double scale, void *stream) {
    LVX_REQUIRE(cam && model && params && img_d && row_stats_d && scratch_d, "null argument");
    LVX_REQUIRE(cam->width >= 1 && cam->height >= 1 && cam->width < 65536 && cam->height < 65536,
                "image dims must be in [1, 65535]");
    if (int rc = wf_check_tiling(tiling)) return rc;
    LVX_REQUIRE(model->rx >= 1 && model->ry >= 1 && model->rz >= 1 && model->counts_d && model->offsets_d &&
                    model->table_d,
                "bad model");
    LVX_REQUIRE(model->rx < 65535 && model->ry < 65535 && model->rz < 65535 &&
                    (i64)model->rx * model->ry * model->rz < ((i64)1 << 31),
                "grid too large to render");
    LVX_REQUIRE(!params->neighbor || (model->nsum_d && model->nmask_d && model->ncell_d),
                "neighbour mode needs the neighbour grids (lvx_neighbor_sums, with the merged cells)");
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
    LVX_REQUIRE(!need_oct || (lod && lod->oct_flat_d && lod->n_levels >= 1 && lod->n_levels <= LVX_MAX_LEVELS),
                "cone shadows / density-rays AO need a density octree");
    LVX_REQUIRE(params->ao_mode != LVX_AO_PRECOMPUTED || (lod && lod->ao_flat_d),
                "precomputed AO requested but no AO field given");
    LVX_REQUIRE((params->ao_mode != LVX_AO_DENSITY && params->ao_mode != LVX_AO_HEMISPHERE) ||
                    (lod && lod->ao_dirs_d && params->ao_n_rays >= 1),
                "density-rays / hemisphere AO need the direction lattice");

    const i64 R = wf_ray_slots(cam, tiling);
    if (R == 0) return LVX_OK;
    LVX_REQUIRE(R < ((i64)1 << 31), "too many rays for one launch");
    const WfLayout L = wf_layout(R, scale);
    LVX_REQUIRE(scratch_bytes >= L.total, "scratch too small: %zu < %zu bytes", scratch_bytes, L.total);
    LVX_REQUIRE(((uintptr_t)scratch_d & 255) == 0, "scratch must be 256-byte aligned");

    WfArgs A;
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
    A.ncell = reinterpret_cast<const unsigned long long *>(model->ncell_d);
    if (lod) {
        A.oc.flat = lod->oct_flat_d;
        A.oc.n_levels = lod->n_levels;
        for (int l = 0; l <= lod->n_levels && l <= LVX_MAX_LEVELS; ++l) A.oc.off[l] = lod->oct_off[l];
        for (int l = 0; l < lod->n_levels * 3 && l < LVX_MAX_LEVELS * 3; ++l) A.oc.dims[l] = (int)lod->oct_dims[l];
        A.ao_flat = lod->ao_flat_d;
        A.ao_dirs = lod->ao_dirs_d;
        if (lod->rep.valid_d) {
            A.rep = LvxRepLevel{lod->rep.valid_d, lod->rep.a_d, lod->rep.b_d, lod->rep.w_d, lod->rep.dims[0],
                                lod->rep.dims[1], lod->rep.dims[2], lod->rep.size};
            A.rep_radius_base = params->tube_r * lod->rep.size;
        }
    }
    A.tl = *tiling;
    {
        const i64 tiles_x = lvx_ceil_div(cam->width, tiling->tile_w);
        A.tiles_x = (int)tiles_x;
        A.n_my_tiles = (int)(R / ((i64)tiling->tile_w * tiling->tile_h));
    }
    A.img = img_d;
    A.row_stats = reinterpret_cast<unsigned long long *>(row_stats_d);
    char *base = (char *)scratch_d;
    A.R = L.R;
    A.ctl = (WfCtl *)(base + L.ctl);
    A.rw = (WfRayWalk *)(base + L.rw);
    A.rp = (WfRayPix *)(base + L.rp);
    A.head = (u32 *)(base + L.head);
    A.rpix = (uint2 *)(base + L.rpix);
    A.tab_seen = (uint2 *)(base + L.tab_seen);
    A.tab_sph = (float4 *)(base + L.tab_sph);
    A.pool_seen = (uint2 *)(base + L.pool_seen);
    A.pool_sph = (float4 *)(base + L.pool_sph);
    A.pool_cap = L.pool_cap;
    A.live[0] = (u32 *)(base + L.live0);
    A.live[1] = (u32 *)(base + L.live1);
    A.win = (WfWindow *)(base + L.win);
    A.cap_win = L.cap_win;
    A.win_over = (u32 *)(base + L.win_over);
    A.item = (uint4 *)(base + L.item);
    A.item_t = (double2 *)(base + L.item_t);
    A.fdir = (float4 *)(base + L.fdir);
    A.span = (double *)(base + L.span);
    A.rdir = (WfRayDir *)(base + L.rdir);
    A.capq_item = L.capq_item;
    A.tube = (WfEntry *)(base + L.tube);
    A.sph = (WfEntry *)(base + L.sph);
    A.capq_surv = L.capq_surv;
    A.hit = (WfHit *)(base + L.hit);
    A.hit_c = (float4 *)(base + L.hit_c);
    A.hit_next = (u32 *)(base + L.hit_next);
    A.capq_hit = L.capq_hit;
    A.hit_slot = (WfHit *)(base + L.hit_slot);
    A.slot_c = (float4 *)(base + L.slot_c);
    A.hcnt = (u32 *)(base + L.hcnt);
    // schedule constants; the LVX_WF_* developer overrides are read ONCE per process
    const WfTuning &tune = wf_tuning();
    A.wn_sched = tune.wn_sched;
    A.cand_budget = tune.cand_budget;
    A.grow_from = tune.grow_from;
    A.grow_bits = tune.grow_bits;
    A.tail_rays = tune.tail_rays;
    A.tail_bits = tune.tail_bits;
    A.tail_mode = tune.tail_mode;
    A.tail_from = tune.tail_from;
    A.wn_shift_max = tune.wn_shift_max;

    const bool debug = tune.debug;
    const bool pdl = tune.pdl && !debug;
    const bool geom = params->shadow_mode == LVX_SHADOW_HARD || params->shadow_mode == LVX_SHADOW_REPLINES ||
                      params->ao_mode == LVX_AO_HEMISPHERE;
    // straight from the encoded records when the caller passes no render records (the geometry
    // secondary rays walk the render records themselves)
    // (a model without segments may pass neither: nothing is dereferenced)
    const bool packed = model->seg_rec_d == nullptr && model->packed_d != nullptr;
    LVX_REQUIRE(!packed || !geom, "frames with geometry secondary rays (hard / replines shadows, hemisphere AO) walk "
                "the render records: pass lvx_seg_record");
    if (packed) {
        LVX_REQUIRE(model->n_bins >= 2 && model->n_bins <= 256 && (model->n_bins & (model->n_bins - 1)) == 0,
                    "bad bin resolution %d of the encoded records", model->n_bins);
        LVX_REQUIRE(((uintptr_t)model->packed_d & 7) == 0, "packed_d must be 8-byte aligned");
        int lb = 0;
        while ((1 << (lb + 1)) <= model->n_bins) ++lb;
        A.pk.bytes = model->packed_d;
        A.pk.lb = lb;
        A.pk.n = model->n_bins;
        A.pk.inv_n = 1.0f / (float)model->n_bins;
        A.pk.width = (2 * (3 + 2 * lb) + 8 + 5 + 7) / 8;  // record_width, voxelizer.py:70-76
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int sms = lvx_sm_count();
    // blocks per SM of the ray-parallel kernels (walk, composite): 8 for a full frame; a screen share of a
    // multi-GPU frame has fewer rays than that launch has threads from the first iteration on, and does
    // better with a smaller one (1080p / 8 ranks: 2.48 -> 2.26 ms, 4K / 8: 4.74 -> 4.54 ms; LVX_WF_GRID_RAYS overrides)
    const int rays_mult = tune.rays_mult > 0 ? tune.rays_mult : (R >= 1500000 ? 8 : (R >= 600000 ? 6 : 4));
    const unsigned grid_rays = (unsigned)(sms * rays_mult), grid_q = (unsigned)(sms * 8);
    A.ray_threads = grid_rays * (unsigned)kThreadsWf;
    const size_t walk_smem = sizeof(WalkStage) + (params->neighbor ? 0 : sizeof(WalkStageT));
    {
        static bool attr_set = false;  // (more than 48 KB of dynamic shared memory is opt-in, once per process)
        if (!attr_set) {
            LVX_CUDA_CHECK(cudaFuncSetAttribute(wf_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(sizeof(WalkStage) + sizeof(WalkStageT))));
            attr_set = true;
        }
    }
    // A HOST image (pinned memory the kernels write through its device mapping): two thirds of a frame
    // like C3 are rays that miss the grid, 22 MB of identical pixels that wf_init would push over PCIe
    // store by store.  A copy engine lays them instead -- the miss pixel repeated over the WHOLE image,
    // from an 8 MB pattern in the scratch buffer, on a second stream while init / walk / candidates /
    // exact run -- and is joined before the first kernel that writes finished pixels (composite).
    WfSide *side = nullptr;
    // (only when this call renders the WHOLE image: a share of an in-place tiled frame must not touch
    // the other shares' pixels)
    if (tune.bg_copy && !debug && !tiling->compact && tiling->tile_step == 1 && tiling->tile_first == 0 &&
        wf_is_host_pointer(img_d))
        side = wf_side();
    bool side_joined = true;
    if (side) {
        float4 *pat = (float4 *)(base + L.bgfill);
        const size_t img_bytes = (size_t)cam->width * cam->height * 16;
        const size_t chunk = img_bytes < kBgChunk ? img_bytes : kBgChunk;
        wf_bgfill_kernel<<<(unsigned)sms, 256, 0, st>>>(A, pat, (u32)(chunk / 16));
        LVX_CUDA_CHECK(cudaEventRecord(side->fork, st));
        LVX_CUDA_CHECK(cudaStreamWaitEvent(side->stream, side->fork, 0));
        for (size_t off = 0; off < img_bytes; off += chunk) {
            const size_t n = img_bytes - off < chunk ? img_bytes - off : chunk;
            LVX_CUDA_CHECK(cudaMemcpyAsync((char *)img_d + off, pat, n, cudaMemcpyDeviceToHost, side->stream));
        }
        LVX_CUDA_CHECK(cudaEventRecord(side->join, side->stream));
        A.skip_miss = 1;
        side_joined = false;
    }
    LVX_CUDA_CHECK(wf_launch(pdl, wf_begin_kernel, 1, 64, 0, st, A));
    LVX_CUDA_CHECK(wf_launch(pdl, wf_init_kernel, (unsigned)lvx_ceil_div(R, kThreadsWf), kThreadsWf, 0, st, A));
    LVX_LAUNCH_CHECK();
    u32 host[4] = {0, 0, 0, 0};
    int it = 0;
    const int first_burst = tune.adaptive_burst ? (g_needed_iterations < 48 ? g_needed_iterations : 48) : 0;
    g_last_launches = 2;
    for (;;) {
        // bursts of iterations between looks at the live-ray count: six at a time (a frame like C3, 10
        // iterations, costs two host read-backs instead of ten; an iteration without rays is five empty
        // launches).  The FIRST burst is as long as the previous frame of this thread turned out to be --
        // consecutive frames of an interactive session need the same number of iterations give or take
        // one --, so a steady sequence of frames reads the count back once, at the end, and launches
        // nothing in vain; a wrong guess costs a few empty launches or one more burst, never a result.
        const int burst = it == 0 && first_burst > 6 ? first_burst : 6;
        for (int b = 0; b < burst; ++b, ++it) {
            const int par = it & 1;
#define WF_DEBUG_SYNC(name)                                                                   \
    if (debug) {                                                                              \
        cudaError_t e_ = cudaStreamSynchronize(st);                                           \
        if (e_ != cudaSuccess) {                                                              \
            lvx_set_error("wavefront iteration %d: %s failed: %s", it, name, cudaGetErrorString(e_)); \
            return LVX_E_CUDA;                                                                \
        }                                                                                     \
    }
            LVX_CUDA_CHECK(wf_launch(pdl, wf_walk_kernel, grid_rays, kThreadsWf, walk_smem, st, A, par));
            WF_DEBUG_SYNC("walk");
            if (packed) LVX_CUDA_CHECK(wf_launch(pdl, wf_cand_kernel<true>, grid_q, kThreadsWf, 0, st, A));
            else LVX_CUDA_CHECK(wf_launch(pdl, wf_cand_kernel<false>, grid_q, kThreadsWf, 0, st, A));
            WF_DEBUG_SYNC("candidates");
            if (geom) LVX_CUDA_CHECK(wf_launch(pdl, wf_exact_kernel<true, false>, grid_q, kThreadsExact, 0, st, A, par));
            else if (packed) LVX_CUDA_CHECK(wf_launch(pdl, wf_exact_kernel<false, true>, grid_q, kThreadsExact, 0, st, A, par));
            else LVX_CUDA_CHECK(wf_launch(pdl, wf_exact_kernel<false, false>, grid_q, kThreadsExact, 0, st, A, par));
            WF_DEBUG_SYNC("exact");
            if (!side_joined) {  // (the background is down before any finished pixel is written)
                LVX_CUDA_CHECK(cudaStreamWaitEvent(st, side->join, 0));
                side_joined = true;
            }
            LVX_CUDA_CHECK(wf_launch(pdl, wf_composite_kernel, grid_rays, kThreadsWf, 0, st, A, par));
            WF_DEBUG_SYNC("composite");
            if (debug) {
                WfCtl c;
                cudaMemcpyAsync(&c, A.ctl, sizeof(c), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                unsigned long long ni = 0, nc = 0, nt = 0, ns = 0, nh = 0;
                for (int q = 0; q < kNQ; ++q) {
                    ni += c.item_cnt[q];
                    nt += c.tube_cnt[q];
                    ns += c.sph_cnt[q];
                    nh += c.hit_cnt[q];
                }
                fprintf(stderr, "wf it %2d: live %8u -> %8u  wn %4u budget %6u  items %10llu  candidates %10llu  tubes %9llu  "
                        "spheres %9llu  listed hits %8llu\n",
                        it, c.n_live[par], c.n_live[par ^ 1], c.wn, c.budget, ni, nc, nt, ns, nh);
#ifdef LVX_WF_STATS
                fprintf(stderr, "      cumulative: owned hits %llu  composited %llu  rays-with-hits %llu  terminated %llu  "
                        "sum n_seen %llu  sum n_sph %llu\n", c.dbg[0], c.dbg[1], c.dbg[3], c.dbg[4], c.dbg[5], c.dbg[6]);
#endif
            }
            LVX_CUDA_CHECK(wf_launch(pdl, wf_next_kernel, 1, 64, 0, st, A, par, it + 1));
        }
        LVX_LAUNCH_CHECK();
        // rays left?  (n_live of the list the next iteration reads, and the error bits)
        LVX_CUDA_CHECK(cudaMemcpyAsync(&host[0], &A.ctl->n_live[it & 1], 4, cudaMemcpyDeviceToHost, st));
        LVX_CUDA_CHECK(cudaMemcpyAsync(&host[1], &A.ctl->err, 4, cudaMemcpyDeviceToHost, st));
        LVX_CUDA_CHECK(cudaMemcpyAsync(&host[2], &A.ctl->done_it, 4, cudaMemcpyDeviceToHost, st));
        LVX_CUDA_CHECK(cudaStreamSynchronize(st));
        if (host[1]) {
            lvx_set_error("wavefront queues overflowed (bits %u): retry with a larger scratch scale", host[1]);
            return LVX_E_RANGE;
        }
        g_last_iterations = it;
        g_needed_iterations = host[2] ? (int)host[2] : it;
        // begin, init (+ the background pattern) + (walk, candidates, exact, composite, next) per iteration
        g_last_launches = 2 + (side ? 1 : 0) + it * 5;
        if (host[0] == 0) break;
        LVX_REQUIRE(it < 100000, "wavefront did not converge");
    }
    return LVX_OK;
}

}  // extern "C"
