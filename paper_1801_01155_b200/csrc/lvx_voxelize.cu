// Voxelizer for sm_100a: edge-parallel clip -> per-voxel counting (atomics) ->
// device prefix sums -> scatter -> per-voxel key ranking -> pack.
//
// Restates, bit for bit, the reference's numpy pipeline
//   _plane_events / _clip_batch   voxelizer.py:174-263
//   _faces_and_bins               voxelizer.py:358-380
//   build_voxel_model             voxelizer.py:397-488
//   _pack_all / _field_layout     voxelizer.py:79-89, 383-394
// The reference sorts all plane-crossing events of a batch (lexsort by edge, s)
// and pairs consecutive events of a curve into chords.  Here every polyline edge
// is one thread: it merges its own x/y/z crossings in the same order (ascending
// s, ties x<y<z), and fetches the one event it cannot produce itself -- the last
// crossing of the nearest earlier edge of the same curve -- by a short look-back.
#include "lvx_common.cuh"

namespace {

constexpr double kMinChord = 1e-9;  // voxelizer.py:37
constexpr double kFaceEps = 1e-9;   // voxelizer.py:361
#ifndef LVX_CLIP_THREADS
#define LVX_CLIP_THREADS 128
#endif
constexpr int kClipThreads = LVX_CLIP_THREADS;
#ifndef LVX_CLIP_TILE
#define LVX_CLIP_TILE 1  // chords built crossing-parallel from a shared-memory tile of events (0: edge-parallel)
#endif

struct Event {
    double pos[3];
    double attr;
    double k;
    int ax;
    bool up;
};

__device__ __forceinline__ double clip01(double s) {
    // np.clip(s, 0, 1), voxelizer.py:200
    s = s < 0.0 ? 0.0 : s;
    s = s > 1.0 ? 1.0 : s;
    return s;
}

// Per-axis crossing bookkeeping of one edge (voxelizer.py:185-200).
struct EdgeAxes {
    double x0[3], d[3], f0[3];
    int cnt[3];
    bool up[3];

    __device__ __forceinline__ void init(const double a0[3], const double a1[3]) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            x0[ax] = a0[ax];
            d[ax] = a1[ax] - a0[ax];
            f0[ax] = floor(a0[ax]);
            double f1 = floor(a1[ax]);
            up[ax] = d[ax] > 0.0;
            double c = up[ax] ? f1 - f0[ax] : f0[ax] - f1;
            long long ci = (long long)c;
            cnt[ax] = ci < 0 ? 0 : (int)ci;
        }
    }
    __device__ __forceinline__ int total() const { return cnt[0] + cnt[1] + cnt[2]; }
    __device__ __forceinline__ double plane(int ax, int j) const {
        return up[ax] ? f0[ax] + 1.0 + (double)j : f0[ax] - (double)j;
    }
    __device__ __forceinline__ double param(int ax, double k) const {
        return clip01((k - x0[ax]) / d[ax]);
    }
};

__device__ __forceinline__ void make_event(Event &ev, const EdgeAxes &E, const double a0[3],
                                           double att0, double att1, bool want_attr, int ax,
                                           double k, double s) {
    // (selects instead of indexing by `ax`: keeps the event in registers)
#pragma unroll
    for (int c = 0; c < 3; ++c) ev.pos[c] = c == ax ? k : a0[c] + s * E.d[c];  // voxelizer.py:228-229
    ev.attr = want_attr ? att0 + s * (att1 - att0) : 0.0;                      // :230
    ev.k = k;
    ev.ax = ax;
    ev.up = ax == 0 ? E.up[0] : (ax == 1 ? E.up[1] : E.up[2]);
}

// Chord voxel + keep test, voxelizer.py:242-250.  Returns the linear voxel index
// or -1 when the chord is dropped.
__device__ __forceinline__ i64 chord_voxel(const Event &a, const Event &b, int rx, int ry, int rz,
                                           long long vox[3]) {
    double m = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double mid = 0.5 * (a.pos[c] + b.pos[c]);
        vox[c] = (long long)floor(mid);
        double dd = fabs(b.pos[c] - a.pos[c]);
        m = dd > m ? dd : m;
    }
    const long long vo = (long long)(b.up ? b.k - 1.0 : b.k);
    const long long vi = (long long)(a.up ? a.k : a.k - 1.0);
    // (selects on the three components, the entry event's axis last: indexing vox[] by a run-time axis
    // puts the array in local memory)
    vox[0] = a.ax == 0 ? vi : (b.ax == 0 ? vo : vox[0]);
    vox[1] = a.ax == 1 ? vi : (b.ax == 1 ? vo : vox[1]);
    vox[2] = a.ax == 2 ? vi : (b.ax == 2 ? vo : vox[2]);
    if (!(m > kMinChord)) return -1;
    if (vox[0] < 0 || vox[0] >= rx || vox[1] < 0 || vox[1] >= ry || vox[2] < 0 || vox[2] >= rz)
        return -1;
    return vox[0] + (i64)rx * (vox[1] + (i64)ry * vox[2]);
}

// _faces_and_bins, voxelizer.py:358-380.  Returns face | code << 3, or ~0 when off
// every face.
__device__ __forceinline__ u32 face_and_bin(const double p[3], const long long vox[3], int n) {
    double local[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) local[c] = p[c] - (double)vox[c];
    int f = -1;
#pragma unroll
    for (int ax = 2; ax >= 0; --ax) {  // lowest face id wins: scan downward, overwrite
        if (local[ax] >= 1.0 - kFaceEps) f = 2 * ax + 1;
        if (local[ax] <= kFaceEps) f = 2 * ax;
    }
    if (f < 0) return 0xFFFFFFFFu;
    int axis = f >> 1;
    double u = axis == 0 ? local[1] : local[0];
    double v = axis == 2 ? local[1] : local[2];
    long long bu = (long long)floor(u * (double)n);
    long long bv = (long long)floor(v * (double)n);
    bu = bu < 0 ? 0 : (bu > n - 1 ? n - 1 : bu);
    bv = bv < 0 ? 0 : (bv > n - 1 ? n - 1 : bv);
    return (u32)f | ((u32)(bu + (long long)n * bv) << 3);
}

// ---------------------------------------------------------------------------
// Single-pass clipper (lvx_voxelize_bound + lvx_voxelize_clip): the polyline vertices are
// read from HBM once.  A block stages its 257 vertices, attributes and curve-start flags in
// shared memory (the look-back to earlier edges stays on chip unless it leaves the block);
// every edge first COUNTS its kept chords, a block scan and one atomic per block reserve a
// contiguous range of the raw-record arrays, then the edge re-derives its chords from the
// staged operands and writes them there (coalesced), bumping the per-voxel counters with
// result-less atomics.  The order of the raw records is irrelevant: the per-voxel order is
// restored from the (edge, ordinal) keys by compact_kernel.
// ---------------------------------------------------------------------------

struct ClipStage {
    double pts[(kClipThreads + 1) * 3];
    double attr[kClipThreads + 1];
    u8 first[kClipThreads + 1];
};

// vertex / attribute / flag of point index p: from the staged block when inside it
struct ClipView {
    const ClipStage &S;
    const double *pts, *attrs;
    const u8 *first;
    i64 base, hi;  // staged range [base, hi)
    __device__ __forceinline__ void vertex(i64 p, double v[3]) const {
        if (p >= base && p < hi) {
#pragma unroll
            for (int c = 0; c < 3; ++c) v[c] = S.pts[3 * (p - base) + c];
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) v[c] = pts[3 * p + c];
        }
    }
    __device__ __forceinline__ double attr(i64 p) const { return p >= base && p < hi ? S.attr[p - base] : attrs[p]; }
    __device__ __forceinline__ bool is_first(i64 p) const { return p >= base && p < hi ? S.first[p - base] : first[p]; }
};

template <bool WANT_ATTR>
__device__ bool lookback_event_v(const ClipView &V, i64 i, Event &ev) {
    i64 ip = i;
    while (!V.is_first(ip)) {
        ip -= 1;
        double a0[3], a1[3];
        V.vertex(ip, a0);
        V.vertex(ip + 1, a1);
        EdgeAxes E;
        E.init(a0, a1);
        if (E.total() == 0) continue;
        int best = -1;
        double bs = 0.0, bk = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (E.cnt[ax] == 0) continue;
            double k = E.plane(ax, E.cnt[ax] - 1);
            double s = E.param(ax, k);
            if (best < 0 || s >= bs) {  // ties: the higher axis sorts last
                best = ax;
                bs = s;
                bk = k;
            }
        }
        double att0 = 0.0, att1 = 0.0;
        if (WANT_ATTR) {
            att0 = V.attr(ip);
            att1 = V.attr(ip + 1);
        }
        make_event(ev, E, a0, att0, att1, WANT_ATTR, best, bk, bs);
        return true;
    }
    return false;
}

constexpr u32 kNoVoxel = 0xFFFFFFFFu;  // raw_lin of a reserved slot that holds no chord

// The chords of edge i in the reference's order, written to raw[slot0 + n] for the n-th
// crossing of the edge (slots of dropped chords keep kNoVoxel) and counted per voxel.
// Returns how many were kept.
__device__ __forceinline__ int clip_edge(const ClipView &V, i64 i, const EdgeAxes &E, const double a0[3],
                                         int rx, int ry, int rz, int n_bins, u32 *__restrict__ vox_cnt,
                                         u64 *__restrict__ raw_key, u64 *__restrict__ raw_q,
                                         u32 *__restrict__ raw_lin, u64 slot0, int *__restrict__ err) {
    const int total = E.total();
    const double att0 = V.attr(i), att1 = V.attr(i + 1);
    Event prev, ev;
    bool have_prev = lookback_event_v<true>(V, i, prev);
    int j[3] = {0, 0, 0};
    double s_next[3], k_next[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        k_next[ax] = E.plane(ax, 0);
        s_next[ax] = E.cnt[ax] > 0 ? E.param(ax, k_next[ax]) : 2.0;
    }
    int kept = 0;
    for (int n = 0; n < total; ++n) {
        // smallest s first; ties resolve x<y<z (stable lexsort, voxelizer.py:224)
        int best = 0;
        double bs = s_next[0];
        if (s_next[1] < bs) {
            best = 1;
            bs = s_next[1];
        }
        if (s_next[2] < bs) {
            best = 2;
            bs = s_next[2];
        }
        const double bk = best == 0 ? k_next[0] : (best == 1 ? k_next[1] : k_next[2]);
        make_event(ev, E, a0, att0, att1, true, best, bk, bs);
        u32 out_lin = kNoVoxel;
        if (have_prev) {
            long long vox[3];
            const i64 lin = chord_voxel(prev, ev, rx, ry, rz, vox);
            if (lin >= 0) {
                // voxelizer.py:439 -- rint is round-half-even
                double av = rint(255.0 * 0.5 * (prev.attr + ev.attr));
                av = av < 0.0 ? 0.0 : (av > 255.0 ? 255.0 : av);
                u32 fin = face_and_bin(prev.pos, vox, n_bins);
                u32 fout = face_and_bin(ev.pos, vox, n_bins);
                if (fin == 0xFFFFFFFFu || fout == 0xFFFFFFFFu) {
                    *err = 1;
                    fin = fout = 0;
                }
                raw_key[slot0 + n] = ((u64)i << 16) | (u64)kept;
                raw_q[slot0 + n] = (u64)fin | ((u64)fout << 19) | ((u64)(u32)av << 38);
                out_lin = (u32)lin;
                atomicAdd(&vox_cnt[lin], 1u);  // result unused: compiles to a reduction
                kept += 1;
            }
        }
        raw_lin[slot0 + n] = out_lin;
        prev = ev;
        have_prev = true;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (ax == best) {
                j[ax] += 1;
                if (j[ax] < E.cnt[ax]) {
                    k_next[ax] = E.plane(ax, j[ax]);
                    s_next[ax] = E.param(ax, k_next[ax]);
                } else {
                    s_next[ax] = 2.0;  // exhausted (valid s are clipped to <= 1)
                }
            }
        }
    }
    return kept;
}

// The edge-parallel path as a call of its own (a block with more than kTileEvents crossings: rare): it
// takes scalars only and rebuilds the edge from the staged vertices, so nothing of the caller's state has
// to live in local memory for it.
__device__ __noinline__ int clip_edge_call(const ClipStage *S, const double *pts, const double *attrs, const u8 *first,
                                           i64 base, i64 hi, i64 i, int rx, int ry, int rz, int n_bins,
                                           u32 *__restrict__ vox_cnt, u64 *__restrict__ raw_key,
                                           u64 *__restrict__ raw_q, u32 *__restrict__ raw_lin, u64 slot0,
                                           int *__restrict__ err) {
    const ClipView V = {*S, pts, attrs, first, base, hi};
    double a0[3], a1[3];
    V.vertex(i, a0);
    V.vertex(i + 1, a1);
    EdgeAxes E;
    E.init(a0, a1);
    return clip_edge(V, i, E, a0, rx, ry, rz, n_bins, vox_cnt, raw_key, raw_q, raw_lin, slot0, err);
}

#ifndef LVX_CLIP_MINB
#define LVX_CLIP_MINB 8
#endif
// The plane-crossing events of a block's edges, in the reference's order (slot order = edge order, then
// the merged (s, axis) order inside an edge), staged in shared memory: every event is computed ONCE, by
// its edge, and every chord -- the pair (event e-1, event e) of one curve -- is then built by its own
// thread, so the chord half of the work (voxel, keep test, two face/bin quantisations, attribute, the
// three stores and the counter) runs with all lanes busy however the crossings are spread over the
// edges (0-3 per edge on the bench scenes: the edge-parallel version ran at 15.8 of 32 lanes and
// computed the last event of every edge twice, once more by the look-back of its successor).
#ifndef LVX_CLIP_TILE_EVENTS
#define LVX_CLIP_TILE_EVENTS 512
#endif
constexpr int kTileEvents = LVX_CLIP_TILE_EVENTS;  // a block whose edges cross more planes takes the edge-parallel path
static_assert(kClipThreads <= 128, "block-local edge and curve-start indices are bytes with 0xFF reserved");
struct ClipTile {
    // (slot kTileEvents: the predecessor of the block's first event when it lies in an earlier block)
    double x[kTileEvents + 1], y[kTileEvents + 1], z[kTileEvents + 1], a[kTileEvents + 1];
    u16 meta[kTileEvents + 1];    // edge (block-local) | axis << 8 | up << 10
    u8 kept[kTileEvents];
    u16 slot0[kClipThreads];      // first event slot of edge t (exclusive prefix of the crossing counts)
    u8 cstart[kClipThreads];      // block-local index of the first point of edge t's curve; 0xFF: before the block
};

__device__ __forceinline__ void tile_event(const ClipTile &T, int e, Event &ev) {
    const u32 m = T.meta[e];
    ev.pos[0] = T.x[e];
    ev.pos[1] = T.y[e];
    ev.pos[2] = T.z[e];
    ev.attr = T.a[e];
    ev.ax = (int)((m >> 8) & 3u);
    ev.up = ((m >> 10) & 1u) != 0;
    ev.k = ev.ax == 0 ? ev.pos[0] : (ev.ax == 1 ? ev.pos[1] : ev.pos[2]);  // make_event: pos[ax] = k
}

__global__ void __launch_bounds__(kClipThreads, LVX_CLIP_MINB)
clip_once_kernel(const double *__restrict__ pts, const double *__restrict__ attrs, const u8 *__restrict__ first,
                 i64 n_points, int rx, int ry, int rz, int n_bins, u64 capacity, u32 *__restrict__ vox_cnt,
                 u64 *__restrict__ raw_key, u64 *__restrict__ raw_q, u32 *__restrict__ raw_lin,
                 unsigned long long *__restrict__ n_slots, u16 *__restrict__ edge_kept, int *__restrict__ err) {
    __shared__ ClipStage S;
#if LVX_CLIP_TILE
    __shared__ ClipTile T;
    __shared__ int s_cw[kClipThreads / 32];  // last curve start seen by each warp
    __shared__ int s_prev0;                  // the block's first event has a predecessor outside the block
#endif
    __shared__ u32 s_warp[kClipThreads / 32];
    __shared__ unsigned long long s_base;
    const i64 base = (i64)blockIdx.x * kClipThreads;
    const i64 hi = min(base + kClipThreads + 1, n_points);
    for (i64 k = base * 3 + threadIdx.x; k < hi * 3; k += kClipThreads) S.pts[k - base * 3] = pts[k];
    for (i64 k = base + threadIdx.x; k < hi; k += kClipThreads) {
        S.attr[k - base] = attrs[k];
        S.first[k - base] = first[k];
    }
    __syncthreads();
    const ClipView V = {S, pts, attrs, first, base, hi};
    const i64 i = base + threadIdx.x;
    const bool edge = i + 1 < n_points && !S.first[threadIdx.x + 1];
    // (only the crossing count is carried over the block scan: the edge is set up again from the staged
    // vertices where its events are listed -- six shared-memory loads and floors against ~25 registers
    // held across two barriers)
    int crossings = 0;
    if (edge) {
        double a0[3], a1[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            a0[c] = S.pts[3 * threadIdx.x + c];
            a1[c] = S.pts[3 * (threadIdx.x + 1) + c];
        }
        EdgeAxes E0;
        E0.init(a0, a1);
        crossings = E0.total();
    }
    // reserve one slot per plane crossing of the block (every chord ends at a crossing)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 inc = (u32)crossings;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
#if LVX_CLIP_TILE
    // the curve of edge t starts at the last first-point at or before t (running maximum over the block)
    int cs = (i < n_points && S.first[threadIdx.x]) ? (int)threadIdx.x : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, cs, o);
        if (lane >= o) cs = max(cs, t);
    }
    if (lane == 31) s_cw[warp] = cs;
#endif
    __syncthreads();
    u32 before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kClipThreads / 32; ++w) {
        const u32 t = s_warp[w];
        if (w < warp) before += t;
        total += t;
    }
    if (threadIdx.x == 0) s_base = total ? atomicAdd(n_slots, (unsigned long long)total) : 0ull;
#if LVX_CLIP_TILE
    if (total != 0 && total <= (u32)kTileEvents) {
#pragma unroll
        for (int w = 0; w < kClipThreads / 32; ++w) {
            if (w < warp) cs = max(cs, s_cw[w]);
        }
        const u32 my0 = before + inc - (u32)crossings;
        T.slot0[threadIdx.x] = (u16)my0;
        T.cstart[threadIdx.x] = cs < 0 ? (u8)0xFF : (u8)cs;
        if (threadIdx.x == 0) s_prev0 = 0;
        __syncthreads();
        const u64 blk0 = s_base;
        if (blk0 + (u64)total > capacity) {  // the caller's bound was wrong
            if (threadIdx.x == 0) *err = 2;
            if (i < n_points && edge_kept) edge_kept[i] = 0;
            return;
        }
        // A: every edge lists its own events in merged (s, axis) order (voxelizer.py:224)
        if (crossings > 0) {
            const double att0 = S.attr[threadIdx.x], att1 = S.attr[threadIdx.x + 1];
            EdgeAxes E;
            {
                double a0[3], a1[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    a0[c] = S.pts[3 * threadIdx.x + c];
                    a1[c] = S.pts[3 * (threadIdx.x + 1) + c];
                }
                E.init(a0, a1);
            }
            // (the plane of the next crossing is recomputed from its ordinal instead of being carried: the
            // kernel is short of registers, not of integer-to-double conversions)
            int j[3] = {0, 0, 0};
            double s_next[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) s_next[ax] = E.cnt[ax] > 0 ? E.param(ax, E.plane(ax, 0)) : 2.0;
            Event ev;
            for (int n = 0; n < crossings; ++n) {
                int best = 0;
                double bs = s_next[0];
                if (s_next[1] < bs) {
                    best = 1;
                    bs = s_next[1];
                }
                if (s_next[2] < bs) {
                    best = 2;
                    bs = s_next[2];
                }
                const double bk = best == 0 ? E.plane(0, j[0]) : (best == 1 ? E.plane(1, j[1]) : E.plane(2, j[2]));
                make_event(ev, E, E.x0, att0, att1, true, best, bk, bs);
                const u32 e = my0 + (u32)n;
                T.x[e] = ev.pos[0];
                T.y[e] = ev.pos[1];
                T.z[e] = ev.pos[2];
                T.a[e] = ev.attr;
                T.meta[e] = (u16)(threadIdx.x | ((u32)best << 8) | ((ev.up ? 1u : 0u) << 10));
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    if (ax == best) {
                        j[ax] += 1;
                        s_next[ax] = j[ax] < E.cnt[ax] ? E.param(ax, E.plane(ax, j[ax])) : 2.0;  // (valid s are <= 1)
                    }
                }
            }
        }
        // the one event that may pair with an event of an earlier block: the block's first, when its curve
        // began before the block (the look-back from the block's first point; the edges between that
        // point and the event's own edge cross nothing)
        if (crossings > 0 && my0 == 0 && cs < 0) {
            Event p0;
            if (lookback_event_v<true>(V, base, p0)) {
                T.x[kTileEvents] = p0.pos[0];
                T.y[kTileEvents] = p0.pos[1];
                T.z[kTileEvents] = p0.pos[2];
                T.a[kTileEvents] = p0.attr;
                T.meta[kTileEvents] = (u16)(((u32)p0.ax << 8) | ((p0.up ? 1u : 0u) << 10));
                s_prev0 = 1;
            }
        }
        __syncthreads();
        // B: one thread per chord
        for (u32 e = threadIdx.x; e < total; e += kClipThreads) {
            Event ev, prev;
            tile_event(T, (int)e, ev);
            const u32 il = T.meta[e] & 0xFFu;
            bool have_prev;
            if (e > 0) {
                tile_event(T, (int)e - 1, prev);
                have_prev = T.cstart[T.meta[e - 1] & 0xFFu] == T.cstart[il];  // same curve
            } else {
                have_prev = s_prev0 != 0;
                if (have_prev) tile_event(T, kTileEvents, prev);
            }
            u32 out_lin = kNoVoxel;
            u8 kept = 0;
            if (have_prev) {
                long long vox[3];
                const i64 lin = chord_voxel(prev, ev, rx, ry, rz, vox);
                if (lin >= 0) {
                    // voxelizer.py:439 -- rint is round-half-even
                    double av = rint(255.0 * 0.5 * (prev.attr + ev.attr));
                    av = av < 0.0 ? 0.0 : (av > 255.0 ? 255.0 : av);
                    u32 fin = face_and_bin(prev.pos, vox, n_bins);
                    u32 fout = face_and_bin(ev.pos, vox, n_bins);
                    if (fin == 0xFFFFFFFFu || fout == 0xFFFFFFFFu) {
                        *err = 1;
                        fin = fout = 0;
                    }
                    raw_q[blk0 + e] = (u64)fin | ((u64)fout << 19) | ((u64)(u32)av << 38);
                    out_lin = (u32)lin;
                    atomicAdd(&vox_cnt[lin], 1u);  // result unused: compiles to a reduction
                    kept = 1;
                }
            }
            raw_lin[blk0 + e] = out_lin;
            T.kept[e] = kept;
        }
        __syncthreads();
        // C: the key of a kept chord carries its ordinal among the kept chords of its edge
        for (u32 e = threadIdx.x; e < total; e += kClipThreads) {
            if (!T.kept[e]) continue;
            const u32 il = T.meta[e] & 0xFFu;
            u32 ord = 0;
            for (u32 k = T.slot0[il]; k < e; ++k) ord += T.kept[k];
            raw_key[blk0 + e] = ((u64)(base + il) << 16) | (u64)ord;
        }
        if (i < n_points && edge_kept) {
            u32 kept = 0;
            for (u32 k = 0; k < (u32)crossings; ++k) kept += T.kept[my0 + k];
            edge_kept[i] = (u16)kept;
        }
        return;
    }
#endif
    __syncthreads();
    int kept = 0;
    if (crossings > 0) {
        const u64 slot0 = s_base + before + inc - (u32)crossings;
        if (slot0 + (u64)crossings > capacity) *err = 2;  // the caller's bound was wrong
        else kept = clip_edge_call(&S, pts, attrs, first, base, hi, i, rx, ry, rz, n_bins, vox_cnt, raw_key, raw_q,
                                   raw_lin, slot0, err);
    }
    if (i < n_points && edge_kept) edge_kept[i] = (u16)kept;
}

// _clip_batch (voxelizer.py:213-263) with its float64 outputs, for the reference op
// clip_curve_to_voxels and the parity tests: one thread per edge, the kept chords are appended
// in any order with their (edge, ordinal) key; the host sorts by key.
__global__ void __launch_bounds__(128)
probe_clip_kernel(const double *__restrict__ pts, const double *__restrict__ attrs, const u8 *__restrict__ first,
                  i64 n_points, int rx, int ry, int rz, u64 capacity, i64 *__restrict__ out_vox,
                  double *__restrict__ out_pin, double *__restrict__ out_pout, double *__restrict__ out_attr,
                  u64 *__restrict__ out_key, unsigned long long *__restrict__ n_out) {
    __shared__ ClipStage S;  // (unused: everything is read from global memory)
    const ClipView V = {S, pts, attrs, first, 0, 0};
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 >= n_points || first[i + 1]) return;
    double a0[3], a1[3];
    V.vertex(i, a0);
    V.vertex(i + 1, a1);
    EdgeAxes E;
    E.init(a0, a1);
    const int total = E.total();
    if (total == 0) return;
    const double att0 = attrs[i], att1 = attrs[i + 1];
    Event prev, ev;
    bool have_prev = lookback_event_v<true>(V, i, prev);
    int j[3] = {0, 0, 0};
    u32 kept = 0;
    for (int n = 0; n < total; ++n) {
        int best = -1;
        double bs = 0.0, bk = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            if (j[ax] >= E.cnt[ax]) continue;
            const double k = E.plane(ax, j[ax]);
            const double sv = E.param(ax, k);
            if (best < 0 || sv < bs) {  // ties resolve x<y<z (stable lexsort, voxelizer.py:224)
                best = ax;
                bs = sv;
                bk = k;
            }
        }
        j[best] += 1;
        make_event(ev, E, a0, att0, att1, true, best, bk, bs);
        if (have_prev) {
            long long vox[3];
            if (chord_voxel(prev, ev, rx, ry, rz, vox) >= 0) {
                const unsigned long long slot = atomicAdd(n_out, 1ull);
                if (slot < capacity) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        out_vox[3 * slot + c] = vox[c];
                        out_pin[3 * slot + c] = prev.pos[c];
                        out_pout[3 * slot + c] = ev.pos[c];
                    }
                    out_attr[2 * slot] = prev.attr;
                    out_attr[2 * slot + 1] = ev.attr;
                    out_key[slot] = ((u64)i << 16) | (u64)kept;
                }
                kept += 1;
            }
        }
        prev = ev;
        have_prev = true;
    }
}

// Upper bound of the chord count: every chord ends at a plane crossing.
__global__ void __launch_bounds__(256)
count_crossings_kernel(const double *__restrict__ pts, const u8 *__restrict__ first, i64 n_points,
                       unsigned long long *__restrict__ total) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long n = 0;
    if (i + 1 < n_points && !first[i + 1]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double d = fabs(floor(pts[3 * (i + 1) + c]) - floor(pts[3 * i + c]));
            n += d < 1e15 ? (unsigned long long)d : 0ull;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, o);
    __shared__ unsigned long long s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += s[w];
        if (t) atomicAdd(total, t);
    }
}

__global__ void mark_starts_kernel(const i64 *__restrict__ curve_off, i64 n_curves,
                                   u8 *__restrict__ first) {
    i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < n_curves) first[curve_off[c]] = 1;
}

// ---------------------------------------------------------------------------
// Device prefix sums (three-phase: tile sums, scan of tile sums, tile rescan).
// ---------------------------------------------------------------------------

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of one u32 per thread; returns the thread's exclusive
// prefix and leaves the block total in *total.
__device__ __forceinline__ u32 block_exclusive_scan(u32 v, u32 *s_warp, u32 *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        u32 w = lane < (kScanThreads / 32) ? s_warp[lane] : 0;
        u32 winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 t = __shfl_up_sync(0xFFFFFFFFu, winc, o);
            if (lane >= o) winc += t;
        }
        if (lane < (kScanThreads / 32)) s_warp[lane] = winc - w;
        if (lane == (kScanThreads / 32) - 1) s_warp[kScanThreads / 32] = winc;
    }
    __syncthreads();
    u32 res = s_warp[warp] + inc - v;
    *total = s_warp[kScanThreads / 32];
    __syncthreads();
    return res;
}

template <typename T>
__device__ __forceinline__ u32 load_count(const T *in, i64 idx, i64 n) {
    return idx < n ? (u32)in[idx] : 0u;
}

// the kScanItems counters of one thread (one 32-byte access when they are u32 and in range)
template <typename T>
__device__ __forceinline__ void load_counts(const T *in, i64 t0, i64 n, u32 v[kScanItems]) {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = load_count(in, t0 + k, n);
}
template <>
__device__ __forceinline__ void load_counts<u32>(const u32 *in, i64 t0, i64 n, u32 v[kScanItems]) {
    static_assert(kScanItems == 8, "one 32-byte vector per thread");
    if (t0 + kScanItems <= n && (reinterpret_cast<uintptr_t>(in) & 31) == 0) {
        u64 a, b, c, d;
        lvx_ld256(in + t0, a, b, c, d);
        v[0] = (u32)a;
        v[1] = (u32)(a >> 32);
        v[2] = (u32)b;
        v[3] = (u32)(b >> 32);
        v[4] = (u32)c;
        v[5] = (u32)(c >> 32);
        v[6] = (u32)d;
        v[7] = (u32)(d >> 32);
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = load_count(in, t0 + k, n);
    }
}

// phase 1: per-tile sums of raw and capped counts
template <typename T, bool CAP>
__global__ void __launch_bounds__(kScanThreads)
scan_tile_sums(const T *__restrict__ in, i64 n, u64 *__restrict__ partial) {
    __shared__ u32 s_warp[kScanThreads / 32 + 1];
    const i64 t0 = (i64)blockIdx.x * kScanTile + (i64)threadIdx.x * kScanItems;
    u32 raw = 0, cap = 0;
    u32 vv[kScanItems];
    load_counts(in, t0, n, vv);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const u32 v = vv[k];
        raw += v;
        cap += CAP ? (v > 255u ? 255u : v) : 0u;
    }
    u32 total;
    block_exclusive_scan(raw, s_warp, &total);
    if (threadIdx.x == 0) partial[2 * (i64)blockIdx.x] = total;
    if (CAP) {
        block_exclusive_scan(cap, s_warp, &total);
        if (threadIdx.x == 0) partial[2 * (i64)blockIdx.x + 1] = total;
    } else if (threadIdx.x == 0) {
        partial[2 * (i64)blockIdx.x + 1] = 0;
    }
}

// phase 2: one block turns the tile sums into exclusive prefixes (u64) in place
__global__ void __launch_bounds__(1024) scan_partials(u64 *partial, i64 n_tiles, u64 *totals) {
    __shared__ u64 s_a[1024], s_b[1024];
    u64 run_a = 0, run_b = 0;
    for (i64 base = 0; base < n_tiles; base += 1024) {
        i64 idx = base + threadIdx.x;
        u64 a = idx < n_tiles ? partial[2 * idx] : 0, b = idx < n_tiles ? partial[2 * idx + 1] : 0;
        s_a[threadIdx.x] = a;
        s_b[threadIdx.x] = b;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            u64 ta = threadIdx.x >= o ? s_a[threadIdx.x - o] : 0;
            u64 tb = threadIdx.x >= o ? s_b[threadIdx.x - o] : 0;
            __syncthreads();
            s_a[threadIdx.x] += ta;
            s_b[threadIdx.x] += tb;
            __syncthreads();
        }
        if (idx < n_tiles) {
            partial[2 * idx] = run_a + s_a[threadIdx.x] - a;
            partial[2 * idx + 1] = run_b + s_b[threadIdx.x] - b;
        }
        run_a += s_a[1023];
        run_b += s_b[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0 && totals) {
        totals[0] = run_a;
        totals[1] = run_b;
    }
}

// phase 3: rescan each tile with its prefix and write the outputs
template <typename T, bool CAP>
__global__ void __launch_bounds__(kScanThreads)
scan_write(const T *__restrict__ in, i64 n, const u64 *__restrict__ partial,
           u32 *__restrict__ out_raw, u32 *__restrict__ out_cap, u8 *__restrict__ out_counts) {
    __shared__ u32 s_warp[kScanThreads / 32 + 1];
    const i64 t0 = (i64)blockIdx.x * kScanTile + (i64)threadIdx.x * kScanItems;
    u32 v[kScanItems];
    u32 raw = 0, cap = 0;
    load_counts(in, t0, n, v);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        raw += v[k];
        cap += CAP ? (v[k] > 255u ? 255u : v[k]) : 0u;
    }
    u32 total;
    u32 pr = block_exclusive_scan(raw, s_warp, &total) + (u32)partial[2 * (i64)blockIdx.x];
    u32 pc = 0;
    if (CAP) pc = block_exclusive_scan(cap, s_warp, &total) + (u32)partial[2 * (i64)blockIdx.x + 1];
    const bool full = t0 + kScanItems <= n && (reinterpret_cast<uintptr_t>(out_raw) & 31) == 0 &&
                      (!CAP || ((reinterpret_cast<uintptr_t>(out_cap) & 31) == 0 &&
                                (reinterpret_cast<uintptr_t>(out_counts) & 7) == 0));
    if (full) {
        // one 32-byte store per output array and thread
        u32 r[kScanItems], c[kScanItems];
        u64 cnt8 = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            r[k] = pr;
            pr += v[k];
            const u32 cc = v[k] > 255u ? 255u : v[k];
            c[k] = pc;
            pc += cc;
            cnt8 |= (u64)cc << (8 * k);
        }
        lvx_st256(out_raw + t0, r[0] | ((u64)r[1] << 32), r[2] | ((u64)r[3] << 32), r[4] | ((u64)r[5] << 32),
                  r[6] | ((u64)r[7] << 32));
        if (CAP) {
            lvx_st256(out_cap + t0, c[0] | ((u64)c[1] << 32), c[2] | ((u64)c[3] << 32), c[4] | ((u64)c[5] << 32),
                      c[6] | ((u64)c[7] << 32));
            *reinterpret_cast<u64 *>(out_counts + t0) = cnt8;
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        i64 idx = t0 + k;
        if (idx < n) {
            out_raw[idx] = pr;
            if (CAP) {
                u32 c = v[k] > 255u ? 255u : v[k];
                out_cap[idx] = pc;
                out_counts[idx] = (u8)c;
                pc += c;
            }
        }
        pr += v[k];
    }
}

// ---------------------------------------------------------------------------
// Compaction: rank every raw record inside its voxel by key, apply the 255 cap,
// assign lid, decode bin centres, pack.  One thread per raw record.
// ---------------------------------------------------------------------------

struct CompactOut {
    u8 *packed;
    float *seg_a, *seg_b;
    u8 *seg_attr, *seg_lid;
    int32_t *seg_voxel;
    u8 *face_in, *face_out;
    u16 *bin_in, *bin_out;
    u64 *seg_key;
    lvx_seg_record *seg_rec;
};

__device__ __forceinline__ void decode_point(u32 face, u32 code, int n, int lb, int vx, int vy,
                                             int vz, float out[3]) {
    // bin centre + voxel, cast to f32 (voxelizer.py:376-380, 477-478)
    const int bu = (int)(code & (u32)(n - 1)), bv = (int)(code >> lb);
    const double cu = ((double)bu + 0.5) / (double)n, cv = ((double)bv + 0.5) / (double)n;
    const int axis = (int)(face >> 1);
    double q[3];
    q[0] = axis == 0 ? (double)(face & 1) : cu;
    q[1] = axis == 1 ? (double)(face & 1) : (axis == 0 ? cu : cv);
    q[2] = axis == 2 ? (double)(face & 1) : cv;
    out[0] = (float)(q[0] + (double)vx);
    out[1] = (float)(q[1] + (double)vy);
    out[2] = (float)(q[2] + (double)vz);
}

__global__ void __launch_bounds__(256)
compact_kernel(const lvx_raw_record *__restrict__ grouped, i64 n_raw, const u32 *__restrict__ vox_cnt,
               const u32 *__restrict__ cursor_end, const u32 *__restrict__ offsets, int rx, int ry,
               int n_bins, int lb, int width, CompactOut o) {
    const i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_raw) return;
    u64 key, q, lin64, unused;
    lvx_ld256(grouped + r, key, q, lin64, unused);
    const u32 lin = (u32)lin64;
    const u32 n = vox_cnt[lin];
    u32 rank = 0;
    if (n > 1) {
        const u32 end = cursor_end[lin];
        // (a record that already has 255 predecessors is dropped whatever the rest of its group
        // holds: the scan of a crowded voxel -- thousands of chords on a coarse grid -- stops there)
        for (u32 k = end - n; k < end && rank < 255u; ++k) rank += grouped[k].key < key ? 1u : 0u;
    }
    if (rank >= 255u) return;  // voxelizer.py:442-448 keep the first 255 in curve order
    const i64 dst = (i64)offsets[lin] + rank;
    const u32 fi = (u32)(q & 7u), bi = (u32)((q >> 3) & 0xFFFFu);
    const u32 fo = (u32)((q >> 19) & 7u), bo = (u32)((q >> 22) & 0xFFFFu);
    const u32 attr = (u32)((q >> 38) & 0xFFu);
    const u32 lid = rank & 31u;  // voxelizer.py:449
    const int vx = (int)(lin % (u32)rx), vy = (int)((lin / (u32)rx) % (u32)ry),
              vz = (int)(lin / ((u32)rx * (u32)ry));
    float a[3], b[3];
    decode_point(fi, bi, n_bins, lb, vx, vy, vz, a);
    decode_point(fo, bo, n_bins, lb, vx, vy, vz, b);
    // _field_layout / _pack_all, voxelizer.py:79-89, 383-394 (LSB first)
    const int bb = 2 * lb;
    const u64 value = (u64)fi | ((u64)bi << 3) | ((u64)fo << (3 + bb)) | ((u64)bo << (6 + bb)) |
                      ((u64)attr << (6 + 2 * bb)) | ((u64)lid << (14 + 2 * bb));
    u8 *pk = o.packed + dst * width;
    for (int k = 0; k < width; ++k) pk[k] = (u8)(value >> (8 * k));
    if (o.seg_a) {
        o.seg_a[3 * dst] = a[0];
        o.seg_a[3 * dst + 1] = a[1];
        o.seg_a[3 * dst + 2] = a[2];
    }
    if (o.seg_b) {
        o.seg_b[3 * dst] = b[0];
        o.seg_b[3 * dst + 1] = b[1];
        o.seg_b[3 * dst + 2] = b[2];
    }
    if (o.seg_attr) o.seg_attr[dst] = (u8)attr;
    if (o.seg_lid) o.seg_lid[dst] = (u8)lid;
    if (o.seg_voxel) {
        o.seg_voxel[3 * dst] = vx;
        o.seg_voxel[3 * dst + 1] = vy;
        o.seg_voxel[3 * dst + 2] = vz;
    }
    if (o.face_in) o.face_in[dst] = (u8)fi;
    if (o.face_out) o.face_out[dst] = (u8)fo;
    if (o.bin_in) o.bin_in[dst] = (u16)bi;
    if (o.bin_out) o.bin_out[dst] = (u16)bo;
    if (o.seg_key) o.seg_key[dst] = key;
    if (o.seg_rec) {
        const float hl = lvx_half_len(a[0], a[1], a[2], b[0], b[1], b[2]);
        lvx_st256(o.seg_rec + dst, (u64)__float_as_uint(a[0]) | ((u64)__float_as_uint(a[1]) << 32),
                  (u64)__float_as_uint(a[2]) | ((u64)(attr | (lid << 8)) << 32),
                  (u64)__float_as_uint(b[0]) | ((u64)__float_as_uint(b[1]) << 32),
                  (u64)__float_as_uint(b[2]) | ((u64)__float_as_uint(hl) << 32));
    }
}

// Inverse of the packer: one thread per voxel walks its records (model_io.py:151-179,
// _decode_records + _bin_centers).  A model that arrives as (counts, offsets, packed) --
// e.g. read from a .vxl file -- gets its render records and, if wanted, the reference's
// per-segment caches without a host-side expansion.
__global__ void __launch_bounds__(128)
decode_packed_kernel(const u8 *__restrict__ packed, const u8 *__restrict__ counts,
                     const u32 *__restrict__ offsets, i64 n_voxels, int rx, int ry, int n_bins, int lb,
                     int width, CompactOut o, int *__restrict__ err) {
    const i64 lin = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (lin >= n_voxels) return;
    const u32 cnt = counts[lin];
    if (cnt == 0) return;
    const i64 base = offsets[lin];
    const int vx = (int)(lin % rx), vy = (int)((lin / rx) % ry), vz = (int)(lin / ((i64)rx * ry));
    const int bb = 2 * lb;
    const u64 bmask = ((u64)1 << bb) - 1;
    for (u32 sgi = 0; sgi < cnt; ++sgi) {
        const i64 dst = base + sgi;
        const u8 *pk = packed + dst * width;
        u64 value = 0;
        for (int k = 0; k < width; ++k) value |= (u64)pk[k] << (8 * k);
        // _field_layout, voxelizer.py:79-89 (LSB first)
        const u32 fi = (u32)(value & 7u), bi = (u32)((value >> 3) & bmask);
        const u32 fo = (u32)((value >> (3 + bb)) & 7u), bo = (u32)((value >> (6 + bb)) & bmask);
        const u32 attr = (u32)((value >> (6 + 2 * bb)) & 0xFFu), lid = (u32)((value >> (14 + 2 * bb)) & 31u);
        if (fi > 5u || fo > 5u) {
            *err = 1;  // model_io.py:277-278: segment record with face ID > 5
            continue;
        }
        float a[3], b[3];
        decode_point(fi, bi, n_bins, lb, vx, vy, vz, a);
        decode_point(fo, bo, n_bins, lb, vx, vy, vz, b);
        if (o.seg_a) {
            o.seg_a[3 * dst] = a[0];
            o.seg_a[3 * dst + 1] = a[1];
            o.seg_a[3 * dst + 2] = a[2];
        }
        if (o.seg_b) {
            o.seg_b[3 * dst] = b[0];
            o.seg_b[3 * dst + 1] = b[1];
            o.seg_b[3 * dst + 2] = b[2];
        }
        if (o.seg_attr) o.seg_attr[dst] = (u8)attr;
        if (o.seg_lid) o.seg_lid[dst] = (u8)lid;
        if (o.seg_voxel) {
            o.seg_voxel[3 * dst] = vx;
            o.seg_voxel[3 * dst + 1] = vy;
            o.seg_voxel[3 * dst + 2] = vz;
        }
        if (o.face_in) o.face_in[dst] = (u8)fi;
        if (o.face_out) o.face_out[dst] = (u8)fo;
        if (o.bin_in) o.bin_in[dst] = (u16)bi;
        if (o.bin_out) o.bin_out[dst] = (u16)bo;
        if (o.seg_rec) {
            const float hl = lvx_half_len(a[0], a[1], a[2], b[0], b[1], b[2]);
            lvx_st256(o.seg_rec + dst, (u64)__float_as_uint(a[0]) | ((u64)__float_as_uint(a[1]) << 32),
                      (u64)__float_as_uint(a[2]) | ((u64)(attr | (lid << 8)) << 32),
                      (u64)__float_as_uint(b[0]) | ((u64)__float_as_uint(b[1]) << 32),
                      (u64)__float_as_uint(b[2]) | ((u64)__float_as_uint(hl) << 32));
        }
    }
}

__global__ void __launch_bounds__(256)
provenance_kernel(const u64 *__restrict__ seg_key, i64 n_seg, const u32 *__restrict__ edge_base,
                  const i64 *__restrict__ curve_off, i64 n_curves, int32_t *__restrict__ seg_curve,
                  int32_t *__restrict__ seg_order) {
    const i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    const u64 key = seg_key[s];
    const i64 e = (i64)(key >> 16);
    const u32 jk = (u32)(key & 0xFFFFu);
    // curve = last c with curve_off[c] <= e
    i64 lo = 0, hi = n_curves;  // invariant: curve_off[lo] <= e < curve_off[hi]
    while (hi - lo > 1) {
        i64 mid = (lo + hi) >> 1;
        if (curve_off[mid] <= e) lo = mid;
        else hi = mid;
    }
    seg_curve[s] = (int32_t)lo;
    // chord index inside the curve after filtering (voxelizer.py:254-262)
    seg_order[s] = (int32_t)(edge_base[e] + jk - edge_base[curve_off[lo]]);
}

__global__ void __launch_bounds__(256)
seg_records_kernel(const float *__restrict__ seg_a, const float *__restrict__ seg_b,
                   const u8 *__restrict__ seg_attr, const u8 *__restrict__ seg_lid, i64 n,
                   lvx_seg_record *__restrict__ rec) {
    const i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    float4 *r = reinterpret_cast<float4 *>(rec + s);
    u32 meta = (u32)seg_attr[s] | ((u32)seg_lid[s] << 8);
    r[0] = make_float4(seg_a[3 * s], seg_a[3 * s + 1], seg_a[3 * s + 2], __uint_as_float(meta));
    r[1] = make_float4(seg_b[3 * s], seg_b[3 * s + 1], seg_b[3 * s + 2],
                       lvx_half_len(seg_a[3 * s], seg_a[3 * s + 1], seg_a[3 * s + 2], seg_b[3 * s],
                                    seg_b[3 * s + 1], seg_b[3 * s + 2]));
}

// Multi-GPU merge: raw records gathered from all ranks (each rank's block is grouped
// by voxel, but the blocks are not interleaved) are scattered into one voxel-grouped
// array through the global per-voxel cursors.  Order inside a voxel is restored by
// the key ranking of compact_kernel.
__global__ void __launch_bounds__(256)
regroup_kernel(const u64 *__restrict__ in_key, const u64 *__restrict__ in_q,
               const u32 *__restrict__ in_lin, i64 n, u32 *__restrict__ cursor,
               lvx_raw_record *__restrict__ out) {
    const i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const u32 lin = in_lin[r];
    if (lin == kNoVoxel) return;  // a reserved slot without a chord
    const u32 slot = atomicAdd(&cursor[lin], 1u);
    // one whole 32-byte sector per record: the scattered write needs no read-modify-write
    lvx_st256(out + slot, in_key[r], in_q[r], (u64)lin, 0ull);
}

int ilog2i(int n) {
    int lb = 0;
    while ((1 << (lb + 1)) <= n) ++lb;
    return lb;
}

int check_dims(const int32_t dims[3]) {
    LVX_REQUIRE(dims && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1, "grid dims must be >= 1");
    const i64 V = (i64)dims[0] * dims[1] * dims[2];
    if (V >= ((i64)1 << 32) || (i64)dims[0] + dims[1] + dims[2] > 65000) {
        lvx_set_error("grid %dx%dx%d exceeds the 2^32-voxel / 65000-plane limits", dims[0],
                      dims[1], dims[2]);
        return LVX_E_RANGE;
    }
    return LVX_OK;
}

int check_bins(int n) {
    LVX_REQUIRE(n >= 2 && n <= 256 && (n & (n - 1)) == 0,
                "bin resolution must be a power of two in [2,256], got %d", n);
    return LVX_OK;
}

}  // namespace

extern "C" {

int lvx_mark_curve_starts(const int64_t *curve_off_d, int64_t n_curves, int64_t n_points,
                          uint8_t *first_d, void *stream) {
    LVX_REQUIRE(curve_off_d && first_d && n_curves >= 0 && n_points >= 0, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    if (n_points == 0) return LVX_OK;
    LVX_CUDA_CHECK(cudaMemsetAsync(first_d, 0, (size_t)n_points, st));
    if (n_curves > 0) {
        mark_starts_kernel<<<(unsigned)lvx_ceil_div(n_curves, 256), 256, 0, st>>>(curve_off_d,
                                                                                 n_curves, first_d);
        LVX_LAUNCH_CHECK();
    }
    return LVX_OK;
}

size_t lvx_scan_scratch_bytes(int64_t n) {
    return (size_t)(lvx_ceil_div(n > 0 ? n : 1, kScanTile) * 2 * sizeof(u64));
}

int lvx_voxel_scan(const uint32_t *vox_cnt_d, int64_t n_voxels, uint32_t *cursor_d,
                   uint32_t *offsets_d, uint8_t *counts_d, uint64_t *totals_d, void *scratch_d,
                   void *stream) {
    LVX_REQUIRE(vox_cnt_d && cursor_d && offsets_d && counts_d && totals_d && scratch_d &&
                    n_voxels > 0,
                "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const i64 tiles = lvx_ceil_div(n_voxels, kScanTile);
    u64 *partial = (u64 *)scratch_d;
    scan_tile_sums<u32, true><<<(unsigned)tiles, kScanThreads, 0, st>>>(vox_cnt_d, n_voxels, partial);
    LVX_LAUNCH_CHECK();
    scan_partials<<<1, 1024, 0, st>>>(partial, tiles, totals_d);
    LVX_LAUNCH_CHECK();
    scan_write<u32, true><<<(unsigned)tiles, kScanThreads, 0, st>>>(vox_cnt_d, n_voxels, partial,
                                                                   cursor_d, offsets_d, counts_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_scan_u16(const uint16_t *in_d, int64_t n, uint32_t *out_d, void *scratch_d, void *stream) {
    LVX_REQUIRE(in_d && out_d && scratch_d && n > 0, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const i64 tiles = lvx_ceil_div(n, kScanTile);
    u64 *partial = (u64 *)scratch_d;
    scan_tile_sums<u16, false><<<(unsigned)tiles, kScanThreads, 0, st>>>(in_d, n, partial);
    LVX_LAUNCH_CHECK();
    scan_partials<<<1, 1024, 0, st>>>(partial, tiles, nullptr);
    LVX_LAUNCH_CHECK();
    scan_write<u16, false><<<(unsigned)tiles, kScanThreads, 0, st>>>(in_d, n, partial, out_d,
                                                                    nullptr, nullptr);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_voxelize_compact(const lvx_raw_record *grouped_d, int64_t n_raw, const uint32_t *vox_cnt_d,
                         const uint32_t *cursor_end_d, const uint32_t *offsets_d,
                         const int32_t dims[3], int32_t n_bins, uint8_t *packed_d, float *seg_a_d,
                         float *seg_b_d, uint8_t *seg_attr_d, uint8_t *seg_lid_d,
                         int32_t *seg_voxel_d, uint8_t *seg_face_in_d, uint16_t *seg_bin_in_d,
                         uint8_t *seg_face_out_d, uint16_t *seg_bin_out_d, uint64_t *seg_key_d,
                         lvx_seg_record *seg_rec_d, void *stream) {
    if (int rc = check_dims(dims)) return rc;
    if (int rc = check_bins(n_bins)) return rc;
    LVX_REQUIRE(n_raw >= 0, "bad arguments");
    if (n_raw == 0) return LVX_OK;
    LVX_REQUIRE(grouped_d && vox_cnt_d && cursor_end_d && offsets_d && packed_d, "null input");
    LVX_REQUIRE(((uintptr_t)grouped_d & 31) == 0 && ((uintptr_t)seg_rec_d & 31) == 0,
                "grouped_d and seg_rec_d must be 32-byte aligned (256-bit accesses)");
    const int lb = ilog2i(n_bins);
    const int width = (2 * (3 + 2 * lb) + 8 + 5 + 7) / 8;  // record_width, voxelizer.py:70-76
    CompactOut o = {packed_d,      seg_a_d,        seg_b_d,      seg_attr_d, seg_lid_d, seg_voxel_d,
                    seg_face_in_d, seg_face_out_d, seg_bin_in_d, seg_bin_out_d, seg_key_d, seg_rec_d};
    compact_kernel<<<(unsigned)lvx_ceil_div(n_raw, 256), 256, 0, (cudaStream_t)stream>>>(
        grouped_d, n_raw, vox_cnt_d, cursor_end_d, offsets_d, dims[0], dims[1], n_bins, lb, width, o);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_raw_regroup(const uint64_t *in_key_d, const uint64_t *in_q_d, const uint32_t *in_lin_d,
                    int64_t n_slots, uint32_t *cursor_d, lvx_raw_record *grouped_d, void *stream) {
    LVX_REQUIRE(n_slots >= 0, "bad arguments");
    if (n_slots == 0) return LVX_OK;
    LVX_REQUIRE(in_key_d && in_q_d && in_lin_d && cursor_d && grouped_d, "null input");
    LVX_REQUIRE(((uintptr_t)grouped_d & 31) == 0, "grouped_d must be 32-byte aligned (256-bit stores)");
    regroup_kernel<<<(unsigned)lvx_ceil_div(n_slots, 256), 256, 0, (cudaStream_t)stream>>>(
        in_key_d, in_q_d, in_lin_d, n_slots, cursor_d, grouped_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_provenance(const uint64_t *seg_key_d, int64_t n_seg, const uint32_t *edge_base_d,
                   const int64_t *curve_off_d, int64_t n_curves, int32_t *seg_curve_d,
                   int32_t *seg_order_d, void *stream) {
    LVX_REQUIRE(n_seg >= 0 && n_curves >= 0, "bad arguments");
    if (n_seg == 0) return LVX_OK;
    LVX_REQUIRE(seg_key_d && edge_base_d && curve_off_d && seg_curve_d && seg_order_d, "null input");
    provenance_kernel<<<(unsigned)lvx_ceil_div(n_seg, 256), 256, 0, (cudaStream_t)stream>>>(
        seg_key_d, n_seg, edge_base_d, curve_off_d, n_curves, seg_curve_d, seg_order_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_build_seg_records(const float *seg_a_d, const float *seg_b_d, const uint8_t *seg_attr_d,
                          const uint8_t *seg_lid_d, int64_t n_seg, lvx_seg_record *seg_rec_d,
                          void *stream) {
    LVX_REQUIRE(n_seg >= 0, "bad arguments");
    if (n_seg == 0) return LVX_OK;
    LVX_REQUIRE(seg_a_d && seg_b_d && seg_attr_d && seg_lid_d && seg_rec_d, "null input");
    seg_records_kernel<<<(unsigned)lvx_ceil_div(n_seg, 256), 256, 0, (cudaStream_t)stream>>>(
        seg_a_d, seg_b_d, seg_attr_d, seg_lid_d, n_seg, seg_rec_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_voxelize_bound(const double *pts_d, const uint8_t *first_d, int64_t n_points,
                       uint64_t *total_d, void *stream) {
    LVX_REQUIRE(total_d && n_points >= 0, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    LVX_CUDA_CHECK(cudaMemsetAsync(total_d, 0, 8, st));
    if (n_points < 2) return LVX_OK;
    LVX_REQUIRE(pts_d && first_d, "null input");
    count_crossings_kernel<<<(unsigned)lvx_ceil_div(n_points, 256), 256, 0, st>>>(
        pts_d, first_d, n_points, reinterpret_cast<unsigned long long *>(total_d));
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_voxelize_clip(const double *pts_d, const double *attrs_d, const uint8_t *first_d,
                      int64_t n_points, const int32_t dims[3], int32_t n_bins, uint64_t capacity,
                      uint32_t *vox_cnt_d, uint64_t *raw_key_d, uint64_t *raw_q_d,
                      uint32_t *raw_lin_d, uint64_t *n_slots_d, uint16_t *edge_kept_d, int32_t *err_d,
                      void *stream) {
    if (int rc = check_dims(dims)) return rc;
    if (int rc = check_bins(n_bins)) return rc;
    LVX_REQUIRE(vox_cnt_d && n_slots_d && err_d && n_points >= 0, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    LVX_CUDA_CHECK(cudaMemsetAsync(n_slots_d, 0, 8, st));
    if (n_points < 2) {
        if (edge_kept_d && n_points > 0) LVX_CUDA_CHECK(cudaMemsetAsync(edge_kept_d, 0, (size_t)n_points * 2, st));
        return LVX_OK;
    }
    LVX_REQUIRE(pts_d && attrs_d && first_d && (capacity == 0 || (raw_key_d && raw_q_d && raw_lin_d)), "null input");
    LVX_REQUIRE(n_points < ((i64)1 << 47), "too many vertices");
    clip_once_kernel<<<(unsigned)lvx_ceil_div(n_points, kClipThreads), kClipThreads, 0, st>>>(
        pts_d, attrs_d, first_d, n_points, dims[0], dims[1], dims[2], n_bins, capacity, vox_cnt_d, raw_key_d,
        raw_q_d, raw_lin_d, reinterpret_cast<unsigned long long *>(n_slots_d), edge_kept_d, err_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_clip(const double *pts_d, const double *attrs_d, const uint8_t *first_d, int64_t n_points,
                   const int32_t dims[3], uint64_t capacity, int64_t *vox_d, double *p_in_d, double *p_out_d,
                   double *attr_d, uint64_t *key_d, uint64_t *n_d, void *stream) {
    if (int rc = check_dims(dims)) return rc;
    LVX_REQUIRE(n_d && n_points >= 0, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    LVX_CUDA_CHECK(cudaMemsetAsync(n_d, 0, 8, st));
    if (n_points < 2) return LVX_OK;
    LVX_REQUIRE(pts_d && attrs_d && first_d && (capacity == 0 || (vox_d && p_in_d && p_out_d && attr_d && key_d)),
                "null input");
    probe_clip_kernel<<<(unsigned)lvx_ceil_div(n_points, 128), 128, 0, st>>>(
        pts_d, attrs_d, first_d, n_points, dims[0], dims[1], dims[2], capacity, vox_d, p_in_d, p_out_d, attr_d, key_d,
        reinterpret_cast<unsigned long long *>(n_d));
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_decode_packed(const uint8_t *packed_d, const uint8_t *counts_d, const uint32_t *offsets_d,
                      const int32_t dims[3], int32_t n_bins, float *seg_a_d, float *seg_b_d,
                      uint8_t *seg_attr_d, uint8_t *seg_lid_d, int32_t *seg_voxel_d,
                      uint8_t *seg_face_in_d, uint16_t *seg_bin_in_d, uint8_t *seg_face_out_d,
                      uint16_t *seg_bin_out_d, lvx_seg_record *seg_rec_d, int32_t *err_d, void *stream) {
    if (int rc = check_dims(dims)) return rc;
    if (int rc = check_bins(n_bins)) return rc;
    LVX_REQUIRE(packed_d && counts_d && offsets_d && err_d, "null input");
    LVX_REQUIRE(((uintptr_t)seg_rec_d & 31) == 0, "seg_rec_d must be 32-byte aligned (256-bit stores)");
    const i64 V = (i64)dims[0] * dims[1] * dims[2];
    const int lb = ilog2i(n_bins);
    const int width = (2 * (3 + 2 * lb) + 8 + 5 + 7) / 8;  // record_width, voxelizer.py:70-76
    CompactOut o = {nullptr,       seg_a_d,        seg_b_d,      seg_attr_d,    seg_lid_d, seg_voxel_d,
                    seg_face_in_d, seg_face_out_d, seg_bin_in_d, seg_bin_out_d, nullptr,   seg_rec_d};
    decode_packed_kernel<<<(unsigned)lvx_ceil_div(V, 128), 128, 0, (cudaStream_t)stream>>>(
        packed_d, counts_d, offsets_d, V, dims[0], dims[1], n_bins, lb, width, o, err_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
