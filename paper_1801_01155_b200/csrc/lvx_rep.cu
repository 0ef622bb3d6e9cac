// Representative lines for sm_100a: one averaged line per coarse voxel and level
// (the "direction" mip of the LoD), the adjacency snap, and the shadow probe.
//
//   _snap_to_face_bin / representative_line   lod.py:122-169
//   _adjacency_snap                           lod.py:176-221
//   build_rep_lines                           lod.py:224-284
//   replines_ray_blocked                      _kernels.py:498-538 (lvx_geom.cuh)
//
// The reference builds a level with Python loops over the occupied parents; nothing in it
// couples two parents, so a level is one thread per parent voxel here.  Inside a parent the
// members are visited in the reference's order (stable sort by parent index = children in
// z,y,x order, each child's segments in stored order): the flip rule (:158-160) and the
// float64 sums depend on it.  The weight is numpy's PAIRWISE float64 sum of the member
// weights (np.add.reduce), restated below.  The adjacency snap touches disjoint endpoints
// for different voxel pairs of one axis pass, so each pass is one thread per lower voxel;
// the three axes run one after the other like in the reference.
#include <math_constants.h>

#include "lvx_geom.cuh"

namespace {

__device__ __forceinline__ double bin_centre(double u, int n) {
    // quantize_point_on_face, voxelizer.py:161-165
    long long b = (long long)floor(u * (double)n);
    b = b < 0 ? 0 : (b > n - 1 ? n - 1 : b);
    return ((double)b + 0.5) / (double)n;
}

// _snap_to_face_bin, lod.py:122-138
__device__ void snap_to_face_bin(const double p[3], int n, double out[3]) {
    double best = 0.0;
    bool have = false;
#pragma unroll
    for (int face = 0; face < 6; ++face) {
        const int axis = face >> 1;
        const int ua = axis == 0 ? 1 : 0, va = axis == 2 ? 1 : 2;  // _FACE_UV, lod.py:24
        double u = p[ua] < 0.0 ? 0.0 : p[ua];
        u = u > 1.0 ? 1.0 : u;
        double v = p[va] < 0.0 ? 0.0 : p[va];
        v = v > 1.0 ? 1.0 : v;
        double cand[3];
        cand[axis] = (double)(face & 1);
        cand[ua] = bin_centre(u, n);
        cand[va] = bin_centre(v, n);
        const double e0 = cand[0] - p[0], e1 = cand[1] - p[1], e2 = cand[2] - p[2];
        const double d = e0 * e0 + e1 * e1 + e2 * e2;
        if (!have || d < best - 1e-15) {
            have = true;
            best = d;
            out[0] = cand[0];
            out[1] = cand[1];
            out[2] = cand[2];
        }
    }
}

// The members of one parent voxel: up to 8 children, each a run of consecutive entries.
struct Members {
    int n_child;
    i64 base[8];
    int cnt[8];
    int total;
    // level 1: runs of segment records; level >= 2: single representatives of the level below
    const lvx_seg_record *rec;
    const float *ca, *cb, *cw;

    __device__ __forceinline__ void locate(int i, i64 &idx) const {
        int c = 0;
        while (i >= cnt[c]) {
            i -= cnt[c];
            ++c;
        }
        idx = base[c] + i;
    }
    __device__ __forceinline__ void endpoints(i64 idx, double a[3], double b[3]) const {
        if (rec) {
            const float4 ra = __ldg(reinterpret_cast<const float4 *>(rec + idx));
            const float4 rb = __ldg(reinterpret_cast<const float4 *>(rec + idx) + 1);
            a[0] = (double)ra.x;
            a[1] = (double)ra.y;
            a[2] = (double)ra.z;
            b[0] = (double)rb.x;
            b[1] = (double)rb.y;
            b[2] = (double)rb.z;
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                a[c] = (double)ca[3 * idx + c];
                b[c] = (double)cb[3 * idx + c];
            }
        }
    }
    __device__ __forceinline__ double weight(int i) const {
        i64 idx;
        locate(i, idx);
        if (rec) {
            // np.linalg.norm(cur_b - cur_a, axis=1), lod.py:239
            double a[3], b[3];
            endpoints(idx, a, b);
            const double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
            return sqrt((d0 * d0 + d1 * d1) + d2 * d2);
        }
        return (double)cw[idx];
    }
};

// numpy's pairwise float64 summation (np.add.reduce over a contiguous vector)
__device__ double pairwise_sum(const Members &M, int start, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res += M.weight(start + i);
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = M.weight(start + j);
        int i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] += M.weight(start + i + j);
        }
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += M.weight(start + i);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(M, start, n2) + pairwise_sum(M, start + n2, n - n2);
}

// One thread per parent voxel of level `level` (size = 2^level grid units).
__global__ void __launch_bounds__(128)
rep_level_kernel(int cdx, int cdy, int cdz,  // child grid (level - 1)
                 const u8 *__restrict__ c_counts, const u32 *__restrict__ c_offsets,
                 const lvx_seg_record *__restrict__ rec,                                     // level 1
                 const u8 *__restrict__ c_valid, const float *__restrict__ c_a,
                 const float *__restrict__ c_b, const float *__restrict__ c_w,              // level >= 2
                 int pdx, int pdy, int pdz, double size, int n_bins, u8 *__restrict__ valid,
                 float *__restrict__ rep_a, float *__restrict__ rep_b, float *__restrict__ rep_w) {
    const i64 lin = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (lin >= (i64)pdx * pdy * pdz) return;
    const int px = (int)(lin % pdx), py = (int)((lin / pdx) % pdy), pz = (int)(lin / ((i64)pdx * pdy));
    Members M;
    M.n_child = 0;
    M.total = 0;
    M.rec = rec;
    M.ca = c_a;
    M.cb = c_b;
    M.cw = c_w;
    // children in ascending child index: z, y, x
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const int x = 2 * px + dx, y = 2 * py + dy, z = 2 * pz + dz;
                if (x >= cdx || y >= cdy || z >= cdz) continue;
                const i64 cl = x + (i64)cdx * (y + (i64)cdy * z);
                int n;
                i64 b;
                if (rec) {
                    n = c_counts[cl];
                    b = c_offsets[cl];
                } else {
                    n = c_valid[cl] ? 1 : 0;
                    b = cl;
                }
                if (n == 0) continue;
                M.base[M.n_child] = b;
                M.cnt[M.n_child] = n;
                M.n_child += 1;
                M.total += n;
            }
    for (int c = M.n_child; c < 8; ++c) {
        M.base[c] = 0;
        M.cnt[c] = 0x7FFFFFFF;  // (never walked past)
    }
    if (M.total == 0) {
        valid[lin] = 0;
        rep_w[lin] = 0.0f;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            rep_a[3 * lin + c] = 0.0f;
            rep_b[3 * lin + c] = 0.0f;
        }
        return;
    }
    // representative_line, lod.py:141-169
    double sa[3] = {0.0, 0.0, 0.0}, sb[3] = {0.0, 0.0, 0.0};
    bool first = true;
    for (int c = 0; c < M.n_child; ++c) {
        for (int k = 0; k < M.cnt[c]; ++k) {
            double a[3], b[3];
            M.endpoints(M.base[c] + k, a, b);
            bool flip = false;
            if (!first) {
                const double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
                const double e0 = sb[0] - sa[0], e1 = sb[1] - sa[1], e2 = sb[2] - sa[2];
                flip = d0 * e0 + d1 * e1 + d2 * e2 < 0.0;
            }
            first = false;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                sa[q] += flip ? b[q] : a[q];
                sb[q] += flip ? a[q] : b[q];
            }
        }
    }
    const double origin[3] = {(double)px * size, (double)py * size, (double)pz * size};
    double la[3], lb[3], qa[3], qb[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        la[q] = (sa[q] / (double)M.total - origin[q]) / size;
        lb[q] = (sb[q] / (double)M.total - origin[q]) / size;
    }
    snap_to_face_bin(la, n_bins, qa);
    snap_to_face_bin(lb, n_bins, qb);
    valid[lin] = 1;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        rep_a[3 * lin + q] = (float)(qa[q] * size + origin[q]);
        rep_b[3 * lin + q] = (float)(qb[q] * size + origin[q]);
    }
    rep_w[lin] = (float)pairwise_sum(M, 0, M.total);
}

// One axis pass of _adjacency_snap (lod.py:176-221): one thread per lower voxel of a pair.
__global__ void __launch_bounds__(128)
rep_adjacency_kernel(int dx, int dy, int dz, int axis, double size, int n_bins, const u8 *__restrict__ valid,
                     float *__restrict__ rep_a, float *__restrict__ rep_b) {
    const i64 lin = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (lin >= (i64)dx * dy * dz || !valid[lin]) return;
    const i64 step = axis == 0 ? 1 : (axis == 1 ? dx : (i64)dx * dy);
    const int n_axis = axis == 0 ? dx : (axis == 1 ? dy : dz);
    const int cx = (int)(lin % dx), cy = (int)((lin / dx) % dy), cz = (int)(lin / ((i64)dx * dy));
    const int coord = axis == 0 ? cx : (axis == 1 ? cy : cz);
    if (coord + 1 >= n_axis) return;
    const i64 nb = lin + step;
    if (!valid[nb]) return;
    // endpoints_on: the first of (a, b) that lies on the shared face, per voxel
    float *mine = nullptr, *theirs = nullptr;
    const double base_lo = (double)coord * size, base_hi = (double)(coord + 1) * size;
    for (int which = 0; which < 2; ++which) {
        float *arr = which == 0 ? rep_a : rep_b;
        if (!mine && fabs(((double)arr[3 * lin + axis] - base_lo) / size - 1.0) <= 1e-9) mine = arr;
        if (!theirs && fabs(((double)arr[3 * nb + axis] - base_hi) / size - 0.0) <= 1e-9) theirs = arr;
    }
    if (!mine || !theirs) return;
    const double base[3] = {(double)cx * size, (double)cy * size, (double)cz * size};
    double avg[3], local[3], snapped[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        avg[c] = 0.5 * ((double)mine[3 * lin + c] + (double)theirs[3 * nb + c]);
        local[c] = (avg[c] - base[c]) / size;
        snapped[c] = avg[c];
    }
    const int ua = axis == 0 ? 1 : 0, va = axis == 2 ? 1 : 2;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        if (c == axis) snapped[c] = base[c] + size;
        else if (c == ua) snapped[c] = base[c] + bin_centre(local[c], n_bins) * size;
        else if (c == va) snapped[c] = base[c] + bin_centre(local[c], n_bins) * size;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        mine[3 * lin + c] = (float)snapped[c];
        theirs[3 * nb + c] = (float)snapped[c];
    }
}

__global__ void __launch_bounds__(64)
probe_replines_kernel(LvxRepLevel rep, const double *__restrict__ rays, const double *__restrict__ max_t,
                      double radius_base, i64 n, int32_t *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *r = rays + 6 * i;
    out[i] = lvx_replines_blocked(r[0], r[1], r[2], r[3], r[4], r[5], max_t[i], rep, radius_base) ? 1 : 0;
}

// numpy's pairwise float64 sum over a plain vector (np.sum of the member lengths, lod.py:168)
__device__ double pairwise_sum_vec(const double *w, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res += w[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = w[j];
        int i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] += w[i + j];
        }
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += w[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum_vec(w, n2) + pairwise_sum_vec(w + n2, n - n2);
}

// representative_line (lod.py:141-169) for one explicit member list: the same flip rule, sums
// and face-bin snap the level kernel applies per parent voxel.  One thread; `len_d` is scratch.
__global__ void probe_rep_line_kernel(const double *__restrict__ starts, const double *__restrict__ ends, int m,
                                      double ox, double oy, double oz, double size, int n_bins,
                                      double *__restrict__ len_d, double *__restrict__ out) {
    double sa[3] = {0.0, 0.0, 0.0}, sb[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < m; ++i) {
        const double *a = starts + 3 * i, *b = ends + 3 * i;
        bool flip = false;
        if (i > 0) {
            const double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
            const double e0 = sb[0] - sa[0], e1 = sb[1] - sa[1], e2 = sb[2] - sa[2];
            flip = d0 * e0 + d1 * e1 + d2 * e2 < 0.0;
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            sa[q] += flip ? b[q] : a[q];
            sb[q] += flip ? a[q] : b[q];
        }
        const double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
        len_d[i] = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    }
    const double origin[3] = {ox, oy, oz};
    double la[3], lb[3], qa[3], qb[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        la[q] = (sa[q] / (double)m - origin[q]) / size;
        lb[q] = (sb[q] / (double)m - origin[q]) / size;
    }
    snap_to_face_bin(la, n_bins, qa);
    snap_to_face_bin(lb, n_bins, qb);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        out[q] = qa[q] * size + origin[q];
        out[3 + q] = qb[q] * size + origin[q];
    }
    out[6] = pairwise_sum_vec(len_d, m);
}

}  // namespace

extern "C" {

int lvx_probe_rep_line(const double *starts_d, const double *ends_d, int64_t m, const double origin[3],
                       double size, int32_t n_bins, double *scratch_d, double *out_d, void *stream) {
    LVX_REQUIRE(starts_d && ends_d && origin && scratch_d && out_d && m >= 1 && m < ((int64_t)1 << 30), "bad arguments");
    LVX_REQUIRE(size > 0.0, "size must be positive");
    LVX_REQUIRE(n_bins >= 2 && n_bins <= 256 && (n_bins & (n_bins - 1)) == 0, "bad bin resolution %d", n_bins);
    probe_rep_line_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(starts_d, ends_d, (int)m, origin[0], origin[1], origin[2],
                                                            size, n_bins, scratch_d, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_rep_level(const int32_t child_dims[3], const uint8_t *c_counts_d, const uint32_t *c_offsets_d,
                  const lvx_seg_record *seg_rec_d, const uint8_t *c_valid_d, const float *c_a_d,
                  const float *c_b_d, const float *c_w_d, int32_t level, int32_t n_bins, int32_t adjacency,
                  uint8_t *valid_d, float *rep_a_d, float *rep_b_d, float *rep_w_d, void *stream) {
    LVX_REQUIRE(child_dims && child_dims[0] >= 1 && child_dims[1] >= 1 && child_dims[2] >= 1, "bad child dims");
    LVX_REQUIRE(level >= 1 && level < 31, "level must be >= 1");
    LVX_REQUIRE(n_bins >= 2 && n_bins <= 256 && (n_bins & (n_bins - 1)) == 0, "bad bin resolution %d", n_bins);
    LVX_REQUIRE(valid_d && rep_a_d && rep_b_d && rep_w_d, "null output");
    const bool from_segments = seg_rec_d != nullptr;
    LVX_REQUIRE(from_segments ? (c_counts_d && c_offsets_d) : (c_valid_d && c_a_d && c_b_d && c_w_d),
                "level 1 needs counts/offsets/records, higher levels the level below");
    const int pdx = (child_dims[0] + 1) / 2, pdy = (child_dims[1] + 1) / 2, pdz = (child_dims[2] + 1) / 2;
    const i64 V = (i64)pdx * pdy * pdz;
    const double size = (double)((i64)1 << level);
    cudaStream_t st = (cudaStream_t)stream;
    rep_level_kernel<<<(unsigned)lvx_ceil_div(V, 128), 128, 0, st>>>(
        child_dims[0], child_dims[1], child_dims[2], c_counts_d, c_offsets_d, seg_rec_d, c_valid_d, c_a_d, c_b_d,
        c_w_d, pdx, pdy, pdz, size, n_bins, valid_d, rep_a_d, rep_b_d, rep_w_d);
    LVX_LAUNCH_CHECK();
    if (adjacency) {
        for (int axis = 0; axis < 3; ++axis) {
            rep_adjacency_kernel<<<(unsigned)lvx_ceil_div(V, 128), 128, 0, st>>>(pdx, pdy, pdz, axis, size, n_bins,
                                                                                 valid_d, rep_a_d, rep_b_d);
            LVX_LAUNCH_CHECK();
        }
    }
    return LVX_OK;
}

int lvx_probe_replines(const lvx_replines *rep, const double *rays_d, const double *max_t_d,
                       double radius_base, int64_t n, int32_t *out_d, void *stream) {
    LVX_REQUIRE(rep && rep->valid_d && rep->a_d && rep->b_d && rep->w_d && rep->dims[0] >= 1 &&
                    rep->dims[1] >= 1 && rep->dims[2] >= 1 && rep->size >= 1.0,
                "bad representative-line level");
    LVX_REQUIRE(n >= 0 && radius_base > 0.0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(rays_d && max_t_d && out_d, "null argument");
    LvxRepLevel R = {rep->valid_d, rep->a_d, rep->b_d, rep->w_d, rep->dims[0], rep->dims[1], rep->dims[2], rep->size};
    probe_replines_kernel<<<(unsigned)lvx_ceil_div(n, 64), 64, 0, (cudaStream_t)stream>>>(R, rays_d, max_t_d,
                                                                                        radius_base, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
