// LoD construction for sm_100a: level-0 density, 2x2x2 mip chain, dilated
// occupancy map.
//
//   compute_density_level0   lod.py:82-94
//   _coarsen / build_octree  lod.py:97-119
//   _occupancy_dilated       raycast.py:351-366
#include <math_constants.h>

#include <cstdlib>

#include "lvx_geom.cuh"

namespace {

// Level-0 density.  np.bincount with weights is a sequential float64 accumulation of the
// per-segment products length * sigma in stored order, one cast to float32 (lod.py:87-94).
//
// A warp owns 64 consecutive voxels per round (two per lane, interleaved so that the header loads
// coalesce).  Their records are one contiguous span of the record array
// (headers are exclusive prefix sums in voxel scan order), so the lanes load the span together --
// one 32-byte record per lane and round, every sector used once, all loads independent -- and
// leave the float64 products in shared memory; each lane then adds up the products of ITS voxel in
// stored order.  The span is worked through in chunks of kDlChunk records, so the accumulation
// order per voxel is the stored order whatever the group sizes.  A model whose offsets are not
// prefix sums (nothing in the reference produces one) takes the per-thread loop.
constexpr int kDlThreads = 256;
constexpr int kDlChunk = 256;  // records per warp and round

__device__ __forceinline__ double density_weight(const float4 a, const float4 b, const float *s_sigma) {
    // endpoints are widened BEFORE the subtraction (lod.py:87-89)
    const double ex = (double)b.x - (double)a.x;
    const double ey = (double)b.y - (double)a.y;
    const double ez = (double)b.z - (double)a.z;
    const double len = sqrt(ex * ex + ey * ey + ez * ez);
    return len * (double)s_sigma[__float_as_uint(a.w) & 0xFFu];
}

#ifndef LVX_DL_CAP
#define LVX_DL_CAP 64
#endif
#ifndef LVX_DL_U1
#define LVX_DL_U1 1
#endif
#ifndef LVX_DL_VOX
#define LVX_DL_VOX 2
#endif
constexpr int kDlVox = LVX_DL_VOX;  // voxels per lane and round

// One encoded record's product.  Used only while every global coordinate (voxel + bin centre) is exact
// in float32 -- then b - a in float64 is the difference of the voxel-local bin centres, whichever voxel
// the record sits in, and the voxel need not be known here.
__device__ __forceinline__ double density_weight_packed(const LvxPacked &P, size_t s, const float *s_sigma) {
    const LvxPackedFields f = lvx_packed_fields(P, lvx_packed_word(P, s));
    float a[3], b[3];
    lvx_packed_point(f.face_in, f.bin_in, P, 0, 0, 0, a);
    lvx_packed_point(f.face_out, f.bin_out, P, 0, 0, 0, b);
    const double ex = (double)b[0] - (double)a[0], ey = (double)b[1] - (double)a[1], ez = (double)b[2] - (double)a[2];
    return sqrt(ex * ex + ey * ey + ez * ez) * (double)s_sigma[f.attr];
}

template <typename CountT, bool PACKED>
__global__ void __launch_bounds__(kDlThreads)
density_l0_kernel(const CountT *__restrict__ counts, const u32 *__restrict__ offsets,
                  const lvx_seg_record *__restrict__ rec, const LvxPacked P, const float *__restrict__ table,
                  i64 n_voxels, float *__restrict__ out) {
    constexpr unsigned FULL = 0xFFFFFFFFu;
    __shared__ float s_sigma[256];
    __shared__ double s_w[kDlThreads / 32][kDlChunk];
    s_sigma[threadIdx.x] = table[4 * threadIdx.x + 3];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 n_warps = ((i64)gridDim.x * blockDim.x) >> 5;
    constexpr int per_round = 32 * kDlVox;
    const bool aligned32 = (reinterpret_cast<uintptr_t>(rec) & 31) == 0;
    for (i64 w = (((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5); w * per_round < n_voxels; w += n_warps) {
        // lane owns voxels vbase + k * 32 + lane, k = 0 .. kDlVox - 1 (every load below is coalesced)
        const i64 vbase = w * per_round;
        const CountT *c = counts + vbase;
        const u32 *o = offsets + vbase;
        float *dst = out + vbase;
        const int nv = (int)(n_voxels - vbase < per_round ? n_voxels - vbase : per_round);
        u32 n[kDlVox], off[kDlVox], first[kDlVox];
        unsigned any = 0;
        // counts AND offsets in one round trip (the offsets of empty voxels are part of the prefix
        // sums and are used below); the headers of the warp's next round are requested now
#pragma unroll
        for (int k = 0; k < kDlVox; ++k) {
            const int i = 32 * k + lane;
            n[k] = i < nv ? (u32)c[i] : 0u;
            off[k] = i < nv ? o[i] : 0u;
            any |= n[k];
        }
        if (vbase + n_warps * per_round + per_round <= n_voxels) {
            const size_t ahead = (size_t)(n_warps * per_round);
            if (lane < 4 * kDlVox) asm volatile("prefetch.global.L2 [%0];" ::"l"(o + ahead + 8 * lane));
            if (lane == 31) asm volatile("prefetch.global.L2 [%0];" ::"l"(c + ahead));
        }
        if (!__any_sync(FULL, any != 0)) {
#pragma unroll
            for (int k = 0; k < kDlVox; ++k)
                if (32 * k + lane < nv) dst[32 * k + lane] = 0.0f;
            continue;
        }
        // The headers of a whole round are exclusive prefix sums exactly when every voxel's offset is
        // its predecessor's offset + count: one shuffle per voxel checks that, and then the span, each
        // voxel's place in it and its length follow from the offsets alone (no scan).
        bool chain = nv == per_round;
#pragma unroll
        for (int k = 0; k < kDlVox; ++k) {
            u32 next = __shfl_down_sync(FULL, off[k], 1);
            if (k + 1 < kDlVox) {
                const u32 wrap = __shfl_sync(FULL, off[k + 1], 0);
                if (lane == 31) next = wrap;
            }
            if (k + 1 < kDlVox || lane < 31) chain = chain && next == off[k] + n[k];
        }
        const bool contiguous = __all_sync(FULL, chain);
        const u32 base = __shfl_sync(FULL, off[0], 0);
        const u32 total = __shfl_sync(FULL, off[kDlVox - 1] + n[kDlVox - 1], 31) - base;
#pragma unroll
        for (int k = 0; k < kDlVox; ++k) first[k] = off[k] - base;
        double acc[kDlVox];
#pragma unroll
        for (int k = 0; k < kDlVox; ++k) acc[k] = 0.0;
        if (contiguous) {
            const float4 *r = reinterpret_cast<const float4 *>(rec + base);
            for (u32 j0 = 0; j0 < total; j0 += kDlChunk) {
                const u32 m = min((u32)kDlChunk, total - j0);
                for (u32 j = lane; j < m; j += 32) {
                    if constexpr (PACKED) {
                        s_w[warp][j] = density_weight_packed(P, (size_t)base + j0 + j, s_sigma);
                        continue;
                    }
                    float4 a, b;
                    if (aligned32) {
                        // one 256-bit load per record: every sector of the span is requested once
                        u64 q0, q1, q2, q3;
                        lvx_ld256(r + 2 * (size_t)(j0 + j), q0, q1, q2, q3);
                        a = make_float4(__uint_as_float((u32)q0), __uint_as_float((u32)(q0 >> 32)), __uint_as_float((u32)q1),
                                        __uint_as_float((u32)(q1 >> 32)));
                        b = make_float4(__uint_as_float((u32)q2), __uint_as_float((u32)(q2 >> 32)), __uint_as_float((u32)q3),
                                        __uint_as_float((u32)(q3 >> 32)));
                    } else {
                        a = __ldg(r + 2 * (size_t)(j0 + j));
                        b = __ldg(r + 2 * (size_t)(j0 + j) + 1);
                    }
                    s_w[warp][j] = density_weight(a, b, s_sigma);
                }
                __syncwarp();
                if (total <= (u32)kDlChunk) {  // the whole span is in shared memory (the usual round)
#pragma unroll
                    for (int k = 0; k < kDlVox; ++k) {
                        const double *p = &s_w[warp][first[k]];
#if LVX_DL_U1
#pragma unroll 1
#endif
                        for (u32 q = 0; q < n[k]; ++q) acc[k] += p[q];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < kDlVox; ++k) {
                        const u32 lo = max(first[k], j0), hi = min(first[k] + n[k], j0 + m);
                        for (u32 q = lo; q < hi; ++q) acc[k] += s_w[warp][q - j0];
                    }
                }
                __syncwarp();
            }
        } else {
#pragma unroll
            for (int k = 0; k < kDlVox; ++k) {
                if constexpr (PACKED) {
                    for (u32 q = 0; q < n[k]; ++q) acc[k] += density_weight_packed(P, (size_t)off[k] + q, s_sigma);
                } else {
                    const float4 *r = reinterpret_cast<const float4 *>(rec + off[k]);
                    for (u32 q = 0; q < n[k]; ++q)
                        acc[k] += density_weight(__ldg(r + 2 * q), __ldg(r + 2 * q + 1), s_sigma);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kDlVox; ++k)
            if (32 * k + lane < nv) dst[32 * k + lane] = (float)acc[k];
    }
}

// The same sums from the ENCODED records (5 bytes per segment at N = 32 instead of the 32-byte render
// record: 2.3x less traffic for the whole kernel at C3).  A lane adds up the records of its own voxels
// in stored order; neighbouring lanes own neighbouring voxels, whose records are neighbours in memory,
// so the 8-byte loads of a warp fall into a handful of sectors.  The endpoints are reconstructed exactly
// as the voxelizer does (bin centre + voxel in float64, cast to float32), so the products are bit-identical.
__global__ void __launch_bounds__(kDlThreads)
density_l0_packed_kernel(const u8 *__restrict__ counts, const u32 *__restrict__ offsets, const LvxPacked P,
                         const float *__restrict__ table, int rx, int ry, i64 n_voxels, float *__restrict__ out) {
    __shared__ float s_sigma[256];
    s_sigma[threadIdx.x] = table[4 * threadIdx.x + 3];
    __syncthreads();
    const i64 stride = (i64)gridDim.x * blockDim.x;
    for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < n_voxels; v += stride) {
        const u32 n = counts[v];
        double acc = 0.0;
        if (n) {
            const u32 base = offsets[v];
            const int vx = (int)(v % rx), vy = (int)((v / rx) % ry), vz = (int)(v / ((i64)rx * ry));
            for (u32 q = 0; q < n; ++q) {
                const LvxPackedFields f = lvx_packed_fields(P, lvx_packed_word(P, base + q));
                float a[3], b[3];
                lvx_packed_point(f.face_in, f.bin_in, P, vx, vy, vz, a);
                lvx_packed_point(f.face_out, f.bin_out, P, vx, vy, vz, b);
                // endpoints are widened BEFORE the subtraction (lod.py:87-89)
                const double ex = (double)b[0] - (double)a[0], ey = (double)b[1] - (double)a[1],
                             ez = (double)b[2] - (double)a[2];
                acc += sqrt(ex * ex + ey * ey + ez * ez) * (double)s_sigma[f.attr];
            }
        }
        out[v] = (float)acc;
    }
}

// Mip chain (lod.py:97-110): a parent is the float32 sum of its (up to) eight existing children in
// the fixed (oz, oy, ox) order divided by the float32 child count.
//
// mip3_kernel: a block owns an 8x8x8 brick of level l+1; it stages the 16x16x16 child brick of level
// l with coalesced row loads and reduces it three times in shared memory, writing its 8^3 / 4^3 /
// 2^3 share of levels l+1, l+2, l+3 (as many of them as exist).  One pass over level l, no re-read of
// the levels in between.
#ifndef LVX_MIP_DIRECT
#define LVX_MIP_DIRECT 1
#endif
constexpr int kMipP = 8;             // brick edge at the first output level
constexpr int kMipC = 2 * kMipP;     // child brick edge

struct MipDims {
    int x, y, z;
};

__device__ __forceinline__ float mip_reduce(const float *s, int pitch_y, int pitch_z, int tx, int ty, int tz, int gx,
                                            int gy, int gz, MipDims child) {
    // children (2g + o) that exist at the child level, (oz, oy, ox) order, float32
    float acc = 0.0f, cnt = 0.0f;
#pragma unroll
    for (int oz = 0; oz < 2; ++oz)
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) {
                if (2 * gz + oz < child.z && 2 * gy + oy < child.y && 2 * gx + ox < child.x) {
                    acc = acc + s[(2 * tz + oz) * pitch_z + (2 * ty + oy) * pitch_y + (2 * tx + ox)];
                    cnt = cnt + 1.0f;
                }
            }
    return acc / cnt;
}

__global__ void __launch_bounds__(kMipP *kMipP *kMipP)
mip3_kernel(const float *__restrict__ src, MipDims d0, float *__restrict__ dst1, MipDims d1,
            float *__restrict__ dst2, MipDims d2, float *__restrict__ dst3, MipDims d3, int n_out, bool vec4) {
    __shared__ float s0[kMipC * kMipC * (kMipC + 1)];
    __shared__ float s1[kMipP * kMipP * (kMipP + 1)];
    __shared__ float s2[4 * 4 * 5];
    const int bx = blockIdx.x * kMipP, by = blockIdx.y * kMipP, bz = blockIdx.z * kMipP;
#if LVX_MIP_DIRECT
    // The first level straight from global memory: a thread's eight children are four aligned pairs
    // (x, x+1) -- four 8-byte loads in flight at once, added in the reference's (oz, oy, ox) order in
    // registers; no staging of the 16^3 child brick, no barrier before the first output.  (The staged
    // path ran at a third of the HBM peak on its instruction count: index arithmetic, four scalar
    // shared-memory stores per 16-byte load, eight shared-memory loads per parent.)
    if (vec4) {  // (rows of an even length, 16-byte aligned base: every pair is 8-byte aligned and in range together)
        const int tx = threadIdx.x % kMipP, ty = (threadIdx.x / kMipP) % kMipP, tz = threadIdx.x / (kMipP * kMipP);
        const int x = bx + tx, y = by + ty, z = bz + tz;
        float v = 0.0f;
        if (x < d1.x && y < d1.y && z < d1.z) {
            float2 c[2][2];
            bool in[2][2];
#pragma unroll
            for (int oz = 0; oz < 2; ++oz)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy) {
                    in[oz][oy] = 2 * z + oz < d0.z && 2 * y + oy < d0.y;
                    c[oz][oy] = make_float2(0.0f, 0.0f);
                    if (in[oz][oy])
                        c[oz][oy] = __ldg(reinterpret_cast<const float2 *>(
                            src + ((i64)(2 * z + oz) * d0.y + (2 * y + oy)) * d0.x + 2 * x));
                }
            float acc = 0.0f, cnt = 0.0f;
#pragma unroll
            for (int oz = 0; oz < 2; ++oz)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy) {
                    if (in[oz][oy]) {  // (d0.x is even here: both x children exist)
                        acc = acc + c[oz][oy].x;
                        cnt = cnt + 1.0f;
                        acc = acc + c[oz][oy].y;
                        cnt = cnt + 1.0f;
                    }
                }
            v = acc / cnt;
            dst1[((i64)z * d1.y + y) * d1.x + x] = v;
        }
        s1[(tz * kMipP + ty) * (kMipP + 1) + tx] = v;
    } else {
#endif
    if (vec4 && 2 * bx + kMipC <= d0.x) {
        // rows of the child brick as four 16-byte loads (the row starts are 64-byte aligned here)
        for (int idx = threadIdx.x; idx < kMipC * kMipC * kMipC / 4; idx += blockDim.x) {
            const int q = idx % (kMipC / 4), ly = (idx / (kMipC / 4)) % kMipC, lz = idx / (kMipC * kMipC / 4);
            const int gy = 2 * by + ly, gz = 2 * bz + lz;
            float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (gy < d0.y && gz < d0.z)
                v = __ldg(reinterpret_cast<const float4 *>(src + ((i64)gz * d0.y + gy) * d0.x + 2 * bx) + q);
            float *row = &s0[(lz * kMipC + ly) * (kMipC + 1) + 4 * q];
            row[0] = v.x;
            row[1] = v.y;
            row[2] = v.z;
            row[3] = v.w;
        }
    } else
    for (int idx = threadIdx.x; idx < kMipC * kMipC * kMipC; idx += blockDim.x) {
        const int lx = idx % kMipC, ly = (idx / kMipC) % kMipC, lz = idx / (kMipC * kMipC);
        const int gx = 2 * bx + lx, gy = 2 * by + ly, gz = 2 * bz + lz;
        float v = 0.0f;
        if (gx < d0.x && gy < d0.y && gz < d0.z) v = src[((i64)gz * d0.y + gy) * d0.x + gx];
        s0[(lz * kMipC + ly) * (kMipC + 1) + lx] = v;
    }
    __syncthreads();
    {
        const int tx = threadIdx.x % kMipP, ty = (threadIdx.x / kMipP) % kMipP, tz = threadIdx.x / (kMipP * kMipP);
        const int x = bx + tx, y = by + ty, z = bz + tz;
        float v = 0.0f;
        if (x < d1.x && y < d1.y && z < d1.z) {
            v = mip_reduce(s0, kMipC + 1, kMipC * (kMipC + 1), tx, ty, tz, x, y, z, d0);
            dst1[((i64)z * d1.y + y) * d1.x + x] = v;
        }
        s1[(tz * kMipP + ty) * (kMipP + 1) + tx] = v;
    }
#if LVX_MIP_DIRECT
    }
#endif
    if (n_out < 2) return;
    __syncthreads();
    if (threadIdx.x < 64) {
        const int tx = threadIdx.x % 4, ty = (threadIdx.x / 4) % 4, tz = threadIdx.x / 16;
        const int x = bx / 2 + tx, y = by / 2 + ty, z = bz / 2 + tz;
        float v = 0.0f;
        if (x < d2.x && y < d2.y && z < d2.z) {
            v = mip_reduce(s1, kMipP + 1, kMipP * (kMipP + 1), tx, ty, tz, x, y, z, d1);
            dst2[((i64)z * d2.y + y) * d2.x + x] = v;
        }
        s2[(tz * 4 + ty) * 5 + tx] = v;
    }
    if (n_out < 3) return;
    __syncthreads();
    if (threadIdx.x < 8) {
        const int tx = threadIdx.x % 2, ty = (threadIdx.x / 2) % 2, tz = threadIdx.x / 4;
        const int x = bx / 4 + tx, y = by / 4 + ty, z = bz / 4 + tz;
        if (x < d3.x && y < d3.y && z < d3.z)
            dst3[((i64)z * d3.y + y) * d3.x + x] = mip_reduce(s2, 5, 20, tx, ty, tz, x, y, z, d2);
    }
}

// The small top of the pyramid (from a level of at most 64^3 cells down to 1x1x1) in ONE block:
// level after level through global memory (L2), a block barrier between levels.
struct MipTail {
    i64 off[LVX_MAX_LEVELS + 1];
    int dims[LVX_MAX_LEVELS * 3];
    int first, n_levels;  // levels first+1 .. n_levels-1 are computed from level `first`
};

__global__ void __launch_bounds__(1024) mip_tail_kernel(float *__restrict__ flat, const MipTail T) {
    for (int l = T.first + 1; l < T.n_levels; ++l) {
        const float *src = flat + T.off[l - 1];
        float *dst = flat + T.off[l];
        const int sx = T.dims[3 * (l - 1)], sy = T.dims[3 * (l - 1) + 1], sz = T.dims[3 * (l - 1) + 2];
        const int px = T.dims[3 * l], py = T.dims[3 * l + 1], pz = T.dims[3 * l + 2];
        const i64 n = (i64)px * py * pz;
        for (i64 i = threadIdx.x; i < n; i += blockDim.x) {
            const int x = (int)(i % px), y = (int)((i / px) % py), z = (int)(i / ((i64)px * py));
            float acc = 0.0f, cnt = 0.0f;
#pragma unroll
            for (int oz = 0; oz < 2; ++oz)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy)
#pragma unroll
                    for (int ox = 0; ox < 2; ++ox) {
                        if (2 * z + oz < sz && 2 * y + oy < sy && 2 * x + ox < sx) {
                            acc = acc + src[((i64)(2 * z + oz) * sy + (2 * y + oy)) * sx + (2 * x + ox)];
                            cnt = cnt + 1.0f;
                        }
                    }
            dst[i] = acc / cnt;
        }
        __syncthreads();  // (block-scope visibility of the level just written)
    }
}

// One thread per cell of the grid padded by one voxel: 1 if the voxel or any of
// its 26 in-grid neighbours holds segments.
__global__ void __launch_bounds__(256)
dilate_kernel(const u8 *__restrict__ counts, int rx, int ry, int rz, u8 *__restrict__ occ) {
    const i64 sx = rx + 2, sy = ry + 2, sz = rz + 2;
    const i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= sx * sy * sz) return;
    // padded cell (px,py,pz) covers voxels [p-2, p] on each axis
    const int px = (int)(c % sx), py = (int)((c / sx) % sy), pz = (int)(c / (sx * sy));
    u8 any = 0;
    for (int z = max(pz - 2, 0); z <= min(pz, rz - 1) && !any; ++z)
        for (int y = max(py - 2, 0); y <= min(py, ry - 1) && !any; ++y)
            for (int x = max(px - 2, 0); x <= min(px, rx - 1); ++x)
                if (counts[((i64)z * ry + y) * rx + x]) {
                    any = 1;
                    break;
                }
    occ[c] = any;
}

// One thread per cell of the padded grid: over the voxel's in-grid 27-neighbourhood,
//   nsum  = sum of `counts` (max 27*255 fits u16): nsum > 0 is exactly the dilated
//           occupancy above, and the value is the number of candidate segments the
//           reference's neighbour gather visits for a window in this cell
//           (_kernels.py:811-821), i.e. what its `intersection_tests` counter adds up;
//   nmask = bit (dz+1)*9 + (dy+1)*3 + (dx+1) set when neighbour (dx,dy,dz) holds
//           segments: bit order == the reference's gather order (z, y, x loops).
__global__ void __launch_bounds__(256)
nsum_kernel(const u8 *__restrict__ counts, int rx, int ry, int rz, u16 *__restrict__ nsum,
            u32 *__restrict__ nmask, u64 *__restrict__ ncell) {
    const i64 sx = rx + 2, sy = ry + 2, sz = rz + 2;
    const i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= sx * sy * sz) return;
    // padded cell p is voxel p-1; its neighbours are voxels p-2 .. p
    const int px = (int)(c % sx), py = (int)((c / sx) % sy), pz = (int)(c / (sx * sy));
    u32 sum = 0, mask = 0;
    for (int dz = 0; dz < 3; ++dz) {
        const int z = pz - 2 + dz;
        if (z < 0 || z >= rz) continue;
        for (int dy = 0; dy < 3; ++dy) {
            const int y = py - 2 + dy;
            if (y < 0 || y >= ry) continue;
            for (int dx = 0; dx < 3; ++dx) {
                const int x = px - 2 + dx;
                if (x < 0 || x >= rx) continue;
                const u32 n = counts[((i64)z * ry + y) * rx + x];
                sum += n;
                if (n) mask |= 1u << (dz * 9 + dy * 3 + dx);
            }
        }
    }
    nsum[c] = (u16)sum;
    if (nmask) nmask[c] = mask;
    if (ncell) ncell[c] = (u64)mask | ((u64)sum << 32);
}

}  // namespace

extern "C" {

int lvx_density_l0(const uint8_t *counts_d, const uint32_t *offsets_d,
                   const lvx_seg_record *seg_rec_d, const float *table_d, int64_t n_voxels,
                   float *level0_d, void *stream) {
    LVX_REQUIRE(counts_d && offsets_d && table_d && level0_d && n_voxels > 0, "bad arguments");
    LVX_REQUIRE(((uintptr_t)seg_rec_d & 15) == 0, "seg_rec_d must be 16-byte aligned");
    // a few warps' worth of voxels per warp keeps the grid at some waves of the 148 SMs
    const i64 warps = lvx_ceil_div(n_voxels, 32 * kDlVox);
    const i64 blocks = lvx_ceil_div(warps, kDlThreads / 32);
    const i64 cap = (i64)lvx_sm_count() * LVX_DL_CAP;
    density_l0_kernel<u8, false><<<(unsigned)(blocks < cap ? blocks : cap), kDlThreads, 0, (cudaStream_t)stream>>>(
        counts_d, offsets_d, seg_rec_d, LvxPacked{}, table_d, n_voxels, level0_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_density_l0_packed(const uint8_t *counts_d, const uint32_t *offsets_d, const uint8_t *packed_d,
                          const int32_t dims[3], int32_t n_bins, const float *table_d, float *level0_d, void *stream) {
    LVX_REQUIRE(counts_d && offsets_d && table_d && level0_d && dims && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1,
                "bad arguments");
    LVX_REQUIRE(n_bins >= 2 && n_bins <= 256 && (n_bins & (n_bins - 1)) == 0, "bad bin resolution %d", n_bins);
    LVX_REQUIRE(((uintptr_t)packed_d & 7) == 0, "packed_d must be 8-byte aligned");
    LvxPacked P;
    int lb = 0;
    while ((1 << (lb + 1)) <= n_bins) ++lb;
    P.bytes = packed_d;
    P.lb = lb;
    P.n = n_bins;
    P.inv_n = 1.0f / (float)n_bins;
    P.width = (2 * (3 + 2 * lb) + 8 + 5 + 7) / 8;  // record_width, voxelizer.py:70-76
    const i64 V = (i64)dims[0] * dims[1] * dims[2];
    const int dmax = dims[0] > dims[1] ? (dims[0] > dims[2] ? dims[0] : dims[2]) : (dims[1] > dims[2] ? dims[1] : dims[2]);
    static const bool force_general = getenv("LVX_DENSITY_GENERAL") != nullptr;  // tests reach the fallback with it
    if (!force_general && (i64)dmax * 2 * n_bins <= (i64)1 << 24) {
        // voxel + bin centre is exact in float32: the warp-cooperative kernel, without the voxel
        const i64 blocks = lvx_ceil_div(lvx_ceil_div(V, (i64)kDlVox), kDlThreads);
        const i64 cap = (i64)lvx_sm_count() * LVX_DL_CAP;
        density_l0_kernel<u8, true><<<(unsigned)(blocks < cap ? blocks : cap), kDlThreads, 0, (cudaStream_t)stream>>>(
            counts_d, offsets_d, nullptr, P, table_d, V, level0_d);
        LVX_LAUNCH_CHECK();
        return LVX_OK;
    }
    const i64 blocks = lvx_ceil_div(V, kDlThreads);
    const i64 cap = (i64)lvx_sm_count() * 256;
    density_l0_packed_kernel<<<(unsigned)(blocks < cap ? blocks : cap), kDlThreads, 0, (cudaStream_t)stream>>>(
        counts_d, offsets_d, P, table_d, dims[0], dims[1], V, level0_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_density_l0_u32(const uint32_t *counts_d, const uint32_t *offsets_d, const lvx_seg_record *seg_rec_d,
                       const float *table_d, int64_t n_voxels, float *level0_d, void *stream) {
    LVX_REQUIRE(counts_d && offsets_d && table_d && level0_d && n_voxels > 0, "bad arguments");
    LVX_REQUIRE(((uintptr_t)seg_rec_d & 15) == 0, "seg_rec_d must be 16-byte aligned");
    const i64 warps = lvx_ceil_div(n_voxels, 32 * kDlVox);
    const i64 blocks = lvx_ceil_div(warps, kDlThreads / 32);
    const i64 cap = (i64)lvx_sm_count() * LVX_DL_CAP;
    density_l0_kernel<u32, false><<<(unsigned)(blocks < cap ? blocks : cap), kDlThreads, 0, (cudaStream_t)stream>>>(
        counts_d, offsets_d, seg_rec_d, LvxPacked{}, table_d, n_voxels, level0_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_octree_layout(const int32_t dims[3], int64_t *off, int64_t *ldims, int32_t *n_levels) {
    LVX_REQUIRE(dims && off && ldims && n_levels && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1,
                "bad arguments");
    i64 d[3] = {dims[0], dims[1], dims[2]};
    int L = 0;
    off[0] = 0;
    for (;;) {
        LVX_REQUIRE(L < LVX_MAX_LEVELS, "too many octree levels");
        ldims[3 * L] = d[0];
        ldims[3 * L + 1] = d[1];
        ldims[3 * L + 2] = d[2];
        off[L + 1] = off[L] + d[0] * d[1] * d[2];
        ++L;
        if (d[0] == 1 && d[1] == 1 && d[2] == 1) break;
        for (int c = 0; c < 3; ++c) d[c] = (d[c] + 1) / 2;
    }
    *n_levels = L;
    return LVX_OK;
}

int lvx_build_octree(float *flat_d, const int32_t dims[3], void *stream) {
    LVX_REQUIRE(flat_d, "null octree buffer");
    i64 off[LVX_MAX_LEVELS + 1], ld[LVX_MAX_LEVELS * 3];
    int32_t L = 0;
    if (int rc = lvx_octree_layout(dims, off, ld, &L)) return rc;
    auto dims_of = [&](int l) {
        MipDims d = {1, 1, 1};
        if (l < L) d = MipDims{(int)ld[3 * l], (int)ld[3 * l + 1], (int)ld[3 * l + 2]};
        return d;
    };
    int l = 0;
    // three levels per pass while the level is large ...
    while (l + 1 < L && ld[3 * l] * ld[3 * l + 1] * ld[3 * l + 2] > 64 * 64 * 64) {
        const int n_out = (L - 1 - l) < 3 ? (L - 1 - l) : 3;
        const MipDims d0 = dims_of(l), d1 = dims_of(l + 1), d2 = dims_of(l + 2), d3 = dims_of(l + 3);
        dim3 grid((unsigned)lvx_ceil_div(d1.x, kMipP), (unsigned)lvx_ceil_div(d1.y, kMipP),
                  (unsigned)lvx_ceil_div(d1.z, kMipP));
        mip3_kernel<<<grid, kMipP * kMipP * kMipP, 0, (cudaStream_t)stream>>>(
            flat_d + off[l], d0, flat_d + off[l + 1], d1, n_out >= 2 ? flat_d + off[l + 2] : nullptr, d2,
            n_out >= 3 ? flat_d + off[l + 3] : nullptr, d3, n_out,
            d0.x % 4 == 0 && ((uintptr_t)(flat_d + off[l]) & 15) == 0);
        LVX_LAUNCH_CHECK();
        l += n_out;
    }
    // ... and the rest of the pyramid in one block
    if (l + 1 < L) {
        MipTail T;
        memset(&T, 0, sizeof(T));
        for (int k = 0; k <= L; ++k) T.off[k] = off[k];
        for (int k = 0; k < 3 * L; ++k) T.dims[k] = (int)ld[k];
        T.first = l;
        T.n_levels = L;
        mip_tail_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(flat_d, T);
        LVX_LAUNCH_CHECK();
    }
    return LVX_OK;
}

int lvx_occupancy_dilate(const uint8_t *counts_d, const int32_t dims[3], uint8_t *occ_d,
                         void *stream) {
    LVX_REQUIRE(counts_d && occ_d && dims && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1,
                "bad arguments");
    const i64 cells = (i64)(dims[0] + 2) * (dims[1] + 2) * (dims[2] + 2);
    dilate_kernel<<<(unsigned)lvx_ceil_div(cells, 256), 256, 0, (cudaStream_t)stream>>>(
        counts_d, dims[0], dims[1], dims[2], occ_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_neighbor_sums(const uint8_t *counts_d, const int32_t dims[3], uint16_t *nsum_d,
                      uint32_t *nmask_d, uint64_t *ncell_d, void *stream) {
    LVX_REQUIRE(counts_d && nsum_d && dims && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1,
                "bad arguments");
    const i64 cells = (i64)(dims[0] + 2) * (dims[1] + 2) * (dims[2] + 2);
    nsum_kernel<<<(unsigned)lvx_ceil_div(cells, 256), 256, 0, (cudaStream_t)stream>>>(
        counts_d, dims[0], dims[1], dims[2], nsum_d, nmask_d, ncell_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
