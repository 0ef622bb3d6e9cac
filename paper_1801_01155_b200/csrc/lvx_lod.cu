// LoD construction for sm_100a: level-0 density, 2x2x2 mip chain, dilated
// occupancy map.
//
//   compute_density_level0   lod.py:82-94
//   _coarsen / build_octree  lod.py:97-119
//   _occupancy_dilated       raycast.py:351-366
#include "lvx_common.cuh"

namespace {

// One thread per voxel; its segments are summed in stored order in float64
// (np.bincount with weights is a sequential f64 accumulation), one cast to f32.
__global__ void __launch_bounds__(256)
density_l0_kernel(const u8 *__restrict__ counts, const u32 *__restrict__ offsets,
                  const lvx_seg_record *__restrict__ rec, const float *__restrict__ table,
                  i64 n_voxels, float *__restrict__ out) {
    __shared__ float s_sigma[256];
    s_sigma[threadIdx.x] = table[4 * threadIdx.x + 3];
    __syncthreads();
    const i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_voxels) return;
    const u32 n = counts[v];
    double acc = 0.0;
    if (n) {
        const float4 *r = reinterpret_cast<const float4 *>(rec + offsets[v]);
        for (u32 k = 0; k < n; ++k) {
            const float4 a = __ldg(r + 2 * k), b = __ldg(r + 2 * k + 1);
            // endpoints are widened BEFORE the subtraction (lod.py:87-89)
            const double ex = (double)b.x - (double)a.x;
            const double ey = (double)b.y - (double)a.y;
            const double ez = (double)b.z - (double)a.z;
            const double len = sqrt(ex * ex + ey * ey + ez * ez);
            const double sigma = (double)s_sigma[__float_as_uint(a.w) & 0xFFu];
            acc += len * sigma;
        }
    }
    out[v] = (float)acc;
}

// Shared-memory staged 2x2x2 reduction.  A block owns an 8x8x8 parent brick; it
// stages the 16x16x16 child brick with coalesced row loads, then every thread
// sums its (up to) eight children in the fixed (oz, oy, ox) order in float32 and
// divides by the float32 child count (lod.py:97-110).
constexpr int kMipP = 8;             // parent brick edge
constexpr int kMipC = 2 * kMipP;     // child brick edge
constexpr int kMipPitch = kMipC + 1; // +1: conflict-free strided reads

__global__ void __launch_bounds__(kMipP *kMipP *kMipP)
mip_kernel(const float *__restrict__ src, int sx, int sy, int sz, float *__restrict__ dst, int px,
           int py, int pz) {
    __shared__ float s[kMipC][kMipC][kMipPitch];
    const int bx = blockIdx.x * kMipP, by = blockIdx.y * kMipP, bz = blockIdx.z * kMipP;
    const int cx0 = 2 * bx, cy0 = 2 * by, cz0 = 2 * bz;
    for (int idx = threadIdx.x; idx < kMipC * kMipC * kMipC; idx += blockDim.x) {
        const int lx = idx % kMipC, ly = (idx / kMipC) % kMipC, lz = idx / (kMipC * kMipC);
        const int gx = cx0 + lx, gy = cy0 + ly, gz = cz0 + lz;
        float v = 0.0f;
        if (gx < sx && gy < sy && gz < sz) v = src[((i64)gz * sy + gy) * sx + gx];
        s[lz][ly][lx] = v;
    }
    __syncthreads();
    const int tx = threadIdx.x % kMipP, ty = (threadIdx.x / kMipP) % kMipP,
              tz = threadIdx.x / (kMipP * kMipP);
    const int x = bx + tx, y = by + ty, z = bz + tz;
    if (x >= px || y >= py || z >= pz) return;
    float acc = 0.0f, cnt = 0.0f;
#pragma unroll
    for (int oz = 0; oz < 2; ++oz)
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) {
                if (2 * z + oz < sz && 2 * y + oy < sy && 2 * x + ox < sx) {
                    acc = acc + s[2 * tz + oz][2 * ty + oy][2 * tx + ox];
                    cnt = cnt + 1.0f;
                }
            }
    dst[((i64)z * py + y) * px + x] = acc / cnt;
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
            u32 *__restrict__ nmask) {
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
}

}  // namespace

extern "C" {

int lvx_density_l0(const uint8_t *counts_d, const uint32_t *offsets_d,
                   const lvx_seg_record *seg_rec_d, const float *table_d, int64_t n_voxels,
                   float *level0_d, void *stream) {
    LVX_REQUIRE(counts_d && offsets_d && table_d && level0_d && n_voxels > 0, "bad arguments");
    density_l0_kernel<<<(unsigned)lvx_ceil_div(n_voxels, 256), 256, 0, (cudaStream_t)stream>>>(
        counts_d, offsets_d, seg_rec_d, table_d, n_voxels, level0_d);
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
    for (int l = 1; l < L; ++l) {
        const int sx = (int)ld[3 * (l - 1)], sy = (int)ld[3 * (l - 1) + 1], sz = (int)ld[3 * (l - 1) + 2];
        const int px = (int)ld[3 * l], py = (int)ld[3 * l + 1], pz = (int)ld[3 * l + 2];
        dim3 grid((unsigned)lvx_ceil_div(px, kMipP), (unsigned)lvx_ceil_div(py, kMipP),
                  (unsigned)lvx_ceil_div(pz, kMipP));
        mip_kernel<<<grid, kMipP * kMipP * kMipP, 0, (cudaStream_t)stream>>>(
            flat_d + off[l - 1], sx, sy, sz, flat_d + off[l], px, py, pz);
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
                      uint32_t *nmask_d, void *stream) {
    LVX_REQUIRE(counts_d && nsum_d && dims && dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1,
                "bad arguments");
    const i64 cells = (i64)(dims[0] + 2) * (dims[1] + 2) * (dims[2] + 2);
    nsum_kernel<<<(unsigned)lvx_ceil_div(cells, 256), 256, 0, (cudaStream_t)stream>>>(
        counts_d, dims[0], dims[1], dims[2], nsum_d, nmask_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
