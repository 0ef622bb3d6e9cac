// AO bake and point probes for sm_100a.
//
//   precompute_ao_kernel / precompute_voxel_ao   _kernels.py:608-620, illumination.py:193-214
//   probes: traverse_voxels raycast.py:170-181, intersect_ray_tube/sphere :184-213,
//           cone_soft_shadow / ao_density_rays / sample_ao illumination.py:142-225
#include <math_constants.h>
#include <stdlib.h>

#include "lvx_geom.cuh"

namespace {

// One thread per voxel.  Occupied voxels integrate n_rays full-sphere density rays
// from the voxel centre (normal (0,0,1)); rays are summed in lattice order in
// float64, the mean is clipped to [0,1] and cast to float32.  The direction lattice
// is staged in shared memory (n_rays * 24 bytes).
__global__ void __launch_bounds__(128)
ao_bake_kernel(const u8 *__restrict__ counts, int rx, int ry, int rz, int n_rays, double radius,
               double step, const double *__restrict__ dirs, const float *__restrict__ l0,
               float *__restrict__ out) {
    extern __shared__ double s_dirs[];
    for (int k = threadIdx.x; k < 3 * n_rays; k += blockDim.x) s_dirs[k] = dirs[k];
    __syncthreads();
    // 4x4x8 voxel bricks per block keep a warp's samples inside a few cache lines
    const int bx = blockIdx.x * 4, by = blockIdx.y * 4, bz = blockIdx.z * 8;
    const int x = bx + (threadIdx.x & 3), y = by + ((threadIdx.x >> 2) & 3), z = bz + (threadIdx.x >> 4);
    if (x >= rx || y >= ry || z >= rz) return;
    const i64 lin = x + (i64)rx * (y + (i64)ry * z);
    float res = 0.0f;
    if (counts[lin] != 0) {
        double v = lvx_ao_density_point((double)x + 0.5, (double)y + 0.5, (double)z + 0.5, 0.0, 0.0,
                                        1.0, n_rays, radius, step, s_dirs, l0, rx, ry, rz);
        v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        res = (float)v;
    }
    out[lin] = res;
}

// Brick version of the bake (used when the halo fits in shared memory).  One block per 8x8x8
// voxel brick: the level-0 density of the brick plus a halo of ceil(radius)+1 voxels is staged
// in shared memory (indices clamped to the grid exactly like sample_field_trilinear does), so
// the 8 loads of every trilinear sample stay on chip.  Occupied voxels are listed; each warp
// takes one voxel at a time and spreads its rays over the lanes (all lanes busy whatever the
// occupancy pattern).  The per-ray results are then summed by one lane in lattice order --
// the reference's float64 summation order (_kernels.py:592-605) -- so the result is
// bit-identical to the one-thread-per-voxel kernel above.
constexpr int kBrick = 8;
constexpr int kBakeWarps = 8;

__device__ __forceinline__ double bake_trilinear(const float *__restrict__ s, int E, int lox, int loy, int loz,
                                                 int ldx, int ldy, int ldz, double x, double y, double z) {
    // sample_field_trilinear (_kernels.py:346-383) at scale 1: x / 1.0 - 0.5 == x - 0.5
    const double qx = x / 1.0 - 0.5, qy = y / 1.0 - 0.5, qz = z / 1.0 - 0.5;
    const double flx = floor(qx), fly = floor(qy), flz = floor(qz);
    const double fx = qx - flx, fy = qy - fly, fz = qz - flz;
    const double hx = (double)(ldx - 1), hy = (double)(ldy - 1), hz = (double)(ldz - 1);
    const int x0 = (int)fmin(fmax(flx, 0.0), hx) - lox, x1 = (int)fmin(fmax(flx + 1.0, 0.0), hx) - lox;
    const int y0 = (int)fmin(fmax(fly, 0.0), hy) - loy, y1 = (int)fmin(fmax(fly + 1.0, 0.0), hy) - loy;
    const int z0 = (int)fmin(fmax(flz, 0.0), hz) - loz, z1 = (int)fmin(fmax(flz + 1.0, 0.0), hz) - loz;
    const int sy = E, sz = E * E;
    const double v000 = (double)s[z0 * sz + y0 * sy + x0], v001 = (double)s[z0 * sz + y0 * sy + x1];
    const double v010 = (double)s[z0 * sz + y1 * sy + x0], v011 = (double)s[z0 * sz + y1 * sy + x1];
    const double v100 = (double)s[z1 * sz + y0 * sy + x0], v101 = (double)s[z1 * sz + y0 * sy + x1];
    const double v110 = (double)s[z1 * sz + y1 * sy + x0], v111 = (double)s[z1 * sz + y1 * sy + x1];
    const double c00 = v000 * (1.0 - fx) + v001 * fx;
    const double c01 = v010 * (1.0 - fx) + v011 * fx;
    const double c10 = v100 * (1.0 - fx) + v101 * fx;
    const double c11 = v110 * (1.0 - fx) + v111 * fx;
    const double c0 = c00 * (1.0 - fy) + c01 * fy;
    const double c1 = c10 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

__global__ void __launch_bounds__(kBakeWarps * 32)
ao_bake_brick_kernel(const u8 *__restrict__ counts, int rx, int ry, int rz, int n_rays, double radius,
                     double step, const double *__restrict__ dirs, const float *__restrict__ l0, int H,
                     float *__restrict__ out) {
    extern __shared__ double s_mem[];
    const int E = kBrick + 2 * H;
    double *s_dirs = s_mem;                            // [3 * n_rays]
    double *s_ray = s_dirs + 3 * n_rays;               // [kBakeWarps][n_rays]
    float *s_l0 = reinterpret_cast<float *>(s_ray + kBakeWarps * n_rays);  // [E^3]
    __shared__ unsigned short s_list[kBrick * kBrick * kBrick];
    __shared__ int s_n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bx = blockIdx.x * kBrick, by = blockIdx.y * kBrick, bz = blockIdx.z * kBrick;
    const int lox = bx - H, loy = by - H, loz = bz - H;
    if (tid == 0) s_n = 0;
    for (int k = tid; k < 3 * n_rays; k += blockDim.x) s_dirs[k] = dirs[k];
    for (int k = tid; k < E * E * E; k += blockDim.x) {
        const int ix = k % E, iy = (k / E) % E, iz = k / (E * E);
        const int gx_ = min(max(lox + ix, 0), rx - 1), gy_ = min(max(loy + iy, 0), ry - 1),
                  gz_ = min(max(loz + iz, 0), rz - 1);
        s_l0[k] = __ldg(l0 + ((i64)gz_ * ry + gy_) * rx + gx_);
    }
    __syncthreads();
    // list the occupied voxels of the brick; empty ones are written now
    for (int k = tid; k < kBrick * kBrick * kBrick; k += blockDim.x) {
        const int x = bx + (k & 7), y = by + ((k >> 3) & 7), z = bz + (k >> 6);
        if (x >= rx || y >= ry || z >= rz) continue;
        const i64 lin = x + (i64)rx * (y + (i64)ry * z);
        if (counts[lin] != 0) s_list[atomicAdd(&s_n, 1)] = (unsigned short)k;
        else out[lin] = 0.0f;
    }
    __syncthreads();
    const int n_occ = s_n;
    const double gx = (double)rx, gy = (double)ry, gz = (double)rz;
    double *my_ray = s_ray + warp * n_rays;
    for (int e = warp; e < n_occ; e += kBakeWarps) {
        const int k = s_list[e];
        const int x = bx + (k & 7), y = by + ((k >> 3) & 7), z = bz + (k >> 6);
        const double px = (double)x + 0.5, py = (double)y + 0.5, pz = (double)z + 0.5;
        // orient_frame for the normal (0,0,1) (_kernels.py:555-569): t = (1,0,0), b = (0,1,0)
        double tf[3], bf[3];
        lvx_orient_frame(0.0, 0.0, 1.0, tf, bf);
        for (int r = lane; r < n_rays; r += 32) {
            const double lx = s_dirs[3 * r], ly = s_dirs[3 * r + 1], lz = s_dirs[3 * r + 2];
            const double dx = lx * tf[0] + ly * bf[0] + lz * 0.0;
            const double dy = lx * tf[1] + ly * bf[1] + lz * 0.0;
            const double dz = lx * tf[2] + ly * bf[2] + lz * 1.0;
            // density_ray_blocking, _kernels.py:425-445
            double acc = 0.0, t_cur = step;
            bool sat = false;
            while (t_cur <= radius) {
                const double sx = px + t_cur * dx, sy_ = py + t_cur * dy, sz_ = pz + t_cur * dz;
                if (sx < 0.0 || sy_ < 0.0 || sz_ < 0.0 || sx > gx || sy_ > gy || sz_ > gz) break;
                acc += bake_trilinear(s_l0, E, lox, loy, loz, rx, ry, rz, sx, sy_, sz_) * step;
                if (acc >= 1.0) {
                    sat = true;
                    break;
                }
                t_cur += step;
            }
            my_ray[r] = sat ? 1.0 : (acc < 1.0 ? acc : 1.0);
        }
        __syncwarp();
        if (lane == 0) {
            double total = 0.0;
            for (int r = 0; r < n_rays; ++r) total += my_ray[r];
            double v = total / (double)n_rays;
            v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
            out[x + (i64)rx * (y + (i64)ry * z)] = (float)v;
        }
        __syncwarp();
    }
}

// Batched brick bake (the default).  Same staging as above; what changes is how the work is dealt:
//  * the (voxel, ray) pairs of up to kBakeBatch occupied voxels are flattened over ALL threads of the
//    block, so every lane marches a ray whatever n_rays and the occupancy pattern are (one warp per
//    voxel left 28 of 32 lanes idle in the last of its four rounds at 100 rays);
//  * the per-ray results of the batch sit in shared memory and ONE THREAD PER VOXEL adds them up in
//    lattice order -- the reference's float64 summation order (_kernels.py:592-605) -- so up to 32 of
//    these 100-step dependent chains run side by side instead of one at a time;
//  * a brick whose halo lies inside the grid (INTERIOR) needs neither the grid-exit test nor the
//    clamp-to-edge of sample_field_trilinear: no sample can leave the staged block;
//  * cell indices are integers from one float64 -> int floor conversion per axis (the reference's
//    floor / clip / int chain is the same integer), the eight corners are one base address plus
//    constant offsets.
// Arithmetic per sample is the reference's, operation for operation; the field is bit-identical.
#ifndef LVX_AO_BATCH
#define LVX_AO_BATCH 32
#endif
#ifndef LVX_AO_F64
#define LVX_AO_F64 0
#endif
#ifndef LVX_AO_TABLE
#define LVX_AO_TABLE 1
#endif
#ifndef LVX_AO_STEPS
#define LVX_AO_STEPS 6
#endif
constexpr int kBakeSteps = LVX_AO_STEPS;  // march steps whose parameters a thread keeps in registers
constexpr int kBakeBatch = LVX_AO_BATCH;
constexpr int kBakeThreads = 256;
// the staged density: float32 as stored (widened per corner load), or widened once at staging
#if LVX_AO_F64
typedef double bake_t;
#else
typedef float bake_t;
#endif

template <bool INTERIOR>
__device__ __forceinline__ double bake_sample(const bake_t *__restrict__ s, int E, int lox, int loy, int loz, int rx,
                                              int ry, int rz, double x, double y, double z) {
    // sample_field_trilinear (_kernels.py:346-383) at scale 1: x / 1.0 - 0.5 == x - 0.5
    const double qx = x / 1.0 - 0.5, qy = y / 1.0 - 0.5, qz = z / 1.0 - 0.5;
    const int ix = __double2int_rd(qx), iy = __double2int_rd(qy), iz = __double2int_rd(qz);  // floor
    const double fx = qx - (double)ix, fy = qy - (double)iy, fz = qz - (double)iz;
    int o000, dx1, dy1, dz1;
    if (INTERIOR) {
        o000 = ((iz - loz) * E + (iy - loy)) * E + (ix - lox);
        dx1 = 1;
        dy1 = E;
        dz1 = E * E;
    } else {
        const int x0 = min(max(ix, 0), rx - 1), x1 = min(max(ix + 1, 0), rx - 1);
        const int y0 = min(max(iy, 0), ry - 1), y1 = min(max(iy + 1, 0), ry - 1);
        const int z0 = min(max(iz, 0), rz - 1), z1 = min(max(iz + 1, 0), rz - 1);
        o000 = ((z0 - loz) * E + (y0 - loy)) * E + (x0 - lox);
        dx1 = x1 - x0;
        dy1 = (y1 - y0) * E;
        dz1 = (z1 - z0) * E * E;
    }
    const bake_t *c = s + o000;
    const double v000 = (double)c[0], v001 = (double)c[dx1];
    const double v010 = (double)c[dy1], v011 = (double)c[dy1 + dx1];
    const double v100 = (double)c[dz1], v101 = (double)c[dz1 + dx1];
    const double v110 = (double)c[dz1 + dy1], v111 = (double)c[dz1 + dy1 + dx1];
    const double gx_ = 1.0 - fx, gy_ = 1.0 - fy, gz_ = 1.0 - fz;
    const double c00 = v000 * gx_ + v001 * fx;
    const double c01 = v010 * gx_ + v011 * fx;
    const double c10 = v100 * gx_ + v101 * fx;
    const double c11 = v110 * gx_ + v111 * fx;
    const double c0 = c00 * gy_ + c01 * fy;
    const double c1 = c10 * gy_ + c11 * fy;
    return c0 * gz_ + c1 * fz;
}

template <bool INTERIOR, bool TABLE>
__device__ __forceinline__ void bake_batches(const bake_t *__restrict__ s_l0, const double *__restrict__ s_d,
                                             double *__restrict__ s_res, const unsigned short *__restrict__ s_list,
                                             int n_occ, int batch, int row, int E, int lox, int loy, int loz, int bx, int by,
                                             int bz, int rx, int ry, int rz, int n_rays, double radius, double step,
                                             float *__restrict__ out) {
    const int tid = threadIdx.x;
    const double gx = (double)rx, gy = (double)ry, gz = (double)rz;
    // The march parameters t_1 = step, t_{k+1} = t_k + step (while t_k <= radius) are the same for every
    // ray: up to kBakeSteps of them are computed ONCE per thread, by the reference's own additions, and
    // kept in registers (the loop below is fully unrolled, so the indices are static).  Per sample that
    // takes the float64 add and compare of the loop control off the FP64 pipe, the kernel's bound; so do
    // multiplying by a step of exactly 1 (x * 1.0 == x) and testing acc >= 1 on the high word (for any
    // acc the final result is the same: a NaN ends as 1.0 either way).
    // (TABLE is the host's decision, lvx_ao_bake: the march has 4 .. kBakeSteps steps; a kernel of its
    // own, so that the plain loop keeps its 60 registers -- 4 blocks per SM at small radii)
    double tk[kBakeSteps];
    int n_steps = 0;
    if (TABLE) {
        double t = step;
#pragma unroll
        for (int k = 0; k < kBakeSteps; ++k) {
            tk[k] = t;
            if (t <= radius) n_steps = k + 1;  // (t grows: the steps that qualify are the leading ones)
            t += step;
        }
    }
    const bool unit_step = step == 1.0;
    for (int e0 = 0; e0 < n_occ; e0 += batch) {
        const int nb = min(batch, n_occ - e0);
        const int items = nb * n_rays;
        if (TABLE) {
            for (int w = tid; w < items; w += kBakeThreads) {
                const int v = w / n_rays, r = w - v * n_rays;
                const int k = s_list[e0 + v];
                const double px = (double)(bx + (k & 7)) + 0.5, py = (double)(by + ((k >> 3) & 7)) + 0.5,
                             pz = (double)(bz + (k >> 6)) + 0.5;
                const double dx = s_d[3 * r], dy = s_d[3 * r + 1], dz = s_d[3 * r + 2];
                // density_ray_blocking, _kernels.py:425-445
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < kBakeSteps; ++q) {
                    if (q >= n_steps) break;
                    const double t_cur = tk[q];
                    const double sx = px + t_cur * dx, sy_ = py + t_cur * dy, sz_ = pz + t_cur * dz;
                    if (!INTERIOR && (sx < 0.0 || sy_ < 0.0 || sz_ < 0.0 || sx > gx || sy_ > gy || sz_ > gz)) break;
                    const double smp = bake_sample<INTERIOR>(s_l0, E, lox, loy, loz, rx, ry, rz, sx, sy_, sz_);
                    acc += unit_step ? smp : smp * step;
                    if (__double2hiint(acc) >= 0x3FF00000) break;  // acc >= 1.0
                }
                s_res[v * row + r] = acc < 1.0 ? acc : 1.0;  // (a saturated ray has acc >= 1)
            }
        } else
        for (int w = tid; w < items; w += kBakeThreads) {
            const int v = w / n_rays, r = w - v * n_rays;
            const int k = s_list[e0 + v];
            const double px = (double)(bx + (k & 7)) + 0.5, py = (double)(by + ((k >> 3) & 7)) + 0.5,
                         pz = (double)(bz + (k >> 6)) + 0.5;
            const double dx = s_d[3 * r], dy = s_d[3 * r + 1], dz = s_d[3 * r + 2];
            // density_ray_blocking, _kernels.py:425-445
            double acc = 0.0, t_cur = step;
            bool sat = false;
            while (t_cur <= radius) {
                const double sx = px + t_cur * dx, sy_ = py + t_cur * dy, sz_ = pz + t_cur * dz;
                if (!INTERIOR && (sx < 0.0 || sy_ < 0.0 || sz_ < 0.0 || sx > gx || sy_ > gy || sz_ > gz)) break;
                acc += bake_sample<INTERIOR>(s_l0, E, lox, loy, loz, rx, ry, rz, sx, sy_, sz_) * step;
                if (acc >= 1.0) {
                    sat = true;
                    break;
                }
                t_cur += step;
            }
            s_res[v * row + r] = sat ? 1.0 : (acc < 1.0 ? acc : 1.0);
        }
        __syncthreads();
        if (tid < nb) {
            const double *mine = s_res + tid * row;
            double total = 0.0;
            for (int r = 0; r < n_rays; ++r) total += mine[r];
            double v = total / (double)n_rays;
            v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
            const int k = s_list[e0 + tid];
            out[(bx + (k & 7)) + (i64)rx * ((by + ((k >> 3) & 7)) + (i64)ry * (bz + (k >> 6)))] = (float)v;
        }
        __syncthreads();
    }
}

// (the table kernel is given the registers of three blocks per SM -- what its shared memory allows at
// R = 5 anyway; left to itself ptxas stops at 64 and spills: 15.4 instead of 14.9 ms)
template <bool TABLE>
__global__ void __launch_bounds__(kBakeThreads, TABLE ? 3 : 4)
ao_bake_batch_kernel(const u8 *__restrict__ counts, int rx, int ry, int rz, int n_rays, double radius, double step,
                     const double *__restrict__ dirs, const float *__restrict__ l0, int H, int batch, int row,
                     float *__restrict__ out) {
    extern __shared__ double s_mem[];
    const int E = kBrick + 2 * H;
    double *s_d = s_mem;                  // [3 * n_rays] ray directions in grid space
    double *s_res = s_d + 3 * n_rays;     // [batch][row] per-ray results of the current batch
    bake_t *s_l0 = reinterpret_cast<bake_t *>(s_res + (size_t)batch * row);  // [E^3]
    __shared__ unsigned short s_list[kBrick * kBrick * kBrick];
    __shared__ int s_n;
    const int tid = threadIdx.x;
    const int bx = blockIdx.x * kBrick, by = blockIdx.y * kBrick, bz = blockIdx.z * kBrick;
    const int lox = bx - H, loy = by - H, loz = bz - H;
    if (tid == 0) s_n = 0;
    __syncthreads();
    // occupied voxels first: an empty brick is done after writing its zeros
    for (int k = tid; k < kBrick * kBrick * kBrick; k += kBakeThreads) {
        const int x = bx + (k & 7), y = by + ((k >> 3) & 7), z = bz + (k >> 6);
        if (x >= rx || y >= ry || z >= rz) continue;
        const i64 lin = x + (i64)rx * (y + (i64)ry * z);
        if (counts[lin] != 0) s_list[atomicAdd(&s_n, 1)] = (unsigned short)k;
        else out[lin] = 0.0f;
    }
    __syncthreads();
    const int n_occ = s_n;
    if (n_occ == 0) return;
    {
        // ray directions: the lattice in the frame of the normal (0,0,1) (orient_frame, _kernels.py:555-569)
        double tf[3], bf[3];
        lvx_orient_frame(0.0, 0.0, 1.0, tf, bf);
        for (int r = tid; r < n_rays; r += kBakeThreads) {
            const double lx = dirs[3 * r], ly = dirs[3 * r + 1], lz = dirs[3 * r + 2];
            s_d[3 * r] = lx * tf[0] + ly * bf[0] + lz * 0.0;
            s_d[3 * r + 1] = lx * tf[1] + ly * bf[1] + lz * 0.0;
            s_d[3 * r + 2] = lx * tf[2] + ly * bf[2] + lz * 1.0;
        }
    }
    for (int k = tid; k < E * E * E; k += kBakeThreads) {
        const int ix = k % E, iy = (k / E) % E, iz = k / (E * E);
        const int gx_ = min(max(lox + ix, 0), rx - 1), gy_ = min(max(loy + iy, 0), ry - 1),
                  gz_ = min(max(loz + iz, 0), rz - 1);
        s_l0[k] = (bake_t)__ldg(l0 + ((i64)gz_ * ry + gy_) * rx + gx_);
    }
    __syncthreads();
    // the warp order of the list is arbitrary (atomics); the result per voxel does not depend on it
    const bool interior = lox >= 0 && loy >= 0 && loz >= 0 && lox + E <= rx && loy + E <= ry && loz + E <= rz;
    if (interior)
        bake_batches<true, TABLE>(s_l0, s_d, s_res, s_list, n_occ, batch, row, E, lox, loy, loz, bx, by, bz, rx, ry, rz, n_rays,
                           radius, step, out);
    else
        bake_batches<false, TABLE>(s_l0, s_d, s_res, s_list, n_occ, batch, row, E, lox, loy, loz, bx, by, bz, rx, ry, rz, n_rays,
                            radius, step, out);
}

__global__ void probe_dda_kernel(double ox, double oy, double oz, double dx, double dy, double dz,
                                 int rx, int ry, int rz, int pad, i64 cap, i64 *out_vox,
                                 double *out_t, i64 *n_out) {
    LvxDda dda;
    dda.init(ox, oy, oz, dx, dy, dz, rx, ry, rz, pad);
    i64 n = 0;
    int wx, wy, wz;
    double t0, t1;
    while (dda.next(wx, wy, wz, t0, t1)) {
        if (n < cap) {
            out_vox[3 * n] = wx;
            out_vox[3 * n + 1] = wy;
            out_vox[3 * n + 2] = wz;
            out_t[2 * n] = t0;
            out_t[2 * n + 1] = t1;
            n += 1;
        }
    }
    *n_out = n;
}

__device__ __forceinline__ void store_hit(double *o, bool hit, const LvxHit &h) {
    o[0] = hit ? 1.0 : 0.0;
    o[1] = hit ? h.t_in : 0.0;
    o[2] = hit ? h.t_out : 0.0;
    o[3] = hit ? h.nx : 0.0;
    o[4] = hit ? h.ny : 0.0;
    o[5] = hit ? h.nz : 0.0;
}

__global__ void probe_tube_kernel(const double *__restrict__ rays, const void *a_, const void *b_,
                                  double r, int f32_axis, i64 n, double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *q = rays + 6 * i;
    LvxHit h;
    bool hit;
    if (f32_axis) {
        const float *a = (const float *)a_ + 3 * i, *b = (const float *)b_ + 3 * i;
        hit = lvx_tube_f32axis(q[0], q[1], q[2], q[3], q[4], q[5], a[0], a[1], a[2], b[0], b[1], b[2], r, h);
    } else {
        const double *a = (const double *)a_ + 3 * i, *b = (const double *)b_ + 3 * i;
        hit = lvx_tube_f64(q[0], q[1], q[2], q[3], q[4], q[5], a[0], a[1], a[2], b[0], b[1], b[2], r, h);
    }
    store_hit(out + 6 * i, hit, h);
}

__global__ void probe_sphere_kernel(const double *__restrict__ rays, const double *__restrict__ c,
                                    double r, i64 n, double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *q = rays + 6 * i;
    LvxHit h;
    const bool hit = lvx_sphere<true>(q[0], q[1], q[2], q[3], q[4], q[5], c[3 * i], c[3 * i + 1],
                                      c[3 * i + 2], r, h);
    store_hit(out + 6 * i, hit, h);
}

__global__ void probe_trilinear_kernel(const float *__restrict__ flat, i64 off, int ldx, int ldy,
                                       int ldz, double scale, const double *__restrict__ pts, i64 n,
                                       double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = lvx_trilinear(flat, off, ldx, ldy, ldz, scale, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

__global__ void probe_cone_kernel(const LvxOctree oc, const double *__restrict__ pts, double lx,
                                  double ly, double lz, double eps, i64 n, double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = lvx_cone_blocking(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], lx, ly, lz, oc,
                               (double)oc.dims[0], (double)oc.dims[1], (double)oc.dims[2], eps);
}

__global__ void probe_ao_kernel(const LvxOctree oc, const double *__restrict__ pts,
                                const double *__restrict__ nrm, int n_rays, double radius,
                                double step, const double *__restrict__ dirs, i64 n,
                                double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = lvx_ao_density_point(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], nrm[3 * i],
                                  nrm[3 * i + 1], nrm[3 * i + 2], n_rays, radius, step, dirs,
                                  oc.flat, oc.dims[0], oc.dims[1], oc.dims[2]);
}

__global__ void probe_shade_kernel(const double *__restrict__ nlv, double ka, double kd, double ks, double shininess,
                                   i64 n, double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *q = nlv + 9 * i;
    out[i] = lvx_shade(q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8], ka, kd, ks, shininess);
}

int fill_octree(LvxOctree &oc, const lvx_lod *lod) {
    LVX_REQUIRE(lod && lod->oct_flat_d && lod->n_levels >= 1 && lod->n_levels <= LVX_MAX_LEVELS,
                "a density octree is required");
    memset(&oc, 0, sizeof(oc));
    oc.flat = lod->oct_flat_d;
    oc.n_levels = lod->n_levels;
    for (int l = 0; l <= lod->n_levels; ++l) oc.off[l] = lod->oct_off[l];
    for (int l = 0; l < lod->n_levels * 3; ++l) oc.dims[l] = (int)lod->oct_dims[l];
    return LVX_OK;
}

}  // namespace

namespace {

__global__ void __launch_bounds__(64)
probe_blocked_kernel(LvxGeomModel M, const double *__restrict__ rays, const double *__restrict__ max_t,
                     double radius, int joints, i64 n, int32_t *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *r = rays + 6 * i;
    out[i] = lvx_geometry_blocked(r[0], r[1], r[2], r[3], r[4], r[5], max_t[i], M, radius, joints != 0) ? 1 : 0;
}

__global__ void __launch_bounds__(64)
probe_ao_hemi_kernel(LvxGeomModel M, const double *__restrict__ pts, const double *__restrict__ nrm, int n_rays,
                     double radius, const double *__restrict__ dirs, double tube_r, i64 n,
                     double *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = lvx_ao_hemisphere_point(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], nrm[3 * i], nrm[3 * i + 1],
                                     nrm[3 * i + 2], n_rays, radius, dirs, M, tube_r);
}

int geom_model(LvxGeomModel &G, const lvx_model *m) {
    LVX_REQUIRE(m && m->rx >= 1 && m->ry >= 1 && m->rz >= 1 && m->counts_d && m->offsets_d && m->nmask_d,
                "geometry rays need counts, offsets and the neighbour grids (lvx_neighbor_sums)");
    G.rx = m->rx;
    G.ry = m->ry;
    G.rz = m->rz;
    G.counts = m->counts_d;
    G.offsets = m->offsets_d;
    G.rec = m->seg_rec_d;
    G.nmask = m->nmask_d;
    return LVX_OK;
}

}  // namespace

extern "C" {

int lvx_ao_bake(const uint8_t *counts_d, const int32_t dims[3], int32_t n_rays, double radius,
                double step, const double *dirs_d, const float *level0_d, float *ao_d,
                void *stream) {
    LVX_REQUIRE(counts_d && dims && dirs_d && level0_d && ao_d, "null argument");
    LVX_REQUIRE(dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1, "grid dims must be >= 1");
    LVX_REQUIRE(n_rays >= 1 && n_rays <= 8192, "n_rays must be in [1, 8192], got %d", n_rays);
    LVX_REQUIRE(radius > 0.0 && step > 0.0, "radius and step must be positive");
    {
        // brick kernels when the halo of the radius of influence fits in shared memory
        const int H = (int)ceil(radius) + 1;
        const size_t E = (size_t)kBrick + 2 * (size_t)H;
        dim3 bgrid((unsigned)lvx_ceil_div(dims[0], kBrick), (unsigned)lvx_ceil_div(dims[1], kBrick),
                   (unsigned)lvx_ceil_div(dims[2], kBrick));
        // batched kernel: as many voxels per batch as 64 KB of per-ray results hold (rows padded to an odd
        // number of doubles: the per-voxel sums then read conflict-free)
        const int row = n_rays | 1;
        int batch = (int)((64 * 1024) / ((size_t)row * sizeof(double)));
        batch = batch > kBakeBatch ? kBakeBatch : batch;
        const size_t need_b = ((size_t)n_rays * 3 + (size_t)(batch > 0 ? batch : 1) * row) * sizeof(double) +
                              E * E * E * sizeof(bake_t);
        static const bool legacy = getenv("LVX_AO_LEGACY") != nullptr;  // developer A/B switch
        if (!legacy && radius < 64.0 && batch >= 1 && need_b <= 200 * 1024) {
            // the march parameters in registers when there are 4 .. kBakeSteps of them (the same float64
            // additions the kernels make; see bake_batches)
            int n_steps = 0;
            {
                double t = step;
                while (t <= radius && n_steps <= kBakeSteps) {
                    n_steps += 1;
                    t += step;
                }
            }
            const bool table = LVX_AO_TABLE && n_steps >= 4 && n_steps <= kBakeSteps;
            auto kernel = table ? ao_bake_batch_kernel<true> : ao_bake_batch_kernel<false>;
            if (need_b > 48 * 1024)
                LVX_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need_b));
            kernel<<<bgrid, kBakeThreads, need_b, (cudaStream_t)stream>>>(
                counts_d, dims[0], dims[1], dims[2], n_rays, radius, step, dirs_d, level0_d, H, batch, row, ao_d);
            LVX_LAUNCH_CHECK();
            return LVX_OK;
        }
        const size_t need = ((size_t)n_rays * 3 + (size_t)kBakeWarps * n_rays) * sizeof(double) + E * E * E * sizeof(float);
        if (radius < 64.0 && need <= 160 * 1024) {
            if (need > 48 * 1024)
                LVX_CUDA_CHECK(cudaFuncSetAttribute(ao_bake_brick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)need));
            ao_bake_brick_kernel<<<bgrid, kBakeWarps * 32, need, (cudaStream_t)stream>>>(
                counts_d, dims[0], dims[1], dims[2], n_rays, radius, step, dirs_d, level0_d, H, ao_d);
            LVX_LAUNCH_CHECK();
            return LVX_OK;
        }
    }
    dim3 grid((unsigned)lvx_ceil_div(dims[0], 4), (unsigned)lvx_ceil_div(dims[1], 4),
              (unsigned)lvx_ceil_div(dims[2], 8));
    const size_t smem = (size_t)n_rays * 3 * sizeof(double);
    if (smem > 48 * 1024)
        LVX_CUDA_CHECK(cudaFuncSetAttribute(ao_bake_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem));
    ao_bake_kernel<<<grid, 128, smem, (cudaStream_t)stream>>>(counts_d, dims[0], dims[1], dims[2],
                                                             n_rays, radius, step, dirs_d, level0_d,
                                                             ao_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_dda(const double o[3], const double d[3], const int32_t dims[3], int32_t pad,
                  int64_t cap, int64_t *out_vox_d, double *out_t_d, int64_t *n_d, void *stream) {
    LVX_REQUIRE(o && d && dims && out_vox_d && out_t_d && n_d && cap >= 0 && pad >= 0, "bad arguments");
    probe_dda_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(o[0], o[1], o[2], d[0], d[1], d[2], dims[0],
                                                       dims[1], dims[2], pad, cap, out_vox_d,
                                                       out_t_d, n_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_tube(const double *rays_d, const void *a_d, const void *b_d, double radius,
                   int32_t f32_axis, int64_t n, double *out_d, void *stream) {
    LVX_REQUIRE(n >= 0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(rays_d && a_d && b_d && out_d, "null argument");
    probe_tube_kernel<<<(unsigned)lvx_ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(
        rays_d, a_d, b_d, radius, f32_axis, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_sphere(const double *rays_d, const double *c_d, double radius, int64_t n,
                     double *out_d, void *stream) {
    LVX_REQUIRE(n >= 0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(rays_d && c_d && out_d, "null argument");
    probe_sphere_kernel<<<(unsigned)lvx_ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(
        rays_d, c_d, radius, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_shade(const double *nlv_d, double ka, double kd, double ks, double shininess, int64_t n,
                    double *out_d, void *stream) {
    LVX_REQUIRE(n >= 0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(nlv_d && out_d, "null argument");
    probe_shade_kernel<<<(unsigned)lvx_ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(nlv_d, ka, kd, ks, shininess, n,
                                                                                        out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_trilinear(const float *flat_d, int64_t off, const int64_t ldims[3], double scale,
                        const double *pts_d, int64_t n, double *out_d, void *stream) {
    LVX_REQUIRE(n >= 0 && ldims, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(flat_d && pts_d && out_d, "null argument");
    probe_trilinear_kernel<<<(unsigned)lvx_ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(
        flat_d, off, (int)ldims[0], (int)ldims[1], (int)ldims[2], scale, pts_d, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_cone(const lvx_lod *lod, const double *pts_d, const double light[3], double eps,
                   int64_t n, double *out_d, void *stream) {
    LvxOctree oc;
    if (int rc = fill_octree(oc, lod)) return rc;
    LVX_REQUIRE(n >= 0 && light, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(pts_d && out_d, "null argument");
    probe_cone_kernel<<<(unsigned)lvx_ceil_div(n, 128), 128, 0, (cudaStream_t)stream>>>(
        oc, pts_d, light[0], light[1], light[2], eps, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_ao_density(const lvx_lod *lod, const double *pts_d, const double *normals_d,
                         int32_t n_rays, double radius, double step, const double *dirs_d,
                         int64_t n, double *out_d, void *stream) {
    LvxOctree oc;
    if (int rc = fill_octree(oc, lod)) return rc;
    LVX_REQUIRE(n >= 0 && n_rays >= 1, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(pts_d && normals_d && dirs_d && out_d, "null argument");
    probe_ao_kernel<<<(unsigned)lvx_ceil_div(n, 64), 64, 0, (cudaStream_t)stream>>>(
        oc, pts_d, normals_d, n_rays, radius, step, dirs_d, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_blocked(const lvx_model *model, const double *rays_d, const double *max_t_d, double radius,
                      int32_t joints, int64_t n, int32_t *out_d, void *stream) {
    LvxGeomModel G;
    if (int rc = geom_model(G, model)) return rc;
    LVX_REQUIRE(n >= 0 && radius > 0.0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(rays_d && max_t_d && out_d, "null argument");
    probe_blocked_kernel<<<(unsigned)lvx_ceil_div(n, 64), 64, 0, (cudaStream_t)stream>>>(G, rays_d, max_t_d, radius,
                                                                                       joints, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_probe_ao_hemisphere(const lvx_model *model, const double *pts_d, const double *normals_d, int32_t n_rays,
                            double radius, const double *dirs_d, double tube_r, int64_t n, double *out_d,
                            void *stream) {
    LvxGeomModel G;
    if (int rc = geom_model(G, model)) return rc;
    LVX_REQUIRE(n >= 0 && n_rays >= 1 && tube_r > 0.0, "bad arguments");
    if (n == 0) return LVX_OK;
    LVX_REQUIRE(pts_d && normals_d && dirs_d && out_d, "null argument");
    probe_ao_hemi_kernel<<<(unsigned)lvx_ceil_div(n, 64), 64, 0, (cudaStream_t)stream>>>(
        G, pts_d, normals_d, n_rays, radius, dirs_d, tube_r, n, out_d);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
