// Device-side geometry shared by the ray-caster, the AO bake and the point probes.
// Each function restates one numba kernel of the reference (_kernels.py) in IEEE
// float64 without FMA contraction (the TU is compiled with -fmad=false).
#pragma once
#include "lvx_common.cuh"

struct LvxHit {
    double t_in, t_out, nx, ny, nz;
};

// ---------------------------------------------------------------------------
// The encoded segment records (voxelizer.py:79-89, model_io.py:151-179): `width` bytes per
// record, LSB first  face_in(3) bin_in(2 lb) face_out(3) bin_out(2 lb) attr(8) lid(5).
// A frame can be rendered straight from them: 5 bytes per segment at N = 32
// instead of the 32-byte render record, so the whole model stays in L2.
// ---------------------------------------------------------------------------
struct LvxPacked {
    const u8 *bytes;  // 8-byte aligned, readable up to the next multiple of 8 bytes
    int width, lb, n;
    float inv_n;      // 1 / n: n is a power of two, so x * inv_n == x / n exactly (float32 and float64)
};

__device__ __forceinline__ u64 lvx_packed_word(const LvxPacked &P, u32 seg) {
    const size_t off = (size_t)seg * (size_t)P.width;
    const u64 *p = reinterpret_cast<const u64 *>(P.bytes) + (off >> 3);
    const int sh = (int)(off & 7) * 8;
    u64 v = __ldg(p) >> sh;
    if (sh + 8 * P.width > 64) v |= __ldg(p + 1) << (64 - sh);
    return v;
}

struct LvxPackedFields {
    u32 face_in, bin_in, face_out, bin_out, attr, lid;
};
__device__ __forceinline__ LvxPackedFields lvx_packed_fields(const LvxPacked &P, u64 v) {
    const int bb = 2 * P.lb;
    const u64 bmask = ((u64)1 << bb) - 1;
    LvxPackedFields f;
    f.face_in = (u32)(v & 7u);
    f.bin_in = (u32)((v >> 3) & bmask);
    f.face_out = (u32)((v >> (3 + bb)) & 7u);
    f.bin_out = (u32)((v >> (6 + bb)) & bmask);
    f.attr = (u32)((v >> (6 + 2 * bb)) & 0xFFu);
    f.lid = (u32)((v >> (14 + 2 * bb)) & 31u);
    return f;
}

// bin centre of (face, code) in the unit cube of its voxel: exact in float32 (dyadic, <= 9 fraction bits)
__device__ __forceinline__ void lvx_packed_local(u32 face, u32 code, const LvxPacked &P, float out[3]) {
    const int bu = (int)(code & (u32)(P.n - 1)), bv = (int)(code >> P.lb);
    const float cu = ((float)bu + 0.5f) * P.inv_n, cv = ((float)bv + 0.5f) * P.inv_n;
    const int axis = (int)(face >> 1);
    const float side = (float)(face & 1);
    out[0] = axis == 0 ? side : cu;
    out[1] = axis == 1 ? side : (axis == 0 ? cu : cv);
    out[2] = axis == 2 ? side : cv;
}

// the reference's reconstructed endpoint: bin centre + voxel in float64, cast to float32
// (voxelizer.py:376-380, 477-478; model_io.py:169-179) -- the value the render records hold
__device__ __forceinline__ void lvx_packed_point(u32 face, u32 code, const LvxPacked &P, int vx, int vy, int vz,
                                                 float out[3]) {
    const int bu = (int)(code & (u32)(P.n - 1)), bv = (int)(code >> P.lb);
    const double cu = ((double)bu + 0.5) * (double)P.inv_n, cv = ((double)bv + 0.5) * (double)P.inv_n;
    const int axis = (int)(face >> 1);
    const double side = (double)(face & 1);
    out[0] = (float)((axis == 0 ? side : cu) + (double)vx);
    out[1] = (float)((axis == 1 ? side : (axis == 0 ? cu : cv)) + (double)vy);
    out[2] = (float)((axis == 2 ? side : cv) + (double)vz);
}

// intersect_tube_raw, _kernels.py:76-134, in the specialisation the frame kernels
// compile to: the endpoints arrive as float32, numba's float(f32) does not widen,
// so axis, length and normalisation run in float32.
__device__ __forceinline__ bool lvx_tube_f32axis(double ox, double oy, double oz, double dx,
                                                 double dy, double dz, float ax, float ay,
                                                 float az, float bx, float by, float bz, double r,
                                                 LvxHit &h) {
    float ux = bx - ax, uy = by - ay, uz = bz - az;
    const float length = sqrtf(ux * ux + uy * uy + uz * uz);
    if ((double)length < 1e-12) return false;
    ux = ux / length;
    uy = uy / length;
    uz = uz / length;
    const double Ux = (double)ux, Uy = (double)uy, Uz = (double)uz, L = (double)length;
    const double mx = ox - (double)ax, my = oy - (double)ay, mz = oz - (double)az;
    const double du = dx * Ux + dy * Uy + dz * Uz;
    const double mu = mx * Ux + my * Uy + mz * Uz;
    const double nx_ = dx - du * Ux, ny_ = dy - du * Uy, nz_ = dz - du * Uz;
    const double qx = mx - mu * Ux, qy = my - mu * Uy, qz = mz - mu * Uz;
    const double a = nx_ * nx_ + ny_ * ny_ + nz_ * nz_;
    const double c = qx * qx + qy * qy + qz * qz - r * r;
    double t0, t1;
    if (a < 1e-14) {
        if (c > 0.0) return false;
        t0 = -CUDART_INF;
        t1 = CUDART_INF;
    } else {
        const double b = 2.0 * (nx_ * qx + ny_ * qy + nz_ * qz);
        const double disc = b * b - 4.0 * a * c;
        if (disc < 0.0) return false;
        const double sq = sqrt(disc);
        t0 = (-b - sq) / (2.0 * a);
        t1 = (-b + sq) / (2.0 * a);
    }
    if (du == 0.0) {
        if (mu < 0.0 || mu > L) return false;
    } else {
        double s0 = (0.0 - mu) / du;
        double s1 = (L - mu) / du;
        if (s0 > s1) {
            const double t = s0;
            s0 = s1;
            s1 = t;
        }
        if (s0 > t0) t0 = s0;
        if (s1 < t1) t1 = s1;
    }
    if (t1 < t0 || t1 < 0.0) return false;
    const double t_in = t0 > 0.0 ? t0 : 0.0;
    const double px = ox + t_in * dx, py = oy + t_in * dy, pz = oz + t_in * dz;
    const double wx = px - (double)ax, wy = py - (double)ay, wz = pz - (double)az;
    const double wu = wx * Ux + wy * Uy + wz * Uz;
    double rx = wx - wu * Ux, ry = wy - wu * Uy, rz = wz - wu * Uz;
    const double rn = sqrt(rx * rx + ry * ry + rz * rz);
    if (rn < 1e-12) {
        rx = -dx;
        ry = -dy;
        rz = -dz;
    } else {
        rx = rx / rn;
        ry = ry / rn;
        rz = rz / rn;
    }
    h.t_in = t_in;
    h.t_out = t1;
    h.nx = rx;
    h.ny = ry;
    h.nz = rz;
    return true;
}

// The all-float64 specialisation reached through the Python-level
// intersect_ray_tube (raycast.py:184-200).
__device__ __forceinline__ bool lvx_tube_f64(double ox, double oy, double oz, double dx, double dy,
                                             double dz, double ax, double ay, double az, double bx,
                                             double by, double bz, double r, LvxHit &h) {
    double ux = bx - ax, uy = by - ay, uz = bz - az;
    const double length = sqrt(ux * ux + uy * uy + uz * uz);
    if (length < 1e-12) return false;
    ux = ux / length;
    uy = uy / length;
    uz = uz / length;
    const double mx = ox - ax, my = oy - ay, mz = oz - az;
    const double du = dx * ux + dy * uy + dz * uz;
    const double mu = mx * ux + my * uy + mz * uz;
    const double nx_ = dx - du * ux, ny_ = dy - du * uy, nz_ = dz - du * uz;
    const double qx = mx - mu * ux, qy = my - mu * uy, qz = mz - mu * uz;
    const double a = nx_ * nx_ + ny_ * ny_ + nz_ * nz_;
    const double c = qx * qx + qy * qy + qz * qz - r * r;
    double t0, t1;
    if (a < 1e-14) {
        if (c > 0.0) return false;
        t0 = -CUDART_INF;
        t1 = CUDART_INF;
    } else {
        const double b = 2.0 * (nx_ * qx + ny_ * qy + nz_ * qz);
        const double disc = b * b - 4.0 * a * c;
        if (disc < 0.0) return false;
        const double sq = sqrt(disc);
        t0 = (-b - sq) / (2.0 * a);
        t1 = (-b + sq) / (2.0 * a);
    }
    if (du == 0.0) {
        if (mu < 0.0 || mu > length) return false;
    } else {
        double s0 = (0.0 - mu) / du;
        double s1 = (length - mu) / du;
        if (s0 > s1) {
            const double t = s0;
            s0 = s1;
            s1 = t;
        }
        if (s0 > t0) t0 = s0;
        if (s1 < t1) t1 = s1;
    }
    if (t1 < t0 || t1 < 0.0) return false;
    const double t_in = t0 > 0.0 ? t0 : 0.0;
    const double px = ox + t_in * dx, py = oy + t_in * dy, pz = oz + t_in * dz;
    const double wx = px - ax, wy = py - ay, wz = pz - az;
    const double wu = wx * ux + wy * uy + wz * uz;
    double rx = wx - wu * ux, ry = wy - wu * uy, rz = wz - wu * uz;
    const double rn = sqrt(rx * rx + ry * ry + rz * rz);
    if (rn < 1e-12) {
        rx = -dx;
        ry = -dy;
        rz = -dz;
    } else {
        rx = rx / rn;
        ry = ry / rn;
        rz = rz / rn;
    }
    h.t_in = t_in;
    h.t_out = t1;
    h.nx = rx;
    h.ny = ry;
    h.nz = rz;
    return true;
}

// intersect_sphere_raw, _kernels.py:137-159.  WANT_NORMAL=false stops after t_in
// (the ownership test needs nothing else).
template <bool WANT_NORMAL>
__device__ __forceinline__ bool lvx_sphere(double ox, double oy, double oz, double dx, double dy,
                                           double dz, double cx, double cy, double cz, double r,
                                           LvxHit &h) {
    const double mx = ox - cx, my = oy - cy, mz = oz - cz;
    const double b = 2.0 * (dx * mx + dy * my + dz * mz);
    const double c = mx * mx + my * my + mz * mz - r * r;
    const double disc = b * b - 4.0 * c;
    if (disc < 0.0) return false;
    const double sq = sqrt(disc);
    const double t0 = (-b - sq) / 2.0;
    const double t1 = (-b + sq) / 2.0;
    if (t1 < 0.0) return false;
    const double t_in = t0 > 0.0 ? t0 : 0.0;
    h.t_in = t_in;
    h.t_out = t1;
    if (WANT_NORMAL) {
        const double px = ox + t_in * dx, py = oy + t_in * dy, pz = oz + t_in * dz;
        double nx_ = px - cx, ny_ = py - cy, nz_ = pz - cz;
        const double nn = sqrt(nx_ * nx_ + ny_ * ny_ + nz_ * nz_);
        if (nn < 1e-12) {
            nx_ = -dx;
            ny_ = -dy;
            nz_ = -dz;
        } else {
            nx_ = nx_ / nn;
            ny_ = ny_ / nn;
            nz_ = nz_ / nn;
        }
        h.nx = nx_;
        h.ny = ny_;
        h.nz = nz_;
    }
    return true;
}

// dda_collect, _kernels.py:164-256, as an incremental walker: init() does the slab
// clip and the start voxel, next() yields one [t0,t1) window at a time in the
// reference's order (zero-length visits dropped, ties x<=y<=z, tmax accumulated by
// repeated addition exactly like the reference).
struct LvxDda {
    double t_cur, t_exit;
    double tmax_x, tmax_y, tmax_z, tdel_x, tdel_y, tdel_z;
    int ix, iy, iz, step_x, step_y, step_z;
    int ilo, ihx, ihy, ihz;
    bool alive;

    __device__ __forceinline__ void init(double ox, double oy, double oz, double dx, double dy,
                                         double dz, int rx, int ry, int rz, int pad) {
        alive = false;
        double t_enter = -CUDART_INF;
        t_exit = CUDART_INF;
        const double lo = -(double)pad;
        const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
        const double hi[3] = {(double)(rx + pad), (double)(ry + pad), (double)(rz + pad)};
#pragma unroll
        for (int axis = 0; axis < 3; ++axis) {
            if (d[axis] == 0.0) {
                if (o[axis] < lo || o[axis] >= hi[axis]) return;
            } else {
                double ta = (lo - o[axis]) / d[axis];
                double tb = (hi[axis] - o[axis]) / d[axis];
                if (ta > tb) {
                    const double t = ta;
                    ta = tb;
                    tb = t;
                }
                if (ta > t_enter) t_enter = ta;
                if (tb < t_exit) t_exit = tb;
            }
        }
        if (t_enter < 0.0) t_enter = 0.0;
        if (t_exit <= t_enter) return;
        const double px = ox + t_enter * dx, py = oy + t_enter * dy, pz = oz + t_enter * dz;
        ilo = -pad;
        ihx = rx + pad - 1;
        ihy = ry + pad - 1;
        ihz = rz + pad - 1;
        // the clamp keeps huge floors from overflowing the int conversion
        const double fx = floor(px), fy = floor(py), fz = floor(pz);
        ix = fx < (double)ilo ? ilo : (fx > (double)ihx ? ihx : (int)fx);
        iy = fy < (double)ilo ? ilo : (fy > (double)ihy ? ihy : (int)fy);
        iz = fz < (double)ilo ? ilo : (fz > (double)ihz ? ihz : (int)fz);
        step_x = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
        step_y = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
        step_z = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
        const double big = CUDART_INF;
        tmax_x = step_x != 0 ? ((double)(ix + (step_x > 0 ? 1 : 0)) - ox) / dx : big;
        tmax_y = step_y != 0 ? ((double)(iy + (step_y > 0 ? 1 : 0)) - oy) / dy : big;
        tmax_z = step_z != 0 ? ((double)(iz + (step_z > 0 ? 1 : 0)) - oz) / dz : big;
        tdel_x = step_x != 0 ? fabs(1.0 / dx) : big;
        tdel_y = step_y != 0 ? fabs(1.0 / dy) : big;
        tdel_z = step_z != 0 ? fabs(1.0 / dz) : big;
        t_cur = t_enter;
        alive = t_cur < t_exit;
    }

    // Advances to the next non-empty window; returns false when the walk is over.
    __device__ __forceinline__ bool next(int &wx, int &wy, int &wz, double &t0, double &t1) {
        while (alive) {
            double t_next;
            int axis;
            if (tmax_x <= tmax_y && tmax_x <= tmax_z) {
                t_next = tmax_x;
                axis = 0;
            } else if (tmax_y <= tmax_z) {
                t_next = tmax_y;
                axis = 1;
            } else {
                t_next = tmax_z;
                axis = 2;
            }
            const double te = t_next < t_exit ? t_next : t_exit;
            const bool emit = te > t_cur;
            wx = ix;
            wy = iy;
            wz = iz;
            t0 = t_cur;
            t1 = te;
            t_cur = te;
            if (axis == 0) {
                ix += step_x;
                tmax_x += tdel_x;
                if (ix < ilo || ix > ihx) alive = false;
            } else if (axis == 1) {
                iy += step_y;
                tmax_y += tdel_y;
                if (iy < ilo || iy > ihy) alive = false;
            } else {
                iz += step_z;
                tmax_z += tdel_z;
                if (iz < ilo || iz > ihz) alive = false;
            }
            if (!(t_cur < t_exit)) alive = false;
            if (emit) return true;
        }
        return false;
    }
};

// sample_field_trilinear, _kernels.py:346-383
__device__ __forceinline__ double lvx_trilinear(const float *__restrict__ flat, i64 off, int ldx,
                                                int ldy, int ldz, double scale, double x, double y,
                                                double z) {
    // x / scale: the scale of a LoD level is a power of two, and dividing by 2^e IS multiplying by 2^-e
    // (the same real operation, rounded the same way) -- three float64 divisions less per sample
    double qx, qy, qz;
    {
        const long long sb = __double_as_longlong(scale);
        const int ef = (int)((sb >> 52) & 0x7FF);
        if ((sb & 0x800FFFFFFFFFFFFFll) == 0 && ef >= 1 && ef <= 2045) {
            const double inv = __longlong_as_double((long long)(2046 - ef) << 52);
            qx = x * inv - 0.5;
            qy = y * inv - 0.5;
            qz = z * inv - 0.5;
        } else {
            qx = x / scale - 0.5;
            qy = y / scale - 0.5;
            qz = z / scale - 0.5;
        }
    }
    const double flx = floor(qx), fly = floor(qy), flz = floor(qz);
    const double fx = qx - flx, fy = qy - fly, fz = qz - flz;
    // clamp in floating point first so far-away queries cannot overflow the int cast (to [-1, dim-1]:
    // the two cell indices are then integer clamps of ix and ix + 1 -- the reference's
    // clip(floor, 0, dim-1) and clip(floor + 1, 0, dim-1))
    const int ix = (int)fmin(fmax(flx, -1.0), (double)(ldx - 1));
    const int iy = (int)fmin(fmax(fly, -1.0), (double)(ldy - 1));
    const int iz = (int)fmin(fmax(flz, -1.0), (double)(ldz - 1));
    const int x0 = max(ix, 0), x1 = min(ix + 1, ldx - 1);
    const int y0 = max(iy, 0), y1 = min(iy + 1, ldy - 1);
    const int z0 = max(iz, 0), z1 = min(iz + 1, ldz - 1);
    const i64 sy = ldx, sz = (i64)ldx * ldy;
    const float *f = flat + off;
    const double v000 = (double)__ldg(f + z0 * sz + y0 * sy + x0), v001 = (double)__ldg(f + z0 * sz + y0 * sy + x1);
    const double v010 = (double)__ldg(f + z0 * sz + y1 * sy + x0), v011 = (double)__ldg(f + z0 * sz + y1 * sy + x1);
    const double v100 = (double)__ldg(f + z1 * sz + y0 * sy + x0), v101 = (double)__ldg(f + z1 * sz + y0 * sy + x1);
    const double v110 = (double)__ldg(f + z1 * sz + y1 * sy + x0), v111 = (double)__ldg(f + z1 * sz + y1 * sy + x1);
    const double c00 = v000 * (1.0 - fx) + v001 * fx;
    const double c01 = v010 * (1.0 - fx) + v011 * fx;
    const double c10 = v100 * (1.0 - fx) + v101 * fx;
    const double c11 = v110 * (1.0 - fx) + v111 * fx;
    const double c0 = c00 * (1.0 - fy) + c01 * fy;
    const double c1 = c10 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

// Octree view passed by value to kernels (from lvx_lod).
struct LvxOctree {
    const float *flat;
    i64 off[LVX_MAX_LEVELS + 1];
    int dims[LVX_MAX_LEVELS * 3];
    int n_levels;
};

// cone_blocking, _kernels.py:386-422.  The reference picks the level with
// floor(log2(width)); width is max(t,1) with t = 0.5 + sum of powers of two, so
// the value equals the binary exponent of width exactly (no libm call needed).
__device__ __forceinline__ double lvx_cone_blocking(double px, double py, double pz, double lx,
                                                    double ly, double lz, const LvxOctree &oc,
                                                    double gx, double gy, double gz, double eps_T) {
    double t_cur = 0.5, T = 1.0;
    const double max_d = sqrt(gx * gx + gy * gy + gz * gz);
    while (t_cur < max_d) {
        const double x = px + t_cur * lx, y = py + t_cur * ly, z = pz + t_cur * lz;
        if (x < 0.0 || y < 0.0 || z < 0.0 || x > gx || y > gy || z > gz) break;
        const double width = t_cur < 1.0 ? 1.0 : t_cur;
        // (width >= 1 is a normal number: its binary exponent is the biased exponent field - 1023)
        int level = (int)((__double_as_longlong(width) >> 52) & 0x7FF) - 1023;
        if (level < 0) level = 0;
        if (level > oc.n_levels - 1) level = oc.n_levels - 1;
        const double step = (double)((i64)1 << level);
        const double rho = lvx_trilinear(oc.flat, oc.off[level], oc.dims[3 * level],
                                         oc.dims[3 * level + 1], oc.dims[3 * level + 2], step, x, y, z);
        double ext = 1.0 - rho * step;
        if (ext < 0.0) ext = 0.0;
        T *= ext;
        if (T <= eps_T) {
            T = 0.0;
            break;
        }
        t_cur += step;
    }
    return 1.0 - T;
}

// density_ray_blocking, _kernels.py:425-445 (level 0 only)
__device__ __forceinline__ double lvx_density_ray(double px, double py, double pz, double dx,
                                                  double dy, double dz, const float *__restrict__ l0,
                                                  int gxi, int gyi, int gzi, double radius,
                                                  double step) {
    const double gx = (double)gxi, gy = (double)gyi, gz = (double)gzi;
    double acc = 0.0, t_cur = step;
    while (t_cur <= radius) {
        const double x = px + t_cur * dx, y = py + t_cur * dy, z = pz + t_cur * dz;
        if (x < 0.0 || y < 0.0 || z < 0.0 || x > gx || y > gy || z > gz) break;
        acc += lvx_trilinear(l0, 0, gxi, gyi, gzi, 1.0, x, y, z) * step;
        if (acc >= 1.0) return 1.0;
        t_cur += step;
    }
    return acc < 1.0 ? acc : 1.0;
}

// orient_frame, _kernels.py:555-569
__device__ __forceinline__ void lvx_orient_frame(double nx, double ny, double nz, double t[3],
                                                 double b[3]) {
    double tx, ty, tz;
    if (fabs(nx) > 0.9) {
        tx = 0.0;
        ty = 1.0;
        tz = 0.0;
    } else {
        tx = 1.0;
        ty = 0.0;
        tz = 0.0;
    }
    const double d = tx * nx + ty * ny + tz * nz;
    tx = tx - d * nx;
    ty = ty - d * ny;
    tz = tz - d * nz;
    const double tn = sqrt(tx * tx + ty * ty + tz * tz);
    tx = tx / tn;
    ty = ty / tn;
    tz = tz / tn;
    t[0] = tx;
    t[1] = ty;
    t[2] = tz;
    b[0] = ny * tz - nz * ty;
    b[1] = nz * tx - nx * tz;
    b[2] = nx * ty - ny * tx;
}

// ao_density_point, _kernels.py:592-605.  `dirs` is the host-built Fibonacci
// lattice (fibonacci_dir with libm cos/sin, bit-identical to the reference).
__device__ __forceinline__ double lvx_ao_density_point(double px, double py, double pz, double nx,
                                                       double ny, double nz, int n_rays,
                                                       double radius, double step,
                                                       const double *__restrict__ dirs,
                                                       const float *__restrict__ l0, int gx, int gy,
                                                       int gz) {
    double total = 0.0, t[3], b[3];
    lvx_orient_frame(nx, ny, nz, t, b);
    for (int i = 0; i < n_rays; ++i) {
        const double lx = dirs[3 * i], ly = dirs[3 * i + 1], lz = dirs[3 * i + 2];
        const double dx = lx * t[0] + ly * b[0] + lz * nx;
        const double dy = lx * t[1] + ly * b[1] + lz * ny;
        const double dz = lx * t[2] + ly * b[2] + lz * nz;
        total += lvx_density_ray(px, py, pz, dx, dy, dz, l0, gx, gy, gz, radius, step);
    }
    return total / (double)n_rays;
}

// ---------------------------------------------------------------------------
// Geometry secondary rays: geometry_ray_blocked / ao_hemisphere_point,
// _kernels.py:450-495, 572-589.
// ---------------------------------------------------------------------------

// What the secondary rays read of the voxel model.
struct LvxGeomModel {
    int rx, ry, rz;
    const u8 *counts;
    const u32 *offsets;
    const lvx_seg_record *rec;
    const u32 *nmask;  // occupancy bits of the 27-neighbourhood over the padded grid (lvx_neighbor_sums)
};

// 27-neighbourhood mask `e` of the cell a walk just left, re-expressed around the cell it
// moved to (step per axis in {-1, 0, 1}); voxels leaving the 3x3x3 frame drop out.
__device__ __forceinline__ u32 lvx_shift_mask27(u32 e, int dx, int dy, int dz) {
    if (dx > 0) e = (e & 0x6DB6DB6u) >> 1;
    else if (dx < 0) e = (e & 0x36DB6DBu) << 1;
    if (dy > 0) e = (e & 0x7E3F1F8u) >> 3;
    else if (dy < 0) e = (e & 0x0FC7E3Fu) << 3;
    if (dz > 0) e = (e & 0x7FFFE00u) >> 9;
    else if (dz < 0) e = (e & 0x003FFFFu) << 9;
    return e;
}

// geometry_ray_blocked, _kernels.py:450-495: true if any tube (or joint sphere) is entered
// by the ray at 1e-9 < t_in < max_t.  The reference walks the padded grid and tests the 27
// neighbours of every window that starts before max_t; the answer is a disjunction over
// (ray, segment) pairs, so each voxel is tested once (the first time a window sees it), only
// voxels within tube radius of the ray piece are listed (a hit's entry point lies in some
// window and within the radius of its segment), and a conservative float32 distance test
// runs ahead of the exact float64 ones.  Same set of hits, same boolean.
__device__ inline bool lvx_geometry_blocked(double ox, double oy, double oz, double dx, double dy,
                                            double dz, double max_t, const LvxGeomModel &M, double radius,
                                            bool joints) {
    LvxDda dda;
    dda.init(ox, oy, oz, dx, dy, dz, M.rx, M.ry, M.rz, 1);
    if (!dda.alive) return false;
    const double cull = radius + 1e-4;
    const float reach_pt = (float)radius + 2e-3f;
    const float fdx = (float)dx, fdy = (float)dy, fdz = (float)dz;
    u32 listed = 0;
    int px = 0, py = 0, pz = 0;
    int wx, wy, wz;
    double t0, t1;
    while (dda.next(wx, wy, wz, t0, t1)) {
        if (t0 >= max_t) break;
        if (listed) {
            const int sx = wx - px, sy = wy - py, sz = wz - pz;
            listed = (sx < -1 || sx > 1 || sy < -1 || sy > 1 || sz < -1 || sz > 1) ? 0u
                                                                                 : lvx_shift_mask27(listed, sx, sy, sz);
        }
        px = wx;
        py = wy;
        pz = wz;
        u32 nm = __ldg(M.nmask + (((i64)(wz + 1) * (M.ry + 2) + (wy + 1)) * (M.rx + 2) + (wx + 1)));
        if (nm == 0) continue;
        const double p0x = ox + t0 * dx, p0y = oy + t0 * dy, p0z = oz + t0 * dz;
        const double p1x = ox + t1 * dx, p1y = oy + t1 * dy, p1z = oz + t1 * dz;
        u32 bx_ = 0x2492492u, by_ = 0x0E07038u, bz_ = 0x003FE00u;
        if (fmin(p0x, p1x) - cull < (double)wx) bx_ |= 0x1249249u;
        if (fmax(p0x, p1x) + cull > (double)(wx + 1)) bx_ |= 0x4924924u;
        if (fmin(p0y, p1y) - cull < (double)wy) by_ |= 0x01C0E07u;
        if (fmax(p0y, p1y) + cull > (double)(wy + 1)) by_ |= 0x70381C0u;
        if (fmin(p0z, p1z) - cull < (double)wz) bz_ |= 0x00001FFu;
        if (fmax(p0z, p1z) + cull > (double)(wz + 1)) bz_ |= 0x7FC0000u;
        nm &= bx_ & by_ & bz_;
        const u32 fresh = nm & ~listed;
        listed |= nm;
        for (u32 mm = fresh; mm; mm &= mm - 1) {
            const int b = __ffs((int)mm) - 1;
            const int bz = b / 9, by = (b - 9 * bz) / 3, bx = b - 9 * bz - 3 * by;
            const int hx = wx + bx - 1, hy = wy + by - 1, hz = wz + bz - 1;
            const u32 lin = (u32)(hx + M.rx * (hy + M.ry * hz));
            const u32 cnt = __ldg(M.counts + lin), base = __ldg(M.offsets + lin);
            // voxel-local float32 frame
            const float q0x = (float)(p0x - (double)hx), q0y = (float)(p0y - (double)hy),
                        q0z = (float)(p0z - (double)hz);
            const float fhx = (float)hx, fhy = (float)hy, fhz = (float)hz;
            for (u32 s = 0; s < cnt; ++s) {
                const float4 ra = __ldg(reinterpret_cast<const float4 *>(M.rec + base + s));
                const float4 rb = __ldg(reinterpret_cast<const float4 *>(M.rec + base + s) + 1);
                {
                    // bounding sphere of the segment (tube and both joints) against the ray's line
                    const float cx = 0.5f * ((ra.x - fhx) + (rb.x - fhx)) - q0x, cy = 0.5f * ((ra.y - fhy) + (rb.y - fhy)) - q0y,
                                cz = 0.5f * ((ra.z - fhz) + (rb.z - fhz)) - q0z;
                    const float tc = cx * fdx + cy * fdy + cz * fdz;
                    const float reach = rb.w + reach_pt;
                    if ((cx * cx + cy * cy + cz * cz) - tc * tc > reach * reach) continue;
                }
                LvxHit h;
                if (lvx_tube_f32axis(ox, oy, oz, dx, dy, dz, ra.x, ra.y, ra.z, rb.x, rb.y, rb.z, radius, h) &&
                    1e-9 < h.t_in && h.t_in < max_t)
                    return true;
                if (joints) {
                    if (lvx_sphere<false>(ox, oy, oz, dx, dy, dz, (double)ra.x, (double)ra.y, (double)ra.z, radius, h) &&
                        1e-9 < h.t_in && h.t_in < max_t)
                        return true;
                    if (lvx_sphere<false>(ox, oy, oz, dx, dy, dz, (double)rb.x, (double)rb.y, (double)rb.z, radius, h) &&
                        1e-9 < h.t_in && h.t_in < max_t)
                        return true;
                }
            }
        }
    }
    return false;
}

// ao_hemisphere_point, _kernels.py:572-589 (jitter 0: `dirs` is the host-built hemisphere
// lattice, see lvx_ao_density_point)
__device__ inline double lvx_ao_hemisphere_point(double px, double py, double pz, double nx, double ny,
                                                 double nz, int n_rays, double radius,
                                                 const double *__restrict__ dirs, const LvxGeomModel &M,
                                                 double tube_r) {
    int blocked = 0;
    double t[3], b[3];
    lvx_orient_frame(nx, ny, nz, t, b);
    const double ox = px + 1e-3 * nx, oy = py + 1e-3 * ny, oz = pz + 1e-3 * nz;
    for (int i = 0; i < n_rays; ++i) {
        const double lx = dirs[3 * i], ly = dirs[3 * i + 1], lz = dirs[3 * i + 2];
        const double dx = lx * t[0] + ly * b[0] + lz * nx;
        const double dy = lx * t[1] + ly * b[1] + lz * ny;
        const double dz = lx * t[2] + ly * b[2] + lz * nz;
        if (lvx_geometry_blocked(ox, oy, oz, dx, dy, dz, radius, M, tube_r, true)) blocked += 1;
    }
    return (double)blocked / (double)n_rays;
}

// One level of the representative-line field (lvx_rep.cu).
struct LvxRepLevel {
    const u8 *valid;
    const float *a, *b, *w;
    int dx, dy, dz;
    double size;  // 2^level grid units
};

// replines_ray_blocked, _kernels.py:498-538: shadow test against one representative line
// per coarse voxel; the radius grows with the aggregated weight (clamped to [1, 4]).  The
// reference walks the coarse grid and tests the 27 neighbours of every window that starts
// before max_t; the answer is a disjunction, so each coarse voxel is tested once.
__device__ inline bool lvx_replines_blocked(double ox, double oy, double oz, double dx, double dy, double dz,
                                            double max_t, const LvxRepLevel &R, double radius_base) {
    LvxDda dda;
    dda.init(ox / R.size, oy / R.size, oz / R.size, dx, dy, dz, R.dx, R.dy, R.dz, 1);
    if (!dda.alive) return false;
    u32 listed = 0;
    int px = 0, py = 0, pz = 0;
    int wx, wy, wz;
    double t0, t1;
    while (dda.next(wx, wy, wz, t0, t1)) {
        if (t0 * R.size >= max_t) break;
        if (listed) {
            const int sx = wx - px, sy = wy - py, sz = wz - pz;
            listed = (sx < -1 || sx > 1 || sy < -1 || sy > 1 || sz < -1 || sz > 1) ? 0u
                                                                                 : lvx_shift_mask27(listed, sx, sy, sz);
        }
        px = wx;
        py = wy;
        pz = wz;
        const u32 fresh = 0x7FFFFFFu & ~listed;
        listed = 0x7FFFFFFu;
        for (u32 mm = fresh; mm; mm &= mm - 1) {
            const int b = __ffs((int)mm) - 1;
            const int bz = b / 9, by = (b - 9 * bz) / 3, bx = b - 9 * bz - 3 * by;
            const int hx = wx + bx - 1, hy = wy + by - 1, hz = wz + bz - 1;
            if (hx < 0 || hy < 0 || hz < 0 || hx >= R.dx || hy >= R.dy || hz >= R.dz) continue;
            const i64 lin = hx + (i64)R.dx * (hy + (i64)R.dy * hz);
            if (!R.valid[lin]) continue;
            double wgt = (double)R.w[lin];
            wgt = wgt < 1.0 ? 1.0 : (wgt > 4.0 ? 4.0 : wgt);
            LvxHit h;
            if (lvx_tube_f32axis(ox, oy, oz, dx, dy, dz, R.a[3 * lin], R.a[3 * lin + 1], R.a[3 * lin + 2], R.b[3 * lin],
                                 R.b[3 * lin + 1], R.b[3 * lin + 2], radius_base * wgt, h) &&
                1e-9 < h.t_in && h.t_in < max_t)
                return true;
        }
    }
    return false;
}

// shade_scalar, _kernels.py:316-329
__device__ __forceinline__ double lvx_shade(double nx, double ny, double nz, double lx, double ly,
                                            double lz, double vx, double vy, double vz, double ka,
                                            double kd, double ks, double shininess) {
    double ndl = nx * lx + ny * ly + nz * lz;
    if (ndl < 0.0) ndl = 0.0;
    const double hx = lx + vx, hy = ly + vy, hz = lz + vz;
    const double hn = sqrt(hx * hx + hy * hy + hz * hz);
    double spec = 0.0;
    if (hn > 1e-12) {
        const double ndh = (nx * hx + ny * hy + nz * hz) / hn;
        if (ndh > 0.0) spec = pow(ndh, shininess);
    }
    return ka + kd * ndl + ks * spec;
}

// _alpha_of, _kernels.py:332-341
__device__ __forceinline__ double lvx_alpha_of(int mode, double base_alpha, double table_alpha,
                                               double t_in, double t_out) {
    if (mode == LVX_OPACITY_CONSTANT) return base_alpha;
    if (mode == LVX_OPACITY_TRANSFER) return table_alpha;
    double span = t_out - t_in;
    if (span < 0.0) span = 0.0;
    return 1.0 - pow(1.0 - base_alpha, span);
}
