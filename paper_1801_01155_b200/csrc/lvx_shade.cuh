// The state-free half of stream_hit (_kernels.py:673-718) shared by the frame engines and the
// brute-force renderer: shadow term, AO term, alpha, Blinn scale of one hit.  `ArgsT` is a
// kernel argument block with the fields p, rx, ry, rz, oc, ao_flat, ao_dirs, table, counts,
// offsets, rec, nmask, rep, rep_radius_base.  GEOM: the frame uses secondary rays against
// geometry (hard / replines shadows, hemisphere AO); kept out of the common instantiations.
#pragma once
#include "lvx_geom.cuh"

template <bool GEOM, class ArgsT>
__device__ __forceinline__ void lvx_shade_hit(const ArgsT &A, double ox, double oy, double oz, double ddx,
                                         double ddy, double ddz, const LvxHit &h, u32 attr,
                                         double &scale_out, double &alpha_out) {
    const lvx_params &p = A.p;
    const double gx = (double)A.rx, gy = (double)A.ry, gz = (double)A.rz;
    const double px = ox + h.t_in * ddx, py = oy + h.t_in * ddy, pz = oz + h.t_in * ddz;
    double shadow_term = 0.0;
    if (p.shadow_mode == LVX_SHADOW_CONE) {
        shadow_term = lvx_cone_blocking(px, py, pz, p.light[0], p.light[1], p.light[2], A.oc, gx, gy, gz, 0.01);
    } else if (GEOM && p.shadow_mode == LVX_SHADOW_HARD) {
        const LvxGeomModel G = {A.rx, A.ry, A.rz, A.counts, A.offsets, A.rec, A.nmask};
        if (lvx_geometry_blocked(px + 1e-3 * h.nx, py + 1e-3 * h.ny, pz + 1e-3 * h.nz, p.light[0], p.light[1],
                                 p.light[2], 1e30, G, p.tube_r, p.joints != 0))
            shadow_term = 1.0;
    } else if (GEOM && p.shadow_mode == LVX_SHADOW_REPLINES) {
        if (lvx_replines_blocked(px + 1e-3 * h.nx, py + 1e-3 * h.ny, pz + 1e-3 * h.nz, p.light[0], p.light[1],
                                 p.light[2], 1e30, A.rep, A.rep_radius_base))
            shadow_term = 1.0;
    }
    double ao_term = 0.0;
    if (p.ao_mode == LVX_AO_PRECOMPUTED) {
        ao_term = lvx_trilinear(A.ao_flat, 0, A.rx, A.ry, A.rz, 1.0, px, py, pz);
        if (ao_term > 1.0) ao_term = 1.0;
        if (ao_term < 0.0) ao_term = 0.0;
    } else if (p.ao_mode == LVX_AO_DENSITY) {
        ao_term = lvx_ao_density_point(px, py, pz, h.nx, h.ny, h.nz, p.ao_n_rays, p.ao_radius, 1.0,
                                       A.ao_dirs, A.oc.flat, A.rx, A.ry, A.rz);
    } else if (GEOM && p.ao_mode == LVX_AO_HEMISPHERE) {
        const LvxGeomModel G = {A.rx, A.ry, A.rz, A.counts, A.offsets, A.rec, A.nmask};
        ao_term = lvx_ao_hemisphere_point(px, py, pz, h.nx, h.ny, h.nz, p.ao_n_rays, p.ao_radius, A.ao_dirs, G,
                                          p.tube_r);
    }
    const float table_alpha = __ldg(A.table + 4 * attr + 3);
    alpha_out = lvx_alpha_of(p.opacity_mode, p.base_alpha, (double)table_alpha, h.t_in, h.t_out);
    double lgx, lgy, lgz;
    if (p.headlight != 0) {
        lgx = -ddx;
        lgy = -ddy;
        lgz = -ddz;
    } else {
        lgx = p.light[0];
        lgy = p.light[1];
        lgz = p.light[2];
    }
    double scale = lvx_shade(h.nx, h.ny, h.nz, lgx, lgy, lgz, -ddx, -ddy, -ddz, p.ka * (1.0 - ao_term),
                             p.kd, p.ks, p.shininess);
    scale *= 1.0 - shadow_term;
    scale_out = scale;
}

