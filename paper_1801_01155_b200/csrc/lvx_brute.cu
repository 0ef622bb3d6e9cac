// Brute-force reference renderer for sm_100a: every primitive tested against every pixel,
// no DDA, no windows, no ownership -- the algorithm of the reference's own brute-force
// renderer
//
//   (all-primitives frame kernel)   _kernels.py:926-1082
//   brute_force_render   metrics.py:58-107
//
// which the reference's tests use to check its accelerated renderer.  It shares nothing
// with the two frame engines except the primitive tests, the shading terms and the
// compositing rules, so agreement between them is evidence about traversal and gathering.
//
//   count      one thread per pixel loops over ALL segments (the whole warp reads the same
//              record: broadcast loads), a conservative midpoint-distance bound, then the exact
//              float64 tests; counts the pixel's hits
//   (scan of the counts on the caller's side -> offsets)
//   fill       the same loop again, now writing the first MAX_PIXEL_HITS hits of the pixel in
//              collection order, each with its state-free shading terms
//   composite  one thread per pixel: hits in the reference's total order (t_in, home voxel,
//              lid, kind, collection order), de-duplication, blending, termination
#include <math_constants.h>

#include "lvx_geom.cuh"
#include "lvx_shade.cuh"

namespace {

constexpr int kMaxPixelHits = 8192;  // _kernels.py:37 MAX_PIXEL_HITS
constexpr int kBruteSort = 64;

struct BruteArgs {
    lvx_camera cam;
    lvx_params p;
    int rx, ry, rz;
    const u8 *counts;
    const u32 *offsets;
    const lvx_seg_record *rec;
    const float *table;
    const u32 *nmask;
    LvxOctree oc;
    const float *ao_flat;
    const double *ao_dirs;
    LvxRepLevel rep;
    double rep_radius_base;
    i64 n_seg;
    const u32 *seg_lin;  // home voxel of every segment
    u32 *hit_count;      // [W*H] hits found (uncapped)
    const i64 *hit_off;  // [W*H] first slot of the pixel's hits
    double *hit_t;       // per hit: t_in
    unsigned long long *hit_key;  // lin << 24 | lid << 19 | (kind != tube) << 18 | index in voxel << 10 | kind3 << 8 | attr
    double *hit_scale, *hit_alpha;
    float *hit_c;        // [3] sphere centre
    float *img;
    unsigned long long *row_stats;
};

__device__ __forceinline__ void pixel_ray(const lvx_camera &cam, int x, int y, double &ddx, double &ddy,
                                          double &ddz) {
    // _kernels.py:958-965
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

// FILL = false: count the hits of every pixel.  FILL = true: store the first kMaxPixelHits.
template <bool FILL, bool GEOM>
__global__ void __launch_bounds__(128) brute_kernel(const BruteArgs A) {
    const int W = A.cam.width, H = A.cam.height;
    const i64 pix = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = pix < (i64)W * H;
    const int x = active ? (int)(pix % W) : 0, y = active ? (int)(pix / W) : 0;
    double ddx, ddy, ddz;
    pixel_ray(A.cam, x, y, ddx, ddy, ddz);
    const double ox = A.cam.o[0], oy = A.cam.o[1], oz = A.cam.o[2];
    const double tube_r = A.p.tube_r;
    const bool joints = A.p.joints != 0;
    // conservative bound (the reference uses the same idea, :970-979): every capsule point lies
    // within half_len + radius of the segment's midpoint (half_len is rounded up, plus a margin)
    const double reach0 = tube_r + 1e-6;
    u32 n = 0;
    const i64 base = FILL && active ? A.hit_off[pix] : 0;
    for (i64 i = 0; i < A.n_seg; ++i) {
        const float4 ra = __ldg(reinterpret_cast<const float4 *>(A.rec + i));
        const float4 rb = __ldg(reinterpret_cast<const float4 *>(A.rec + i) + 1);
        if (!active) continue;
        {
            // |w x d|^2 = squared distance of the midpoint to the ray's line (float64: the
            // camera is far from the grid, a float32 form would cancel)
            const double wx = 0.5 * ((double)ra.x + (double)rb.x) - ox, wy = 0.5 * ((double)ra.y + (double)rb.y) - oy,
                         wz = 0.5 * ((double)ra.z + (double)rb.z) - oz;
            const double cxd = wy * ddz - wz * ddy, cyd = wz * ddx - wx * ddz, czd = wx * ddy - wy * ddx;
            const double reach = (double)rb.w + reach0;
            if (cxd * cxd + cyd * cyd + czd * czd > reach * reach) continue;
        }
        const u32 rmeta = __float_as_uint(ra.w);
        const u32 attr = rmeta & 0xFFu, lid = (rmeta >> 8) & 31u;
#pragma unroll 1
        for (u32 kind3 = 0; kind3 < (joints ? 3u : 1u); ++kind3) {
            LvxHit h;
            bool hit;
            float cx = 0.0f, cy = 0.0f, cz = 0.0f;
            if (kind3 == 0) {
                hit = lvx_tube_f32axis(ox, oy, oz, ddx, ddy, ddz, ra.x, ra.y, ra.z, rb.x, rb.y, rb.z, tube_r, h);
            } else {
                cx = kind3 == 1 ? ra.x : rb.x;
                cy = kind3 == 1 ? ra.y : rb.y;
                cz = kind3 == 1 ? ra.z : rb.z;
                hit = lvx_sphere<true>(ox, oy, oz, ddx, ddy, ddz, (double)cx, (double)cy, (double)cz, tube_r, h);
            }
            if (!hit) continue;
            if (FILL && n < (u32)kMaxPixelHits) {
                const u32 lin = A.seg_lin[i];
                const u32 rank = (u32)(i - (i64)A.offsets[lin]);
                double scale, alpha;
                lvx_shade_hit<GEOM>(A, ox, oy, oz, ddx, ddy, ddz, h, attr, scale, alpha);
                const i64 e = base + n;
                A.hit_t[e] = h.t_in;
                A.hit_key[e] = ((unsigned long long)lin << 24) | ((unsigned long long)lid << 19) |
                               (kind3 ? 1ull << 18 : 0ull) | ((unsigned long long)(rank & 255u) << 10) |
                               ((unsigned long long)kind3 << 8) | attr;
                A.hit_scale[e] = scale;
                A.hit_alpha[e] = alpha;
                A.hit_c[3 * e] = cx;
                A.hit_c[3 * e + 1] = cy;
                A.hit_c[3 * e + 2] = cz;
            }
            n += 1;
        }
    }
    if (!FILL && active) A.hit_count[pix] = n;
}

__device__ __forceinline__ bool brute_before(double ta, unsigned long long ka, double tb, unsigned long long kb) {
    // _hit_before (_kernels.py:261-270), ties in collection order
    return ta < tb || (ta == tb && (ka >> 8) < (kb >> 8));
}

struct BrutePixel {
    double acc[4];
    int n_seen, n_sph;
    u32 seen_key[LVX_MAX_SEEN], seen_mask[LVX_MAX_SEEN];
    float sph[LVX_MAX_SEEN][3];
};

// stream_hit's stateful half (_kernels.py:666-670, 719-730)
__device__ __forceinline__ void brute_accumulate(BrutePixel &S, const float *table, double scale, double alpha,
                                                 u32 lin, u32 lid, u32 attr, bool is_sphere, float cx, float cy,
                                                 float cz) {
    if (is_sphere) {
        for (int i = 0; i < S.n_sph; ++i)
            if (S.sph[i][0] == cx && S.sph[i][1] == cy && S.sph[i][2] == cz) return;
    }
    {
        const u32 bit = 1u << lid;
        bool found = false;
        for (int i = 0; i < S.n_seen; ++i) {
            if (S.seen_key[i] == lin) {
                if (S.seen_mask[i] & bit) return;
                S.seen_mask[i] |= bit;
                found = true;
                break;
            }
        }
        if (!found && S.n_seen < LVX_MAX_SEEN) {
            S.seen_key[S.n_seen] = lin;
            S.seen_mask[S.n_seen] = bit;
            S.n_seen += 1;
        }
    }
    const float4 col = __ldg(reinterpret_cast<const float4 *>(table) + attr);
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
    }
}

__global__ void __launch_bounds__(64) brute_composite_kernel(const BruteArgs A) {
    const int W = A.cam.width, H = A.cam.height;
    const i64 pix = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= (i64)W * H) return;
    const u32 found = A.hit_count[pix];
    const u32 n = found < (u32)kMaxPixelHits ? found : (u32)kMaxPixelHits;
    const i64 base = A.hit_off[pix];
    BrutePixel S;
    S.acc[0] = S.acc[1] = S.acc[2] = S.acc[3] = 0.0;
    S.n_seen = 0;
    S.n_sph = 0;
    const double tau = A.p.tau;
    auto composite = [&](i64 e) {
        const unsigned long long k = A.hit_key[e];
        brute_accumulate(S, A.table, A.hit_scale[e], A.hit_alpha[e], (u32)(k >> 24), (u32)(k >> 19) & 31u,
                         (u32)k & 0xFFu, ((k >> 8) & 3ull) != 0, A.hit_c[3 * e], A.hit_c[3 * e + 1], A.hit_c[3 * e + 2]);
        return S.acc[3] >= tau;
    };
    if (n <= (u32)kBruteSort) {
        double s_t[kBruteSort];
        unsigned long long s_k[kBruteSort];
        u32 s_i[kBruteSort];
        for (u32 j = 0; j < n; ++j) {
            const double t = A.hit_t[base + j];
            const unsigned long long k = A.hit_key[base + j];
            int pos = (int)j;
            while (pos > 0 && brute_before(t, k, s_t[pos - 1], s_k[pos - 1])) {
                s_t[pos] = s_t[pos - 1];
                s_k[pos] = s_k[pos - 1];
                s_i[pos] = s_i[pos - 1];
                --pos;
            }
            s_t[pos] = t;
            s_k[pos] = k;
            s_i[pos] = j;
        }
        for (u32 j = 0; j < n; ++j)
            if (composite(base + s_i[j])) break;
    } else {
        // selection: repeatedly the smallest key after the last composited one
        bool have_last = false;
        double lt = 0.0;
        unsigned long long lk = 0;
        for (;;) {
            i64 best = -1;
            double bt = 0.0;
            unsigned long long bk = 0;
            for (u32 j = 0; j < n; ++j) {
                const double t = A.hit_t[base + j];
                const unsigned long long k = A.hit_key[base + j];
                if (have_last && !brute_before(lt, lk, t, k)) continue;
                if (best < 0 || brute_before(t, k, bt, bk)) {
                    best = base + j;
                    bt = t;
                    bk = k;
                }
            }
            if (best < 0) break;
            if (composite(best)) break;
            have_last = true;
            lt = bt;
            lk = bk;
        }
    }
    // _kernels.py:1070-1074
    const lvx_params &p = A.p;
    const double a = S.acc[3];
    float4 outp;
    outp.x = (float)(S.acc[0] + (1.0 - a) * p.bg[3] * p.bg[0]);
    outp.y = (float)(S.acc[1] + (1.0 - a) * p.bg[3] * p.bg[1]);
    outp.z = (float)(S.acc[2] + (1.0 - a) * p.bg[3] * p.bg[2]);
    outp.w = (float)(a + (1.0 - a) * p.bg[3]);
    reinterpret_cast<float4 *>(A.img)[pix] = outp;
    if (found > n) atomicAdd(A.row_stats + 3 * (pix / W) + 2, (unsigned long long)(found - n));
}

__global__ void brute_row_stats_kernel(unsigned long long *row_stats, int H, unsigned long long tests_per_row) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y < H) row_stats[3 * y + 1] = tests_per_row;  // definitional (:1076-1080)
}

int fill_args(BruteArgs &A, const lvx_camera *cam, const lvx_model *model, const lvx_params *params,
              const lvx_lod *lod) {
    LVX_REQUIRE(cam && model && params, "null argument");
    LVX_REQUIRE(cam->width >= 1 && cam->height >= 1, "image dims must be >= 1");
    LVX_REQUIRE(model->rx >= 1 && model->ry >= 1 && model->rz >= 1 && model->counts_d && model->offsets_d &&
                    model->table_d,
                "bad model");
    LVX_REQUIRE(params->opacity_mode >= 0 && params->opacity_mode <= 2, "bad opacity mode");
    LVX_REQUIRE(params->shadow_mode >= LVX_SHADOW_NONE && params->shadow_mode <= LVX_SHADOW_CONE, "bad shadow_mode");
    LVX_REQUIRE(params->ao_mode >= LVX_AO_NONE && params->ao_mode <= LVX_AO_PRECOMPUTED, "bad ao_mode");
    LVX_REQUIRE((params->shadow_mode != LVX_SHADOW_HARD && params->ao_mode != LVX_AO_HEMISPHERE) || model->nmask_d,
                "geometry secondary rays need the neighbour grids (lvx_neighbor_sums)");
    LVX_REQUIRE(params->shadow_mode != LVX_SHADOW_REPLINES || (lod && lod->rep.valid_d),
                "replines shadows need a representative-line level (lvx_lod.rep)");
    const bool need_oct = params->shadow_mode == LVX_SHADOW_CONE || params->ao_mode == LVX_AO_DENSITY;
    LVX_REQUIRE(!need_oct || (lod && lod->oct_flat_d && lod->n_levels >= 1 && lod->n_levels <= LVX_MAX_LEVELS),
                "cone shadows / density-rays AO need a density octree");
    LVX_REQUIRE(params->ao_mode != LVX_AO_PRECOMPUTED || (lod && lod->ao_flat_d), "precomputed AO needs the AO field");
    LVX_REQUIRE((params->ao_mode != LVX_AO_DENSITY && params->ao_mode != LVX_AO_HEMISPHERE) ||
                    (lod && lod->ao_dirs_d && params->ao_n_rays >= 1),
                "density-rays / hemisphere AO need the direction lattice");
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
    A.nmask = model->nmask_d;
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
    return LVX_OK;
}

}  // namespace

extern "C" {

int lvx_brute_count(const lvx_camera *cam, const lvx_model *model, const lvx_params *params, int64_t n_seg,
                    uint32_t *hit_count_d, void *stream) {
    BruteArgs A;
    LVX_REQUIRE(params, "null argument");
    lvx_params q = *params;  // (the count pass runs no shading: no illumination inputs needed)
    q.shadow_mode = LVX_SHADOW_NONE;
    q.ao_mode = LVX_AO_NONE;
    if (int rc = fill_args(A, cam, model, &q, nullptr)) return rc;
    LVX_REQUIRE(hit_count_d && n_seg >= 0 && (n_seg == 0 || model->seg_rec_d), "bad arguments");
    A.n_seg = n_seg;
    A.hit_count = hit_count_d;
    const i64 px = (i64)cam->width * cam->height;
    brute_kernel<false, false><<<(unsigned)lvx_ceil_div(px, 128), 128, 0, (cudaStream_t)stream>>>(A);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_brute_render(const lvx_camera *cam, const lvx_model *model, const lvx_params *params, const lvx_lod *lod,
                     int64_t n_seg, const uint32_t *seg_lin_d, uint32_t *hit_count_d, const int64_t *hit_off_d,
                     double *hit_t_d, uint64_t *hit_key_d, double *hit_scale_d, double *hit_alpha_d, float *hit_c_d,
                     float *img_d, int64_t *row_stats_d, void *stream) {
    BruteArgs A;
    if (int rc = fill_args(A, cam, model, params, lod)) return rc;
    LVX_REQUIRE(hit_count_d && hit_off_d && img_d && row_stats_d && n_seg >= 0, "bad arguments");
    LVX_REQUIRE(n_seg == 0 || (model->seg_rec_d && seg_lin_d && hit_t_d && hit_key_d && hit_scale_d && hit_alpha_d &&
                               hit_c_d),
                "null hit buffers");
    A.n_seg = n_seg;
    A.seg_lin = seg_lin_d;
    A.hit_count = hit_count_d;
    A.hit_off = hit_off_d;
    A.hit_t = hit_t_d;
    A.hit_key = reinterpret_cast<unsigned long long *>(hit_key_d);
    A.hit_scale = hit_scale_d;
    A.hit_alpha = hit_alpha_d;
    A.hit_c = hit_c_d;
    A.img = img_d;
    A.row_stats = reinterpret_cast<unsigned long long *>(row_stats_d);
    cudaStream_t st = (cudaStream_t)stream;
    const i64 px = (i64)cam->width * cam->height;
    const bool geom = params->shadow_mode == LVX_SHADOW_HARD || params->shadow_mode == LVX_SHADOW_REPLINES ||
                      params->ao_mode == LVX_AO_HEMISPHERE;
    if (geom) brute_kernel<true, true><<<(unsigned)lvx_ceil_div(px, 128), 128, 0, st>>>(A);
    else brute_kernel<true, false><<<(unsigned)lvx_ceil_div(px, 128), 128, 0, st>>>(A);
    LVX_LAUNCH_CHECK();
    brute_composite_kernel<<<(unsigned)lvx_ceil_div(px, 64), 64, 0, st>>>(A);
    LVX_LAUNCH_CHECK();
    const unsigned long long per_row = (unsigned long long)(params->joints ? 3 : 1) * (unsigned long long)n_seg *
                                       (unsigned long long)cam->width;
    brute_row_stats_kernel<<<(unsigned)lvx_ceil_div(cam->height, 128), 128, 0, st>>>(A.row_stats, cam->height, per_row);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
