// Shared host/device helpers for liblinevox_b200.so (sm_100a only).
//
// Arithmetic contract: the reference is IEEE float64 (and a few float32 islands)
// with NO fused multiply-add.  Every translation unit is compiled with
// -fmad=false so `a*b+c` stays two roundings; f32 divide/sqrt keep the default
// IEEE-exact (-prec-div/-prec-sqrt) code paths.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/linevox_b200.h"

typedef int64_t i64;
typedef uint8_t u8;
typedef uint16_t u16;
typedef uint32_t u32;
typedef uint64_t u64;

void lvx_set_error(const char *fmt, ...);

#define LVX_CUDA_CHECK(expr)                                                            \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            lvx_set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,                 \
                          cudaGetErrorString(_e));                                      \
            return LVX_E_CUDA;                                                          \
        }                                                                               \
    } while (0)

#define LVX_LAUNCH_CHECK() LVX_CUDA_CHECK(cudaGetLastError())

#define LVX_REQUIRE(cond, ...)                                                          \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            lvx_set_error(__VA_ARGS__);                                                 \
            return LVX_E_INVALID;                                                       \
        }                                                                               \
    } while (0)

static inline i64 lvx_ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }

// number of SMs of the current device (148 on B200); grids of persistent-style
// kernels are sized as a multiple of it
int lvx_sm_count();

// Upper bound of half the segment length (bounding-sphere radius about the midpoint),
// stored in lvx_seg_record::half_len for the frame kernel's conservative pre-reject.
__host__ __device__ __forceinline__ float lvx_half_len(float ax, float ay, float az, float bx,
                                                       float by, float bz) {
    const float ux = bx - ax, uy = by - ay, uz = bz - az;
    return 0.5f * sqrtf(ux * ux + uy * uy + uz * uz) * 1.0001f + 1e-6f;
}

#ifdef __CUDACC__
// 32-byte (one sector) global accesses: sm_100 has 256-bit vector loads/stores
// (LDG/STG.E.ENL2.256).  `p` must be 32-byte aligned.
__device__ __forceinline__ void lvx_st256(void *p, u64 a, u64 b, u64 c, u64 d) {
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void lvx_ld256(const void *p, u64 &a, u64 &b, u64 &c, u64 &d) {
    asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
#endif
