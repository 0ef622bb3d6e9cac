// Library-wide pieces of the C ABI: error channel, device check, host helpers.
#include <math.h>
#include <stdarg.h>

#include "lvx_common.cuh"

static thread_local char g_err[512] = "";

void lvx_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int lvx_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return n > 0 ? n : 148;
}

extern "C" {

int lvx_abi_version(void) { return LVX_ABI_VERSION; }

const char *lvx_last_error(void) { return g_err; }

int lvx_device_check(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        lvx_set_error("no CUDA device visible: liblinevox_b200 has no CPU fallback");
        return LVX_E_NO_DEVICE;
    }
    int dev = 0, major = 0;
    LVX_CUDA_CHECK(cudaGetDevice(&dev));
    LVX_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) {
        lvx_set_error("device %d has compute capability %d.x; this library is built for sm_100a only",
                      dev, major);
        return LVX_E_NO_DEVICE;
    }
    return LVX_OK;
}

// fibonacci_dir, _kernels.py:541-552, evaluated on the host with libm so the table
// is bit-identical to what the reference's numba code computes per ray.
int lvx_fibonacci_dirs(int32_t n, int32_t hemisphere, double jitter, double *out_host) {
    LVX_REQUIRE(n >= 1 && out_host, "bad arguments");
    const double golden = 2.399963229728653;
    for (int i = 0; i < n; ++i) {
        double z;
        if (hemisphere != 0) z = 1.0 - ((double)i + 0.5) / (double)n;
        else z = 1.0 - 2.0 * ((double)i + 0.5) / (double)n;
        const double rho = sqrt(fmax(0.0, 1.0 - z * z));
        const double phi = golden * (double)i + jitter * 6.283185307179586;
        out_host[3 * i] = rho * cos(phi);
        out_host[3 * i + 1] = rho * sin(phi);
        out_host[3 * i + 2] = z;
    }
    return LVX_OK;
}

}  // extern "C"
