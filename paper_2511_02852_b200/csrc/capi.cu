// C ABI bookkeeping: error strings, ABI version, device properties.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include "hs_common.cuh"

namespace hs {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

#ifdef HS_EXP_SKIP
bool hs_exp_skip(const char* tag) {
    const char* e = getenv("HS_EXP_SKIP");
    return e && strstr(e, tag) != nullptr;
}
#endif

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < HS_MAX_DEVICES ? dev : 0;
}

int num_sms() {
    static int cached[HS_MAX_DEVICES] = {0};
    const int dev = current_device();
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

}  // namespace hs

extern "C" int hs_abi_version(void) { return HS_ABI_VERSION; }

extern "C" const char* hs_last_error(void) { return hs::g_err; }

// sizeof of each ABI struct, so the ctypes mirror can verify its layout
extern "C" HS_API int hs_struct_size(int which) {
    switch (which) {
        case 0: return (int)sizeof(HsBucket);
        case 1: return (int)sizeof(HsPatch);
        case 2: return (int)sizeof(HsLayer);
        case 3: return (int)sizeof(HsPool);
        case 4: return (int)sizeof(HsFftArgs);
        case 5: return (int)sizeof(HsInjectArgs);
        case 6: return (int)sizeof(HsAdvectArgs);
        case 7: return (int)sizeof(HsSplatArgs);
        case 8: return (int)sizeof(HsSmoothArgs);
        case 9: return (int)sizeof(HsComposeArgs);
        case 10: return (int)sizeof(HsSampleArgs);
        case 11: return (int)sizeof(HsCompositeArgs);
        case 12: return (int)sizeof(HsFinishArgs);
        case 13: return (int)sizeof(HsResidentArgs);
        case 14: return (int)sizeof(HsLayoutArgs);
        case 15: return (int)sizeof(HsSource);
        case 16: return (int)sizeof(HsEmitArgs);
        case 17: return (int)sizeof(HsBody);
        case 18: return (int)sizeof(HsBodyArgs);
        case 19: return (int)sizeof(HsInitArgs);
        case 20: return (int)sizeof(HsBoxArgs);
        default: return -1;
    }
}

extern "C" HS_API int hs_configure_device(void) {
    int rc = 0;
    if (!rc) rc = hs::fft_configure();
    if (!rc) rc = hs::smooth_configure();
    if (!rc) rc = hs::compose_configure();
    if (!rc) rc = hs::particles_configure();
    return rc;
}

// Streams owned by one Simulation (side branches, graph capture), created
// here rather than taken from a framework's shared round-robin pool, so no
// other component (e.g. a collective library) ever issues work on them.
extern "C" HS_API int hs_stream_create(void** stream, int priority) {
    HS_CHECK_ARG(stream != nullptr, "hs_stream_create: null output");
    cudaStream_t s = nullptr;
    HS_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
    *stream = (void*)s;
    return 0;
}

extern "C" HS_API int hs_stream_destroy(void* stream) {
    if (stream) HS_CUDA(cudaStreamDestroy((cudaStream_t)stream));
    return 0;
}
