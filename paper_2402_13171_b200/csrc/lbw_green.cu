// lbw_green.cu — SM partition between the sweep and the actuator chain.
//
// The actuator chain (kinematics, sampling / blade forces, fill) of step
// n+1 runs beside sweep n.  On a shared SM its single warp per point
// competes with five resident sweep CTAs for the FP64 pipe and waits on a
// saturated memory system (2-3x slower than alone, tools/trace_timeline.py),
// and on small lattices that latency, not the sweep, sets the step time.
// With a partition the chain owns a few SMs (a green context) and the sweep
// the rest: the sweep is HBM-bound, so it loses nothing measurable, and the
// chain runs at its unloaded speed.  Streams of both green contexts share
// the primary context's memory and events, so nothing else changes.
//
// The partition costs the sweep 8 of 148 SMs (~1.7 % at C2), so by default
// it is used only on slabs small enough for the chain's latency to matter
// (< 3.5 M cells: a sweep under ~230 us).  LBW_ALM_SMS (env) overrides:
// 0 never, N > 0 always with N SMs.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "lbw_domain.h"

namespace lbw {
namespace {

struct GreenApi {
    decltype(&cuDeviceGetDevResource) get_resource = nullptr;
    decltype(&cuDevSmResourceSplitByCount) split = nullptr;
    decltype(&cuDevResourceGenerateDesc) gen_desc = nullptr;
    decltype(&cuGreenCtxCreate) create = nullptr;
    decltype(&cuGreenCtxStreamCreate) stream_create = nullptr;
    decltype(&cuGreenCtxDestroy) destroy = nullptr;
    decltype(&cuDeviceGet) device_get = nullptr;
    bool ok = false;
};

const GreenApi& api() {
    static GreenApi a = [] {
        GreenApi g;
        auto load = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || !*fn) {
                cudaGetLastError();
                *fn = nullptr;
            }
        };
        load("cuDeviceGetDevResource", (void**)&g.get_resource);
        load("cuDevSmResourceSplitByCount", (void**)&g.split);
        load("cuDevResourceGenerateDesc", (void**)&g.gen_desc);
        load("cuGreenCtxCreate", (void**)&g.create);
        load("cuGreenCtxStreamCreate", (void**)&g.stream_create);
        load("cuGreenCtxDestroy", (void**)&g.destroy);
        load("cuDeviceGet", (void**)&g.device_get);
        g.ok = g.get_resource && g.split && g.gen_desc && g.create && g.stream_create &&
               g.destroy && g.device_get;
        return g;
    }();
    return a;
}

}  // namespace

// A profiler or sanitizer injected into the process (ncu, compute-sanitizer)
// serialises kernels: no partition then, so no sweep ever waits in-kernel
// for a chain kernel that the tool has not run yet.
// (ncu and compute-sanitizer load an injection library into the target:
// look for it among the mapped objects, and for the variables they use.)
bool tool_injected() {
    static const bool injected = [] {
        if (getenv("CUDA_INJECTION64_PATH") || getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR"))
            return true;
        FILE* f = fopen("/proc/self/maps", "r");
        if (!f) return false;
        char line[4096];
        bool hit = false;
        while (!hit && fgets(line, sizeof line, f))
            hit = strstr(line, "injection") != nullptr || strstr(line, "Injection") != nullptr ||
                  strstr(line, "sanitizer") != nullptr;
        fclose(f);
        return hit;
    }();
    return injected;
}

int alm_sm_count(const lbw_domain* d) {
    if (tool_injected()) return 0;
    const char* e = getenv("LBW_ALM_SMS");
    if (e) return atoi(e);
    const int64_t cells = (int64_t)d->g.nxl * d->g.ny * d->g.nz;
    return cells < 3500000 ? 8 : 0;
}

int green_partition(lbw_domain* d, int alm_sms) {
    if (d->green_sweep || alm_sms <= 0) return LBW_OK;
    const GreenApi& g = api();
    if (!g.ok) return LBW_OK;   // no green contexts: keep the shared streams
    CUdevice dev;
    if (g.device_get(&dev, d->device) != CUDA_SUCCESS) return LBW_OK;
    CUdevResource all, part, rest;
    unsigned nb = 1;
    if (g.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
        all.sm.smCount < (unsigned)(4 * alm_sms) ||
        g.split(&part, &nb, &all, &rest, 0, (unsigned)alm_sms) != CUDA_SUCCESS || nb != 1)
        return LBW_OK;
    CUdevResourceDesc dp, dr;
    CUgreenCtx gp = nullptr, gr = nullptr;
    if (g.gen_desc(&dp, &part, 1) != CUDA_SUCCESS || g.gen_desc(&dr, &rest, 1) != CUDA_SUCCESS ||
        g.create(&gp, dp, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
        return LBW_OK;
    if (g.create(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) {
        g.destroy(gp);
        return LBW_OK;
    }
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUstream sm = nullptr, sa = nullptr;
    if (g.stream_create(&sm, gr, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
        g.stream_create(&sa, gp, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) {
        if (sm) cudaStreamDestroy((cudaStream_t)sm);
        g.destroy(gp);
        g.destroy(gr);
        return LBW_OK;
    }
    // swap the domain's streams (everything queued so far has completed)
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    cudaStreamDestroy(d->stream);
    cudaStreamDestroy(d->alm_stream);
    d->stream = (cudaStream_t)sm;
    d->alm_stream = (cudaStream_t)sa;
    d->green_sweep = gr;
    d->green_alm = gp;
    d->alm_sms = (int)part.sm.smCount;
    return LBW_OK;
}

// a further stream on the chain's SMs (the kinematics stream), or nullptr
cudaStream_t green_alm_stream(lbw_domain* d) {
    if (!d->green_alm) return nullptr;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUstream s = nullptr;
    if (api().stream_create(&s, (CUgreenCtx)d->green_alm, CU_STREAM_NON_BLOCKING, hi) !=
        CUDA_SUCCESS)
        return nullptr;
    return (cudaStream_t)s;
}

void green_release(lbw_domain* d) {
    if (d->stream && d->green_sweep) {
        cudaStreamSynchronize(d->stream);
        cudaStreamDestroy(d->stream);
        d->stream = nullptr;
    }
    if (d->alm_stream && d->green_alm) {
        cudaStreamSynchronize(d->alm_stream);
        cudaStreamDestroy(d->alm_stream);
        d->alm_stream = nullptr;
    }
    if (api().ok) {
        if (d->green_sweep) api().destroy((CUgreenCtx)d->green_sweep);
        if (d->green_alm) api().destroy((CUgreenCtx)d->green_alm);
    }
    d->green_sweep = d->green_alm = nullptr;
}

}  // namespace lbw
