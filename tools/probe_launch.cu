// probe_launch.cu — back-to-back kernel gaps on a plain stream vs a green-
// context stream, alone and with a second stream busy beside it (used to
// find where the 64^3 rotor step loses time between kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_launch tools/probe_launch.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// every CTA spins `ns` from its own start; CTA 0 / the last CTA record the
// kernel's first start and last end
__global__ void spin(unsigned long long ns, unsigned long long* rec, int i) {
    const unsigned long long t0 = gtime();
    if (threadIdx.x == 0) atomicMin(&rec[2 * i], t0);
    while (gtime() - t0 < ns) {
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&rec[2 * i + 1], gtime());
}

#define CK(x)                                                               \
    do {                                                                    \
        auto e = (x);                                                       \
        if (e != 0) {                                                       \
            printf("error %d at %s:%d\n", (int)e, __FILE__, __LINE__);      \
            return 1;                                                       \
        }                                                                   \
    } while (0)

static void report(const char* name, const std::vector<unsigned long long>& r, int n) {
    double gap = 0, dur = 0;
    int k = 0;
    for (int i = 5; i < n; ++i, ++k) {
        gap += (double)(r[2 * i] - r[2 * (i - 1) + 1]) * 1e-3;
        dur += (double)(r[2 * i + 1] - r[2 * i]) * 1e-3;
    }
    printf("%-44s kernel %6.2f us, gap to previous %6.2f us\n", name, dur / k, gap / k);
}

int run(const char* name, cudaStream_t a, cudaStream_t b, int ctas_a, int ctas_b, bool events,
        unsigned long long* rec_a, unsigned long long* rec_b) {
    const int n = 60;
    std::vector<unsigned long long> init(2 * n);
    for (int i = 0; i < n; ++i) init[2 * i] = ~0ull, init[2 * i + 1] = 0;
    CK(cudaMemcpy(rec_a, init.data(), 16 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(rec_b, init.data(), 16 * n, cudaMemcpyHostToDevice));
    cudaEvent_t ea[n], eb[n];
    for (int i = 0; i < n; ++i) {
        cudaEventCreateWithFlags(&ea[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&eb[i], cudaEventDisableTiming);
    }
    CK(cudaDeviceSynchronize());
    for (int i = 0; i < n; ++i) {
        if (events && i > 0) CK(cudaStreamWaitEvent(a, eb[i - 1], 0));
        spin<<<ctas_a, 128, 0, a>>>(18000, rec_a, i);
        if (events) CK(cudaEventRecord(ea[i], a));
        if (b) {
            if (events) CK(cudaStreamWaitEvent(b, ea[i], 0));
            spin<<<ctas_b, 32, 0, b>>>(12000, rec_b, i);
            if (events) CK(cudaEventRecord(eb[i], b));
        }
    }
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> ra(2 * n), rb(2 * n);
    CK(cudaMemcpy(ra.data(), rec_a, 16 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rb.data(), rec_b, 16 * n, cudaMemcpyDeviceToHost));
    char buf[128];
    snprintf(buf, sizeof buf, "%s: A", name);
    report(buf, ra, n);
    if (b) {
        snprintf(buf, sizeof buf, "%s: B", name);
        report(buf, rb, n);
    }
    for (int i = 0; i < n; ++i) {
        cudaEventDestroy(ea[i]);
        cudaEventDestroy(eb[i]);
    }
    return 0;
}

int main() {
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    unsigned long long *ra, *rb;
    CK(cudaMalloc(&ra, 16 * 64));
    CK(cudaMalloc(&rb, 16 * 64));
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi));
    // 140 SMs x 5 CTAs: one wave
    if (run("plain stream", s1, nullptr, 700, 0, false, ra, rb)) return 1;
    if (run("plain + hi-prio stream", s1, s2, 700, 18, false, ra, rb)) return 1;
    if (run("plain + hi-prio stream, events", s1, s2, 700, 18, true, ra, rb)) return 1;

    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all, part, rest;
    unsigned nb = 1;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    CK(cuDevSmResourceSplitByCount(&part, &nb, &all, &rest, 0, 8));
    CUdevResourceDesc dp, dr;
    CUgreenCtx gp, gr;
    CK(cuDevResourceGenerateDesc(&dp, &part, 1));
    CK(cuDevResourceGenerateDesc(&dr, &rest, 1));
    CK(cuGreenCtxCreate(&gp, dp, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream g1, g2;
    CK(cuGreenCtxStreamCreate(&g1, gr, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&g2, gp, CU_STREAM_NON_BLOCKING, hi));
    printf("partition: %u + %u SMs\n", part.sm.smCount, rest.sm.smCount);
    if (run("green stream", (cudaStream_t)g1, nullptr, 700, 0, false, ra, rb)) return 1;
    if (run("green + green(8 SMs) stream", (cudaStream_t)g1, (cudaStream_t)g2, 700, 18, false, ra,
            rb))
        return 1;
    if (run("green + green(8 SMs) stream, events", (cudaStream_t)g1, (cudaStream_t)g2, 700, 18,
            true, ra, rb))
        return 1;
    // the rotor pipeline's stream shape without cross-stream dependencies
    // of the main stream: A sweeps back to back; B (8 SMs) a chain kernel +
    // an event record per step; C (8 SMs) a kinematics kernel waiting on
    // B's event of the step before
    CUstream g3;
    CK(cuGreenCtxStreamCreate(&g3, gp, CU_STREAM_NON_BLOCKING, hi));
    {
        const int n = 60;
        unsigned long long* rc;
        CK(cudaMalloc(&rc, 16 * 64));
        std::vector<unsigned long long> init(2 * n);
        for (int i = 0; i < n; ++i) init[2 * i] = ~0ull, init[2 * i + 1] = 0;
        for (int variant = 0; variant < 3; ++variant) {
            CK(cudaMemcpy(ra, init.data(), 16 * n, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(rb, init.data(), 16 * n, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(rc, init.data(), 16 * n, cudaMemcpyHostToDevice));
            cudaEvent_t eb[n];
            for (int i = 0; i < n; ++i) cudaEventCreateWithFlags(&eb[i], cudaEventDisableTiming);
            CK(cudaDeviceSynchronize());
            for (int i = 0; i < n; ++i) {
                spin<<<700, 128, 0, (cudaStream_t)g1>>>(18000, ra, i);
                if (variant >= 1) {
                    spin<<<18, 32, 0, (cudaStream_t)g2>>>(12000, rb, i);
                    CK(cudaEventRecord(eb[i], (cudaStream_t)g2));
                }
                if (variant >= 2) {
                    if (i > 0) CK(cudaStreamWaitEvent((cudaStream_t)g3, eb[i - 1], 0));
                    spin<<<1, 256, 0, (cudaStream_t)g3>>>(8000, rc, i);
                }
            }
            CK(cudaDeviceSynchronize());
            std::vector<unsigned long long> va(2 * n), vb(2 * n), vc(2 * n);
            CK(cudaMemcpy(va.data(), ra, 16 * n, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(vb.data(), rb, 16 * n, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(vc.data(), rc, 16 * n, cudaMemcpyDeviceToHost));
            printf("pipeline variant %d\n", variant);
            report("  A (sweep-like)", va, n);
            if (variant >= 1) report("  B (chain-like + record)", vb, n);
            if (variant >= 2) report("  C (kin-like, waits B)", vc, n);
        }
    }
    return 0;
}
