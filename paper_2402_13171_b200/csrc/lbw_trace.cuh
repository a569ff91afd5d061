// lbw_trace.cuh — optional kernel timeline (build with EXTRA=-DLBW_TRACE):
// the first block start and the last block end of each kernel, per step, in
// %globaltimer ns, kept per translation unit and read back by
// lbw_trace_dump_<tu>().  Compiled out of the normal library.
#pragma once
#ifdef LBW_TRACE
static __device__ unsigned long long lbw_trace_tab[8][64][2];
__device__ __forceinline__ unsigned long long lbw_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define LBW_TRACE_BEGIN(id, step)                                                   \
    do {                                                                            \
        if (threadIdx.x == 0 && threadIdx.y == 0)                                   \
            atomicMin(&lbw_trace_tab[id][(step) & 63][0], lbw_gtime());             \
    } while (0)
#define LBW_TRACE_END(id, step)                                                     \
    do {                                                                            \
        if (threadIdx.x == 0 && threadIdx.y == 0)                                   \
            atomicMax(&lbw_trace_tab[id][(step) & 63][1], lbw_gtime());             \
    } while (0)
// recorded by the calling thread (the caller picks one)
#define LBW_TRACE_END_HERE(id, step) \
    atomicMax(&lbw_trace_tab[id][(step) & 63][1], lbw_gtime())
#define LBW_TRACE_EXPORT(tu)                                                        \
    extern "C" int lbw_trace_dump_##tu(unsigned long long* out) {                  \
        cudaDeviceSynchronize();                                                    \
        return (int)cudaMemcpyFromSymbol(out, lbw_trace_tab, sizeof(lbw_trace_tab)); \
    }                                                                               \
    extern "C" int lbw_trace_reset_##tu(void) {                                     \
        static unsigned long long init[8][64][2];                                   \
        for (int i = 0; i < 8; ++i)                                                 \
            for (int j = 0; j < 64; ++j) init[i][j][0] = ~0ull, init[i][j][1] = 0;  \
        cudaDeviceSynchronize();                                                    \
        return (int)cudaMemcpyToSymbol(lbw_trace_tab, init, sizeof(init));          \
    }
#else
#define LBW_TRACE_BEGIN(id, step) \
    do {                          \
    } while (0)
#define LBW_TRACE_END(id, step) \
    do {                        \
    } while (0)
#define LBW_TRACE_END_HERE(id, step) \
    do {                             \
    } while (0)
#define LBW_TRACE_EXPORT(tu)
#endif
