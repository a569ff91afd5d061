// lbw_kernels_fast.cu — FMA flavour of the collide kernels (LBW_MODE_FAST).
// Compiled with contraction enabled (default -fmad=true).
#define LBW_FAST 1
#include <cstdlib>

#include "lbw_sweep.cuh"
#include "lbw_fused.cuh"

namespace lbw {

cudaError_t launch_fused_fast(int op, bool pull, const FusedArgs& a, size_t smem, cudaStream_t s) {
    const cudaError_t e = launch_fused<5>(op, pull, a, smem, s);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t preload_sweep_cb_fast(int op, bool single) {
    const char* e = getenv("LBW_SWEEP_MINB");
    const int minb = e ? atoi(e) : 5;
    if (single)
        return minb == 6 ? preload_k_sweep_cb<6, float>(op)
               : minb == 4 ? preload_k_sweep_cb<4, float>(op) : preload_k_sweep_cb<5, float>(op);
    return minb == 6 ? preload_k_sweep_cb<6, double>(op)
           : minb == 4 ? preload_k_sweep_cb<4, double>(op) : preload_k_sweep_cb<5, double>(op);
}

cudaError_t launch_sweep_fast(int op, bool pull, const SweepArgs& a, cudaStream_t s) {
    const dim3 blk = sweep_block(a.g);
    const dim3 grd((a.g.nz + blk.x - 1) / blk.x, (a.g.ny + blk.y - 1) / blk.y, a.x_end - a.x_begin);
    if (grd.z == 0) return cudaSuccess;
    SweepArgs b = a;
    b.halo.edge_ctas = grd.x * grd.y * (grd.z < 2 ? grd.z : 2u);
    // occupancy variant of the hot kernel (LBW_SWEEP_MINB=4|5|6 CTAs/SM)
    static const int minb = [] {
        const char* e = getenv("LBW_SWEEP_MINB");
        return e ? atoi(e) : 5;
    }();
    if (a.g.single) {
        if (minb == 6) launch_k_sweep<6, float>(op, pull, grd, blk, b, s);
        else if (minb == 4) launch_k_sweep<4, float>(op, pull, grd, blk, b, s);
        else launch_k_sweep<5, float>(op, pull, grd, blk, b, s);
    } else {
        if (minb == 6) launch_k_sweep<6, double>(op, pull, grd, blk, b, s);
        else if (minb == 4) launch_k_sweep<4, double>(op, pull, grd, blk, b, s);
        else launch_k_sweep<5, double>(op, pull, grd, blk, b, s);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_batch_fast(int op, double* f2, const double* F2, double* macro2, int64_t n,
                              Relax r, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    if (op == 1) k_batch<1><<<blocks, 128, 0, s>>>(f2, F2, macro2, n, r);
    else k_batch<0><<<blocks, 128, 0, s>>>(f2, F2, macro2, n, r);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_block_collide_fast(int op, double* f, const double* force, double* macro,
                                      int64_t nx, int64_t ny, int64_t nz, Relax r,
                                      cudaStream_t s) {
    const int64_t n = nx * ny * nz;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    if (op == 1) k_block_collide<1><<<blocks, 128, 0, s>>>(f, force, macro, nx, ny, nz, r);
    else k_block_collide<0><<<blocks, 128, 0, s>>>(f, force, macro, nx, ny, nz, r);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lbw

LBW_TRACE_EXPORT(fast)
