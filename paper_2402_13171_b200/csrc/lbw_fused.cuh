// lbw_fused.cuh — the fused time step: ONE launch per step on a single slab
// with device kinematics and at most 64 actuator points (on-the-fly force
// sums).  Included by each flavour's translation unit after lbw_sweep.cuh.
//
// Launch m (step m) carries three kinds of CTA, told apart by block index:
//
//   KK      CTA 0 (when the pipeline is full): kinematics of step m+2
//           (turbine-tree walk + point frames, turbine.py:227-311) and its
//           flow-independent geometry -- deposit cells / Roma weights, the
//           force rows it will tag, the rows of its sampling cubes
//           (fs_geometry).  Step m+2 is two launches away, so nothing in
//           this launch reads what it writes.
//   helper  the next ceil(P/4) CTAs: each warp claims point tasks K4(m)
//           (sample the macro of collide m-1 at the trilinear cube, blade
//           element force from the polar, lattice force; actuator.py:70-146,
//           sim.py:193-235) from a counter until none is left.
//   sweep   the rest: pull-stream-collide of one tile, exactly k_sweep.  A
//           tile whose rows carry step m's force (row tag m+1, set by KK(m))
//           needs every point force first: it claims any task still
//           unclaimed itself, then waits for the done counter.  Every
//           claimed task is executed by a running warp, so the wait cannot
//           deadlock whatever order the CTAs are scheduled in (no CTA ever
//           waits for a CTA that may not be resident).  Tiles holding rows
//           of step m+1's sampling cubes store the (rho, u) their collide
//           computes into the sample pool, so K4(m+1) reads 8 x 4 values per
//           point from L2 instead of re-streaming 8 x 27 populations.
//
// Launches follow each other with programmatic dependent launch: launch
// m+1 starts its CTAs while launch m drains, and reads nothing before
// launch m has completed (griddepcontrol.wait).
#pragma once

#include "lbw_chain.cuh"

namespace lbw {
namespace LBW_FLAVOR {
namespace {

// The actuator paths run out of line with their inputs passed BY VALUE:
// a reference into the kernel's parameter block would make the compiler
// copy the whole block (~1.5 KB) to local memory at kernel entry in every
// thread, and inlined they would share (and spill) the sweep's registers.
// The copies are made at the call sites only, i.e. in the rare branches.

// A warp claims point tasks K4(m) until none is left (all lanes call).
__device__ __forceinline__ unsigned long long fs_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __noinline__ void fs_claim_tasks(const AlmDev a, const Geom g, const MacroDev md,
                                            const FsPool pool, int use_pool, uint32_t* ctr,
                                            int lane, unsigned long long* prof) {
    const FsPool* pp = use_pool ? &pool : nullptr;
    while (true) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(ctr, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= (uint32_t)a.n) break;
        const PointInputs in = load_point_inputs(a, (int)t, lane);
        ForceSet none{};   // the rows were tagged by KK(m): nothing to tag here
        CubeArgs cube{};
        point_warp(a, g, md, none, 0, cube, (int)t, lane, in, pp, false);
        __syncwarp();
        if (lane == 0) {
            __threadfence();   // this task's stores before its completion count
            const uint32_t done = atomicAdd(ctr + 1, 1u);
            if (prof && done + 1 == (uint32_t)a.n) prof[3] = fs_now();
        }
    }
}

__device__ __forceinline__ void fs_claim(const FusedArgs& A, int lane) {
    fs_claim_tasks(A.a, A.sw.g, A.md, A.pool, A.use_pool, A.ctr, lane, A.prof);
}

// KK(m+2): kinematics, then the geometry of that step (whole CTA)
__device__ __noinline__ void fs_kk(const KinDev k, const AlmDev ak, const Geom g,
                                   const FsGeom geo, int per_x, double* sm, int tid, int nthr) {
    kinematics_cta(k, ak, g, per_x, 1, sm, tid, nthr);
    __syncthreads();
    fs_geometry(geo, ak, g, per_x, tid, nthr);
}

// Whole CTA: help with the point tasks, then wait until all are done.
__device__ __forceinline__ void fs_help_and_wait(const FusedArgs& A, int tid) {
    fs_claim(A, tid & 31);
    if (tid == 0) {
        const uint32_t* done = A.ctr + 1;
        const uint32_t n = (uint32_t)A.a.n;
        while (true) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
            if (v >= n) break;
            __nanosleep(32);
        }
        if (A.prof) atomicMax(A.prof + 4, fs_now());
    }
    __syncthreads();
}

template <int OP, bool PULL, class T>
__device__ __forceinline__ void fused_tile(const FusedArgs& A, int x, int y, int z, bool valid,
                                           int tid) {
    const SweepArgs& a = A.sw;
    const Geom& g = a.g;
    uint64_t key = 0ull, skey = 0ull;
    if (valid) {
        key = a.fv.row_key[(int64_t)x * g.ny + y];
        skey = A.skey_next[(int64_t)x * g.ny + y];
    }
    // tiles holding force rows of step m need every point force first (the
    // wait comes before the population loads: nothing large is live across it)
    const bool need = valid && (uint32_t)(key >> 32) == a.fv.tag;
    if (__syncthreads_or(need)) fs_help_and_wait(A, tid);
    if (!valid) return;
    const T* src = static_cast<const T*>(a.src);
    double f[27];
    if (PULL && pull_is_simple(g, x, y, z)) load_cell_simple(src, g, x, y, z, f);
    else load_cell<PULL>(src, g, x, y, z, f);
    double Fx, Fy, Fz;
    force_from_key<T>(a.fv, g, key, x, y, z, Fx, Fy, Fz);
    const Macro m = collide_cell<OP>(f, Fx, Fy, Fz, a.r);
    flag_nonfinite<T>(a.nan_key, a.step, ((g.x0 + x) * g.ny + y) * (int64_t)g.nz + z, m);
    T* d = static_cast<T*>(a.dst) + buf_index(g, x + 1, 0, y, z);
#pragma unroll
    for (int i = 0; i < 27; ++i) st_pop(d + i * (int)g.dir_stride, f[i]);
    if ((uint32_t)(skey >> 32) == A.store_tag) {
        // the macro this collide wrote (sim.py:27-28) for step m+1's sampling
        const Macro ms = stored_macro(g, m);
        double* b = A.spool_next + (int64_t)(uint32_t)skey * 4 * g.zp + z;
        b[0] = ms.rho;
        b[g.zp] = ms.ux;
        b[2 * g.zp] = ms.uy;
        b[3 * g.zp] = ms.uz;
    }
}

template <int OP, bool PULL, int MINB, class T>
__global__ void __launch_bounds__(kSweepThreads, MINB) k_step_fused(FusedArgs A) {
    extern __shared__ double fs_sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int tid = (int)(threadIdx.x + threadIdx.y * blockDim.x);
    const int nthr = (int)(blockDim.x * blockDim.y);
    int b = (int)blockIdx.x;
    if (A.prof && tid == 0) atomicMin(A.prof, fs_now());
    if (b == 0 && tid == 0) {
        // the next launch's task counters (nothing in this launch uses them)
        A.ctr_next[0] = 0u;
        A.ctr_next[1] = 0u;
        if (A.prof_next) {
            A.prof_next[0] = ~0ull;
            for (int k = 1; k < 8; ++k) A.prof_next[k] = 0ull;
        }
    }
    if (b < A.n_kk) {
        if (A.prof && tid == 0) A.prof[1] = fs_now();
        fs_kk(A.k, A.a_kk, A.sw.g, A.geo, A.per_x, fs_sm, tid, nthr);
        if (A.prof && tid == 0) A.prof[2] = fs_now();
        return;
    }
    b -= A.n_kk;
    if (b < A.n_help) {
        fs_claim(A, tid & 31);
        return;
    }
    b -= A.n_help;
    const Geom& g = A.sw.g;
    const uint32_t bx = (uint32_t)b % A.tiles_x;
    const uint32_t by = ((uint32_t)b / A.tiles_x) % A.tiles_y;
    const int bz = (int)((uint32_t)b / (A.tiles_x * A.tiles_y));
    const int z = (int)(bx * blockDim.x + threadIdx.x);
    const int y = (int)(by * blockDim.y + threadIdx.y);
    const int np = A.sw.x_end - A.sw.x_begin;
    const int x = A.sw.x_begin + (A.sw.reverse ? np - 1 - bz : bz);
    fused_tile<OP, PULL, T>(A, x, y, z, z < g.nz && y < g.ny, tid);
    if (A.prof) {
        __syncthreads();
        if (tid == 0) atomicMax(A.prof + 5, fs_now());
    }
}

template <int OP, bool PULL, int MINB, class T>
cudaError_t launch_fused_one(const FusedArgs& A, unsigned grid, dim3 blk, size_t smem,
                             cudaStream_t s) {
    auto kern = k_step_fused<OP, PULL, MINB, T>;
    if (smem > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = blk;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = sweep_pdl() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, A);
}

template <int MINB>
cudaError_t launch_fused(int op, bool pull, const FusedArgs& A0, size_t smem, cudaStream_t s) {
    const dim3 blk = sweep_block(A0.sw.g);
    FusedArgs A = A0;
    A.tiles_x = (A.sw.g.nz + blk.x - 1) / blk.x;
    A.tiles_y = (A.sw.g.ny + blk.y - 1) / blk.y;
    const unsigned planes = (unsigned)(A.sw.x_end - A.sw.x_begin);
    const unsigned grid = (unsigned)(A.n_kk + A.n_help) + A.tiles_x * A.tiles_y * planes;
    const bool single = A.sw.g.single != 0;
    if (op == 1) {
        if (pull) return single ? launch_fused_one<1, true, MINB, float>(A, grid, blk, smem, s)
                                : launch_fused_one<1, true, MINB, double>(A, grid, blk, smem, s);
        return single ? launch_fused_one<1, false, MINB, float>(A, grid, blk, smem, s)
                      : launch_fused_one<1, false, MINB, double>(A, grid, blk, smem, s);
    }
    if (pull) return single ? launch_fused_one<0, true, MINB, float>(A, grid, blk, smem, s)
                            : launch_fused_one<0, true, MINB, double>(A, grid, blk, smem, s);
    return single ? launch_fused_one<0, false, MINB, float>(A, grid, blk, smem, s)
                  : launch_fused_one<0, false, MINB, double>(A, grid, blk, smem, s);
}

}  // namespace
}  // namespace LBW_FLAVOR
}  // namespace lbw
