// lbw_sweep.cuh — kernel templates shared by the exact and fast translation
// units.  Each TU defines LBW_FAST (0/1) before including this header and
// instantiates only its own flavour, so the exact kernels never see a
// contracting compiler (-fmad=false is a per-TU flag).
#pragma once
#include <cstdlib>

#include "lbw_internal.h"
#include "lbw_trace.cuh"

#ifndef LBW_FAST
#error "define LBW_FAST before including lbw_sweep.cuh"
#endif

// Kernels get a per-flavour namespace: identical template kernels in two
// translation units would share one weak host stub, and the runtime would
// launch whichever TU's cubin registered that stub (an ODR trap that once
// ran the FMA kernel for LBW_MODE_EXACT).
#if LBW_FAST
#define LBW_FLAVOR fast
#else
#define LBW_FLAVOR exact
#endif

namespace lbw {
namespace LBW_FLAVOR {

constexpr int kSweepThreads = 128;

template <int OP>
__device__ __forceinline__ Macro collide_cell(double (&f)[27], double Fx, double Fy, double Fz,
                                              const Relax& r) {
#if LBW_FAST
    if constexpr (OP == 1) return cumulant_fast(f, Fx, Fy, Fz, r);
    else return bgk_fast(f, Fx, Fy, Fz, r);
#else
    if constexpr (OP == 1) return cumulant_exact(f, Fx, Fy, Fz, r);
    else return bgk_exact(f, Fx, Fy, Fz, r);
#endif
}

// Where population i of cell (x,y,z) streams from (pull: x - c_i), with the
// x-face rules of XSource and the y/z wrap (periodic) or zero-ghost
// (non-periodic) rule of the reference's ghost ring (halo.py:92-160).
struct PullSrc {
    int64_t xoff[3];  // plane offset for cx = -1, 0, +1
    int32_t xkind[3]; // 0 memory, 1 constant inflow, 2 zero
    int32_t yoff[3];  // ys*zp for cy = -1, 0, +1
    int32_t zs[3];
    bool yok[3], zok[3];
    int8_t ywall[3], zwall[3];  // LBW_WALL_* of the face a failing source crosses
    bool any_wall;              // some source of this cell lies beyond a wall
};

__device__ __forceinline__ void x_source(const Geom& g, int x, int cx, int64_t& off, int32_t& kind) {
    int xs = x - cx;
    kind = 0;
    if (xs < 0 || xs >= g.nxl) {
        const int mode = xs < 0 ? g.lo_src : g.hi_src;
        if (mode == XS_WRAP) xs = xs < 0 ? g.nxl - 1 : 0;
        else if (mode == XS_CLAMP) xs = xs < 0 ? 0 : g.nxl - 1;
        else if (mode == XS_CONST) kind = 1;
        else if (mode == XS_ZERO) kind = 2;
        // XS_GHOST: plane -1 / nxl are the ghost planes 0 / nxl+1
    }
    off = (int64_t)(xs + 1) * g.plane_stride;
}

__device__ __forceinline__ void make_pull(const Geom& g, int x, int y, int z, PullSrc& s) {
    s.any_wall = false;
#pragma unroll
    for (int c = -1; c <= 1; ++c) {
        x_source(g, x, c, s.xoff[c + 1], s.xkind[c + 1]);
        int ys = y - c;
        bool yok = true;
        if (ys < 0) { if (g.per_y) ys += g.ny; else yok = false; }
        else if (ys >= g.ny) { if (g.per_y) ys -= g.ny; else yok = false; }
        s.yoff[c + 1] = yok ? ys * g.zp : 0;
        s.yok[c + 1] = yok;
        s.ywall[c + 1] = yok ? 0 : (int8_t)g.walls[ys < 0 ? 0 : 1];
        s.any_wall |= s.ywall[c + 1] != 0;
        int zs = z - c;
        bool zok = true;
        if (zs < 0) { if (g.per_z) zs += g.nz; else zok = false; }
        else if (zs >= g.nz) { if (g.per_z) zs -= g.nz; else zok = false; }
        s.zs[c + 1] = zok ? zs : 0;
        s.zok[c + 1] = zok;
        s.zwall[c + 1] = zok ? 0 : (int8_t)g.walls[zs < 0 ? 2 : 3];
        s.any_wall |= s.zwall[c + 1] != 0;
    }
}

#ifndef LBW_STREAM_HINTS
#define LBW_STREAM_HINTS 0
#endif
// Streaming cache hints for the single-use population traffic: loads skip
// L1 allocation, stores are marked evict-first.  Storage is double or
// float (precision: single); values are widened on load and rounded to
// nearest on store, as numpy/numba do for float32 fields (_kernels.py:5-7).
__device__ __forceinline__ double ld_pop(const double* p) {
#if LBW_STREAM_HINTS
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double ld_pop(const float* p) { return (double)__ldg(p); }
__device__ __forceinline__ void st_pop(double* p, double v) {
#if LBW_STREAM_HINTS
    __stcs(p, v);
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_pop(float* p, double v) { *p = (float)v; }

// the value a store of v into storage type T reads back as
template <class T>
__device__ __forceinline__ double stored(double v) {
    return (double)(T)v;
}

// Pull of a cell with some source beyond a y / z wall (rare: cells next to
// walled faces), a separate branch so the common path stays the plain one.
template <class T>
__device__ __forceinline__ void load_cell_walls(const T* __restrict__ src, const Geom& g,
                                             const PullSrc& s, int x, int y, int z,
                                             double (&f)[27]) {
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        const int a = cx_of(i) + 1, b = cy_of(i) + 1, c = cz_of(i) + 1;
        const bool yo = !s.yok[b], zo = !s.zok[c];
        const bool out = yo || zo;
        const bool wall = out && !(yo && s.ywall[b] == 0) && !(zo && s.zwall[c] == 0);
        const bool noslip = wall && ((yo && s.ywall[b] == 1) || (zo && s.zwall[c] == 1));
        const bool mirror = wall && !noslip;
        // free-slip: the crossed components of c_i negated
        const int iy = (a * 3 + (2 - b)) * 3 + c, iz = (a * 3 + b) * 3 + (2 - c);
        const int iyz = (a * 3 + (2 - b)) * 3 + (2 - c);
        const int ip = !mirror ? i : (yo && zo ? iyz : (yo ? iy : iz));
        const int xk = s.xkind[a];
        const bool is_const = !noslip && (xk == 1 || xk == 2 || (out && !wall));
        const double feq =
            !mirror ? g.feq_in[i] : (yo && zo ? g.feq_in[iyz] : (yo ? g.feq_in[iy] : g.feq_in[iz]));
        const double cval = xk == 1 ? feq : 0.0;
        const T* p = noslip ? src + buf_index(g, x + 1, 26 - i, y, z)
                            : src + s.xoff[a] + (int64_t)ip * g.dir_stride +
                                  ((mirror && yo) ? y * g.zp : s.yoff[b]) +
                                  ((mirror && zo) ? z : s.zs[c]);
        const double v = ld_pop(is_const ? src : p);
        f[i] = is_const ? cval : v;
    }
}

template <bool PULL, class T>
__device__ __forceinline__ void load_cell(const T* __restrict__ src, const Geom& g, int x, int y,
                                          int z, double (&f)[27]) {
    if constexpr (!PULL) {
        const T* p = src + buf_index(g, x + 1, 0, y, z);
#pragma unroll
        for (int i = 0; i < 27; ++i) f[i] = ld_pop(p + (int64_t)i * g.dir_stride);
    } else {
        PullSrc s;
        make_pull(g, x, y, z, s);
        if (s.any_wall) {
            load_cell_walls(src, g, s, x, y, z, f);
            return;
        }
        // Every direction's source is selected without branches and all 27
        // loads are issued back to back (a constant -- inflow equilibrium or
        // a zero ghost -- loads a harmless dummy and is selected after).
#pragma unroll
        for (int i = 0; i < 27; ++i) {
            const int a = cx_of(i) + 1, b = cy_of(i) + 1, c = cz_of(i) + 1;
            const bool out = !s.yok[b] || !s.zok[c];
            const int xk = s.xkind[a];
            const bool is_const = xk == 1 || xk == 2 || out;
            const double cval = xk == 1 ? g.feq_in[i] : 0.0;
            const T* p = src + s.xoff[a] + (int64_t)i * g.dir_stride + s.yoff[b] + s.zs[c];
            const double v = ld_pop(is_const ? src : p);
            f[i] = is_const ? cval : v;
        }
    }
}

// Pull with every source in memory (no inflow constant, no zero ghost):
// true for all cells except those at a non-periodic y/z face or an
// inflow / unbounded x face.  Branch-free: one 32-bit offset per
// direction inside its source plane (a plane is < 2^31 doubles).
__device__ __forceinline__ bool pull_is_simple(const Geom& g, int x, int y, int z) {
    const bool xs = !((x == 0 && (g.lo_src == XS_CONST || g.lo_src == XS_ZERO)) ||
                      (x == g.nxl - 1 && (g.hi_src == XS_CONST || g.hi_src == XS_ZERO)));
    const bool ys = g.per_y || (y > 0 && y < g.ny - 1);
    const bool zs = g.per_z || (z > 0 && z < g.nz - 1);
    return xs && ys && zs;
}

template <class T>
__device__ __forceinline__ void load_cell_simple(const T* __restrict__ src, const Geom& g,
                                                 int x, int y, int z, double (&f)[27]) {
    const T* px[3];
#pragma unroll
    for (int c = -1; c <= 1; ++c) {
        int64_t off;
        int32_t kind;
        x_source(g, x, c, off, kind);
        px[c + 1] = src + off;
    }
    LBW_CHECK(x >= 0 && x < g.nxl && y >= 0 && y < g.ny && z >= 0 && z < g.nz);
    const int ym = (y + 1 < g.ny ? y + 1 : y + 1 - g.ny) * g.zp;  // cy = -1: y+1
    const int y0 = y * g.zp;
    const int yp = (y > 0 ? y - 1 : y - 1 + g.ny) * g.zp;        // cy = +1: y-1
    const int zm = z + 1 < g.nz ? z + 1 : z + 1 - g.nz;           // cz = -1: z+1
    const int zp = z > 0 ? z - 1 : z - 1 + g.nz;                  // cz = +1: z-1
    const int ds = (int)g.dir_stride;
    const int yo[3] = {ym, y0, yp};
    const int zo[3] = {zm, z, zp};
#pragma unroll
    for (int i = 0; i < 27; ++i)
        f[i] = ld_pop(px[cx_of(i) + 1] + (i * ds + yo[cy_of(i) + 1] + zo[cz_of(i) + 1]));
}

// Roma spreading evaluated at one cell (actuator.py:190-247): the sum over
// the points whose 3x3x3 support holds the cell, in ascending id, each
// adding ((wx*wy)*wz)*F_lat; with float storage every addition is rounded
// as `+=` on the reference's float32 force array rounds it.
template <class T, int KW>
__device__ __forceinline__ void actuator_force_k(const ForceView& fv, int64_t xg, int y, int z,
                                              double& Fx, double& Fy, double& Fz) {
    double F[3] = {0.0, 0.0, 0.0};
    const int kw = KW > 0 ? KW : fv.kw;   // 3 (Roma) unrolled, else the run's width
    for (int p = 0; p < fv.npts; ++p) {
        const int32_t* dc = fv.dep_cell + (int64_t)p * 3 * kw;
        const double* dw = fv.dep_w + (int64_t)p * 3 * kw;
        double wx = 0.0, wy = 0.0;
        bool hx = false, hy = false;
        for (int t = 0; t < kw; ++t) {
            if (dc[t] == xg) { hx = true; wx = dw[t]; }
            if (dc[kw + t] == y) { hy = true; wy = dw[kw + t]; }
        }
        if (!(hx && hy)) continue;
        // explicit roundings: no FMA contraction in either flavour's TU
        const double wxy = __dmul_rn(wx, wy);
        for (int t = 0; t < kw; ++t) {
            if (dc[2 * kw + t] == z) {
                const double w = __dmul_rn(wxy, dw[2 * kw + t]);
                for (int c = 0; c < 3; ++c)
                    // plain (L1-coherent) loads: flat is written by another
                    // kernel or, in the flag-ordered / fused steps, by
                    // another CTA whose completion flag this CTA acquired
                    // (the acquire invalidates this SM's L1) -- never
                    // ld.global.nc here
                    F[c] = (double)(T)__dadd_rn(F[c], __dmul_rn(w, fv.flat[p * 3 + c]));
            }
        }
    }
    Fx = F[0];
    Fy = F[1];
    Fz = F[2];
}

template <class T>
__device__ __forceinline__ void actuator_force(const ForceView& fv, int64_t xg, int y, int z,
                                            double& Fx, double& Fy, double& Fz) {
    if (fv.kw == 3) actuator_force_k<T, 3>(fv, xg, y, z, Fx, Fy, Fz);
    else actuator_force_k<T, 0>(fv, xg, y, z, Fx, Fy, Fz);
}

// force of cell (x,y,z) given its row's key (ForceView)
template <class T>
__device__ __forceinline__ void force_from_key(const ForceView& fv, const Geom& g, uint64_t key,
                                               int x, int y, int z, double& Fx, double& Fy,
                                               double& Fz) {
    Fx = Fy = Fz = 0.0;
    const int32_t slot = (int32_t)(uint32_t)key;
    if (fv.row_key == nullptr || (uint32_t)(key >> 32) != fv.tag || slot < 0) return;
    LBW_CHECK(x >= 0 && x < g.nxl && y >= 0 && y < g.ny && z >= 0 && z < g.nz);
    if (fv.pool != nullptr) {
        const T* p = static_cast<const T*>(fv.pool) + (int64_t)slot * 3 * g.zp + z;
        Fx = (double)p[0];
        Fy = (double)p[g.zp];
        Fz = (double)p[2 * g.zp];
    } else {
        actuator_force<T>(fv, g.x0 + x, y, z, Fx, Fy, Fz);
    }
}

template <class T>
__device__ __forceinline__ void load_force(const ForceView& fv, const Geom& g, int x, int y, int z,
                                           double& Fx, double& Fy, double& Fz) {
    LBW_CHECK(x >= 0 && x < g.nxl && y >= 0 && y < g.ny);
    const uint64_t key = fv.row_key != nullptr ? fv.row_key[(int64_t)x * g.ny + y] : 0ull;
    force_from_key<T>(fv, g, key, x, y, z, Fx, Fy, Fz);
}

// runtime storage dispatch for the non-hot paths (actuator sampling, output)
template <bool PULL>
__device__ __forceinline__ void load_cell_any(const void* src, const Geom& g, int x, int y, int z,
                                              double (&f)[27]) {
    if (g.single) load_cell<PULL>(static_cast<const float*>(src), g, x, y, z, f);
    else load_cell<PULL>(static_cast<const double*>(src), g, x, y, z, f);
}
__device__ __forceinline__ void load_force_any(const ForceView& fv, const Geom& g, int x, int y,
                                               int z, double& Fx, double& Fy, double& Fz) {
    if (g.single) load_force<float>(fv, g, x, y, z, Fx, Fy, Fz);
    else load_force<double>(fv, g, x, y, z, Fx, Fy, Fz);
}
// macro as the reference's macro array of the storage dtype holds it
__device__ __forceinline__ Macro stored_macro(const Geom& g, Macro m) {
    if (g.single) {
        m.rho = stored<float>(m.rho);
        m.ux = stored<float>(m.ux);
        m.uy = stored<float>(m.uy);
        m.uz = stored<float>(m.uz);
    }
    return m;
}

// Non-finite macro -> atomicMin of (step, global cell, density-ok bit)
// (sim.py:254-262: first offending cell in C order, "density" when rho is bad).
// The reference checks its macro array, i.e. the values rounded to T.
template <class T>
__device__ __forceinline__ void flag_nonfinite(unsigned long long* key, int64_t step,
                                               int64_t cell, const Macro& m) {
    const bool rho_ok = isfinite(stored<T>(m.rho));
    if (!(rho_ok && isfinite(stored<T>(m.ux)) && isfinite(stored<T>(m.uy)) &&
          isfinite(stored<T>(m.uz)))) {
        const unsigned long long k = ((unsigned long long)step << 40) |
                                     ((unsigned long long)cell << 1) | (rho_ok ? 1ull : 0ull);
        atomicMin(key, k);
    }
}

// Called by every thread of an edge-plane CTA after its halo stores: the
// CTA's last arrival on the edge counter of this sweep publishes the
// step's completion value to both neighbours over NVLink.  The counter
// grows by edge_ctas per sweep, so no reset is needed.
__device__ __forceinline__ void edge_done(const HaloOut& h) {
    __threadfence_system();  // this thread's peer stores before the CTA's arrival
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence_system();
        const unsigned long long old = atomicAdd(h.edge_counter, 1ull);
        if ((old + 1) % h.edge_ctas == 0) {
            __threadfence_system();
            for (int s = 0; s < 2; ++s)
                if (h.peer_flag[s])
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(h.peer_flag[s]),
                                 "r"(h.value)
                                 : "memory");
        }
    }
}

template <int OP, bool PULL, class T>
__device__ __forceinline__ void sweep_cell(const SweepArgs& a, int x, int y, int z) {
    const Geom& g = a.g;
    const T* src = static_cast<const T*>(a.src);
    double f[27];
    if (PULL && pull_is_simple(g, x, y, z)) load_cell_simple(src, g, x, y, z, f);
    else load_cell<PULL>(src, g, x, y, z, f);
    double Fx, Fy, Fz;
    load_force<T>(a.fv, g, x, y, z, Fx, Fy, Fz);
    const Macro m = collide_cell<OP>(f, Fx, Fy, Fz, a.r);
    flag_nonfinite<T>(a.nan_key, a.step, ((g.x0 + x) * g.ny + y) * (int64_t)g.nz + z, m);
    T* d = static_cast<T*>(a.dst) + buf_index(g, x + 1, 0, y, z);
#pragma unroll
    for (int i = 0; i < 27; ++i) st_pop(d + i * (int)g.dir_stride, f[i]);
    // edge planes: the outgoing directions go straight into the neighbour
    // slab's ghost plane (NVLink stores; halo pointers are peer mappings)
    if (x == 0 && a.halo.lo != nullptr) {
        T* h = static_cast<T*>(a.halo.lo) + (int64_t)y * g.zp + z;
#pragma unroll
        for (int i = 0; i < 9; ++i) h[(int64_t)i * g.dir_stride] = (T)f[i];
    }
    if (x == g.nxl - 1 && a.halo.hi != nullptr) {
        T* h = static_cast<T*>(a.halo.hi) + (int64_t)y * g.zp + z;
#pragma unroll
        for (int i = 18; i < 27; ++i) h[(int64_t)(i - 18) * g.dir_stride] = (T)f[i];
    }
}

// In-kernel wait for the actuator chain of this step (see SweepArgs gate):
// bounded; an expired wait raises the gate error flag (reported by the host
// as LBW_ECUDA) and lets the CTA finish rather than trapping the context.
__device__ __forceinline__ void gate_wait(const uint32_t* flag, uint32_t value, int32_t* err,
                                          int32_t site = 1) {
    long long n = 0;
    while (true) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= value) break;
        __nanosleep(32);
        if (++n > 40000000LL) {
            if (err) atomicCAS(err, 0, site);   // the first expired wait's site
            break;
        }
    }
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Chain-B cell update (SweepArgs kin_flag != nullptr): warp-uniform control
// flow (valid = the lane has a cell).  The K4 flag is waited for and the
// sample stores are counted per warp -- a warp is 32 z-cells of one row, so
// a row's keys are warp-uniform -- with no CTA barrier: lane 0 acquires and
// __syncwarp orders the other lanes behind it.
template <int OP, bool PULL, class T>
__device__ __forceinline__ void sweep_cell_chain(const SweepArgs& a, int x, int y, int z, bool valid,
                                                 int tid) {
    const Geom& g = a.g;
    const T* src = static_cast<const T*>(a.src);
    const int64_t row = (int64_t)x * g.ny + y;
    const int lane = tid & 31;
    // the geometry of steps m (force rows) and m+1 (sampling rows) is
    // visible from the start (k_sweep_cb): keys and populations load together
    uint64_t key = 0ull, skey = 0ull;
    double f[27];
    if (valid) {
        key = __ldcg(reinterpret_cast<const unsigned long long*>(a.fv.row_key) + row);
        skey = __ldcg(reinterpret_cast<const unsigned long long*>(a.skey) + row);
        if (PULL && pull_is_simple(g, x, y, z)) load_cell_simple(src, g, x, y, z, f);
        else load_cell<PULL>(src, g, x, y, z, f);
    }
    // rows of step m+1's sampling cubes: store the force-free half of this
    // collide's macro (rho, sum f c) now -- the sampling of step m+1
    // completes u with this step's force -- so the next step's chain can
    // start before this tile has its force
    const bool store = valid && (uint32_t)(skey >> 32) == a.store_tag;
    if (store) {
        double rho, mx, my, mz;
        raw_sums_exact(f, rho, mx, my, mz);
        double* b = a.spool + (int64_t)(uint32_t)skey * 4 * g.zp + z;
        b[0] = rho;
        b[g.zp] = mx;
        b[2 * g.zp] = my;
        b[3 * g.zp] = mz;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0 &&
        *(const volatile int32_t*)a.pool_tiles == 0) {
        // no sampling row in this slab: nothing to wait for
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.box_flag), "r"(a.box_value)
                     : "memory");
    }
    if (__any_sync(0xffffffffu, store)) {
        LBW_TRACE_BEGIN(7, a.step);
        LBW_TRACE_END(7, a.step);
        __syncwarp();
        if (lane == 0) {
            // the last sample warp publishes "the samples of step m+1 are stored"
            const uint32_t target = (uint32_t)*(const volatile int32_t*)a.pool_tiles;
            __threadfence();
            const uint32_t done = atomicAdd(a.pool_cnt, 1u) + 1u;
            if (done == target) {
                *a.pool_cnt = 0u;   // for the next sweep (it starts after this one completes)
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.box_flag),
                             "r"(a.box_value)
                             : "memory");
                LBW_TRACE_END_HERE(5, a.step);
            }
        }
    }
    // a warp with force rows of step m waits for the point forces of step m
    const bool need = valid && (uint32_t)(key >> 32) == a.fv.tag;
    if (__any_sync(0xffffffffu, need)) {
        LBW_TRACE_BEGIN(6, a.step);
        if (lane == 0) gate_wait(a.k4_flag, a.k4_value, a.gate_error, 12);
        __syncwarp();
        LBW_TRACE_END(6, a.step);
    }
    if (valid) {
        double Fx, Fy, Fz;
        force_from_key<T>(a.fv, g, key, x, y, z, Fx, Fy, Fz);
        const Macro m = collide_cell<OP>(f, Fx, Fy, Fz, a.r);
        flag_nonfinite<T>(a.nan_key, a.step, ((g.x0 + x) * g.ny + y) * (int64_t)g.nz + z, m);
        T* d = static_cast<T*>(a.dst) + buf_index(g, x + 1, 0, y, z);
#pragma unroll
        for (int i = 0; i < 27; ++i) st_pop(d + i * (int)g.dir_stride, f[i]);
    }
}

// K1: fused pull-stream + collide (+Guo) over local planes [x_begin, x_end).
// One thread per cell, z fastest.  PULL=false collides the stored state in
// place position (first step after an upload of pre-collision data).
template <int OP, bool PULL, int MINB, class T>
__global__ void __launch_bounds__(kSweepThreads, MINB) k_sweep(SweepArgs a) {
    const Geom& g = a.g;
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    // the two edge planes come first in dispatch order so their halo stores
    // (and the completion signal) are issued at the start of the sweep
    const int bz = (int)blockIdx.z;
    // edge planes first; the interior ascending or, on alternate steps,
    // descending x, so a sweep starts on the planes the previous one wrote
    // last (still in L2)
    const int xi = a.reverse ? g.nxl - bz : bz - 1;
    const int x = a.x_begin + (bz == 0 ? 0 : (bz == 1 ? g.nxl - 1 : xi));
    const bool edge = bz < 2 && a.halo.edge_counter != nullptr;
    // Programmatic dependent launch: when this sweep directly follows the
    // previous one in the stream it is launched before that one finishes;
    // nothing is read or written before the previous grid has completed and
    // its stores are visible (no-op for an ordinary launch).  The next
    // sweep may then be scheduled as soon as every CTA of this one runs.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (a.gate_flag != nullptr) {   // uniform per CTA
        if (x >= a.gate_box[0] && x <= a.gate_box[1]) {
            if (threadIdx.x == 0 && threadIdx.y == 0) gate_wait(a.gate_flag, a.gate_value, a.gate_error);
            __syncthreads();
        }
    }
    LBW_TRACE_BEGIN(0, a.step);
    if (z < g.nz && y < g.ny) sweep_cell<OP, PULL, T>(a, x, y, z);
    if (edge) edge_done(a.halo);  // whole CTA, uniform branch
    LBW_TRACE_END(0, a.step);
}

// K1 with the flag-ordered actuator chain (single slab, SweepArgs kin_flag):
// the same plane order (ascending / alternating), no halo, no box gate.
template <int OP, bool PULL, int MINB, class T>
__global__ void __launch_bounds__(kSweepThreads, MINB) k_sweep_cb(SweepArgs a) {
    const Geom& g = a.g;
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int bz = (int)blockIdx.z;
    const int np = a.x_end - a.x_begin;
    // rotated plane order: the rotor's planes first (single slab: np == nxl;
    // the host keeps 0 <= x_first < np and 1 <= x_len <= np, so r lies in
    // (-np, 2 np) and one wrap suffices)
    int r = a.reverse ? a.x_first + a.x_len - 1 - bz : a.x_first + bz;
    r += r < 0 ? np : (r >= np ? -np : 0);
    const int x = a.x_begin + r;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    LBW_TRACE_BEGIN(0, a.step);
    const int tid = (int)(threadIdx.x + threadIdx.y * blockDim.x);
    sweep_cell_chain<OP, PULL, T>(a, x, y, z, z < g.nz && y < g.ny, tid);
    // The next sweep reads the geometry of step m+2 without waiting: CTA 0
    // acquires it here, and that sweep's griddepcontrol.wait (or stream
    // order) follows this grid's completion.  KK computes it three steps
    // ahead, so this normally finds the flag set; it depends on sweeps up
    // to m-2 only.  Acquiring at the start of every CTA instead put an
    // acquire and a dependent key load (two round trips) before each CTA's
    // arithmetic (~0.7-1 us per 64^3 step).
    if (bz == 0 && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0)
        gate_wait(a.kin_flag, a.kin_value, a.gate_error, 11);
    LBW_TRACE_END(0, a.step);
}

// K0: batch collide of (n,27) rows (_kernels.py:400-427)
template <int OP>
__global__ void __launch_bounds__(128) k_batch(double* __restrict__ f2, const double* __restrict__ F2,
                                               double* __restrict__ macro2, int64_t n, Relax r) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double f[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) f[i] = f2[k * 27 + i];
    const Macro m = collide_cell<OP>(f, F2[k * 3], F2[k * 3 + 1], F2[k * 3 + 2], r);
#pragma unroll
    for (int i = 0; i < 27; ++i) f2[k * 27 + i] = f[i];
    macro2[k * 4] = m.rho;
    macro2[k * 4 + 1] = m.ux;
    macro2[k * 4 + 2] = m.uy;
    macro2[k * 4 + 3] = m.uz;
}

// collide of every interior cell of a ghosted AoS block (_kernels.py:304-354)
template <int OP>
__global__ void __launch_bounds__(128) k_block_collide(double* __restrict__ f,
                                                       const double* __restrict__ force,
                                                       double* __restrict__ macro, int64_t nx,
                                                       int64_t ny, int64_t nz, Relax r) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nx * ny * nz) return;
    const int64_t z = t % nz + 1, y = (t / nz) % ny + 1, x = t / (nz * ny) + 1;
    const int64_t c = (x * (ny + 2) + y) * (nz + 2) + z;
    double fl[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) fl[i] = f[c * 27 + i];
    const Macro m = collide_cell<OP>(fl, force[c * 3], force[c * 3 + 1], force[c * 3 + 2], r);
#pragma unroll
    for (int i = 0; i < 27; ++i) f[c * 27 + i] = fl[i];
    macro[c * 4] = m.rho;
    macro[c * 4 + 1] = m.ux;
    macro[c * 4 + 2] = m.uy;
    macro[c * 4 + 3] = m.uz;
}

inline dim3 sweep_block(const Geom& g) {
    int bz = 32;
    while (bz < g.nz && bz < kSweepThreads) bz *= 2;
    return dim3(bz, kSweepThreads / bz, 1);
}

// launch K1 for one (operator, pull, storage) combination
// (LBW_SWEEP_PDL=0: ordinary launches, for A/B runs)
inline bool sweep_pdl() {
    static const bool on = [] {
        const char* e = getenv("LBW_SWEEP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// one K1 launch, programmatic stream serialisation allowed (see k_sweep)
template <int OP, bool PULL, int MINB, class T>
void launch_k_sweep_pdl(dim3 grd, dim3 blk, const SweepArgs& b, cudaStream_t s) {
    auto kern = b.kin_flag ? k_sweep_cb<OP, PULL, MINB, T> : k_sweep<OP, PULL, MINB, T>;
    if (!sweep_pdl() || !b.pdl) {
        kern<<<grd, blk, 0, s>>>(b);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grd;
    cfg.blockDim = blk;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, b);
}

template <int MINB, class T>
void launch_k_sweep(int op, bool pull, dim3 grd, dim3 blk, const SweepArgs& b, cudaStream_t s) {
    if (op == 1) {
        if (pull) launch_k_sweep_pdl<1, true, MINB, T>(grd, blk, b, s);
        else launch_k_sweep_pdl<1, false, MINB, T>(grd, blk, b, s);
    } else {
        if (pull) launch_k_sweep_pdl<0, true, MINB, T>(grd, blk, b, s);
        else launch_k_sweep_pdl<0, false, MINB, T>(grd, blk, b, s);
    }
}

// load the chain-B sweep kernels of an operator now: with lazy module loading
// the first launch of a kernel waits for the kernels already running, and a
// resident chain kernel spinning on a flag that only this sweep will set
// would never finish
template <int MINB, class T>
cudaError_t preload_k_sweep_cb(int op) {
    cudaFuncAttributes fa;
    cudaError_t e = op == 1 ? cudaFuncGetAttributes(&fa, k_sweep_cb<1, true, MINB, T>)
                            : cudaFuncGetAttributes(&fa, k_sweep_cb<0, true, MINB, T>);
    if (e == cudaSuccess)
        e = op == 1 ? cudaFuncGetAttributes(&fa, k_sweep_cb<1, false, MINB, T>)
                    : cudaFuncGetAttributes(&fa, k_sweep_cb<0, false, MINB, T>);
    return e;
}

}  // namespace LBW_FLAVOR
using namespace LBW_FLAVOR;
}  // namespace lbw
