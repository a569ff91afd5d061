// lbw_internal.h — structures shared by the host driver and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lbw_cell.cuh"

namespace lbw {

// Source of a pulled population whose x plane lies outside the owned slab.
enum XSource : int {
    XS_GHOST = 0,  // ghost plane in memory, written by the neighbouring slab
    XS_WRAP = 1,   // periodic x on one domain: the plane at the other end
    XS_CONST = 2,  // velocity inflow: polynomial equilibrium feq_in (halo.py:151-156)
    XS_CLAMP = 3,  // zero-gradient outflow: the adjacent interior plane (halo.py:157-160)
    XS_ZERO = 4,   // non-periodic face without a boundary condition: never-written ghost (0)
};

// Device layout of one population buffer: planes p = 0 .. nxl+1 (p = x+1,
// planes 0 and nxl+1 are ghosts), each plane [27][ny][zp] with z fastest.
struct Geom {
    int32_t nxl, ny, nz, zp;   // local x planes, y, z, z pitch
    int64_t dir_stride;        // ny*zp
    int64_t plane_stride;      // 27*ny*zp
    int64_t x0, nxg;           // first global x, global x size
    int32_t per_y, per_z;
    int32_t lo_src, hi_src;    // XSource for x-1 at x=0 and x+1 at x=nxl-1
    int32_t single;            // populations / force stored fp32 (LBW_PREC_SINGLE)
    int32_t walls[4];          // LBW_WALL_* of the y_lo, y_hi, z_lo, z_hi faces
    double feq_in[27];         // already rounded to the storage type
};

// LBW_BOUNDS builds (EXTRA=-DLBW_BOUNDS) trap on any out-of-range index of
// the population buffers, force rows and actuator arrays: the bounds-checked
// library the GPU tests can run against (LBW_LIB) in place of a sanitizer.
#ifdef LBW_BOUNDS
#define LBW_CHECK(cond)          \
    do {                         \
        if (!(cond)) __trap();   \
    } while (0)
#else
#define LBW_CHECK(cond) \
    do {                \
    } while (0)
#endif

__host__ __device__ inline int64_t buf_index(const Geom& g, int p, int i, int y, int z) {
#if defined(LBW_BOUNDS) && defined(__CUDA_ARCH__)
    LBW_CHECK(p >= 0 && p < g.nxl + 2 && i >= 0 && i < 27 && y >= 0 && y < g.ny && z >= 0 &&
              z < g.zp);
#endif
    return (int64_t)p * g.plane_stride + (int64_t)i * g.dir_stride + (int64_t)y * g.zp + z;
}

// Storage element of populations and forces: double, or float when
// g.single (arithmetic stays fp64; values are rounded on store).
__host__ __device__ inline size_t elem_bytes(const Geom& g) { return g.single ? 4 : 8; }

// Force density of the cells that carry one: rows (x,y) with a slot hold
// [3][zp] storage elements in the pool; every other cell has F = 0.
// Row keys are (tag << 32 | slot): a row carries force for this view only
// when its tag matches, so a force set is re-used step after step without
// clearing (the actuator chain tags its claims with step + 1; a caller-set
// body force uses tag 0).
struct ForceView {
    const uint64_t* row_key;  // (nxl*ny); nullptr = no force anywhere
    const void* pool;         // [slot][3][zp] of the storage type, or nullptr:
    uint32_t tag;
    // ... actuator view: a tagged row's force is summed from the points'
    // deposit cells in ascending id at the cell (few points, see lbw_alm.cu)
    int32_t npts;
    int32_t kw;               // deposit cells per axis (3: Roma)
    const int32_t* dep_cell;  // (npts, 3 axes, kw) global cell or -1
    const double* dep_w;      // (npts, 3, kw) kernel weights
    const double* flat;       // (npts, 3) lattice force on the fluid
};
__host__ __device__ inline uint64_t row_key_of(uint32_t tag, int32_t slot) {
    return ((uint64_t)tag << 32) | (uint32_t)slot;
}

// A sparse force field: rows (x,y) of the slab that carry force own a slot
// of [3][zp] storage elements in the pool (keys: see ForceView).
struct ForceSet {
    uint64_t* row_key = nullptr;   // (nxl*ny)
    void* pool = nullptr;          // (cap, 3, zp) of the storage type
    uint32_t tag = 0;              // tag of the filling step
    int32_t flag_rows = 0;         // actuator set without a pool: K4 tags the rows
    int64_t cap = 0;               // slots: user set one per row, actuator set 9 per point
    ForceView view(uint32_t t) const { return ForceView{row_key, pool, t}; }
};

enum MacroKind { MS_UNIFORM = 0, MS_DENSE = 1, MS_GATHER = 2 };
struct HaloOut {
    void* lo;  // receives dirs 0..8 of plane x=0   ([9][ny][zp]), or nullptr
    void* hi;  // receives dirs 18..26 of plane x=nxl-1, or nullptr
    // in-kernel completion signal: the last CTA of the two edge planes
    // (scheduled first) release-stores `value` into both neighbours' flags
    uint32_t* peer_flag[2];
    unsigned long long* edge_counter;  // local, monotonically increasing
    uint32_t edge_ctas;                // CTAs covering planes 0 and nxl-1
    uint32_t value;
};

// kernel launchers (defined in the .cu translation units)
struct SweepArgs {
    const void* src;   // storage type per g.single
    void* dst;
    Geom g;
    ForceView fv;
    Relax r;
    int32_t x_begin, x_end;   // local planes [x_begin, x_end)
    unsigned long long* nan_key;
    int64_t step;
    HaloOut halo;
    // optional gate: CTAs of planes in [gate_box[0], gate_box[1]] wait until
    // *gate_flag >= gate_value (the actuator chain of this step is done)
    const uint32_t* gate_flag;
    const int32_t* gate_box;
    uint32_t gate_value;
    int32_t reverse;   // interior planes in descending x (alternate steps)
    // programmatic dependent launch allowed: only when the previous stream
    // operation is the preceding sweep (single slab; a linked slab has a
    // peer-flag wait between its sweeps)
    int32_t pdl;
    // gate timeout: set to 1 by a CTA whose bounded wait expired (the host
    // reports it as an error instead of the kernel trapping)
    int32_t* gate_error;
    // Flag-ordered actuator chain (lbw_alm.cu, "chain B"; kin_flag != nullptr):
    // the geometry of steps m / m+1 is visible when the sweep starts (its
    // predecessor sweep completed after acquiring it, see k_sweep_cb); CTA 0
    // acquires the geometry of step m+2 (*kin_flag >= kin_value) before it
    // ends, for the next sweep; a warp holding force rows waits for the point
    // forces of step m (*k4_flag >= k4_value), tiles holding rows of step
    // m+1's sampling cubes store their collide's (rho, u) into spool, and the
    // last of those tiles (*pool_tiles of them) publishes *box_flag = box_value.
    const uint32_t* kin_flag;
    uint32_t kin_value;
    const uint32_t* k4_flag;
    uint32_t k4_value;
    const uint64_t* skey;
    double* spool;
    uint32_t store_tag;
    uint32_t* pool_cnt;
    const int32_t* pool_tiles;
    uint32_t* box_flag;
    uint32_t box_value;
    // plane order of the chain-B sweep: ascending from x_first (descending
    // from x_first + x_len - 1 when reverse), both mod nxl, so the planes
    // around the rotor (a hint from KK, x_len of them) are swept first
    int32_t x_first, x_len;
};

// exact flavour (lbw_kernels_exact.cu, -fmad=false)
cudaError_t launch_sweep_exact(int op, bool pull, const SweepArgs& a, cudaStream_t s);
cudaError_t preload_sweep_cb_exact(int op, bool single);
cudaError_t launch_batch_exact(int op, double* f2, const double* F2, double* macro2, int64_t n,
                               Relax r, cudaStream_t s);
cudaError_t launch_block_collide_exact(int op, double* f, const double* force, double* macro,
                                       int64_t nx, int64_t ny, int64_t nz, Relax r,
                                       cudaStream_t s);
// fast flavour (lbw_kernels_fast.cu)
cudaError_t launch_sweep_fast(int op, bool pull, const SweepArgs& a, cudaStream_t s);
cudaError_t preload_sweep_cb_fast(int op, bool single);
cudaError_t launch_batch_fast(int op, double* f2, const double* F2, double* macro2, int64_t n,
                              Relax r, cudaStream_t s);
cudaError_t launch_block_collide_fast(int op, double* f, const double* force, double* macro,
                                      int64_t nx, int64_t ny, int64_t nz, Relax r,
                                      cudaStream_t s);

// data movement / moments (lbw_kernels_exact.cu)
cudaError_t launch_block_moments(const double* f, const double* force, double* macro, int64_t nx,
                                 int64_t ny, int64_t nz, double dt, cudaStream_t s);
cudaError_t launch_block_stream(const double* fsrc, double* fdst, int64_t nx, int64_t ny,
                                int64_t nz, cudaStream_t s);
// population buffers / force pools are of the storage type (g.single);
// the AoS host-side arrays are always fp64
cudaError_t launch_aos_to_soa(const double* aos, void* buf, const Geom& g, cudaStream_t s);
cudaError_t launch_fill_uniform(const double (&f27)[27], void* buf, const Geom& g,
                                cudaStream_t s);
// equilibrium of (rho, u0 + sum of sine modes) in every owned cell, macro too
cudaError_t launch_init_modes(double rho, const double (&u0)[3], int32_t n_modes,
                              const double* modes_dev, int product, void* buf, double* macro,
                              const Geom& g, cudaStream_t s);
cudaError_t launch_gather_aos(bool pull, const void* buf, const Geom& g, double* aos,
                              cudaStream_t s);
cudaError_t launch_moments_soa(bool pull, const void* buf, const Geom& g, ForceView fv,
                               double dt, double* macro_aos, cudaStream_t s);
cudaError_t launch_force_to_aos(ForceView fv, const Geom& g, double* aos, cudaStream_t s);
cudaError_t launch_force_from_aos(const double* aos, const Geom& g, uint64_t* row_key,
                                  void* pool, cudaStream_t s);

void count_launch(int n = 1);

}  // namespace lbw
