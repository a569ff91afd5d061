// lbw_kernels_exact.cu — bit-exact flavour (LBW_MODE_EXACT) + data movement.
// Compiled with -fmad=false: no FMA contraction anywhere in this TU.
#define LBW_FAST 0
#include "lbw_sweep.cuh"
#include "lbw_fused.cuh"

namespace lbw {

cudaError_t launch_fused_exact(int op, bool pull, const FusedArgs& a, size_t smem,
                               cudaStream_t s) {
    const cudaError_t e = launch_fused<4>(op, pull, a, smem, s);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t preload_sweep_cb_exact(int op, bool single) {
    return single ? preload_k_sweep_cb<4, float>(op) : preload_k_sweep_cb<4, double>(op);
}

cudaError_t launch_sweep_exact(int op, bool pull, const SweepArgs& a, cudaStream_t s) {
    const dim3 blk = sweep_block(a.g);
    const dim3 grd((a.g.nz + blk.x - 1) / blk.x, (a.g.ny + blk.y - 1) / blk.y, a.x_end - a.x_begin);
    if (grd.z == 0) return cudaSuccess;
    SweepArgs b = a;
    b.halo.edge_ctas = grd.x * grd.y * (grd.z < 2 ? grd.z : 2u);
    if (a.g.single) launch_k_sweep<4, float>(op, pull, grd, blk, b, s);
    else launch_k_sweep<4, double>(op, pull, grd, blk, b, s);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_batch_exact(int op, double* f2, const double* F2, double* macro2, int64_t n,
                              Relax r, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    if (op == 1) k_batch<1><<<blocks, 128, 0, s>>>(f2, F2, macro2, n, r);
    else k_batch<0><<<blocks, 128, 0, s>>>(f2, F2, macro2, n, r);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_block_collide_exact(int op, double* f, const double* force, double* macro,
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

// ------------------------------------------------------------------------
// Data movement and moments.  All exact (no arithmetic beyond the moment
// sums, which follow _kernels.py:357-380 bit for bit).
namespace lbw {
namespace {

__device__ __forceinline__ bool cell_of(const Geom& g, int64_t t, int& x, int& y, int& z) {
    const int64_t n = (int64_t)g.nxl * g.ny * g.nz;
    if (t >= n) return false;
    z = (int)(t % g.nz);
    y = (int)((t / g.nz) % g.ny);
    x = (int)(t / ((int64_t)g.nz * g.ny));
    return true;
}

__global__ void k_block_moments(const double* __restrict__ f, const double* __restrict__ force,
                                double* __restrict__ macro, int64_t nx, int64_t ny, int64_t nz,
                                double dt) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nx * ny * nz) return;
    const int64_t z = t % nz + 1, y = (t / nz) % ny + 1, x = t / (nz * ny) + 1;
    const int64_t c = (x * (ny + 2) + y) * (nz + 2) + z;
    double fl[27];
#pragma unroll
    for (int i = 0; i < 27; ++i) fl[i] = f[c * 27 + i];
    const Macro m = moments_exact(fl, force[c * 3], force[c * 3 + 1], force[c * 3 + 2], dt);
    macro[c * 4] = m.rho;
    macro[c * 4 + 1] = m.ux;
    macro[c * 4 + 2] = m.uy;
    macro[c * 4 + 3] = m.uz;
}

__global__ void k_block_stream(const double* __restrict__ fsrc, double* __restrict__ fdst,
                               int64_t nx, int64_t ny, int64_t nz) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nx * ny * nz) return;
    const int64_t z = t % nz + 1, y = (t / nz) % ny + 1, x = t / (nz * ny) + 1;
    const int64_t c = (x * (ny + 2) + y) * (nz + 2) + z;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        const int64_t s = ((x - cx_of(i)) * (ny + 2) + (y - cy_of(i))) * (nz + 2) + (z - cz_of(i));
        fdst[c * 27 + i] = fsrc[s * 27 + i];
    }
}

template <class T>
__global__ void k_aos_to_soa(const double* __restrict__ aos, T* __restrict__ buf, Geom g) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    T* d = buf + buf_index(g, x + 1, 0, y, z);
#pragma unroll
    for (int i = 0; i < 27; ++i) st_pop(d + (int64_t)i * g.dir_stride, aos[t * 27 + i]);
}

struct F27 {
    double v[27];
};

template <class T>
__global__ void k_fill_uniform(F27 f, T* __restrict__ buf, Geom g) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    T* d = buf + buf_index(g, x + 1, 0, y, z);
#pragma unroll
    for (int i = 0; i < 27; ++i) st_pop(d + (int64_t)i * g.dir_stride, f.v[i]);
}

// collision.py:54-100 for one cell: polynomial w rho (1 + 3cu + 4.5cu^2 -
// 1.5u.u) or product rho g(ux) g(uy) g(uz)
template <class T>
__global__ void k_init_modes(double rho, double ux0, double uy0, double uz0, int32_t n_modes,
                             const double* __restrict__ modes, int product, T* __restrict__ buf,
                             double* __restrict__ macro, Geom g) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    const double X = (double)(g.x0 + x) + 0.5, Y = (double)y + 0.5, Z = (double)z + 0.5;
    double u[3] = {ux0, uy0, uz0};
    for (int m = 0; m < n_modes; ++m) {
        const double* md = modes + (int64_t)m * 7;
        const double sn = sin(md[0] * X + md[1] * Y + md[2] * Z + md[6]);
        for (int c = 0; c < 3; ++c) u[c] += md[3 + c] * sn;
    }
    double f[27];
    if (product) {
        double gx[3][3];
        for (int c = 0; c < 3; ++c) {
            const double uu = u[c] * u[c];
            gx[c][0] = 0.5 * (uu - u[c] + 1.0 / 3.0);
            gx[c][1] = 1.0 - uu - 1.0 / 3.0;
            gx[c][2] = 0.5 * (uu + u[c] + 1.0 / 3.0);
        }
        for (int i = 0; i < 27; ++i)
            f[i] = rho * gx[0][cx_of(i) + 1] * gx[1][cy_of(i) + 1] * gx[2][cz_of(i) + 1];
    } else {
        const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
        for (int i = 0; i < 27; ++i) {
            const double cu = cx_of(i) * u[0] + cy_of(i) * u[1] + cz_of(i) * u[2];
            f[i] = w_of(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        }
    }
    T* d = buf + buf_index(g, x + 1, 0, y, z);
#pragma unroll
    for (int i = 0; i < 27; ++i) st_pop(d + (int64_t)i * g.dir_stride, f[i]);
    macro[t * 4] = rho;
    for (int c = 0; c < 3; ++c) macro[t * 4 + 1 + c] = u[c];
}

template <bool PULL, class T>
__global__ void k_gather_aos(const T* __restrict__ buf, Geom g, double* __restrict__ aos) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    double f[27];
    load_cell<PULL>(buf, g, x, y, z, f);
#pragma unroll
    for (int i = 0; i < 27; ++i) aos[t * 27 + i] = f[i];
}

template <bool PULL, class T>
__global__ void k_moments_soa(const T* __restrict__ buf, Geom g, ForceView fv, double dt,
                              double* __restrict__ macro) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    double f[27];
    load_cell<PULL>(buf, g, x, y, z, f);
    double Fx, Fy, Fz;
    load_force<T>(fv, g, x, y, z, Fx, Fy, Fz);
    const Macro m = stored_macro(g, moments_exact(f, Fx, Fy, Fz, dt));
    macro[t * 4] = m.rho;
    macro[t * 4 + 1] = m.ux;
    macro[t * 4 + 2] = m.uy;
    macro[t * 4 + 3] = m.uz;
}

__global__ void k_force_to_aos(ForceView fv, Geom g, double* __restrict__ aos) {
    int x, y, z;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (!cell_of(g, t, x, y, z)) return;
    double Fx, Fy, Fz;
    load_force_any(fv, g, x, y, z, Fx, Fy, Fz);
    aos[t * 3] = Fx;
    aos[t * 3 + 1] = Fy;
    aos[t * 3 + 2] = Fz;
}

// one CTA per (x,y) row: copy the row into pool slot == row index and give
// the row a slot only when some component is non-zero.
template <class T>
__global__ void k_force_from_aos(const double* __restrict__ aos, Geom g, uint64_t* __restrict__ row_key,
                                 T* __restrict__ pool) {
    const int64_t row = blockIdx.x;
    bool nz_any = false;
    for (int z = threadIdx.x; z < g.nz; z += blockDim.x) {
        const int64_t t = row * g.nz + z;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T v = (T)aos[t * 3 + c];
            pool[(row * 3 + c) * g.zp + z] = v;
            nz_any |= (v != (T)0);
        }
    }
    const int any = __syncthreads_or(nz_any);
    if (threadIdx.x == 0) row_key[row] = row_key_of(0, any ? (int32_t)row : -1);
}

inline unsigned cells_blocks(const Geom& g, int threads) {
    const int64_t n = (int64_t)g.nxl * g.ny * g.nz;
    return (unsigned)((n + threads - 1) / threads);
}

}  // namespace

cudaError_t launch_block_moments(const double* f, const double* force, double* macro, int64_t nx,
                                 int64_t ny, int64_t nz, double dt, cudaStream_t s) {
    const int64_t n = nx * ny * nz;
    if (n == 0) return cudaSuccess;
    k_block_moments<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(f, force, macro, nx, ny, nz, dt);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_block_stream(const double* fsrc, double* fdst, int64_t nx, int64_t ny,
                                int64_t nz, cudaStream_t s) {
    const int64_t n = nx * ny * nz;
    if (n == 0) return cudaSuccess;
    k_block_stream<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(fsrc, fdst, nx, ny, nz);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_aos_to_soa(const double* aos, void* buf, const Geom& g, cudaStream_t s) {
    if (g.single) k_aos_to_soa<<<cells_blocks(g, 128), 128, 0, s>>>(aos, (float*)buf, g);
    else k_aos_to_soa<<<cells_blocks(g, 128), 128, 0, s>>>(aos, (double*)buf, g);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform(const double (&f27)[27], void* buf, const Geom& g,
                                cudaStream_t s) {
    F27 f;
    for (int i = 0; i < 27; ++i) f.v[i] = f27[i];
    if (g.single) k_fill_uniform<<<cells_blocks(g, 128), 128, 0, s>>>(f, (float*)buf, g);
    else k_fill_uniform<<<cells_blocks(g, 128), 128, 0, s>>>(f, (double*)buf, g);
    count_launch();
    return cudaGetLastError();
}

template <class T>
void gather_aos_t(bool pull, const T* buf, const Geom& g, double* aos, cudaStream_t s) {
    if (pull) k_gather_aos<true><<<cells_blocks(g, 128), 128, 0, s>>>(buf, g, aos);
    else k_gather_aos<false><<<cells_blocks(g, 128), 128, 0, s>>>(buf, g, aos);
}
template <class T>
void moments_soa_t(bool pull, const T* buf, const Geom& g, ForceView fv, double dt, double* m,
                   cudaStream_t s) {
    if (pull) k_moments_soa<true><<<cells_blocks(g, 128), 128, 0, s>>>(buf, g, fv, dt, m);
    else k_moments_soa<false><<<cells_blocks(g, 128), 128, 0, s>>>(buf, g, fv, dt, m);
}

cudaError_t launch_init_modes(double rho, const double (&u0)[3], int32_t n_modes,
                              const double* modes_dev, int product, void* buf, double* macro,
                              const Geom& g, cudaStream_t s) {
    const unsigned nb = cells_blocks(g, 128);
    if (g.single)
        k_init_modes<<<nb, 128, 0, s>>>(rho, u0[0], u0[1], u0[2], n_modes, modes_dev, product,
                                        (float*)buf, macro, g);
    else
        k_init_modes<<<nb, 128, 0, s>>>(rho, u0[0], u0[1], u0[2], n_modes, modes_dev, product,
                                        (double*)buf, macro, g);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gather_aos(bool pull, const void* buf, const Geom& g, double* aos,
                              cudaStream_t s) {
    if (g.single) gather_aos_t(pull, (const float*)buf, g, aos, s);
    else gather_aos_t(pull, (const double*)buf, g, aos, s);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_moments_soa(bool pull, const void* buf, const Geom& g, ForceView fv,
                               double dt, double* macro_aos, cudaStream_t s) {
    if (g.single) moments_soa_t(pull, (const float*)buf, g, fv, dt, macro_aos, s);
    else moments_soa_t(pull, (const double*)buf, g, fv, dt, macro_aos, s);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_force_to_aos(ForceView fv, const Geom& g, double* aos, cudaStream_t s) {
    k_force_to_aos<<<cells_blocks(g, 128), 128, 0, s>>>(fv, g, aos);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_force_from_aos(const double* aos, const Geom& g, uint64_t* row_key,
                                  void* pool, cudaStream_t s) {
    const unsigned rows = (unsigned)((int64_t)g.nxl * g.ny);
    if (rows == 0) return cudaSuccess;
    if (g.single) k_force_from_aos<<<rows, 128, 0, s>>>(aos, g, row_key, (float*)pool);
    else k_force_from_aos<<<rows, 128, 0, s>>>(aos, g, row_key, (double*)pool);
    count_launch();
    return cudaGetLastError();
}

}  // namespace lbw
LBW_TRACE_EXPORT(exact)
