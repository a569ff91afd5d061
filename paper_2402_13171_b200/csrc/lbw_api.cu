// lbw_api.cu — C ABI of liblbw.so: host-array kernel entry points and the
// device-resident domain (one x-slab on one GPU).  See include/lbw.h.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "lbw_domain.h"

namespace lbw {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {

Relax make_relax(double omega, double w3, double w4, double w5, double w6, double dt) {
    Relax r;
    r.omega = omega;
    r.w3 = w3;
    r.w4 = w4;
    r.w5 = w5;
    r.w6 = w6;
    r.dt = dt;
    return r;
}

// RAII device scratch for the host-array entry points
struct DevBuf {
    void* p = nullptr;
    cudaError_t alloc(size_t n) { return n ? cudaMalloc(&p, n) : cudaSuccess; }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int collide_batch(int op, double* f2, const double* F2, double* macro2, int64_t n, Relax r,
                  int mode) {
    LBW_REQ(n >= 0, "n must be >= 0");
    LBW_REQ(mode == LBW_MODE_EXACT || mode == LBW_MODE_FAST, "unknown mode");
    if (n == 0) return LBW_OK;
    LBW_REQ(f2 && F2 && macro2, "null array");
    DevBuf df, dF, dm;
    LBW_CK(df.alloc(n * 27 * sizeof(double)));
    LBW_CK(dF.alloc(n * 3 * sizeof(double)));
    LBW_CK(dm.alloc(n * 4 * sizeof(double)));
    LBW_CK(cudaMemcpy(df.p, f2, n * 27 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dF.p, F2, n * 3 * sizeof(double), cudaMemcpyHostToDevice));
    if (mode == LBW_MODE_EXACT)
        LBW_CK(launch_batch_exact(op, df.as<double>(), dF.as<double>(), dm.as<double>(), n, r, 0));
    else
        LBW_CK(launch_batch_fast(op, df.as<double>(), dF.as<double>(), dm.as<double>(), n, r, 0));
    LBW_CK(cudaMemcpy(f2, df.p, n * 27 * sizeof(double), cudaMemcpyDeviceToHost));
    LBW_CK(cudaMemcpy(macro2, dm.p, n * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    return LBW_OK;
}

int collide_block(int op, double* f, const double* force, double* macro, int64_t nx, int64_t ny,
                  int64_t nz, Relax r, int mode) {
    LBW_REQ(nx >= 1 && ny >= 1 && nz >= 1, "block size must be positive");
    LBW_REQ(mode == LBW_MODE_EXACT || mode == LBW_MODE_FAST, "unknown mode");
    LBW_REQ(f && force && macro, "null array");
    const int64_t cells = (nx + 2) * (ny + 2) * (nz + 2);
    DevBuf df, dF, dm;
    LBW_CK(df.alloc(cells * 27 * sizeof(double)));
    LBW_CK(dF.alloc(cells * 3 * sizeof(double)));
    LBW_CK(dm.alloc(cells * 4 * sizeof(double)));
    LBW_CK(cudaMemcpy(df.p, f, cells * 27 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dF.p, force, cells * 3 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dm.p, macro, cells * 4 * sizeof(double), cudaMemcpyHostToDevice));
    if (mode == LBW_MODE_EXACT)
        LBW_CK(launch_block_collide_exact(op, df.as<double>(), dF.as<double>(), dm.as<double>(), nx,
                                          ny, nz, r, 0));
    else
        LBW_CK(launch_block_collide_fast(op, df.as<double>(), dF.as<double>(), dm.as<double>(), nx,
                                         ny, nz, r, 0));
    LBW_CK(cudaMemcpy(f, df.p, cells * 27 * sizeof(double), cudaMemcpyDeviceToHost));
    LBW_CK(cudaMemcpy(macro, dm.p, cells * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    return LBW_OK;
}

}  // namespace

int ensure_stage(lbw_domain* d, size_t bytes) {
    if (d->stage_bytes >= bytes) return LBW_OK;
    if (d->stage) {
        LBW_CK(cudaStreamSynchronize(d->stream));
        cudaFree(d->stage);
        d->bytes -= (int64_t)d->stage_bytes;
        d->stage = nullptr;
        d->stage_bytes = 0;
    }
    if (cudaMalloc(&d->stage, bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error("cannot allocate transfer staging buffer");
        return LBW_ENOMEM;
    }
    d->stage_bytes = bytes;
    d->bytes += (int64_t)bytes;
    return LBW_OK;
}

}  // namespace lbw

using namespace lbw;

// ============================================================== C entry points
extern "C" {

int lbw_abi_version(void) { return LBW_ABI_VERSION; }
const char* lbw_last_error(void) { return g_err.c_str(); }
int lbw_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
int64_t lbw_kernel_launches(void) { return g_launches.load(); }

int lbw_collide_cumulant_batch(double* f2, const double* F2, double* macro2, int64_t n,
                               double omega, double w3, double w4, double w5, double w6,
                               double dt, int mode) {
    return collide_batch(1, f2, F2, macro2, n, make_relax(omega, w3, w4, w5, w6, dt), mode);
}
int lbw_collide_bgk_batch(double* f2, const double* F2, double* macro2, int64_t n, double omega,
                          double dt, int mode) {
    return collide_batch(0, f2, F2, macro2, n, make_relax(omega, 1, 1, 1, 1, dt), mode);
}
int lbw_collide_cumulant_block(double* f, const double* force, double* macro, int64_t nx,
                               int64_t ny, int64_t nz, double omega, double w3, double w4,
                               double w5, double w6, double dt, int mode) {
    return collide_block(1, f, force, macro, nx, ny, nz, make_relax(omega, w3, w4, w5, w6, dt),
                         mode);
}
int lbw_collide_bgk_block(double* f, const double* force, double* macro, int64_t nx, int64_t ny,
                          int64_t nz, double omega, double dt, int mode) {
    return collide_block(0, f, force, macro, nx, ny, nz, make_relax(omega, 1, 1, 1, 1, dt), mode);
}
int lbw_moments_block(const double* f, const double* force, double* macro, int64_t nx,
                      int64_t ny, int64_t nz, double dt) {
    LBW_REQ(nx >= 1 && ny >= 1 && nz >= 1, "block size must be positive");
    LBW_REQ(f && force && macro, "null array");
    const int64_t cells = (nx + 2) * (ny + 2) * (nz + 2);
    DevBuf df, dF, dm;
    LBW_CK(df.alloc(cells * 27 * sizeof(double)));
    LBW_CK(dF.alloc(cells * 3 * sizeof(double)));
    LBW_CK(dm.alloc(cells * 4 * sizeof(double)));
    LBW_CK(cudaMemcpy(df.p, f, cells * 27 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dF.p, force, cells * 3 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dm.p, macro, cells * 4 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(launch_block_moments(df.as<double>(), dF.as<double>(), dm.as<double>(), nx, ny, nz, dt, 0));
    LBW_CK(cudaMemcpy(macro, dm.p, cells * 4 * sizeof(double), cudaMemcpyDeviceToHost));
    return LBW_OK;
}
int lbw_stream_pull_block(const double* fsrc, double* fdst, int64_t nx, int64_t ny, int64_t nz) {
    LBW_REQ(nx >= 1 && ny >= 1 && nz >= 1, "block size must be positive");
    LBW_REQ(fsrc && fdst, "null array");
    const int64_t cells = (nx + 2) * (ny + 2) * (nz + 2);
    DevBuf ds, dd;
    LBW_CK(ds.alloc(cells * 27 * sizeof(double)));
    LBW_CK(dd.alloc(cells * 27 * sizeof(double)));
    LBW_CK(cudaMemcpy(ds.p, fsrc, cells * 27 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(cudaMemcpy(dd.p, fdst, cells * 27 * sizeof(double), cudaMemcpyHostToDevice));
    LBW_CK(launch_block_stream(ds.as<double>(), dd.as<double>(), nx, ny, nz, 0));
    LBW_CK(cudaMemcpy(fdst, dd.p, cells * 27 * sizeof(double), cudaMemcpyDeviceToHost));
    return LBW_OK;
}

// ------------------------------------------------------------------ domain

static int alloc_dev(lbw_domain* d, void** p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error("device allocation of " + std::to_string(bytes) + " bytes failed");
        return LBW_ENOMEM;
    }
    d->bytes += (int64_t)bytes;
    return LBW_OK;
}

static void free_domain(lbw_domain* d) {
    if (!d) return;
    cudaSetDevice(d->device);
    if (d->stream) cudaStreamSynchronize(d->stream);
    if (d->alm_stream) cudaStreamSynchronize(d->alm_stream);
    alm_sync_side(d);
    alm_destroy(d);
    for (void*& b : d->buf)
        if (b) cudaFree(b);
    if (d->user.row_key) cudaFree(d->user.row_key);
    if (d->user.pool) cudaFree(d->user.pool);
    if (d->macro_dense) cudaFree(d->macro_dense);
    if (d->d_nan) cudaFree(d->d_nan);
    if (d->h_nan) cudaFreeHost(d->h_nan);
    if (d->nan_event) cudaEventDestroy(d->nan_event);
    if (d->stage) cudaFree(d->stage);
    for (cudaEvent_t ev : d->ev_pool) cudaEventDestroy(ev);
    peer_close(d);
    for (cudaEvent_t ev : {d->ev_main, d->ev_ready, d->ev_ready_prev, d->ev_alm_done})
        if (ev) cudaEventDestroy(ev);
    green_release(d);
    if (d->alm_stream) cudaStreamDestroy(d->alm_stream);
    if (d->stream) cudaStreamDestroy(d->stream);
    delete d;
}

static void polynomial_equilibrium(double rho, const double u[3], double out[27]) {
    // equilibrium_pdf (collision.py:54-67) for a single (rho, u); the host
    // wrapper passes the numpy-evaluated values instead when it has them.
    const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < 27; ++i) {
        const double cu = cx_of(i) * u[0] + cy_of(i) * u[1] + cz_of(i) * u[2];
        out[i] = w_of(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
    }
}

int lbw_domain_create(const lbw_domain_desc* desc, lbw_domain** out) {
    LBW_REQ(desc && out, "null argument");
    *out = nullptr;
    const lbw_domain_desc& s = *desc;
    for (int k = 0; k < 3; ++k) LBW_REQ(s.cells[k] >= 1, "cells must be positive");
    LBW_REQ(s.cells[1] <= (1 << 30) && s.cells[2] <= (1 << 30), "y/z extent too large");
    LBW_REQ(s.slab_nx >= 1 && s.slab_x0 >= 0 && s.slab_x0 + s.slab_nx <= s.cells[0],
            "slab outside the x extent");
    LBW_REQ(s.op == LBW_OP_BGK || s.op == LBW_OP_CUMULANT, "unknown collision operator");
    LBW_REQ(s.mode == LBW_MODE_EXACT || s.mode == LBW_MODE_FAST, "unknown arithmetic mode");
    LBW_REQ(s.boundary == LBW_BC_PERIODIC || s.boundary == LBW_BC_INFLOW_OUTFLOW,
            "unknown boundary kind");
    LBW_REQ(s.omega > 0.0 && s.omega < 2.0, "omega must lie in (0, 2)");
    for (int k = 0; k < 4; ++k)
        LBW_REQ(s.rates[k] >= 0.0 && s.rates[k] <= 2.0, "higher-order rate outside [0, 2]");
    LBW_REQ(!(s.boundary == LBW_BC_INFLOW_OUTFLOW && s.periodic[0]),
            "velocity_inflow_outflow needs a non-periodic x axis");
    LBW_REQ(s.nranks >= 1 && s.rank >= 0 && s.rank < s.nranks, "bad rank/nranks");
    LBW_REQ(s.precision == LBW_PREC_DOUBLE || s.precision == LBW_PREC_SINGLE,
            "unknown storage precision");
    for (int k = 0; k < 4; ++k) {
        LBW_REQ(s.walls[k] >= LBW_WALL_NONE && s.walls[k] <= LBW_WALL_FREE_SLIP, "unknown wall kind");
        LBW_REQ(s.walls[k] == LBW_WALL_NONE || !s.periodic[1 + k / 2],
                "walls need a non-periodic axis");
    }
    const int ndev = lbw_device_count();
    LBW_REQ(ndev > 0, "no CUDA device visible");
    LBW_REQ(s.device >= 0 && s.device < ndev, "device ordinal out of range");

    lbw_domain* d = new lbw_domain();
    d->desc = s;
    {
        // LBW_PRELAUNCH=0: queue each actuator chain only when its step runs
        // (diagnostics: the serial chain + sweep time)
        const char* e = getenv("LBW_PRELAUNCH");
        d->prelaunch = !(e && e[0] == '0');
        const char* alt = getenv("LBW_SWEEP_ALT");   // 0 disables (A/B)
        d->sweep_alt = !(alt && alt[0] == '0');
        // LBW_FUSED=1: one fused launch per actuator step (lbw_fused.cuh);
        // off by default until its chain latency beats the standalone chain
        const char* fu = getenv("LBW_FUSED");
        d->fused = fu && fu[0] == '1';
        const char* cb = getenv("LBW_CHAIN_FLAGS");  // 0: event-ordered chain (A/B)
        d->chainb = !(cb && cb[0] == '0');
        d->chainb_forced = cb && cb[0] == '1';
        // one resident chain kernel per multi-step call (lbw_alm.cu
        // k_cb_persist): by default with the FMA arithmetic, where the
        // per-step chain launches set the small-slab step time; the exact
        // flavour's slower sweep hides them.
        // LBW_CHAIN_LOOP=0/1 forces it off / on.
        const char* lp = getenv("LBW_CHAIN_LOOP");
        d->chain_loop = lp ? lp[0] == '1' : s.mode == LBW_MODE_FAST;
    }
    d->device = s.device;
    if (cudaSetDevice(d->device) != cudaSuccess) {
        cudaGetLastError();
        delete d;
        set_error("cudaSetDevice failed");
        return LBW_ECUDA;
    }
    Geom& g = d->g;
    g.nxl = (int32_t)s.slab_nx;
    g.ny = (int32_t)s.cells[1];
    g.nz = (int32_t)s.cells[2];
    g.single = s.precision == LBW_PREC_SINGLE ? 1 : 0;
    for (int k = 0; k < 4; ++k) g.walls[k] = s.walls[k];
    const int row_elems = g.single ? 32 : 16;   // 128-byte aligned z rows
    g.zp = (g.nz + row_elems - 1) / row_elems * row_elems;
    if (g.nz < row_elems) g.zp = g.nz;
    g.dir_stride = (int64_t)g.ny * g.zp;
    g.plane_stride = 27 * g.dir_stride;
    g.x0 = s.slab_x0;
    g.nxg = s.cells[0];
    g.per_y = s.periodic[1] ? 1 : 0;
    g.per_z = s.periodic[2] ? 1 : 0;
    const bool at_lo = s.slab_x0 == 0, at_hi = s.slab_x0 + s.slab_nx == s.cells[0];
    auto face = [&](bool lo) -> int {
        const bool edge = lo ? at_lo : at_hi;
        if (!edge) return XS_GHOST;
        if (s.boundary == LBW_BC_INFLOW_OUTFLOW) return lo ? XS_CONST : XS_CLAMP;
        if (!s.periodic[0]) return XS_ZERO;
        return s.nranks == 1 ? XS_WRAP : XS_GHOST;
    };
    g.lo_src = face(true);
    g.hi_src = face(false);
    if (s.feq_in_given)
        for (int i = 0; i < 27; ++i) g.feq_in[i] = s.feq_in[i];
    else
        polynomial_equilibrium(1.0, s.u_in, g.feq_in);
    // the reference stores the inflow ghost in the field's dtype (halo.py:152-156)
    if (g.single)
        for (int i = 0; i < 27; ++i) g.feq_in[i] = (double)(float)g.feq_in[i];
    d->relax = make_relax(s.omega, s.rates[0], s.rates[1], s.rates[2], s.rates[3], 1.0);

    int rc = LBW_OK;
    const size_t buf_bytes = (size_t)(g.nxl + 2) * g.plane_stride * elem_bytes(g);
    if (cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking) != cudaSuccess ||
        // the actuator chain runs beside the sweep: highest priority so its
        // few CTAs are dispatched ahead of the sweep's remaining ones
        [&] {
            int lo = 0, hi = 0;
            cudaDeviceGetStreamPriorityRange(&lo, &hi);
            return cudaStreamCreateWithPriority(&d->alm_stream, cudaStreamNonBlocking, hi);
        }() != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_main, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_ready_prev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_alm_done, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        free_domain(d);
        set_error("stream/event creation failed");
        return LBW_ECUDA;
    }
    for (int b = 0; b < 2 && rc == LBW_OK; ++b) rc = alloc_dev(d, (void**)&d->buf[b], buf_bytes);
    if (rc == LBW_OK) rc = alloc_dev(d, (void**)&d->d_nan, sizeof(unsigned long long));
    if (rc != LBW_OK) {
        free_domain(d);
        return rc;
    }
    if (cudaMallocHost(&d->h_nan, sizeof(unsigned long long)) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->nan_event, cudaEventDisableTiming) != cudaSuccess ||
        cudaMemsetAsync(d->buf[0], 0, buf_bytes, d->stream) != cudaSuccess ||
        cudaMemsetAsync(d->buf[1], 0, buf_bytes, d->stream) != cudaSuccess ||
        cudaMemsetAsync(d->d_nan, 0xff, sizeof(unsigned long long), d->stream) != cudaSuccess ||
        cudaStreamSynchronize(d->stream) != cudaSuccess) {
        cudaGetLastError();
        free_domain(d);
        set_error("domain initialisation failed");
        return LBW_ECUDA;
    }
    *d->h_nan = ~0ull;
    // inflow ghost data is constant: feq_in lives in the kernel parameters.
    *out = d;
    return LBW_OK;
}

int lbw_domain_destroy(lbw_domain* d) {
    free_domain(d);
    return LBW_OK;
}

int lbw_domain_stream(lbw_domain* d, void** s) {
    LBW_REQ(d && s, "null argument");
    *s = (void*)d->stream;
    return LBW_OK;
}

int64_t lbw_domain_device_bytes(lbw_domain* d) { return d ? d->bytes : 0; }

static size_t interior_cells(const lbw_domain* d) {
    return (size_t)d->g.nxl * d->g.ny * d->g.nz;
}

// The ALM samples a macro field defined by buffers the caller is about to
// overwrite: freeze it into the dense snapshot first.
static int freeze_macro_if(lbw_domain* d, bool touches_buf_cur, bool touches_user_force) {
    if (!alm_active(d) || d->msrc.kind != MS_GATHER) return LBW_OK;
    const bool hit = (touches_buf_cur && d->msrc.buf == d->cur) ||
                     (touches_user_force && d->msrc.fv.row_key == d->user.row_key &&
                      d->user.row_key != nullptr);
    if (!hit) return LBW_OK;
    if (!d->macro_dense) {
        int rc = alloc_dev(d, (void**)&d->macro_dense, interior_cells(d) * 4 * sizeof(double));
        if (rc) return rc;
    }
    LBW_CK(launch_moments_soa(d->msrc.pull, d->buf[d->msrc.buf], d->g, d->msrc.fv, 1.0,
                              d->macro_dense, d->stream));
    d->msrc.kind = MS_DENSE;
    return LBW_OK;
}

int lbw_domain_upload_pdf(lbw_domain* d, const double* f_aos) {
    LBW_REQ(d && f_aos, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    const size_t bytes = interior_cells(d) * 27 * sizeof(double);
    int rc = ensure_stage(d, bytes);
    if (rc) return rc;
    rc = freeze_macro_if(d, true, false);
    if (rc) return rc;
    LBW_CK(cudaMemcpyAsync(d->stage, f_aos, bytes, cudaMemcpyHostToDevice, d->stream));
    LBW_CK(launch_aos_to_soa(d->stage, d->buf[d->cur], d->g, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    d->state_pre = true;
    return LBW_OK;
}

int lbw_domain_fill_uniform(lbw_domain* d, const double* f27) {
    LBW_REQ(d && f27, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    int rc = freeze_macro_if(d, true, false);
    if (rc) return rc;
    double v[27];
    for (int i = 0; i < 27; ++i) v[i] = f27[i];
    LBW_CK(launch_fill_uniform(v, d->buf[d->cur], d->g, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    d->state_pre = true;
    return LBW_OK;
}

int lbw_domain_init_modes(lbw_domain* d, double rho, const double* u0, int32_t n_modes,
                          const double* modes, int32_t product) {
    LBW_REQ(d && u0, "null argument");
    LBW_REQ(n_modes >= 0 && (n_modes == 0 || modes), "bad mode table");
    LBW_REQ(rho > 0.0, "density must be positive");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    int rc = freeze_macro_if(d, true, false);
    if (rc) return rc;
    if (!d->macro_dense) {
        rc = alloc_dev(d, (void**)&d->macro_dense, interior_cells(d) * 4 * sizeof(double));
        if (rc) return rc;
    }
    double* dmodes = nullptr;
    const size_t mb = (size_t)(n_modes > 0 ? n_modes : 1) * 7 * sizeof(double);
    LBW_CK(cudaMalloc(&dmodes, mb));
    if (n_modes > 0)
        LBW_CK(cudaMemcpyAsync(dmodes, modes, (size_t)n_modes * 7 * sizeof(double),
                               cudaMemcpyHostToDevice, d->stream));
    const double u[3] = {u0[0], u0[1], u0[2]};
    const cudaError_t e = launch_init_modes(rho, u, n_modes, dmodes, product ? 1 : 0,
                                            d->buf[d->cur], d->macro_dense, d->g, d->stream);
    const cudaError_t e2 = cudaStreamSynchronize(d->stream);
    cudaFree(dmodes);
    LBW_CK(e);
    LBW_CK(e2);
    d->state_pre = true;
    d->msrc.kind = MS_DENSE;
    d->user_active = false;
    d->shown_fv = ForceView{nullptr, nullptr, 0};
    return LBW_OK;
}

int lbw_domain_upload_pdf_device(lbw_domain* d, const double* f_aos_dev) {
    LBW_REQ(d && f_aos_dev, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    int rc = freeze_macro_if(d, true, false);
    if (rc) return rc;
    LBW_CK(launch_aos_to_soa(f_aos_dev, d->buf[d->cur], d->g, d->stream));
    d->state_pre = true;
    return LBW_OK;
}

int lbw_domain_download_pdf(lbw_domain* d, double* f_aos) {
    LBW_REQ(d && f_aos, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = peer_wait(d, d->stream, 0, (uint32_t)d->steps_done);
        if (rc_) return rc_;
    }
    const size_t bytes = interior_cells(d) * 27 * sizeof(double);
    int rc = ensure_stage(d, bytes);
    if (rc) return rc;
    // post-collision state -> the reference's post-stream state (stream only)
    LBW_CK(launch_gather_aos(!d->state_pre, d->buf[d->cur], d->g, d->stage, d->stream));
    LBW_CK(cudaMemcpyAsync(f_aos, d->stage, bytes, cudaMemcpyDeviceToHost, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    return LBW_OK;
}

int lbw_domain_set_force(lbw_domain* d, const double* force_aos) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    int rc = freeze_macro_if(d, false, true);
    if (rc) return rc;
    if (!force_aos) {
        d->user_active = false;
        d->shown_fv = ForceView{nullptr, nullptr, 0};
        return LBW_OK;
    }
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    if (!d->user.row_key) {
        rc = alloc_dev(d, (void**)&d->user.row_key, rows * sizeof(uint64_t));
        if (!rc) rc = alloc_dev(d, (void**)&d->user.pool, rows * 3 * d->g.zp * elem_bytes(d->g));
        if (rc) return rc;
        d->user.cap = rows;
    }
    const size_t bytes = interior_cells(d) * 3 * sizeof(double);
    rc = ensure_stage(d, bytes);
    if (rc) return rc;
    LBW_CK(cudaMemcpyAsync(d->stage, force_aos, bytes, cudaMemcpyHostToDevice, d->stream));
    LBW_CK(launch_force_from_aos(d->stage, d->g, d->user.row_key, d->user.pool, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    d->user_active = true;
    d->shown_fv = d->user.view(0);
    return LBW_OK;
}

int lbw_domain_download_force(lbw_domain* d, double* force_aos) {
    LBW_REQ(d && force_aos, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    const size_t bytes = interior_cells(d) * 3 * sizeof(double);
    int rc = ensure_stage(d, bytes);
    if (rc) return rc;
    LBW_CK(launch_force_to_aos(d->shown_fv, d->g, d->stage, d->stream));
    LBW_CK(cudaMemcpyAsync(force_aos, d->stage, bytes, cudaMemcpyDeviceToHost, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    return LBW_OK;
}

int lbw_domain_set_macro(lbw_domain* d, const double* macro_aos, const double* uniform4) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    if (uniform4) {
        d->msrc.kind = MS_UNIFORM;
        for (int k = 0; k < 4; ++k) d->msrc.uniform[k] = uniform4[k];
        return LBW_OK;
    }
    if (!macro_aos) return LBW_OK;
    const size_t bytes = interior_cells(d) * 4 * sizeof(double);
    if (!d->macro_dense) {
        int rc = alloc_dev(d, (void**)&d->macro_dense, bytes);
        if (rc) return rc;
    }
    LBW_CK(cudaMemcpyAsync(d->macro_dense, macro_aos, bytes, cudaMemcpyHostToDevice, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    d->msrc.kind = MS_DENSE;
    return LBW_OK;
}

int lbw_domain_download_macro(lbw_domain* d, double* macro_aos) {
    LBW_REQ(d && macro_aos, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = peer_wait(d, d->stream, 0, (uint32_t)d->steps_done);
        if (rc_) return rc_;
    }
    const size_t n = interior_cells(d);
    if (d->msrc.kind == MS_UNIFORM) {
        for (size_t c = 0; c < n; ++c)
            for (int k = 0; k < 4; ++k) macro_aos[c * 4 + k] = d->msrc.uniform[k];
        return LBW_OK;
    }
    const size_t bytes = n * 4 * sizeof(double);
    if (d->msrc.kind == MS_DENSE) {
        LBW_CK(cudaMemcpyAsync(macro_aos, d->macro_dense, bytes, cudaMemcpyDeviceToHost, d->stream));
    } else {
        int rc = ensure_stage(d, bytes);
        if (rc) return rc;
        LBW_CK(launch_moments_soa(d->msrc.pull, d->buf[d->msrc.buf], d->g, d->msrc.fv, 1.0,
                                  d->stage, d->stream));
        LBW_CK(cudaMemcpyAsync(macro_aos, d->stage, bytes, cudaMemcpyDeviceToHost, d->stream));
    }
    LBW_CK(cudaStreamSynchronize(d->stream));
    return LBW_OK;
}

int lbw_domain_recompute_moments(lbw_domain* d, double* macro_aos) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    {
        int rc_ = alm_invalidate(d);
        if (rc_) return rc_;
    }
    {
        int rc_ = peer_wait(d, d->stream, 0, (uint32_t)d->steps_done);
        if (rc_) return rc_;
    }
    const size_t bytes = interior_cells(d) * 4 * sizeof(double);
    int rc = ensure_stage(d, bytes);
    if (rc) return rc;
    const ForceView fv = d->shown_fv;
    LBW_CK(launch_moments_soa(!d->state_pre, d->buf[d->cur], d->g, fv, 1.0, d->stage, d->stream));
    if (macro_aos)
        LBW_CK(cudaMemcpyAsync(macro_aos, d->stage, bytes, cudaMemcpyDeviceToHost, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    // _recompute_moments overwrites PdfField.macro (sim.py:160-165): the
    // next actuator step samples these moments.
    d->msrc.kind = MS_GATHER;
    d->msrc.buf = d->cur;
    d->msrc.pull = !d->state_pre;
    d->msrc.fv = fv;
    return LBW_OK;
}

int lbw_domain_step(lbw_domain* d, int32_t nsteps) {
    LBW_REQ(d, "null domain");
    LBW_REQ(nsteps >= 0, "nsteps must be >= 0");
    LBW_CK(cudaSetDevice(d->device));
    for (int32_t s = 0; s < nsteps; ++s) {
        ForceView fv = d->user_active ? d->user.view(0) : ForceView{nullptr, nullptr, 0};
        const uint32_t* gate_flag = nullptr;
        const int32_t* gate_box = nullptr;
        uint32_t gate_value = 0;
        // neighbours must have finished the previous sweep: it filled our
        // ghost planes and stopped reading theirs (which we overwrite now)
        {
            int rc = peer_wait(d, d->stream, 0, (uint32_t)d->steps_done);
            if (rc) return rc;
        }
        std::swap(d->ev_ready, d->ev_ready_prev);
        LBW_CK(cudaEventRecord(d->ev_ready, d->stream));
        if (alm_active(d) && alm_fused_eligible(d)) {
            // one launch: sweep + this step's point forces + the kinematics
            // of step+2 (lbw_fused.cuh)
            const bool pull = !d->state_pre;
            if (d->timing) {
                while (d->ev_pool.size() < d->ev_used + 2) {
                    cudaEvent_t ev;
                    LBW_CK(cudaEventCreate(&ev));
                    d->ev_pool.push_back(ev);
                }
                LBW_CK(cudaEventRecord(d->ev_pool[d->ev_used], d->stream));
            }
            int rc = alm_fused_launch(d, pull, &fv);
            if (rc) return rc;
            if (d->timing) {
                LBW_CK(cudaEventRecord(d->ev_pool[d->ev_used + 1], d->stream));
                d->ev_used += 2;
            }
            d->msrc.kind = MS_GATHER;
            d->msrc.buf = d->cur;
            d->msrc.pull = pull;
            d->msrc.fv = fv;
            d->last_fv = fv;
            d->shown_fv = fv;
            d->touched = false;
            d->cur = 1 - d->cur;
            d->state_pre = false;
            d->step += 1;
            d->steps_done += 1;
            continue;
        }
        // flag-ordered actuator chain (chain B): no stream waits on the main stream
        const bool cb = alm_active(d) && alm_chainb_eligible(d);
        if (alm_active(d) && !cb) {
            // The actuator chain of this step normally was queued on the
            // actuator stream while the previous sweep ran.  Otherwise (host
            // kinematics, first step) queue it now: it needs the sweep two
            // steps back (ev_ready_prev: its sampled state and force set)
            // unless a call changed state since the last step, in which case
            // it waits for everything already on the main stream.
            if (!alm_ready(d, d->step)) {
                if (d->touched || alm_after_fused(d) || alm_after_chainb(d)) {
                    LBW_CK(cudaEventRecord(d->ev_main, d->stream));
                    LBW_CK(cudaStreamWaitEvent(d->alm_stream, d->ev_main, 0));
                } else {
                    LBW_CK(cudaStreamWaitEvent(d->alm_stream, d->ev_ready_prev, 0));
                }
                int rc = alm_launch(d, d->step);
                if (rc) return rc;
            }
            const uint32_t* gflag = nullptr;
            const int32_t* gbox = nullptr;
            uint32_t gvalue = 0;
            cudaEvent_t kev = nullptr;
            if (alm_gate(d, d->step, &gflag, &gvalue, &gbox, &kev)) {
                // the sweep starts right away; its CTAs in the chain's x range
                // wait in-kernel for the chain (needs this step's x range)
                LBW_CK(cudaStreamWaitEvent(d->stream, kev, 0));
                gate_flag = gflag;
                gate_box = gbox;
                gate_value = gvalue;
            } else {
                LBW_CK(cudaStreamWaitEvent(d->stream, d->ev_alm_done, 0));
            }
            fv = alm_force_view(d, d->step);
        }
        SweepArgs a{};
        a.src = d->buf[d->cur];
        a.dst = d->buf[1 - d->cur];
        a.g = d->g;
        a.fv = fv;
        a.r = d->relax;
        a.x_begin = 0;
        a.x_end = d->g.nxl;
        a.nan_key = d->d_nan;
        a.step = d->step;
        a.reverse = (d->sweep_alt && (d->step & 1)) ? 1 : 0;
        a.halo = d->halo[1 - d->cur];
        a.gate_flag = gate_flag;
        a.gate_box = gate_box;
        a.gate_value = gate_value;
        a.gate_error = gate_flag ? reinterpret_cast<int32_t*>(const_cast<uint32_t*>(gate_flag) + 1)
                                 : nullptr;
        a.pdl = d->linked ? 0 : 1;
        if (d->linked) {
            // the sweep itself tells the neighbours when its edge planes
            // (halo stores included) are done: flag value = sweeps completed
            a.halo.peer_flag[0] = d->nb_rank[0] >= 0 ? d->nb_flags[0] + 1 : nullptr;
            a.halo.peer_flag[1] = d->nb_rank[1] >= 0 ? d->nb_flags[1] + 0 : nullptr;
            a.halo.edge_counter = d->edge_counter;
            a.halo.value = (uint32_t)(d->steps_done + 1);
        }
        if (cb) {
            int rc = alm_chainb_before(d, &a);
            if (rc) return rc;
            fv = a.fv;
        }
        const bool pull = !d->state_pre;
        if (d->timing) {
            while (d->ev_pool.size() < d->ev_used + 2) {
                cudaEvent_t ev;
                LBW_CK(cudaEventCreate(&ev));
                d->ev_pool.push_back(ev);
            }
            LBW_CK(cudaEventRecord(d->ev_pool[d->ev_used], d->stream));
        }
        const cudaError_t e = d->desc.mode == LBW_MODE_FAST
                                  ? launch_sweep_fast(d->desc.op, pull, a, d->stream)
                                  : launch_sweep_exact(d->desc.op, pull, a, d->stream);
        LBW_CK(e);
        if (d->timing) {
            LBW_CK(cudaEventRecord(d->ev_pool[d->ev_used + 1], d->stream));
            d->ev_used += 2;
        }
        // the next step samples moments(pre-collision f, F) of this collide
        d->msrc.kind = MS_GATHER;
        d->msrc.buf = d->cur;
        d->msrc.pull = pull;
        d->msrc.fv = fv;
        d->last_fv = fv;
        d->shown_fv = fv;
        d->touched = false;
        d->cur = 1 - d->cur;
        d->state_pre = false;
        d->step += 1;
        d->steps_done += 1;
        // Queue the next step's actuator chain now: it reads only this
        // sweep's source buffer (ghost planes included) and force set, both
        // read-only during the sweep, and rewrites the force set of the sweep
        // before — exactly the preconditions of this sweep (ev_ready) — so it
        // overlaps this sweep.
        if (cb) {
            int rc = alm_chainb_after(d, d->step - 1, nsteps - s);
            if (rc) return rc;
        } else if (alm_active(d) && alm_can_prelaunch(d)) {
            LBW_CK(cudaStreamWaitEvent(d->alm_stream, d->ev_ready, 0));
            int rc = alm_launch(d, d->step);
            if (rc) return rc;
        }
    }
    if (nsteps > 0) {
        LBW_CK(cudaMemcpyAsync(d->h_nan, d->d_nan, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, d->stream));
        LBW_CK(cudaEventRecord(d->nan_event, d->stream));
        d->nan_pending = true;
    }
    return LBW_OK;
}

int64_t lbw_domain_step_index(lbw_domain* d) { return d ? d->step : -1; }
int lbw_domain_set_step_index(lbw_domain* d, int64_t step) {
    LBW_REQ(d && step >= 0, "bad argument");
    LBW_CK(cudaSetDevice(d->device));
    int rc = alm_invalidate(d);
    if (rc) return rc;
    LBW_REQ(!alm_active(d) || step == d->step,
            "the step index of a domain with actuator points cannot be changed");
    d->step = step;
    return LBW_OK;
}

int lbw_domain_poll_nonfinite(lbw_domain* d, int wait, int64_t* step, int64_t* cell3,
                              int32_t* field) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    if (d->nan_pending) {
        if (wait) {
            LBW_CK(cudaEventSynchronize(d->nan_event));
            d->nan_pending = false;
        } else {
            const cudaError_t q = cudaEventQuery(d->nan_event);
            if (q == cudaSuccess) d->nan_pending = false;
            else if (q != cudaErrorNotReady) LBW_CK(q);
            else cudaGetLastError();
        }
    }
    const unsigned long long k = *d->h_nan;
    if (k == ~0ull) return 0;
    const int64_t cell = (int64_t)((k >> 1) & ((1ull << 39) - 1));
    if (step) *step = (int64_t)(k >> 40);
    if (cell3) {
        const int64_t ny = d->g.ny, nz = d->g.nz;
        cell3[0] = cell / (ny * nz);
        cell3[1] = (cell / nz) % ny;
        cell3[2] = cell % nz;
    }
    if (field) *field = (k & 1ull) ? 1 : 0;
    return 1;
}

int lbw_domain_hold_collided(lbw_domain* d) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    int rc = alm_invalidate(d);
    if (rc) return rc;
    // buf[cur] holds the last collide's output; marking it pre-collision
    // makes downloads return it as is (no stream) -- the reference's f after
    // the abort -- and a further step collides it again, as the reference's
    // next step() would.  The sampled macro (msrc) stays that collide's.
    d->state_pre = true;
    return LBW_OK;
}

int lbw_domain_sync(lbw_domain* d) {
    LBW_REQ(d, "null domain");
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    return alm_check_gate(d);
}

int lbw_domain_sweep_timing(lbw_domain* d, int enable) {
    LBW_REQ(d, "null domain");
    d->timing = enable != 0;
    d->ev_used = 0;
    return LBW_OK;
}

int lbw_domain_sweep_time(lbw_domain* d, double* ms_total, int64_t* launches) {
    LBW_REQ(d && ms_total && launches, "null argument");
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    double total = 0.0;
    for (size_t k = 0; k + 1 < d->ev_used; k += 2) {
        float ms = 0.0f;
        LBW_CK(cudaEventElapsedTime(&ms, d->ev_pool[k], d->ev_pool[k + 1]));
        total += ms;
    }
    *ms_total = total;
    *launches = (int64_t)(d->ev_used / 2);
    return LBW_OK;
}

}  // extern "C"
