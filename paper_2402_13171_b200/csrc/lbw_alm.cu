// lbw_alm.cu — actuator-line coupling on the device (compiled with
// -fmad=false, like the exact sweep: the per-point arithmetic follows the
// reference expression order).
//
//   K4  k_alm_sample_force   one thread per point: trilinear sampling of the
//                            previous step's macro field (recomputed from the
//                            retained population buffer, App. A.7 of
//                            SURVEY.md), angle of attack, polar lookup,
//                            blade-element force, lattice force
//                            (actuator.py:70-146, polars.py:65-80,
//                            sim.py:210-235, units.py:69-70)
//   K5a k_alm_clear          forget the rows used two steps ago
//   K5b k_alm_mark           per point: Roma weights per axis with periodic
//                            images (actuator.py:100-110, 190-195, 297-341);
//                            claim a pool slot for every touched (x,y) row
//   K5c k_alm_fill           one CTA per touched row: per cell, sum
//                            (wx*wy)*wz*F over the points in ascending
//                            global id starting from 0.0 (actuator.py:204-247)
//                            — deterministic, no float atomics.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "lbw_domain.h"

#define LBW_FAST 0
#include "lbw_sweep.cuh"

namespace lbw {

constexpr int kKin = 15;  // pos_lat(3) vel(3) e_chord(3) e_normal(3) e_span(3)
constexpr int kRing = 8;

struct AlmDev {
    int32_t n;
    const double* chord;
    const double* elen;
    const double* twist;
    const int32_t* polar_index;
    const int32_t* polar_offset;
    const int32_t* polar_rows;
    const double* p_alpha;
    const double* p_cl;
    const double* p_cd;
    double vscale, rho_ref, dt2, den;
    const double* kin;     // (P,15)
    double* samples;       // (P,4)
    double* blade;         // (P,3)
    double* flat;          // (P,3) lattice force on the fluid
    int32_t* dep_cell;     // (P,3 axes,3) global cell or -1
    double* dep_w;         // (P,3,3)
    int32_t* clamp_flags;  // (n_polars)
    int32_t* error_flags;  // bit 0: non-positive sampled density
};

struct AlmState {
    int32_t n = 0, n_polars = 0;
    double *chord = nullptr, *elen = nullptr, *twist = nullptr;
    int32_t *polar_index = nullptr, *polar_offset = nullptr, *polar_rows = nullptr;
    double *p_alpha = nullptr, *p_cl = nullptr, *p_cd = nullptr;
    double* kin = nullptr;
    double *samples = nullptr, *blade = nullptr, *flat = nullptr;
    int32_t* dep_cell = nullptr;
    double* dep_w = nullptr;
    int32_t *clamp_flags = nullptr, *error_flags = nullptr;
    double vscale = 0, rho_ref = 0, dt2 = 0, den = 0;
    ForceSet set[2];
    double* h_ring = nullptr;   // pinned (kRing, P, 15)
    cudaEvent_t ring_ev[kRing] = {};
    int ring_pos = 0;
    bool kin_queued = false;
    bool stepped = false;       // apply_outer_boundary has run at least once
    int flip = 0;               // force set written by the next actuator step
    std::vector<void*> allocs;
    AlmDev dev() const {
        AlmDev a;
        a.n = n;
        a.chord = chord;
        a.elen = elen;
        a.twist = twist;
        a.polar_index = polar_index;
        a.polar_offset = polar_offset;
        a.polar_rows = polar_rows;
        a.p_alpha = p_alpha;
        a.p_cl = p_cl;
        a.p_cd = p_cd;
        a.vscale = vscale;
        a.rho_ref = rho_ref;
        a.dt2 = dt2;
        a.den = den;
        a.kin = kin;
        a.samples = samples;
        a.blade = blade;
        a.flat = flat;
        a.dep_cell = dep_cell;
        a.dep_w = dep_w;
        a.clamp_flags = clamp_flags;
        a.error_flags = error_flags;
        return a;
    }
};

// How the macro field sampled at this step is obtained (MacroSource).
struct MacroDev {
    int kind;
    double uniform[4];
    const double* buf;
    int pull;
    ForceView fv;
    const double* dense;
    int bc_set;        // the x-face BC has written its macro ghosts (after step 0)
    double u_in[3];
    int inflow;        // velocity_inflow_outflow
    int per_x;
};

namespace {

// Macro (rho, u) of global cell (gx,gy,gz), following the ghost semantics
// of PdfField.macro (fields.py:35-36, halo.py:144-160).  Returns false when
// the cell belongs to another slab.
__device__ bool macro_at(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                         double out[4]) {
    const double ghost0[4] = {1.0, 0.0, 0.0, 0.0};
    auto put = [&](const double* v) {
        for (int k = 0; k < 4; ++k) out[k] = v[k];
    };
    if (gx < 0 || gx >= g.nxg) {
        if (m.per_x) {
            gx = gx < 0 ? gx + g.nxg : gx - g.nxg;
        } else if (m.inflow && gx < 0) {
            if (m.bc_set) {
                out[0] = 1.0;
                out[1] = m.u_in[0];
                out[2] = m.u_in[1];
                out[3] = m.u_in[2];
            } else {
                put(ghost0);
            }
            return true;
        } else if (m.inflow && gx >= g.nxg && m.bc_set) {
            gx = g.nxg - 1;
        } else {
            put(ghost0);
            return true;
        }
    }
    if (gy < 0 || gy >= g.ny) {
        if (!g.per_y) { put(ghost0); return true; }
        gy = gy < 0 ? gy + g.ny : gy - g.ny;
    }
    if (gz < 0 || gz >= g.nz) {
        if (!g.per_z) { put(ghost0); return true; }
        gz = gz < 0 ? gz + g.nz : gz - g.nz;
    }
    const int64_t x = gx - g.x0;
    if (x < 0 || x >= g.nxl) return false;
    if (m.kind == MS_UNIFORM) {
        put(m.uniform);
        return true;
    }
    const int64_t cell = (x * g.ny + gy) * g.nz + gz;
    if (m.kind == MS_DENSE) {
        put(m.dense + cell * 4);
        return true;
    }
    double f[27];
    if (m.pull) load_cell<true>(m.buf, g, (int)x, (int)gy, (int)gz, f);
    else load_cell<false>(m.buf, g, (int)x, (int)gy, (int)gz, f);
    double Fx, Fy, Fz;
    load_force(m.fv, g, (int)x, (int)gy, (int)gz, Fx, Fy, Fz);
    const Macro mm = moments_exact(f, Fx, Fy, Fz, 1.0);
    out[0] = mm.rho;
    out[1] = mm.ux;
    out[2] = mm.uy;
    out[3] = mm.uz;
    return true;
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// np.interp on one value (numpy compiled_base.c arr_interp semantics)
__device__ double interp1(double x, const double* xp, const double* fp, int n) {
    if (isnan(x)) return x;
    int j;
    if (x < xp[0]) return fp[0];
    if (x > xp[n - 1]) return fp[n - 1];
    if (x == xp[n - 1]) return fp[n - 1];
    int lo = 0, hi = n - 1;  // xp[lo] <= x < xp[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (xp[mid] <= x) lo = mid;
        else hi = mid;
    }
    j = lo;
    if (xp[j] == x) return fp[j];
    const double slope = (fp[j + 1] - fp[j]) / (xp[j + 1] - xp[j]);
    double r = slope * (x - xp[j]) + fp[j];
    if (isnan(r)) {
        r = slope * (x - xp[j + 1]) + fp[j + 1];
        if (isnan(r) && fp[j] == fp[j + 1]) r = fp[j];
    }
    return r;
}

// Roma 3-point kernel (actuator.py:100-110)
__device__ __forceinline__ double roma(double r) {
    const double a = fabs(r);
    if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * (a * a))) / 3.0;
    if (a <= 1.5) {
        const double b = 1.0 - a;
        return (5.0 - 3.0 * a - sqrt(1.0 - 3.0 * (b * b))) / 6.0;
    }
    return 0.0;
}

__global__ void k_alm_sample_force(AlmDev a, Geom g, MacroDev m) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.n) return;
    const double* kin = a.kin + (int64_t)p * kKin;
    // --- trilinear sampling (actuator.py:77-93)
    int64_t j0[3];
    double t[3];
    for (int k = 0; k < 3; ++k) {
        const double fl = floor(kin[k] - 0.5);
        j0[k] = (int64_t)fl;
        t[k] = kin[k] - 0.5 - fl;
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int dx = 0; dx < 2; ++dx) {
        const double wx = dx ? t[0] : 1.0 - t[0];
        for (int dy = 0; dy < 2; ++dy) {
            const double wy = dy ? t[1] : 1.0 - t[1];
            for (int dz = 0; dz < 2; ++dz) {
                const double wz = dz ? t[2] : 1.0 - t[2];
                const double w = wx * wy * wz;
                double v[4];
                macro_at(g, m, j0[0] + dx, j0[1] + dy, j0[2] + dz, v);
                for (int c = 0; c < 4; ++c) acc[c] += w * v[c];
            }
        }
    }
    for (int c = 0; c < 4; ++c) a.samples[p * 4 + c] = acc[c];

    // --- blade element (actuator.py:117-146, sim.py:218-235)
    double blade[3] = {0.0, 0.0, 0.0};
    const int pid = a.polar_index[p];
    if (pid >= 0) {
        const double* vel = kin + 3;
        const double* ec = kin + 6;
        const double* en = kin + 9;
        const double* es = kin + 12;
        double urel[3];
        for (int c = 0; c < 3; ++c) urel[c] = acc[1 + c] * a.vscale - vel[c];
        const double along = dot3(urel, es);
        double up[3];
        for (int c = 0; c < 3; ++c) up[c] = urel[c] - along * es[c];
        const double speed = sqrt(dot3(up, up));
        if (speed >= 1e-12) {  // DEGENERATE_SPEED (actuator.py:30)
            const double phi = atan2(dot3(up, en), dot3(up, ec));
            double alpha = phi - a.twist[p];
            double ed[3], el[3];
            for (int c = 0; c < 3; ++c) ed[c] = up[c] / speed;
            el[0] = es[1] * ed[2] - es[2] * ed[1];
            el[1] = es[2] * ed[0] - es[0] * ed[2];
            el[2] = es[0] * ed[1] - es[1] * ed[0];
            const int off = a.polar_offset[pid], rows = a.polar_rows[pid];
            const double* xp = a.p_alpha + off;
            if (alpha < xp[0] || alpha > xp[rows - 1]) {
                atomicOr(&a.clamp_flags[pid], 1);
                alpha = fmin(fmax(alpha, xp[0]), xp[rows - 1]);
            }
            const double cl = interp1(alpha, xp, a.p_cl + off, rows);
            const double cd = interp1(alpha, xp, a.p_cd + off, rows);
            const double rho_phys = acc[0] * a.rho_ref;
            if (!(rho_phys > 0.0)) atomicOr(a.error_flags, 1);
            const double scale = 0.5 * rho_phys * speed * speed * a.chord[p] * a.elen[p];
            for (int c = 0; c < 3; ++c) blade[c] = scale * (cl * el[c] + cd * ed[c]);
        }
    }
    for (int c = 0; c < 3; ++c) {
        a.blade[p * 3 + c] = blade[c];
        // fluid force = -blade, to lattice units (units.py:69)
        a.flat[p * 3 + c] = -blade[c] * a.dt2 / a.den;
    }
}

__global__ void k_alm_clear(ForceSet s) {
    const int32_t n = *s.count;
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) s.row_slot[s.slot_row[i]] = -1;
    __syncthreads();
    if (threadIdx.x == 0) *s.count = 0;
}

// per point: deposit cells + Roma weights per axis, images across periodic
// faces computed from the shifted position pos - w*L (actuator.py:330-332)
__global__ void k_alm_mark(AlmDev a, Geom g, int per_x, ForceSet s) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.n) return;
    const double* kin = a.kin + (int64_t)p * kKin;
    const int64_t dims[3] = {g.nxg, g.ny, g.nz};
    const int per[3] = {per_x, g.per_y, g.per_z};
    int32_t* dc = a.dep_cell + (int64_t)p * 9;
    double* dw = a.dep_w + (int64_t)p * 9;
    for (int k = 0; k < 3; ++k) {
        int cnt = 0;
        for (int q = 0; q < 3; ++q) { dc[k * 3 + q] = -1; dw[k * 3 + q] = 0.0; }
        const int nimg = per[k] ? 3 : 1;
        for (int im = 0; im < nimg; ++im) {
            const double w = im == 0 ? 0.0 : (im == 1 ? 1.0 : -1.0);
            const double x = im == 0 ? kin[k] : kin[k] - w * (double)dims[k];
            const double n0f = floor(x);
            const int64_t n0 = (int64_t)n0f;
            const double r[3] = {x - (n0f - 0.5), x - (n0f + 0.5), x - (n0f + 1.5)};
            for (int q = 0; q < 3; ++q) {
                const int64_t c = n0 - 1 + q;
                if (c < 0 || c >= dims[k]) continue;
                const double wt = roma(r[q]);
                if (wt == 0.0 || cnt >= 3) continue;
                dc[k * 3 + cnt] = (int32_t)c;
                dw[k * 3 + cnt] = wt;
                ++cnt;
            }
        }
    }
    // claim the (x,y) rows of this slab
    for (int i = 0; i < 3; ++i) {
        const int32_t cxg = dc[i];
        if (cxg < 0) continue;
        const int64_t x = cxg - g.x0;
        if (x < 0 || x >= g.nxl) continue;
        for (int j = 0; j < 3; ++j) {
            const int32_t cy = dc[3 + j];
            if (cy < 0) continue;
            const int64_t row = x * g.ny + cy;
            if (atomicCAS(&s.row_slot[row], -1, -2) == -1) {
                const int32_t slot = atomicAdd(s.count, 1);
                s.slot_row[slot] = (int32_t)row;
                s.row_slot[row] = slot;
            }
        }
    }
}

// one CTA per used slot; dynamic shared memory holds (point, wxy) pairs
__global__ void k_alm_fill(AlmDev a, Geom g, ForceSet s) {
    extern __shared__ unsigned char smem[];
    const int32_t slot = blockIdx.x;
    if (slot >= *s.count) return;
    const int32_t row = s.slot_row[slot];
    const int64_t xg = row / g.ny + g.x0;
    const int32_t y = row % g.ny;
    int32_t* list_p = reinterpret_cast<int32_t*>(smem);
    double* list_w = reinterpret_cast<double*>(smem + ((a.n * 4 + 15) / 16) * 16);
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    // ordered compaction of the points touching row (xg, y)
    for (int c0 = 0; c0 < a.n; c0 += blockDim.x) {
        const int p = c0 + threadIdx.x;
        bool hit = false;
        double wxy = 0.0;
        if (p < a.n) {
            const int32_t* dc = a.dep_cell + (int64_t)p * 9;
            const double* dw = a.dep_w + (int64_t)p * 9;
            double wx = 0.0, wy = 0.0;
            bool hx = false, hy = false;
            for (int q = 0; q < 3; ++q) {
                if (dc[q] == xg) { hx = true; wx = dw[q]; }
                if (dc[3 + q] == y) { hy = true; wy = dw[3 + q]; }
            }
            hit = hx && hy;
            wxy = wx * wy;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) warp_tot[warp] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int w = 0; w < warp; ++w) off += warp_tot[w];
        off += __popc(bal & ((1u << lane) - 1u));
        if (hit) {
            list_p[off] = p;
            list_w[off] = wxy;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < nwarp; ++w) tot += warp_tot[w];
            base += tot;
        }
        __syncthreads();
    }
    const int nlist = base;
    double* dst = s.pool + (int64_t)slot * 3 * g.zp;
    for (int z = threadIdx.x; z < g.nz; z += blockDim.x) {
        double F[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < nlist; ++q) {
            const int p = list_p[q];
            const int32_t* dc = a.dep_cell + (int64_t)p * 9 + 6;
            const double* dw = a.dep_w + (int64_t)p * 9 + 6;
            for (int k = 0; k < 3; ++k) {
                if (dc[k] == z) {
                    const double w = list_w[q] * dw[k];
                    for (int c = 0; c < 3; ++c) F[c] += w * a.flat[p * 3 + c];
                }
            }
        }
        for (int c = 0; c < 3; ++c) dst[(int64_t)c * g.zp + z] = F[c];
    }
}

template <class T>
int dev_alloc(lbw_domain* d, AlmState* s, T** p, size_t count) {
    if (count == 0) count = 1;
    if (cudaMalloc((void**)p, count * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        set_error("ALM device allocation failed");
        return LBW_ENOMEM;
    }
    s->allocs.push_back(*p);
    d->bytes += (int64_t)(count * sizeof(T));
    return LBW_OK;
}

}  // namespace

bool alm_active(const lbw_domain* d) { return d->alm != nullptr && d->alm->n > 0; }

void alm_destroy(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s) return;
    for (void* p : s->allocs) cudaFree(p);
    for (auto& e : s->ring_ev)
        if (e) cudaEventDestroy(e);
    if (s->h_ring) cudaFreeHost(s->h_ring);
    delete s;
    d->alm = nullptr;
}

int alm_before_collide(lbw_domain* d, ForceView* fv_out) {
    AlmState* s = d->alm;
    if (!s->kin_queued) {
        set_error("actuator step without kinematics: call lbw_alm_set_kinematics first");
        return LBW_ESTATE;
    }
    s->kin_queued = false;
    const Geom& g = d->g;
    MacroDev m{};
    m.kind = d->msrc.kind;
    for (int k = 0; k < 4; ++k) m.uniform[k] = d->msrc.uniform[k];
    m.buf = d->buf[d->msrc.buf];
    m.pull = d->msrc.pull ? 1 : 0;
    m.fv = d->msrc.fv;
    m.dense = d->macro_dense;
    m.bc_set = s->stepped ? 1 : 0;
    for (int k = 0; k < 3; ++k) m.u_in[k] = d->desc.u_in[k];
    m.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    m.per_x = d->desc.periodic[0] ? 1 : 0;
    const AlmDev a = s->dev();
    const int threads = 64;
    const unsigned blocks = (unsigned)((s->n + threads - 1) / threads);
    k_alm_sample_force<<<blocks, threads, 0, d->stream>>>(a, g, m);
    count_launch();
    LBW_CK(cudaGetLastError());
    ForceSet& fs = s->set[s->flip];
    s->flip ^= 1;
    k_alm_clear<<<1, 256, 0, d->stream>>>(fs);
    k_alm_mark<<<blocks, threads, 0, d->stream>>>(a, g, m.per_x, fs);
    const size_t shm = ((size_t)(s->n * 4 + 15) / 16) * 16 + (size_t)s->n * 8;
    k_alm_fill<<<(unsigned)fs.cap, 128, shm, d->stream>>>(a, g, fs);
    count_launch(3);
    LBW_CK(cudaGetLastError());
    s->stepped = true;
    *fv_out = fs.view();
    return LBW_OK;
}

}  // namespace lbw

using namespace lbw;

extern "C" {

int lbw_alm_configure(lbw_domain* d, const lbw_alm_desc* desc) {
    LBW_REQ(d && desc, "null argument");
    LBW_REQ(desc->n_points >= 0 && desc->n_points <= 16384, "n_points outside [0, 16384]");
    LBW_REQ(desc->n_polars >= 0, "n_polars must be >= 0");
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    alm_destroy(d);
    const int P = desc->n_points;
    if (P == 0) return LBW_OK;
    for (int p = 0; p < P; ++p)
        LBW_REQ(desc->polar_index[p] >= -1 && desc->polar_index[p] < desc->n_polars,
                "polar index out of range");
    int64_t total_rows = 0;
    for (int k = 0; k < desc->n_polars; ++k) {
        LBW_REQ(desc->polar_rows[k] >= 2, "polar needs at least 2 rows");
        total_rows = std::max<int64_t>(total_rows, (int64_t)desc->polar_offset[k] + desc->polar_rows[k]);
    }
    AlmState* s = new AlmState();
    d->alm = s;
    s->n = P;
    s->n_polars = desc->n_polars;
    s->vscale = desc->velocity_scale;
    s->rho_ref = desc->rho_ref;
    s->dt2 = desc->force_dt2;
    s->den = desc->force_den;
    int rc = LBW_OK;
    auto A = [&](auto** p, size_t n) {
        if (rc == LBW_OK) rc = dev_alloc(d, s, p, n);
    };
    A(&s->chord, P);
    A(&s->elen, P);
    A(&s->twist, P);
    A(&s->polar_index, P);
    A(&s->polar_offset, std::max(1, desc->n_polars));
    A(&s->polar_rows, std::max(1, desc->n_polars));
    A(&s->p_alpha, std::max<int64_t>(1, total_rows));
    A(&s->p_cl, std::max<int64_t>(1, total_rows));
    A(&s->p_cd, std::max<int64_t>(1, total_rows));
    A(&s->kin, (size_t)P * kKin);
    A(&s->samples, (size_t)P * 4);
    A(&s->blade, (size_t)P * 3);
    A(&s->flat, (size_t)P * 3);
    A(&s->dep_cell, (size_t)P * 9);
    A(&s->dep_w, (size_t)P * 9);
    A(&s->clamp_flags, std::max(1, desc->n_polars));
    A(&s->error_flags, 1);
    // sparse force sets: a point touches at most 3x3 (x,y) rows
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    const int64_t cap = std::min<int64_t>(rows, (int64_t)9 * P);
    for (auto& fs : s->set) {
        A(&fs.row_slot, rows);
        A(&fs.pool, (size_t)cap * 3 * d->g.zp);
        A(&fs.slot_row, cap);
        A(&fs.count, 1);
        fs.cap = cap;
    }
    if (rc) {
        alm_destroy(d);
        return rc;
    }
    auto H = [&](void* dst, const void* src, size_t bytes) {
        if (rc == LBW_OK && bytes &&
            cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            set_error("ALM upload failed");
            rc = LBW_ECUDA;
        }
    };
    H(s->chord, desc->chord, P * 8);
    H(s->elen, desc->element_length, P * 8);
    H(s->twist, desc->twist, P * 8);
    H(s->polar_index, desc->polar_index, P * 4);
    if (desc->n_polars) {
        H(s->polar_offset, desc->polar_offset, desc->n_polars * 4);
        H(s->polar_rows, desc->polar_rows, desc->n_polars * 4);
        H(s->p_alpha, desc->polar_alpha, total_rows * 8);
        H(s->p_cl, desc->polar_cl, total_rows * 8);
        H(s->p_cd, desc->polar_cd, total_rows * 8);
    }
    if (rc == LBW_OK) {
        for (auto& fs : s->set) {
            if (cudaMemset(fs.row_slot, 0xff, rows * 4) != cudaSuccess ||
                cudaMemset(fs.count, 0, 4) != cudaSuccess) {
                cudaGetLastError();
                rc = LBW_ECUDA;
            }
        }
        if (cudaMemset(s->clamp_flags, 0, std::max(1, desc->n_polars) * 4) != cudaSuccess ||
            cudaMemset(s->error_flags, 0, 4) != cudaSuccess ||
            cudaMemset(s->samples, 0, (size_t)P * 32) != cudaSuccess ||
            cudaMemset(s->blade, 0, (size_t)P * 24) != cudaSuccess ||
            cudaMallocHost(&s->h_ring, (size_t)kRing * P * kKin * 8) != cudaSuccess) {
            cudaGetLastError();
            set_error("ALM initialisation failed");
            rc = LBW_ECUDA;
        }
        for (auto& e : s->ring_ev)
            if (rc == LBW_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                rc = LBW_ECUDA;
            }
    }
    if (rc) {
        alm_destroy(d);
        return rc;
    }
    return LBW_OK;
}

int lbw_alm_set_kinematics(lbw_domain* d, const double* kin) {
    LBW_REQ(d && kin, "null argument");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    const int slot = s->ring_pos;
    s->ring_pos = (s->ring_pos + 1) % kRing;
    LBW_CK(cudaEventSynchronize(s->ring_ev[slot]));
    double* h = s->h_ring + (size_t)slot * s->n * kKin;
    std::memcpy(h, kin, (size_t)s->n * kKin * 8);
    LBW_CK(cudaMemcpyAsync(s->kin, h, (size_t)s->n * kKin * 8, cudaMemcpyHostToDevice, d->stream));
    LBW_CK(cudaEventRecord(s->ring_ev[slot], d->stream));
    s->kin_queued = true;
    return LBW_OK;
}

int lbw_alm_get(lbw_domain* d, double* rho, double* u, double* blade_force) {
    LBW_REQ(d, "null domain");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    std::vector<double> smp((size_t)s->n * 4);
    LBW_CK(cudaMemcpyAsync(smp.data(), s->samples, smp.size() * 8, cudaMemcpyDeviceToHost, d->stream));
    if (blade_force)
        LBW_CK(cudaMemcpyAsync(blade_force, s->blade, (size_t)s->n * 24, cudaMemcpyDeviceToHost,
                               d->stream));
    int32_t err = 0;
    LBW_CK(cudaMemcpyAsync(&err, s->error_flags, 4, cudaMemcpyDeviceToHost, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    for (int p = 0; p < s->n; ++p) {
        if (rho) rho[p] = smp[p * 4];
        if (u)
            for (int c = 0; c < 3; ++c) u[p * 3 + c] = smp[p * 4 + 1 + c];
    }
    if (err & 1) {
        set_error("density must be positive at an actuator point");
        return LBW_EINVAL;
    }
    return LBW_OK;
}

int lbw_alm_clamp_flags(lbw_domain* d, int32_t* per_polar) {
    LBW_REQ(d && per_polar, "null argument");
    if (!alm_active(d)) return LBW_OK;
    LBW_CK(cudaSetDevice(d->device));
    const int n = std::max(1, d->alm->n_polars);
    LBW_CK(cudaMemcpyAsync(per_polar, d->alm->clamp_flags, d->alm->n_polars * 4,
                           cudaMemcpyDeviceToHost, d->stream));
    LBW_CK(cudaStreamSynchronize(d->stream));
    (void)n;
    return LBW_OK;
}

}  // extern "C"
