// lbw_alm.cu — actuator-line coupling on the device (compiled with
// -fmad=false like the exact sweep: the per-point arithmetic follows the
// reference expression order).  Per step, three small launches precede
// the sweep:
//
//   KK  k_kinematics       (device kinematics mode) one CTA: advance every
//                          component's spin by R(axis, rate dt), compose the
//                          world frames down the tree, then every point's
//                          position, velocity and chord/normal/span frame
//                          (turbine.py:227-311, sim.py:167-191)
//   K4  k_alm_points       one warp per point: lanes 0-7 recompute the
//                          previous step's macro at the 8 sampling-cube cells
//                          from the retained population buffer (SURVEY.md
//                          App. A.7); lane 0 interpolates, evaluates angle of
//                          attack, polar and blade-element force
//                          (actuator.py:70-146, polars.py:65-80,
//                          sim.py:210-235); lanes 0-2 build the per-axis Roma
//                          deposit lists with periodic images
//                          (actuator.py:100-110, 190-195, 297-341); lane 0
//                          claims a pool slot for every touched (x,y) row
//   K5  k_alm_fill         one CTA per claimed row: per cell, the sum of
//                          (wx*wy)*wz*F over the points in ascending global id
//                          from 0.0 (actuator.py:204-247) — deterministic, no
//                          float atomics.  CTA 0 also clears the other force
//                          set (last read by this step's K4) for the next step.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "lbw_domain.h"

#define LBW_FAST 0
#include "lbw_sweep.cuh"

namespace lbw {

constexpr int kKin = 18;  // pos_lat(3) vel(3) e_chord(3) e_normal(3) e_span(3) pos_m(3)
constexpr int kRing = 8;
// per-component device state: world p(3) T(9) v(3) w(3) spin_axis(3) has_axis(1)
// start_p(3) start_T(9) v_start(3) w_start(3) R(9)
constexpr int kCS = 49;
enum { CS_P = 0, CS_T = 3, CS_V = 12, CS_W = 15, CS_AX = 18, CS_HAX = 21, CS_SP = 22,
       CS_ST = 25, CS_VS = 34, CS_WS = 37, CS_R = 40 };

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
    double* kin;           // (P,18)
    double* samples;       // (P,4)
    double* blade;         // (P,3)
    double* flat;          // (P,3) lattice force on the fluid
    int32_t* dep_cell;     // (P,3 axes,kw) global cell or -1
    double* dep_w;         // (P,3,kw)
    int32_t kw;            // deposit cells per axis (3: Roma)
    int32_t kernel;        // LBW_SPREAD_*
    double eps;            // Gaussian width (cells)
    int32_t halo_x;        // support half-width in x (cells), for slab relevance
    int32_t* clamp_flags;  // (n_polars)
    const int32_t* point_ring;  // (P) disk ring id or -1
    const double* area;         // (P)
    int32_t n_rings;
    const int32_t* ring_first;
    const int32_t* ring_count;
    const double* ring_ct;
    int32_t* error_flags;  // bit 0: non-positive density, bit 1: point outside domain,
                           // bit 2: an actuator disk spans more than three slabs
    int64_t step;             // the step this view serves (diagnostics)
    double* ring_samples;     // (P,4) disk samples for the ring averages
    int32_t* ring_sample_ok;  // (P)
};

struct KinDev {
    int32_t nc;
    const int32_t* parent;
    const double* rel_p;
    const double* rel_T;
    const double* axis;
    const double* rate;
    const double* rstep;
    double* spin;
    const int32_t* line_first;
    const int32_t* line_count;
    const int32_t* point_comp;
    const double* off;
    const double* orient;
    const double* lframe;
    const int32_t* is_disk;
    const double* disk_center;
    double* cs;
    double* spin_hist;   // (3, nc, 9): spin state of step j in slot j % 3
    double* cs_hist;     // (3, nc, kCS)
    int32_t hist_slot;
    int32_t* box;           // (2): x planes this step's chain reads / writes (gate)
    int32_t box_halo;       // spreading half-width + 2
    int32_t stage_points;   // per-point constants fit in shared memory
    const int32_t* order;        // (nc) components by tree depth
    const int32_t* level_start;  // (nlevels+1) into order
    int32_t nlevels;
    const int32_t* is_static;    // (nc) world transform constant in time
    int32_t skip_static;         // their state from the previous launch is valid
    double dx;
};

struct AlmState {
    int32_t n = 0, n_polars = 0;
    double *chord = nullptr, *elen = nullptr, *twist = nullptr;
    int32_t *polar_index = nullptr, *polar_offset = nullptr, *polar_rows = nullptr;
    double *p_alpha = nullptr, *p_cl = nullptr, *p_cd = nullptr;
    double* kin = nullptr;       // (3,P,18): slot m % 3 (kinematics run a step ahead)
    double *samples = nullptr;   // (2,P,4)
    double *blade = nullptr;     // (2,P,3)
    double *flat = nullptr;      // (P,3)
    double* cube = nullptr;      // (2,P,8,4) sampled cube values + (2,P,8) tags (multi-slab)
    double* ring_samples = nullptr;
    int32_t* ring_sample_ok = nullptr;
    int32_t* dep_cell = nullptr;
    double* dep_w = nullptr;
    int32_t *clamp_flags = nullptr, *error_flags = nullptr;
    int32_t *point_ring = nullptr, *ring_first = nullptr, *ring_count = nullptr;
    double *area = nullptr, *ring_ct = nullptr;
    int32_t n_rings = 0;
    double vscale = 0, rho_ref = 0, dt2 = 0, den = 0;
    ForceSet set[2];
    // Few points: the sweep sums a tagged cell's force from the points'
    // deposit data itself (no fill kernel, no pool); many points: K5 fills
    // per-row pools.
    bool on_the_fly = false;
    int32_t kw = 3, kernel = 0, halo_x = 1;
    double eps = 0.0;
    double* h_ring = nullptr;   // pinned (kRing, P, 18)
    cudaEvent_t ring_ev[kRing] = {};
    int ring_pos = 0;
    int64_t kin_queued_step = -1;  // host kinematics uploaded for this step
    int64_t ready_step = -1;       // step whose actuator chain is queued and valid
    // device kinematics run on their own stream, one step ahead
    cudaStream_t kin_stream = nullptr;
    cudaEvent_t ev_kin_done = nullptr;
    cudaEvent_t ev_chain_done[2] = {nullptr, nullptr};  // chain of a step parity done
    int64_t kin_valid[3] = {-1, -1, -1};  // step whose kinematics kin[slot] holds
    // sweep gate (alm_gate): chain-done flag, per-slot x range of each step's
    // deposits and sampling, KK completion per slot
    uint32_t* gate_flag = nullptr;
    int32_t* gate_box = nullptr;     // (3, 2) local planes, inclusive
    cudaEvent_t ev_kin_step[3] = {nullptr, nullptr, nullptr};
    // per-step blade-force series (lbw_alm_record_loads)
    double* h_loads = nullptr;   // pinned (loads_cap, P, 3)
    int64_t loads_cap = 0, loads_from = 0;
    // device kinematics
    bool kin_device = false;
    int32_t nc = 0;
    int32_t *k_parent = nullptr, *k_line_first = nullptr, *k_line_count = nullptr;
    int32_t* k_point_comp = nullptr;
    double *k_rel_p = nullptr, *k_rel_T = nullptr, *k_axis = nullptr, *k_rate = nullptr;
    double *k_rstep = nullptr, *k_spin = nullptr, *k_off = nullptr, *k_orient = nullptr;
    double *k_lframe = nullptr, *k_cs = nullptr;
    double *k_spin_hist = nullptr, *k_cs_hist = nullptr;
    int32_t* k_is_disk = nullptr;
    double* k_disk_center = nullptr;
    double k_dx = 1.0;
    int64_t kin_state_step = 0;  // step whose kinematics the device spins represent
    bool kin_stage_points = false;
    int32_t *k_order = nullptr, *k_level_start = nullptr, *k_static = nullptr;
    int32_t k_nlevels = 0;
    bool kin_static_ready = false;   // static components' state computed once
    size_t kin_smem = 0;
    std::vector<void*> allocs;

    // device view for step m: outputs by parity, kinematics by m % 3
    AlmDev dev(int64_t m) const {
        const int parity = (int)(m & 1);
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
        a.kin = kin + (size_t)(m % 3) * n * kKin;
        a.samples = samples + (size_t)parity * n * 4;
        a.blade = blade + (size_t)parity * n * 3;
        a.flat = flat + (size_t)parity * n * 3;
        a.dep_cell = dep_cell + (size_t)parity * n * 3 * kw;
        a.dep_w = dep_w + (size_t)parity * n * 3 * kw;
        a.kw = kw;
        a.kernel = kernel;
        a.eps = eps;
        a.halo_x = halo_x;
        a.clamp_flags = clamp_flags;
        a.step = m;
        a.ring_samples = ring_samples;
        a.ring_sample_ok = ring_sample_ok;
        a.error_flags = error_flags;
        a.point_ring = point_ring;
        a.area = area;
        a.n_rings = n_rings;
        a.ring_first = ring_first;
        a.ring_count = ring_count;
        a.ring_ct = ring_ct;
        return a;
    }
    KinDev kdev() const {
        KinDev k;
        k.nc = nc;
        k.parent = k_parent;
        k.rel_p = k_rel_p;
        k.rel_T = k_rel_T;
        k.axis = k_axis;
        k.rate = k_rate;
        k.rstep = k_rstep;
        k.spin = k_spin;
        k.line_first = k_line_first;
        k.line_count = k_line_count;
        k.point_comp = k_point_comp;
        k.off = k_off;
        k.orient = k_orient;
        k.lframe = k_lframe;
        k.is_disk = k_is_disk;
        k.disk_center = k_disk_center;
        k.cs = k_cs;
        k.spin_hist = k_spin_hist;
        k.cs_hist = k_cs_hist;
        k.hist_slot = 0;
        k.box = nullptr;
        k.box_halo = halo_x + 2;
        k.stage_points = kin_stage_points ? 1 : 0;
        k.order = k_order;
        k.level_start = k_level_start;
        k.nlevels = k_nlevels;
        k.is_static = k_static;
        k.skip_static = 0;
        k.dx = k_dx;
        return k;
    }
};

// How the macro field sampled at this step is obtained (MacroSource).
struct MacroDev {
    int kind;
    double uniform[4];
    const void* buf;   // population buffer (storage type per g.single)
    int pull;
    ForceView fv;
    const double* dense;
    int bc_set;        // the x-face BC has written its macro ghosts (after step 0)
    double u_in[3];
    int inflow;        // velocity_inflow_outflow
    int per_x;
};

namespace {

// ------------------------------------------------------------ 3x3 algebra
// row-major 3x3; C = A B with a fixed (a0 b0 + a1 b1) + a2 b2 order
__device__ void mm3(const double* A, const double* B, double* C) {
    double t[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            t[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
    for (int k = 0; k < 9; ++k) C[k] = t[k];
}
__device__ void mv3(const double* A, const double* v, double* out) {
    double t[3];
    for (int i = 0; i < 3; ++i) t[i] = A[i * 3] * v[0] + A[i * 3 + 1] * v[1] + A[i * 3 + 2] * v[2];
    for (int i = 0; i < 3; ++i) out[i] = t[i];
}
__device__ void cross3(const double* a, const double* b, double* out) {
    const double c0 = a[1] * b[2] - a[2] * b[1];
    const double c1 = a[2] * b[0] - a[0] * b[2];
    const double c2 = a[0] * b[1] - a[1] * b[0];
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
}
// Gram-Schmidt on the columns (turbine.py:83-90)
__device__ void reorth(double* T) {
    double c0[3] = {T[0], T[3], T[6]}, c1[3] = {T[1], T[4], T[7]};
    const double n0 = sqrt(c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2]);
    for (int i = 0; i < 3; ++i) c0[i] /= n0;
    const double d = c0[0] * c1[0] + c0[1] * c1[1] + c0[2] * c1[2];
    for (int i = 0; i < 3; ++i) c1[i] = c1[i] - d * c0[i];
    const double n1 = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] /= n1;
    double c2[3];
    cross3(c0, c1, c2);
    for (int i = 0; i < 3; ++i) {
        T[i * 3] = c0[i];
        T[i * 3 + 1] = c1[i];
        T[i * 3 + 2] = c2[i];
    }
}
// numpy float remainder (npy_divmod): result takes the divisor's sign
__device__ double np_mod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0) != (m < 0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// Warp-cooperative 3x3 algebra on shared memory for the tree walk: every
// lane of the warp calls; lanes 0..8 (0..2) own one entry each, with the
// per-entry arithmetic of mm3 / mv3 / cross3 / drifted (bit-identical).
__device__ void wmm3(const double* A, const double* B, double* C, int lane) {
    double t = 0.0;
    if (lane < 9) {
        const int i = lane / 3, j = lane % 3;
        t = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
    }
    __syncwarp();
    if (lane < 9) C[lane] = t;
    __syncwarp();
}
__device__ void wmv3(const double* A, const double* v, double* out, int lane) {
    double t = 0.0;
    if (lane < 3) t = A[lane * 3] * v[0] + A[lane * 3 + 1] * v[1] + A[lane * 3 + 2] * v[2];
    __syncwarp();
    if (lane < 3) out[lane] = t;
    __syncwarp();
}
__device__ void wcross3(const double* a, const double* b, double* out, int lane) {
    double t = 0.0;
    if (lane == 0) t = a[1] * b[2] - a[2] * b[1];
    if (lane == 1) t = a[2] * b[0] - a[0] * b[2];
    if (lane == 2) t = a[0] * b[1] - a[1] * b[0];
    __syncwarp();
    if (lane < 3) out[lane] = t;
    __syncwarp();
}
// max |T^T T - I| > 1e-12 (turbine.py:_DRIFT_TOL)
__device__ bool wdrifted(const double* T, int lane) {
    bool over = false;
    if (lane < 9) {
        const int i = lane / 3, j = lane % 3;
        double s = T[i] * T[j] + T[3 + i] * T[3 + j] + T[6 + i] * T[6 + j];
        if (i == j) s -= 1.0;
        over = fabs(s) > 1e-12;   // max(...) > tol, NaN entries ignored as fmax does
    }
    return __any_sync(0xffffffffu, over);
}
__device__ void wreorth(double* T, int lane) {
    __syncwarp();
    if (lane == 0) reorth(T);
    __syncwarp();
}

// parameters per component in the kinematics CTA's shared memory:
// rel_p 3, rel_T 9, axis 3, rate 1, rstep 9, spin 9, parent 1, first 1, is_disk 1, disk p 3, T 9
constexpr int kKP = 49;

// One component of the tree walk (turbine.py:259-311, sim.py:167-191) by
// one warp: lanes 0..8 own the entries of each 3x3 product (the per-entry
// arithmetic of mm3 / mv3 / cross3, bit-identical to a serial walk).
__device__ void walk_component(const KinDev& k, double* prm, double* cs, int c, int advance,
                               const double* off, const double* orient, double* wt,
                               const double* I3s, const double* zero3s, int lane) {
    double* tmp9 = wt;
    double* tmp9b = wt + 9;
    double* tmp3 = wt + 18;
    double* tmp3b = wt + 21;
    double* q = prm + c * kKP;
    double* s = cs + c * kCS;
    const int par = (int)q[34];
    const double* Pp = par >= 0 ? cs + par * kCS + CS_P : zero3s;
    const double* PT = par >= 0 ? cs + par * kCS + CS_T : I3s;
    const double* Pv = par >= 0 ? cs + par * kCS + CS_V : zero3s;
    const double* Pw = par >= 0 ? cs + par * kCS + CS_W : zero3s;
    double* spin = q + 25;
    const double rate = q[15];
    if (advance && rate != 0.0) {
        wmm3(spin, q + 16, spin, lane);
        if (wdrifted(spin, lane)) wreorth(spin, lane);
    }
    double* Tp_rp = tmp3;
    double* Tp_Tr = tmp9;
    wmv3(PT, q, Tp_rp, lane);
    wmm3(PT, q + 3, Tp_Tr, lane);
    if (lane < 3) s[CS_P + lane] = Pp[lane] + Tp_rp[lane];
    wmm3(Tp_Tr, spin, s + CS_T, lane);
    if (wdrifted(s + CS_T, lane)) wreorth(s + CS_T, lane);
    wcross3(Pw, Tp_rp, tmp3b, lane);
    if (lane < 3) {
        s[CS_V + lane] = Pv[lane] + tmp3b[lane];
        s[CS_W + lane] = Pw[lane];
        s[CS_AX + lane] = par >= 0 ? cs[par * kCS + CS_AX + lane] : 0.0;
    }
    if (lane == 0) s[CS_HAX] = par >= 0 ? cs[par * kCS + CS_HAX] : 0.0;
    __syncwarp();
    if (rate != 0.0) {
        wmv3(Tp_Tr, q + 12, s + CS_AX, lane);
        if (lane == 0) s[CS_HAX] = 1.0;
        if (lane < 3) s[CS_W + lane] = s[CS_W + lane] + s[CS_AX + lane] * rate;
        __syncwarp();
    }
    if (lane < 9) s[CS_R + lane] = spin[lane];
    __syncwarp();
    const int first = (int)q[35];
    if (q[36] != 0.0) {
        // disk centre (update_disk, turbine.py:237-241) and its velocity
        double* Tc_p = tmp3;
        double* TcT = tmp9b;
        wmv3(s + CS_T, q + 37, Tc_p, lane);
        if (lane < 3) s[CS_SP + lane] = s[CS_P + lane] + Tc_p[lane];
        wmm3(s + CS_T, q + 40, TcT, lane);
        wmm3(TcT, spin, s + CS_ST, lane);
        wcross3(s + CS_W, Tc_p, tmp3b, lane);
        if (lane < 3) s[CS_VS + lane] = s[CS_V + lane] + tmp3b[lane];
        __syncwarp();
    } else if (first >= 0) {
        const double* W = s + CS_T;
        double* Tp_o0 = tmp3;
        double* Tp_O0 = tmp9b;
        wmv3(W, off + (int64_t)first * 3, Tp_o0, lane);
        if (lane < 3) s[CS_SP + lane] = s[CS_P + lane] + Tp_o0[lane];
        wmm3(W, orient + (int64_t)first * 9, Tp_O0, lane);
        wmm3(Tp_O0, spin, s + CS_ST, lane);
        wcross3(s + CS_W, Tp_o0, tmp3b, lane);
        if (lane < 3) {
            s[CS_VS + lane] = s[CS_V + lane] + tmp3b[lane];
            s[CS_WS + lane] = s[CS_W + lane];
        }
        __syncwarp();
        if (rate != 0.0) {
            wmv3(Tp_O0, q + 12, tmp3b, lane);
            if (lane < 3) s[CS_WS + lane] = s[CS_WS + lane] + tmp3b[lane] * rate;
            __syncwarp();
        }
    }
}

// KK: tree walk + point kinematics, one CTA.  The component parameters and
// state are staged in shared memory (the walk itself is one thread: a chain
// of dependent 3x3 products down the tree); points are then evaluated in
// parallel.  Layout per component in smem: params[kKP] then state[kCS].
// rel_p 3, rel_T 9, axis 3, rate 1, rstep 9, spin 9, parent 1, first 1, is_disk 1, disk p 3, T 9
__device__ void kinematics_cta(const KinDev& k, const AlmDev& a, const Geom& g, int per_x,
                               int advance, double* ksm) {
#ifdef LBW_KK_PROF
    long long t0 = clock64();
#endif
    double* prm = ksm;                         // (nc, kKP)
    double* cs = ksm + (size_t)k.nc * kKP;     // (nc, kCS)
    // per-point constants staged too when they fit (k.stage_points): every
    // global load of the kernel is then issued in this one parallel pass
    double* sm_off = cs + (size_t)k.nc * kCS;            // (P,3)
    double* sm_orient = sm_off + (size_t)a.n * 3;        // (P,9)
    double* sm_lframe = sm_orient + (size_t)a.n * 9;     // (P,9)
    int32_t* sm_comp = reinterpret_cast<int32_t*>(sm_lframe + (size_t)a.n * 9);  // (P)
    // walk schedule (always staged, after the point block or after cs)
    int32_t* sm_order = k.stage_points ? sm_comp + a.n
                                       : reinterpret_cast<int32_t*>(cs + (size_t)k.nc * kCS);
    int32_t* sm_static = sm_order + k.nc;
    int32_t* sm_lstart = sm_static + k.nc;
    for (int i = threadIdx.x; i < k.nc; i += blockDim.x) {
        sm_order[i] = k.order[i];
        sm_static[i] = k.is_static[i];
    }
    for (int i = threadIdx.x; i <= k.nlevels; i += blockDim.x) sm_lstart[i] = k.level_start[i];
    if (k.skip_static)
        for (int i = threadIdx.x; i < k.nc * kCS; i += blockDim.x)
            if (k.is_static[i / kCS]) cs[i] = k.cs[i];
    const double* off = k.stage_points ? sm_off : k.off;
    const double* orient = k.stage_points ? sm_orient : k.orient;
    const double* lframe = k.stage_points ? sm_lframe : k.lframe;
    const int32_t* point_comp = k.stage_points ? sm_comp : k.point_comp;
    if (k.stage_points) {
        for (int i = threadIdx.x; i < a.n * 3; i += blockDim.x) sm_off[i] = k.off[i];
        for (int i = threadIdx.x; i < a.n * 9; i += blockDim.x) {
            sm_orient[i] = k.orient[i];
            sm_lframe[i] = k.lframe[i];
        }
        for (int i = threadIdx.x; i < a.n; i += blockDim.x) sm_comp[i] = k.point_comp[i];
    }
    for (int i = threadIdx.x; i < k.nc * kKP; i += blockDim.x) {
        const int c = i / kKP, j = i % kKP;
        double v;
        if (j < 3) v = k.rel_p[c * 3 + j];
        else if (j < 12) v = k.rel_T[c * 9 + j - 3];
        else if (j < 15) v = k.axis[c * 3 + j - 12];
        else if (j < 16) v = k.rate[c];
        else if (j < 25) v = k.rstep[c * 9 + j - 16];
        else if (j < 34) v = k.spin[c * 9 + j - 25];
        else if (j < 35) v = (double)k.parent[c];
        else if (j < 36) v = (double)k.line_first[c];
        else if (j < 37) v = (double)k.is_disk[c];
        else v = k.disk_center[c * 12 + j - 37];
        prm[i] = v;
    }
    __syncthreads();
#ifdef LBW_KK_PROF
    long long t1 = clock64();
#endif
    {
        // level by level: the components of one depth in parallel, one warp
        // each.  Components whose world transform never changes (no
        // rotation on their path) keep the state of the first launch.
        __shared__ double I3s[9], zero3s[3];
        __shared__ double wtmp[8][24];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
        if (threadIdx.x < 9) I3s[threadIdx.x] = (threadIdx.x % 4 == 0) ? 1.0 : 0.0;
        if (threadIdx.x < 3) zero3s[threadIdx.x] = 0.0;
        __syncthreads();
        for (int L = 0; L < k.nlevels; ++L) {
            for (int j = sm_lstart[L] + warp; j < sm_lstart[L + 1]; j += nwarp) {
                const int c = sm_order[j];
                if (k.skip_static && sm_static[c]) continue;
                walk_component(k, prm, cs, c, advance, off, orient, wtmp[warp], I3s, zero3s, lane);
            }
            __syncthreads();
        }
    }
#ifdef LBW_KK_PROF
    long long t2 = clock64();
#endif
    // persist spin + component state (downloadable), evaluate the points
    for (int i = threadIdx.x; i < k.nc * 9; i += blockDim.x)
        k.spin[i] = k.spin_hist[(int64_t)k.hist_slot * k.nc * 9 + i] =
            prm[(i / 9) * kKP + 25 + i % 9];
    for (int i = threadIdx.x; i < k.nc * kCS; i += blockDim.x)
        k.cs[i] = k.cs_hist[(int64_t)k.hist_slot * k.nc * kCS + i] = cs[i];
#ifdef LBW_KK_PROF
    long long t3 = clock64();
#endif
    const int64_t dims[3] = {g.nxg, g.ny, g.nz};
    const int per[3] = {per_x, g.per_y, g.per_z};
    __shared__ int box_lo, box_hi;
    if (threadIdx.x == 0) {
        box_lo = INT_MAX;
        box_hi = INT_MIN;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < a.n; p += blockDim.x) {
        const int c = point_comp[p];
        const double* s = cs + c * kCS;
        const int kk = p - k.line_first[c];
        double pos[3], fr[9], vel[3];
        const bool disk = prm[c * kKP + 36] != 0.0;
        if (disk) {
            // world = centre.p + offs @ centre.T^T (sim.py:182-187); the disk
            // axis (centre frame +x) rides in the e_chord slot
            double rel[3];
            mv3(s + CS_ST, off + (int64_t)p * 3, rel);
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i] + rel[i];
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i];
            const double fr_d[9] = {s[CS_ST], s[CS_ST + 3], s[CS_ST + 6], 0, 1, 0, 0, 0, 1};
            for (int i = 0; i < 9; ++i) fr[i] = fr_d[i];
        } else if (kk == 0) {
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i];
            for (int i = 0; i < 9; ++i) fr[i] = s[CS_ST + i];
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i];
        } else {
            double rel[3], tmp[9], cr[3];
            mv3(s + CS_ST, off + (int64_t)p * 3, rel);
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i] + rel[i];
            mm3(s + CS_ST, orient + (int64_t)p * 9, tmp);
            mm3(tmp, s + CS_R, fr);
            cross3(s + CS_WS, rel, cr);
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i] + cr[i];
        }
        double* out = a.kin + (int64_t)p * kKin;
        for (int i = 0; i < 3; ++i) {
            double lat = pos[i] / k.dx;
            if (per[i]) lat = np_mod(lat, (double)dims[i]);
            else if (!(lat >= 0.0 && lat < (double)dims[i])) atomicOr(a.error_flags, 2);
            out[i] = lat;
            out[3 + i] = vel[i];
            out[15 + i] = pos[i];
            if (i == 0 && k.box) {
                // planes the chain reads (sampling cube + pull sources) or
                // writes (deposit rows) for this point
                const int64_t n0 = (int64_t)floor(lat);
                int64_t lo = n0 - k.box_halo - g.x0, hi = n0 + k.box_halo - g.x0;
                if (lo < 0 || hi >= g.nxl) {   // wraps or leaves the slab: gate all planes
                    if (per_x || lo < 0) lo = 0;
                    if (per_x || hi >= g.nxl) hi = g.nxl - 1;
                }
                atomicMin(&box_lo, (int)(lo < 0 ? 0 : lo));
                atomicMax(&box_hi, (int)(hi > g.nxl - 1 ? g.nxl - 1 : hi));
            }
        }
        if (disk) {
            for (int i = 0; i < 9; ++i) out[6 + i] = fr[i];
        } else {
            for (int f = 0; f < 3; ++f) mv3(fr, lframe + (int64_t)p * 9 + f * 3, out + 6 + 3 * f);
        }
    }
    if (k.box) {
        __syncthreads();
        if (threadIdx.x == 0) {
            k.box[0] = box_lo;
            k.box[1] = box_hi;
        }
    }
#ifdef LBW_KK_PROF
    __syncthreads();
    if (threadIdx.x == 0)
        printf("KKPROF stage %lld walk %lld persist %lld points %lld\n", t1 - t0, t2 - t1, t3 - t2,
               clock64() - t3);
#endif
}

__global__ void k_kinematics(KinDev k, AlmDev a, Geom g, int per_x, int advance) {
    extern __shared__ double ksm[];
    LBW_TRACE_BEGIN(1, a.step);
    kinematics_cta(k, a, g, per_x, advance, ksm);
    LBW_TRACE_END(1, a.step);
}

__device__ __noinline__ void load_cell_general(const void* buf, const Geom& g, bool pull, int x,
                                               int y, int z, double (&f)[27]) {
    if (pull) load_cell_any<true>(buf, g, x, y, z, f);
    else load_cell_any<false>(buf, g, x, y, z, f);
}

// Macro (rho, u) of global cell (gx,gy,gz), following the ghost semantics
// of PdfField.macro (fields.py:35-36, halo.py:144-160).  Returns MA_REMOTE
// (nothing written) when the cell belongs to another slab, MA_OWNED for a
// cell of this slab, MA_CONST for a ghost value every slab knows.  Values
// are those the reference's macro array of the storage dtype holds.
enum { MA_REMOTE = 0, MA_OWNED = 1, MA_CONST = 2 };
__device__ int macro_at_raw(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                            double out[4]);
__device__ int macro_at(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                        double out[4]) {
    const int code = macro_at_raw(g, m, gx, gy, gz, out);
    if (code != MA_REMOTE && g.single)
        for (int k = 0; k < 4; ++k) out[k] = stored<float>(out[k]);
    return code;
}
__device__ int macro_at_raw(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
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
            return MA_CONST;
        } else if (m.inflow && gx >= g.nxg && m.bc_set) {
            gx = g.nxg - 1;
        } else {
            put(ghost0);
            return MA_CONST;
        }
    }
    if (gy < 0 || gy >= g.ny) {
        if (!g.per_y) { put(ghost0); return MA_CONST; }
        gy = gy < 0 ? gy + g.ny : gy - g.ny;
    }
    if (gz < 0 || gz >= g.nz) {
        if (!g.per_z) { put(ghost0); return MA_CONST; }
        gz = gz < 0 ? gz + g.nz : gz - g.nz;
    }
    const int64_t x = gx - g.x0;
    if (x < 0 || x >= g.nxl) return MA_REMOTE;
    if (m.kind == MS_UNIFORM) {
        put(m.uniform);
        return MA_OWNED;
    }
    const int64_t cell = (x * g.ny + gy) * g.nz + gz;
    if (m.kind == MS_DENSE) {
        put(m.dense + cell * 4);
        return MA_OWNED;
    }
    // the row key and the 27 populations are loaded together (one DRAM
    // round trip); the force sum over the staged deposit data follows
    const uint64_t key = m.fv.row_key ? m.fv.row_key[x * g.ny + gy] : 0ull;
    double f[27];
    // interior cells take the compact branch-free pull; cells at boundaries
    // (x faces, non-periodic y / z, walls) the general one, out of line so
    // this kernel's code stays small
    if (m.pull && pull_is_simple(g, (int)x, (int)gy, (int)gz)) {
        if (g.single)
            load_cell_simple(static_cast<const float*>(m.buf), g, (int)x, (int)gy, (int)gz, f);
        else
            load_cell_simple(static_cast<const double*>(m.buf), g, (int)x, (int)gy, (int)gz, f);
    } else {
        load_cell_general(m.buf, g, m.pull != 0, (int)x, (int)gy, (int)gz, f);
    }
    double Fx, Fy, Fz;
    if (g.single) force_from_key<float>(m.fv, g, key, (int)x, (int)gy, (int)gz, Fx, Fy, Fz);
    else force_from_key<double>(m.fv, g, key, (int)x, (int)gy, (int)gz, Fx, Fy, Fz);
    const Macro mm = moments_exact(f, Fx, Fy, Fz, 1.0);
    out[0] = mm.rho;
    out[1] = mm.ux;
    out[2] = mm.uy;
    out[3] = mm.uz;
    return MA_OWNED;
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// np.interp on one value (numpy compiled_base.c arr_interp semantics)
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

// Per-point data that does not depend on the flow, loaded at the start of
// K4 so its latency overlaps the sampling loads: the point's polar table
// sits in registers (one row per lane) when it has at most 32 rows.
struct PointStatic {
    int pid, off, rows;
    double chord, elen, twist;
    double xl, cll, cdl;   // this lane's polar row
};
__device__ __forceinline__ PointStatic load_static(const AlmDev& a, int p, int lane) {
    PointStatic ps;
    ps.pid = a.polar_index[p];
    ps.chord = a.chord[p];
    ps.elen = a.elen[p];
    ps.twist = a.twist[p];
    ps.off = ps.rows = 0;
    ps.xl = ps.cll = ps.cdl = 0.0;
    if (ps.pid >= 0) {
        ps.off = a.polar_offset[ps.pid];
        ps.rows = a.polar_rows[ps.pid];
        if (lane < ps.rows) {
            ps.xl = a.p_alpha[ps.off + lane];
            ps.cll = a.p_cl[ps.off + lane];
            ps.cdl = a.p_cd[ps.off + lane];
        }
    }
    return ps;
}

// polar row r of the point: from the lanes' registers (<= 32 rows) or memory
__device__ __forceinline__ void polar_row(const AlmDev& a, const PointStatic& ps, int r,
                                          double& x, double& cl, double& cd) {
    if (ps.rows <= 32) {
        x = __shfl_sync(0xffffffffu, ps.xl, r);
        cl = __shfl_sync(0xffffffffu, ps.cll, r);
        cd = __shfl_sync(0xffffffffu, ps.cdl, r);
    } else {
        x = a.p_alpha[ps.off + r];
        cl = a.p_cl[ps.off + r];
        cd = a.p_cd[ps.off + r];
    }
}

// np.interp (polars.py:65-80) of cl and cd at x for the whole warp: the
// bracketing row (largest j with xp[j] <= x; tables are increasing) is
// counted with a ballot instead of a binary search of dependent loads.
__device__ void polar_interp(const AlmDev& a, const PointStatic& ps, double x, int lane,
                             double& cl, double& cd) {
    const int n = ps.rows;
    double x0, c0l, c0d, xn, cnl, cnd;
    polar_row(a, ps, 0, x0, c0l, c0d);
    polar_row(a, ps, n - 1, xn, cnl, cnd);
    int cnt = 0;
    if (n <= 32) {
        cnt = __popc(__ballot_sync(0xffffffffu, lane < n && ps.xl <= x));
    } else {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            cnt += __popc(__ballot_sync(0xffffffffu, k < n && a.p_alpha[ps.off + k] <= x));
        }
    }
    const int j = cnt > 0 ? (cnt - 1 < n - 2 ? cnt - 1 : n - 2) : 0;
    double xa, cla, cda, xb, clb, cdb;
    polar_row(a, ps, j, xa, cla, cda);
    polar_row(a, ps, j + 1, xb, clb, cdb);
    auto one = [&](double fa, double fb, double f0, double fn) -> double {
        if (isnan(x)) return x;
        if (x < x0) return f0;
        if (x > xn) return fn;
        if (x == xn) return fn;
        if (xa == x) return fa;
        const double slope = (fb - fa) / (xb - xa);
        double r = slope * (x - xa) + fa;
        if (isnan(r)) {
            r = slope * (x - xb) + fb;
            if (isnan(r) && fa == fb) r = fa;
        }
        return r;
    };
    cl = one(cla, clb, c0l, cnl);
    cd = one(cda, cdb, c0d, cnd);
}

// blade-element force on the BLADE (actuator.py:117-146, sim.py:218-235),
// evaluated by a whole warp (identical values on every lane; lane 0 raises
// the flags).  kr: the point's kinematics row.
__device__ void blade_force_warp(const AlmDev& a, const PointStatic& ps, const double* kr,
                                 const double* acc, double* blade, int lane) {
    blade[0] = blade[1] = blade[2] = 0.0;
    if (ps.pid < 0) return;
    const double* vel = kr + 3;
    const double* ec = kr + 6;
    const double* en = kr + 9;
    const double* es = kr + 12;
    double urel[3];
    for (int c = 0; c < 3; ++c) urel[c] = acc[1 + c] * a.vscale - vel[c];
    const double along = dot3(urel, es);
    double up[3];
    for (int c = 0; c < 3; ++c) up[c] = urel[c] - along * es[c];
    const double speed = sqrt(dot3(up, up));
    if (!(speed >= 1e-12)) return;  // DEGENERATE_SPEED (actuator.py:30)
    const double phi = atan2(dot3(up, en), dot3(up, ec));
    double alpha = phi - ps.twist;
    double ed[3], el[3];
    for (int c = 0; c < 3; ++c) ed[c] = up[c] / speed;
    cross3(es, ed, el);
    double x0, c0l, c0d, xn, cnl, cnd;
    polar_row(a, ps, 0, x0, c0l, c0d);
    polar_row(a, ps, ps.rows - 1, xn, cnl, cnd);
    if (alpha < x0 || alpha > xn) {
        if (lane == 0) atomicOr(&a.clamp_flags[ps.pid], 1);
        alpha = fmin(fmax(alpha, x0), xn);
    }
    double cl, cd;
    polar_interp(a, ps, alpha, lane, cl, cd);
    const double rho_phys = acc[0] * a.rho_ref;
    if (!(rho_phys > 0.0) && lane == 0) atomicOr(a.error_flags, 1);
    const double scale = 0.5 * rho_phys * speed * speed * ps.chord * ps.elen;
    for (int c = 0; c < 3; ++c) blade[c] = scale * (cl * el[c] + cd * ed[c]);
}

// per-axis deposit cells + weights, images across periodic faces computed
// from the shifted position pos - w*L (actuator.py:190-195, 330-332)
// Gaussian kernel (extension): cells j with |x - (j + 1/2)| <= 3 eps,
// weights exp(-(r/eps)^2) normalised over that support (per axis, so the
// deposited momentum equals the point force for interior points).
constexpr int kMaxKw = 13;   // eps <= 2 -> at most floor(6 eps * 2) + 1 cells
__device__ __forceinline__ void gaussian_support(double xs, double eps, int64_t& jlo,
                                                 int64_t& jhi, double& inv_sum) {
    const double R = 3.0 * eps;
    jlo = (int64_t)ceil(xs - 0.5 - R);
    jhi = (int64_t)floor(xs - 0.5 + R);
    double sum = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) {
        const double r = (xs - ((double)j + 0.5)) / eps;
        sum += exp(-r * r);
    }
    inv_sum = 1.0 / sum;
}

__device__ void deposit_axis(double x, int64_t L, int periodic, int kernel, double eps, int kw,
                             int32_t* dc, double* dw) {
    int cnt = 0;
    for (int q = 0; q < kw; ++q) {
        dc[q] = -1;
        dw[q] = 0.0;
    }
    const int nimg = periodic ? 3 : 1;
    for (int im = 0; im < nimg; ++im) {
        const double w = im == 0 ? 0.0 : (im == 1 ? 1.0 : -1.0);
        const double xs = im == 0 ? x : x - w * (double)L;
        if (kernel == LBW_SPREAD_GAUSSIAN) {
            int64_t jlo, jhi;
            double inv_sum;
            gaussian_support(xs, eps, jlo, jhi, inv_sum);
            for (int64_t j = jlo; j <= jhi; ++j) {
                if (j < 0 || j >= L || cnt >= kw) continue;
                const double r = (xs - ((double)j + 0.5)) / eps;
                dc[cnt] = (int32_t)j;
                dw[cnt] = exp(-r * r) * inv_sum;
                ++cnt;
            }
            continue;
        }
        const double n0f = floor(xs);
        const int64_t n0 = (int64_t)n0f;
        const double r[3] = {xs - (n0f - 0.5), xs - (n0f + 0.5), xs - (n0f + 1.5)};
        for (int q = 0; q < 3; ++q) {
            const int64_t c = n0 - 1 + q;
            if (c < 0 || c >= L) continue;
            const double wt = roma(r[q]);
            if (wt == 0.0 || cnt >= kw) continue;
            dc[cnt] = (int32_t)c;
            dw[cnt] = wt;
            ++cnt;
        }
    }
}

// (x,y) row of deposit pair q = p*9 + k (k: 3 x-cells x 3 y-cells of point
// p) as a slab row index, or -1 when it is not a cell of this slab.
__device__ __forceinline__ int32_t pair_row(const AlmDev& a, const Geom& g, int q) {
    const int kw = a.kw, kk = kw * kw;
    const int32_t* dc = a.dep_cell + (int64_t)(q / kk) * 3 * kw;
    const int k = q % kk;
    const int32_t cxg = dc[k / kw], cy = dc[kw + k % kw];
    const int64_t x = (int64_t)cxg - g.x0;
    if (cxg < 0 || cy < 0 || x < 0 || x >= g.nxl) return -1;
    return (int32_t)(x * g.ny + cy);
}

constexpr int kOnTheFlyMaxPoints = 64;

// deposit cells of a wide (Gaussian) kernel, stored straight to the point's
// deposit arrays; out of line to keep the Roma path of K4 compact
__device__ __noinline__ void deposit_axis_wide(const AlmDev& a, int p, int k, double x, int64_t L,
                                               int per) {
    const int kw = a.kw;
    int32_t dc[kMaxKw];
    double dw[kMaxKw];
    deposit_axis(x, L, per, a.kernel, a.eps, kw, dc, dw);
    for (int q = 0; q < kw; ++q) {
        a.dep_cell[(int64_t)p * 3 * kw + kw * k + q] = dc[q];
        a.dep_w[(int64_t)p * 3 * kw + kw * k + q] = dw[q];
    }
}

// K4: one warp per point
// phase 0: single slab, everything in one pass.  Multi-slab: phase 1 only
// computes the cube values of this slab's cells and stores them into the
// local and both neighbours' cube buffers; phase 2 (after the neighbours'
// stores are visible) continues from the cube buffer.
struct CubeArgs {
    double* local;   // (P,8,4) of this step's parity
    double* peer[2];
    // per cube cell: epoch of the launch that wrote it (same allocation,
    // after the values), so a reader knows which cells are this step's
    int32_t* tag_local;  // (P,8)
    int32_t* tag_peer[2];
    int32_t epoch;
};

// Flow-independent per-point inputs, loaded by the kernel before anything
// that waits (kinematics row one value per lane, polar / chord data).
struct PointInputs {
    double kv;
    PointStatic ps;
    bool disk;
#ifdef LBW_K4_PROF
    long long t0, t1;
#endif
};
__device__ __forceinline__ PointInputs load_point_inputs(const AlmDev& a, int p, int lane) {
    PointInputs in;
    in.kv = lane < 15 ? a.kin[(int64_t)p * kKin + lane] : 0.0;
    in.ps = load_static(a, p, lane);
    in.disk = a.point_ring != nullptr && a.point_ring[p] >= 0;
    return in;
}

__device__ void point_warp(const AlmDev& a, const Geom& g, const MacroDev& m, const ForceSet& s,
                           int phase, const CubeArgs& cube, int p, int lane,
                           const PointInputs& in) {
    const PointStatic& ps = in.ps;
    const bool disk = in.disk;
    double kr[15];
    for (int k = 0; k < 15; ++k) kr[k] = __shfl_sync(0xffffffffu, in.kv, k);
#ifdef LBW_K4_PROF
    const long long t2 = clock64();   // kinematics row available
#endif
    const double* kin = kr;
    // deposit cells / Roma weights per axis (lanes 8..10), kept in registers
    // for the row tags below and stored for the sweep / fill / next sample
    const int kw = a.kw;
    int32_t dcl[3] = {-1, -1, -1};   // Roma: kept in registers for the row tags
    if (phase != 1 && lane >= 8 && lane <= 10) {
        const int k = lane - 8;
        const int64_t L = k == 0 ? g.nxg : (k == 1 ? g.ny : g.nz);
        const int per = k == 0 ? m.per_x : (k == 1 ? g.per_y : g.per_z);
        if (kw == 3) {
            double dwl[3];
            deposit_axis(kin[k], L, per, LBW_SPREAD_ROMA, 0.0, 3, dcl, dwl);
            for (int q = 0; q < 3; ++q) {
                a.dep_cell[(int64_t)p * 9 + 3 * k + q] = dcl[q];
                a.dep_w[(int64_t)p * 9 + 3 * k + q] = dwl[q];
            }
        } else {
            deposit_axis_wide(a, p, k, kin[k], L, per);
        }
    }
    int64_t j0[3];
    double t[3];
    for (int k = 0; k < 3; ++k) {
        const double fl = floor(kin[k] - 0.5);
        j0[k] = (int64_t)fl;
        t[k] = kin[k] - 0.5 - fl;
    }
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    bool have = true;  // this lane's cube cell is this step's value
    if (phase == 2) {
        if (lane < 8) {
            for (int q = 0; q < 4; ++q) v[q] = cube.local[((int64_t)p * 8 + lane) * 4 + q];
            have = cube.tag_local[(int64_t)p * 8 + lane] == cube.epoch;
        }
    } else if (lane < 8) {
        const int code = macro_at(g, m, j0[0] + ((lane >> 2) & 1), j0[1] + ((lane >> 1) & 1),
                                  j0[2] + (lane & 1), v);
        if (phase == 1) {
            const int64_t o = ((int64_t)p * 8 + lane) * 4;
            if (code != MA_REMOTE) {
                for (int q = 0; q < 4; ++q) cube.local[o + q] = v[q];
                cube.tag_local[(int64_t)p * 8 + lane] = cube.epoch;
            }
            if (code == MA_OWNED)
                for (int side = 0; side < 2; ++side)
                    if (cube.peer[side]) {
                        for (int q = 0; q < 4; ++q) cube.peer[side][o + q] = v[q];
                        cube.tag_peer[side][(int64_t)p * 8 + lane] = cube.epoch;
                    }
        }
    }
    if (phase == 1) return;
    const bool complete = __all_sync(0xffffffffu, have);
#ifdef LBW_K4_PROF
    const long long t3 = clock64();   // cube macro done
#endif
    // lane 0: trilinear sum in (dx,dy,dz) lexicographic order (actuator.py:88-92)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < 8; ++c) {
        double vc[4];
        for (int q = 0; q < 4; ++q) vc[q] = __shfl_sync(0xffffffffu, v[q], c);
        const double wx = (c >> 2) & 1 ? t[0] : 1.0 - t[0];
        const double wy = (c >> 1) & 1 ? t[1] : 1.0 - t[1];
        const double wz = c & 1 ? t[2] : 1.0 - t[2];
        const double w = wx * wy * wz;
        for (int q = 0; q < 4; ++q) acc[q] += w * vc[q];
    }
    if (s.flag_rows && phase != 1) {
        // tag this step's rows (benign race: equal values); for the Roma
        // kernel the x / y cells come from lanes 8 / 9 by shuffle
        if (kw == 3) {
            int32_t cx[3], cy[3];
            for (int q = 0; q < 3; ++q) {
                cx[q] = __shfl_sync(0xffffffffu, dcl[q], 8);
                cy[q] = __shfl_sync(0xffffffffu, dcl[q], 9);
            }
            if (lane < 9) {
                const int32_t cxg = cx[lane / 3], cyy = cy[lane % 3];
                const int64_t x = (int64_t)cxg - g.x0;
                LBW_CHECK(cyy < g.ny);
                if (cxg >= 0 && cyy >= 0 && x >= 0 && x < g.nxl)
                    s.row_key[x * g.ny + cyy] = row_key_of(s.tag, 0);
            }
        } else {
            __syncwarp();   // the deposit cells stored above are visible to the warp
            for (int t = lane; t < kw * kw; t += 32) {
                const int32_t row = pair_row(a, g, p * kw * kw + t);
                if (row >= 0) s.row_key[row] = row_key_of(s.tag, 0);
            }
        }
    }
    // Multi-slab: only points whose Roma support reaches this slab (their
    // sampling cube is then complete: own + neighbour cells) are evaluated;
    // per-point outputs come from the slab owning floor(x).  (Warp-uniform.)
    const int64_t n0 = (int64_t)floor(kin[0]);
    const int64_t ox = n0 - g.x0;
    const bool owner = phase == 0 || (ox >= 0 && ox < g.nxl);
    bool relevant = phase == 0;
    for (int dxc = -a.halo_x; dxc <= a.halo_x && !relevant; ++dxc) {
        int64_t c = n0 + dxc;
        if (m.per_x) c = (c % g.nxg + g.nxg) % g.nxg;
        relevant = c - g.x0 >= 0 && c - g.x0 < g.nxl;
    }
    double blade[3] = {0.0, 0.0, 0.0};
    if (relevant && !disk) blade_force_warp(a, ps, kin, acc, blade, lane);
#ifdef LBW_K4_PROF
    const long long t4 = clock64();
    if (lane == 0 && p == 0 && (a.step % 50) == 0)
        printf("K4PROF step %lld inputs+stage %lld kin %lld cube %lld blade %lld\n", (long long)a.step,
               in.t1 - in.t0, t2 - in.t1, t3 - t2, t4 - t3);
#endif
    if (lane == 0) {
        for (int q = 0; q < 4; ++q) a.samples[p * 4 + q] = owner ? acc[q] : 0.0;
        for (int c = 0; c < 3; ++c) {
            a.blade[p * 3 + c] = owner ? blade[c] : 0.0;
            a.flat[p * 3 + c] = -blade[c] * a.dt2 / a.den;  // units.py:69
        }
        if (disk) {
            // ring averages need every sample of the ring, owned or not
            for (int q = 0; q < 4; ++q) a.ring_samples[p * 4 + q] = acc[q];
            a.ring_sample_ok[p] = complete ? 1 : 0;
        }
    }
}

__global__ void k_alm_points(AlmDev a, Geom g, MacroDev m, ForceSet s, int phase, CubeArgs cube) {
    extern __shared__ double alm_sm[];
    const int p = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    LBW_TRACE_BEGIN(2, a.step);
    // The sampled cells lie in the rows the previous step's points forced:
    // their force is summed from that step's deposit data (actuator view),
    // which is staged in shared memory first -- one parallel load instead
    // of a dependent global load per point inside every cube cell.
    // flow-independent loads of this warp's point are issued first, so their
    // latency overlaps the staging below
    const int lane = threadIdx.x & 31;
    PointInputs in{};
#ifdef LBW_K4_PROF
    const long long t0 = clock64();
#endif
    if (p < a.n) in = load_point_inputs(a, p, lane);
    const ForceView& fv = m.fv;
    if (fv.row_key != nullptr && fv.pool == nullptr && fv.npts > 0 && fv.npts <= kOnTheFlyMaxPoints &&
        phase != 2) {
        const int n = fv.npts, nd = n * 3 * fv.kw;
        double* w = alm_sm;                                   // (n, 3, kw)
        double* fl = w + nd;                                  // (n, 3)
        int32_t* dc = reinterpret_cast<int32_t*>(fl + n * 3); // (n, 3, kw)
        // every load of a thread is issued before its first shared store
        // (one DRAM round trip, not one per loop iteration)
        constexpr int U = 8;
        const int nb = (int)blockDim.x, n3 = n * 3;
        for (int i0 = threadIdx.x; i0 < nd || i0 < n3; i0 += U * nb) {
            double wv[U], flv[U];
            int32_t cv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nb;
                if (i < nd) {
                    wv[u] = fv.dep_w[i];
                    cv[u] = fv.dep_cell[i];
                }
                if (i < n3) flv[u] = fv.flat[i];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nb;
                if (i < nd) {
                    w[i] = wv[u];
                    dc[i] = cv[u];
                }
                if (i < n3) fl[i] = flv[u];
            }
        }
        __syncthreads();
        m.fv.dep_w = w;
        m.fv.flat = fl;
        m.fv.dep_cell = dc;
    }
    if (p >= a.n) return;  // uniform per warp
#ifdef LBW_K4_PROF
    in.t0 = t0;
    in.t1 = clock64();
#endif
    point_warp(a, g, m, s, phase, cube, p, lane, in);
    LBW_TRACE_END(2, a.step);
}

// K4d: actuator-disk rings (actuator.py:149-183), one thread per ring, fixed
// summation order.  Fluid force per sample = direction * thrust/area_ring *
// area_i * axis; the blade force is its negation (sim.py:236-244).
// Slab-local view of a disk point (multi-slab): its Roma support reaches
// this slab / floor(x) lies in it.
__device__ bool point_relevant(const Geom& g, int per_x, int halo, double x) {
    const int64_t n0 = (int64_t)floor(x);
    for (int dxc = -halo; dxc <= halo; ++dxc) {
        int64_t c = n0 + dxc;
        if (per_x) c = (c % g.nxg + g.nxg) % g.nxg;
        if (c - g.x0 >= 0 && c - g.x0 < g.nxl) return true;
    }
    return false;
}

__device__ void disk_ring(const AlmDev& a, const Geom& g, int per_x, int linked, int r) {
    const int first = a.ring_first[r], cnt = a.ring_count[r];
    const double ct = a.ring_ct[r];
    if (linked) {
        // across slabs: the ring's samples must all be known here (owned by
        // this slab or a neighbour) if any of its forces land here
        bool all_ok = true, needed = false;
        for (int i = 0; i < cnt; ++i) {
            const int p = first + i;
            all_ok &= a.ring_sample_ok[p] != 0;
            needed |= point_relevant(g, per_x, a.halo_x, a.kin[(int64_t)p * kKin]);
        }
        if (!needed) {
            for (int i = 0; i < cnt; ++i)
                for (int c = 0; c < 3; ++c) {
                    a.blade[(first + i) * 3 + c] = 0.0;
                    a.flat[(first + i) * 3 + c] = 0.0;
                }
            return;
        }
        if (!all_ok) {
            atomicOr(a.error_flags, 4);
            return;
        }
    }
    const double* k0 = a.kin + (int64_t)first * kKin;
    double axis[3] = {k0[6], k0[7], k0[8]};
    const double nrm = sqrt(dot3(axis, axis));
    for (int c = 0; c < 3; ++c) axis[c] = axis[c] / nrm;
    if (ct == 0.0) return;  // forces stay zero
    const double ind = (1.0 - sqrt(1.0 - ct)) / 2.0;
    double ring_area = 0.0, su = 0.0, srho = 0.0;
    for (int i = 0; i < cnt; ++i) {
        const int p = first + i;
        const double ar = a.area[p];
        double up[3];
        for (int c = 0; c < 3; ++c) up[c] = a.ring_samples[p * 4 + 1 + c] * a.vscale;
        ring_area += ar;
        su += dot3(up, axis) * ar;
        srho += a.ring_samples[p * 4] * a.rho_ref * ar;
    }
    const double u_d = su / ring_area;
    const double rho = srho / ring_area;
    const double u_inf = u_d / (1.0 - ind);
    const double thrust = 0.5 * rho * u_inf * u_inf * ct * ring_area;
    const double direction = u_d != 0.0 ? (u_d > 0.0 ? -1.0 : 1.0) : 0.0;
    const double per_area = thrust / ring_area;
    for (int i = 0; i < cnt; ++i) {
        const int p = first + i;
        const int64_t ox = (int64_t)floor(a.kin[(int64_t)p * kKin]) - g.x0;
        const bool owner = !linked || (ox >= 0 && ox < g.nxl);
        for (int c = 0; c < 3; ++c) {
            const double f = direction * per_area * a.area[p] * axis[c];
            a.blade[p * 3 + c] = owner ? -f : 0.0;
            a.flat[p * 3 + c] = f * a.dt2 / a.den;
        }
    }
}

__global__ void k_alm_disks(AlmDev a, Geom g, int per_x, int linked) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    LBW_TRACE_BEGIN(3, a.step);
    if (r < a.n_rings) disk_ring(a, g, per_x, linked, r);
    LBW_TRACE_END(3, a.step);
}

// K5: one warp per deposit pair q.  The lowest pair touching a row owns it:
// it writes the row's force into pool slot q (per cell, the sum over all
// points touching the row in ascending id, as the reference's spreading
// loop adds them, actuator.py:241-246) and tags the row for this step.  No
// claims, counters or clearing: rows of earlier steps just keep old tags.
constexpr int kFillSmemPairs = 4096;
__global__ void k_alm_fill(AlmDev a, Geom g, ForceSet s) {
    __shared__ int32_t rows_sm[kFillSmemPairs];
    LBW_TRACE_BEGIN(4, a.step);
    const int kw = a.kw, npairs = a.n * kw * kw;
    const bool staged = npairs <= kFillSmemPairs;
    if (staged)
        for (int q = threadIdx.x; q < npairs; q += blockDim.x) rows_sm[q] = pair_row(a, g, q);
    __syncthreads();
    const int q = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= npairs) return;  // uniform per warp
    const int32_t row = staged ? rows_sm[q] : pair_row(a, g, q);
    if (row < 0) return;
    bool dup = false;
    for (int c0 = 0; c0 < q && !dup; c0 += 32) {
        const int q2 = c0 + lane;
        const bool same = q2 < q && (staged ? rows_sm[q2] : pair_row(a, g, q2)) == row;
        dup = __any_sync(0xffffffffu, same);
    }
    if (dup) return;
    const int64_t xg = row / g.ny + g.x0;
    const int32_t y = row % g.ny;
    LBW_CHECK(q >= 0 && q < npairs && row >= 0 && row < (int64_t)g.nxl * g.ny);
    const int64_t row0 = (int64_t)q * 3 * g.zp;
    for (int z0 = 0; z0 < g.nz; z0 += 32) {
        const int z = z0 + lane;
        double F[3] = {0.0, 0.0, 0.0};
        for (int c0 = 0; c0 < a.n; c0 += 32) {
            const int pl = c0 + lane;
            bool hit = false;
            double wxy = 0.0;
            if (pl < a.n) {
                const int32_t* dc = a.dep_cell + (int64_t)pl * 3 * kw;
                const double* dw = a.dep_w + (int64_t)pl * 3 * kw;
                double wx = 0.0, wy = 0.0;
                bool hx = false, hy = false;
                for (int t = 0; t < kw; ++t) {
                    if (dc[t] == xg) { hx = true; wx = dw[t]; }
                    if (dc[kw + t] == y) { hy = true; wy = dw[kw + t]; }
                }
                hit = hx && hy;
                wxy = wx * wy;
            }
            unsigned bal = __ballot_sync(0xffffffffu, hit);
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const double w2 = __shfl_sync(0xffffffffu, wxy, src);
                const int p = c0 + src;
                if (z < g.nz) {
                    const int32_t* dc = a.dep_cell + (int64_t)p * 3 * kw + 2 * kw;
                    const double* dw = a.dep_w + (int64_t)p * 3 * kw + 2 * kw;
                    for (int t = 0; t < kw; ++t) {
                        if (dc[t] == z) {
                            const double w = w2 * dw[t];
                            // `force[c] += w * F_lat` on an array of the storage
                            // dtype rounds after every addition (actuator.py:246)
                            if (g.single)
                                for (int c = 0; c < 3; ++c)
                                    F[c] = stored<float>(F[c] + w * a.flat[p * 3 + c]);
                            else
                                for (int c = 0; c < 3; ++c) F[c] += w * a.flat[p * 3 + c];
                        }
                    }
                }
            }
        }
        if (z < g.nz) {
            if (g.single) {
                float* dst = static_cast<float*>(s.pool) + row0;
                for (int c = 0; c < 3; ++c) dst[(int64_t)c * g.zp + z] = (float)F[c];
            } else {
                double* dst = static_cast<double*>(s.pool) + row0;
                for (int c = 0; c < 3; ++c) dst[(int64_t)c * g.zp + z] = F[c];
            }
        }
    }
    if (lane == 0) s.row_key[row] = row_key_of(s.tag, q);
    LBW_TRACE_END(4, a.step);
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

int alm_support_halo(const lbw_domain* d) { return alm_active(d) ? d->alm->halo_x : 0; }

double* alm_cube(const lbw_domain* d) { return alm_active(d) ? d->alm->cube : nullptr; }

void alm_destroy(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s) return;
    if (s->kin_stream) cudaStreamSynchronize(s->kin_stream);
    for (void* p : s->allocs) cudaFree(p);
    for (auto& e : s->ring_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {s->ev_kin_done, s->ev_chain_done[0], s->ev_chain_done[1],
                          s->ev_kin_step[0], s->ev_kin_step[1], s->ev_kin_step[2]})
        if (e) cudaEventDestroy(e);
    if (s->kin_stream) cudaStreamDestroy(s->kin_stream);
    if (s->h_ring) cudaFreeHost(s->h_ring);
    if (s->h_loads) cudaFreeHost(s->h_loads);
    delete s;
    d->alm = nullptr;
}

bool alm_ready(const lbw_domain* d, int64_t m) { return d->alm->ready_step == m; }

int alm_check_gate(lbw_domain* d) {
    if (!alm_active(d) || !d->alm->gate_flag) return LBW_OK;
    int32_t err = 0;
    LBW_CK(cudaMemcpy(&err, d->alm->gate_flag + 1, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) {
        set_error("a sweep's in-kernel wait for the actuator chain expired (results invalid)");
        return LBW_ECUDA;
    }
    return LBW_OK;
}

bool alm_can_prelaunch(const lbw_domain* d) { return d->prelaunch && d->alm->kin_device; }

bool alm_gate(lbw_domain* d, int64_t m, const uint32_t** flag, uint32_t* value,
              const int32_t** box, cudaEvent_t* kin_event) {
    const AlmState* s = d->alm;
    // only with the chain on its own SMs (the waiting CTAs cannot starve
    // it), one slab, device kinematics, and the chain of step m queued last
    if (!s || !s->gate_flag || !d->green_alm || d->linked || !s->kin_device ||
        s->ready_step != m || s->kin_valid[m % 3] != m)
        return false;
    *flag = s->gate_flag;
    *value = (uint32_t)d->alm_launches;
    *box = s->gate_box + 2 * (m % 3);
    *kin_event = s->ev_kin_step[m % 3];
    return true;
}

ForceView alm_force_view(const lbw_domain* d, int64_t m) {
    const AlmState* s = d->alm;
    ForceView v = s->set[m & 1].view((uint32_t)(m + 1));
    if (s->on_the_fly) {
        const AlmDev a = s->dev(m);
        v.pool = nullptr;
        v.npts = s->n;
        v.kw = s->kw;
        v.dep_cell = a.dep_cell;
        v.dep_w = a.dep_w;
        v.flat = a.flat;
    }
    return v;
}

int alm_invalidate(lbw_domain* d) {
    d->touched = true;
    if (!alm_active(d)) return LBW_OK;
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    if (d->alm->kin_stream) LBW_CK(cudaStreamSynchronize(d->alm->kin_stream));
    d->alm->ready_step = -1;
    return LBW_OK;
}

// KK for step j on the kinematics stream.  Kinematics do not depend on the
// flow, so step j+1's are computed while step j's chain and sweep run; the
// buffer kin[j&1] is free once the chain of step j-2 (its last reader) is
// done.
static int kin_launch(lbw_domain* d, int64_t j) {
    AlmState* s = d->alm;
    if (j < s->kin_state_step || j > s->kin_state_step + 1) {
        set_error("device kinematics can only advance one step at a time");
        return LBW_ESTATE;
    }
    const int advance = j > s->kin_state_step ? 1 : 0;
    LBW_CK(cudaStreamWaitEvent(s->kin_stream, s->ev_chain_done[j & 1], 0));
    const size_t ksm = s->kin_smem;
    KinDev kd = s->kdev();
    kd.hist_slot = (int32_t)(j % 3);
    kd.box = s->gate_box ? s->gate_box + 2 * (j % 3) : nullptr;
    kd.skip_static = s->kin_static_ready ? 1 : 0;
    k_kinematics<<<1, 256, ksm, s->kin_stream>>>(kd, s->dev(j), d->g,
                                                  d->desc.periodic[0] ? 1 : 0, advance);
    count_launch();
    LBW_CK(cudaGetLastError());
    LBW_CK(cudaEventRecord(s->ev_kin_done, s->kin_stream));
    if (s->ev_kin_step[j % 3]) LBW_CK(cudaEventRecord(s->ev_kin_step[j % 3], s->kin_stream));
    s->kin_static_ready = true;
    s->kin_state_step = j;
    s->kin_valid[j % 3] = j;
    return LBW_OK;
}

int alm_launch(lbw_domain* d, int64_t m) {
    AlmState* s = d->alm;
    const Geom& g = d->g;
    cudaStream_t st = d->alm_stream;
    const int par = (int)(m & 1);
    const AlmDev a = s->dev(m);
    const int per_x = d->desc.periodic[0] ? 1 : 0;
    // this step's use of force set m&1: rows tagged m+1
    ForceSet fs = s->set[par];
    fs.tag = (uint32_t)(m + 1);
    fs.flag_rows = s->on_the_fly ? 1 : 0;
    if (s->kin_device) {
        if (s->kin_valid[m % 3] != m) {
            int rc = kin_launch(d, m);
            if (rc) return rc;
        }
        LBW_CK(cudaStreamWaitEvent(st, s->ev_kin_done, 0));
    } else if (s->kin_queued_step != m) {
        set_error("actuator step without kinematics: call lbw_alm_set_kinematics first");
        return LBW_ESTATE;
    }
    MacroDev md{};
    md.kind = d->msrc.kind;
    for (int k = 0; k < 4; ++k) md.uniform[k] = d->msrc.uniform[k];
    md.buf = d->buf[d->msrc.buf];
    md.pull = d->msrc.pull ? 1 : 0;
    md.fv = d->msrc.fv;
    md.dense = d->macro_dense;
    md.bc_set = d->steps_done > 0 ? 1 : 0;
    for (int k = 0; k < 3; ++k) md.u_in[k] = d->desc.u_in[k];
    md.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    md.per_x = per_x;
    // one warp per CTA: fits in the registers a full sweep leaves free
    const int threads = 32;
    const size_t pts_smem =
        (md.fv.row_key != nullptr && md.fv.pool == nullptr && md.fv.npts <= kOnTheFlyMaxPoints)
            ? (size_t)md.fv.npts * ((3 * md.fv.kw + 3) * sizeof(double) +
                                    3 * md.fv.kw * sizeof(int32_t))
            : 0;
    const unsigned blocks = (unsigned)((s->n * 32 + threads - 1) / threads);
    CubeArgs cube{};
    if (d->linked) {
        const size_t off = (size_t)par * s->n * 32;
        const size_t tags = (size_t)2 * s->n * 32;   // tags follow the values
        const size_t toff = (size_t)par * s->n * 8;
        cube.local = s->cube + off;
        cube.tag_local = reinterpret_cast<int32_t*>(s->cube + tags) + toff;
        for (int side = 0; side < 2; ++side) {
            cube.peer[side] = d->nb_cube[side] ? d->nb_cube[side] + off : nullptr;
            cube.tag_peer[side] = d->nb_cube[side]
                                      ? reinterpret_cast<int32_t*>(d->nb_cube[side] + tags) + toff
                                      : nullptr;
        }
        // epochs count this domain's chain launches: a chain re-launched
        // after a state change (collective on every rank, as SlabSimulation's
        // calls are) waits for the neighbours' re-launch, not their first
        // launch of the same step, whose cube values may be stale
        cube.epoch = (int32_t)(d->alm_launches + 1);
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 1, cube);
        count_launch();
        LBW_CK(cudaGetLastError());
        const uint32_t epoch = (uint32_t)(d->alm_launches + 1);
        int rc = peer_signal(d, st, 1, epoch);
        if (!rc) rc = peer_wait(d, st, 1, epoch);
        if (rc) return rc;
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 2, cube);
    } else {
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 0, cube);
    }
    d->alm_launches += 1;
    if (s->n_rings > 0) {
        k_alm_disks<<<(unsigned)((s->n_rings + 63) / 64), 64, 0, st>>>(a, g, per_x,
                                                                       d->linked ? 1 : 0);
        count_launch();
    }
    if (!s->on_the_fly) {
        k_alm_fill<<<(unsigned)((s->n * s->kw * s->kw + 3) / 4), 128, 0, st>>>(a, g, fs);
        count_launch();
    }
    count_launch();
    LBW_CK(cudaGetLastError());
    LBW_CK(cudaEventRecord(d->ev_alm_done, st));
    if (s->gate_flag) {
        int rc = stream_write32(st, s->gate_flag, (uint32_t)d->alm_launches);
        if (rc) return rc;
    }
    if (s->loads_cap > 0)
        LBW_CK(cudaMemcpyAsync(s->h_loads + (size_t)(m % s->loads_cap) * s->n * 3, a.blade,
                               (size_t)s->n * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (s->kin_device) {
        LBW_CK(cudaEventRecord(s->ev_chain_done[par], st));
        // prefetch the next step's kinematics while this chain and sweep run
        if (alm_can_prelaunch(d) && s->kin_state_step == m) {
            int rc = kin_launch(d, m + 1);
            if (rc) return rc;
        }
    }
    s->ready_step = m;
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
    d->touched = true;
    if (desc->n_points > 0) {
        int rc_ = green_partition(d, alm_sm_count(d));
        if (rc_) return rc_;
    }
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    alm_destroy(d);
    const int P = desc->n_points;
    if (P == 0) return LBW_OK;
    for (int p = 0; p < P; ++p)
        LBW_REQ(desc->polar_index[p] >= -1 && desc->polar_index[p] < desc->n_polars,
                "polar index out of range");
    if (desc->point_ring) {
        LBW_REQ(desc->area && desc->n_rings >= 0, "disk rings need areas");
        for (int r = 0; r < desc->n_rings; ++r) {
            LBW_REQ(desc->ring_first[r] >= 0 && desc->ring_count[r] >= 1 &&
                        desc->ring_first[r] + desc->ring_count[r] <= P,
                    "disk ring point range out of bounds");
            LBW_REQ(desc->ring_ct[r] >= 0.0 && desc->ring_ct[r] < 1.0,
                    "thrust coefficient must lie in [0, 1)");
        }
    }
    LBW_REQ(desc->spread_kernel == LBW_SPREAD_ROMA || desc->spread_kernel == LBW_SPREAD_GAUSSIAN,
            "unknown spreading kernel");
    LBW_REQ(desc->spread_kernel != LBW_SPREAD_GAUSSIAN ||
                (desc->spread_epsilon > 0.0 && desc->spread_epsilon <= 2.0),
            "Gaussian spreading width must lie in (0, 2] lattice cells");
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
    s->kernel = desc->spread_kernel;
    if (s->kernel == LBW_SPREAD_GAUSSIAN) {
        s->eps = desc->spread_epsilon;
        s->kw = (int32_t)floor(6.0 * s->eps) + 1;      // cells within 3 eps of a point
        s->halo_x = (int32_t)ceil(3.0 * s->eps) + 1;
    }
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
    A(&s->kin, (size_t)3 * P * kKin);
    A(&s->samples, (size_t)2 * P * 4);
    A(&s->blade, (size_t)2 * P * 3);
    A(&s->flat, (size_t)2 * P * 3);
    A(&s->cube, (size_t)2 * P * 32 + (size_t)2 * P * 4);   // values, then (2,P,8) int32 tags
    A(&s->ring_samples, (size_t)P * 4);
    A(&s->ring_sample_ok, P);
    A(&s->dep_cell, (size_t)2 * P * 3 * s->kw);
    A(&s->dep_w, (size_t)2 * P * 3 * s->kw);
    A(&s->clamp_flags, std::max(1, desc->n_polars));
    A(&s->error_flags, 1);
    const int R = desc->point_ring ? desc->n_rings : 0;
    if (desc->point_ring) {
        A(&s->point_ring, P);
        A(&s->area, P);
        A(&s->ring_first, std::max(1, R));
        A(&s->ring_count, std::max(1, R));
        A(&s->ring_ct, std::max(1, R));
    }
    // sparse force sets: a point touches at most 3x3 (x,y) rows
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    s->on_the_fly = P <= kOnTheFlyMaxPoints;
    const int64_t cap = s->on_the_fly ? 0 : (int64_t)s->kw * s->kw * P;   // slot = deposit pair
    for (auto& fs : s->set) {
        A(&fs.row_key, rows);
        if (cap) {
            char* pool = nullptr;
            A(&pool, (size_t)cap * 3 * d->g.zp * elem_bytes(d->g));
            fs.pool = pool;
        }
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
    if (desc->point_ring) {
        H(s->point_ring, desc->point_ring, P * 4);
        H(s->area, desc->area, P * 8);
        if (R) {
            H(s->ring_first, desc->ring_first, R * 4);
            H(s->ring_count, desc->ring_count, R * 4);
            H(s->ring_ct, desc->ring_ct, R * 8);
        }
        s->n_rings = R;
    }
    if (desc->n_polars) {
        H(s->polar_offset, desc->polar_offset, desc->n_polars * 4);
        H(s->polar_rows, desc->polar_rows, desc->n_polars * 4);
        H(s->p_alpha, desc->polar_alpha, total_rows * 8);
        H(s->p_cl, desc->polar_cl, total_rows * 8);
        H(s->p_cd, desc->polar_cd, total_rows * 8);
    }
    if (rc == LBW_OK) {
        for (auto& fs : s->set) {
            // keys with tag 0xffffffff match no step (chain tags are step+1)
            if (cudaMemset(fs.row_key, 0xff, rows * 8) != cudaSuccess) {
                cudaGetLastError();
                rc = LBW_ECUDA;
            }
        }
        if (cudaMemset(s->clamp_flags, 0, std::max(1, desc->n_polars) * 4) != cudaSuccess ||
            cudaMemset(s->error_flags, 0, 4) != cudaSuccess ||
            cudaMemset(s->cube, 0, ((size_t)2 * P * 32 + (size_t)2 * P * 4) * 8) != cudaSuccess ||
            cudaMemset(s->samples, 0, (size_t)2 * P * 32) != cudaSuccess ||
            cudaMemset(s->blade, 0, (size_t)2 * P * 24) != cudaSuccess ||
            cudaMemset(s->kin, 0, (size_t)3 * P * kKin * 8) != cudaSuccess ||
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

int lbw_alm_configure_kinematics(lbw_domain* d, const lbw_kin_desc* kd) {
    LBW_REQ(d && kd, "null argument");
    LBW_REQ(alm_active(d), "configure the actuator points first");
    AlmState* s = d->alm;
    const int C = kd->n_components, P = s->n;
    LBW_REQ(C >= 1 && C <= 256, "need 1..256 turbine components");
    LBW_REQ(kd->dx > 0.0, "dx must be positive");
    for (int c = 0; c < C; ++c) {
        LBW_REQ(kd->parent[c] >= -1 && kd->parent[c] < c, "components must be in pre-order");
        LBW_REQ(kd->line_first[c] >= -1 && kd->line_first[c] + kd->line_count[c] <= P,
                "line point range out of bounds");
    }
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    std::vector<int32_t> point_comp(P, -1);
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < kd->line_count[c]; ++k) point_comp[kd->line_first[c] + k] = c;
    for (int p = 0; p < P; ++p)
        LBW_REQ(point_comp[p] >= 0, "point without a line or disk component");
    int rc = LBW_OK;
    auto A = [&](auto** p, size_t n) {
        if (rc == LBW_OK) rc = dev_alloc(d, s, p, n);
    };
    A(&s->k_parent, C);
    A(&s->k_line_first, C);
    A(&s->k_line_count, C);
    A(&s->k_point_comp, P);
    A(&s->k_rel_p, (size_t)C * 3);
    A(&s->k_rel_T, (size_t)C * 9);
    A(&s->k_axis, (size_t)C * 3);
    A(&s->k_rate, C);
    A(&s->k_rstep, (size_t)C * 9);
    A(&s->k_spin, (size_t)C * 9);
    A(&s->k_off, (size_t)P * 3);
    A(&s->k_orient, (size_t)P * 9);
    A(&s->k_lframe, (size_t)P * 9);
    A(&s->k_cs, (size_t)C * kCS);
    A(&s->k_spin_hist, (size_t)3 * C * 9);
    A(&s->k_cs_hist, (size_t)3 * C * kCS);
    A(&s->k_is_disk, C);
    A(&s->k_disk_center, (size_t)C * 12);
    A(&s->k_order, C);
    A(&s->k_static, C);
    A(&s->k_level_start, (size_t)C + 1);
    if (rc) return rc;
    // walk schedule: components by depth (parents precede children), and
    // which ones never move (no rotation on the path from the root)
    std::vector<int32_t> depth(C), stat(C), order, lstart;
    for (int c = 0; c < C; ++c) {
        const int pa = kd->parent[c];
        depth[c] = pa < 0 ? 0 : depth[pa] + 1;
        stat[c] = kd->rate[c] == 0.0 && (pa < 0 || stat[pa]);
    }
    const int maxd = *std::max_element(depth.begin(), depth.end());
    for (int L = 0; L <= maxd; ++L) {
        lstart.push_back((int32_t)order.size());
        for (int c = 0; c < C; ++c)
            if (depth[c] == L) order.push_back(c);
    }
    lstart.push_back((int32_t)order.size());
    s->k_nlevels = maxd + 1;
    auto H = [&](void* dst, const void* src, size_t bytes) {
        if (rc == LBW_OK && cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            set_error("kinematics upload failed");
            rc = LBW_ECUDA;
        }
    };
    H(s->k_parent, kd->parent, C * 4);
    H(s->k_line_first, kd->line_first, C * 4);
    H(s->k_line_count, kd->line_count, C * 4);
    H(s->k_point_comp, point_comp.data(), P * 4);
    H(s->k_rel_p, kd->rel_p, C * 24);
    H(s->k_rel_T, kd->rel_T, C * 72);
    H(s->k_axis, kd->axis, C * 24);
    H(s->k_rate, kd->rate, C * 8);
    H(s->k_rstep, kd->step_rotation, C * 72);
    H(s->k_spin, kd->spin, C * 72);
    H(s->k_off, kd->offsets, (size_t)P * 24);
    H(s->k_orient, kd->orientations, (size_t)P * 72);
    H(s->k_lframe, kd->local_frames, (size_t)P * 72);
    H(s->k_order, order.data(), (size_t)C * 4);
    H(s->k_static, stat.data(), (size_t)C * 4);
    H(s->k_level_start, lstart.data(), lstart.size() * 4);
    {
        std::vector<int32_t> isd(C, 0);
        std::vector<double> dcen((size_t)C * 12, 0.0);
        for (int c = 0; c < C; ++c) {
            if (kd->is_disk) isd[c] = kd->is_disk[c] ? 1 : 0;
            if (kd->disk_center && isd[c])
                for (int i = 0; i < 12; ++i) dcen[(size_t)c * 12 + i] = kd->disk_center[(size_t)c * 12 + i];
        }
        H(s->k_is_disk, isd.data(), C * 4);
        H(s->k_disk_center, dcen.data(), (size_t)C * 96);
    }
    if (rc) return rc;
    size_t ksm = (size_t)C * (kKP + kCS) * sizeof(double) + (size_t)(3 * C + 1) * 4;
    const size_t kpts = (size_t)P * 21 * sizeof(double) + (size_t)P * sizeof(int32_t);
    s->kin_stage_points = ksm + kpts <= 160 * 1024;
    if (s->kin_stage_points) ksm += kpts;
    if (ksm > 48 * 1024 &&
        cudaFuncSetAttribute(k_kinematics, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ksm) != cudaSuccess) {
        cudaGetLastError();
        set_error("too many turbine components for the kinematics CTA");
        return LBW_EINVAL;
    }
    s->kin_smem = ksm;
    if (!s->kin_stream) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        s->kin_stream = green_alm_stream(d);   // on the chain's SMs when partitioned
        if ((!s->kin_stream &&
             cudaStreamCreateWithPriority(&s->kin_stream, cudaStreamNonBlocking, hi) != cudaSuccess) ||
            cudaEventCreateWithFlags(&s->ev_kin_done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_chain_done[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_chain_done[1], cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            set_error("kinematics stream/event creation failed");
            return LBW_ECUDA;
        }
    }
    LBW_CK(cudaStreamSynchronize(s->kin_stream));
    // sweep gate (alm_gate): only when the chain has SMs of its own
    const char* ge = getenv("LBW_SWEEP_GATE");
    if (d->green_alm && !(ge && ge[0] == '0') && !s->gate_flag) {
        int rcg = LBW_OK;
        auto G = [&](auto** p, size_t n) {
            if (rcg == LBW_OK) rcg = dev_alloc(d, s, p, n);
        };
        G(&s->gate_flag, 2);   // [0] chain launches done, [1] sweep wait expired
        G(&s->gate_box, 6);
        if (rcg) return rcg;
        for (auto& e : s->ev_kin_step)
            LBW_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        LBW_CK(cudaMemset(s->gate_flag, 0, 2 * sizeof(uint32_t)));
    }
    s->nc = C;
    s->k_dx = kd->dx;
    s->kin_device = true;
    s->kin_state_step = d->step - (kd->advance_first ? 1 : 0);
    s->kin_valid[0] = s->kin_valid[1] = s->kin_valid[2] = -1;
    s->kin_static_ready = false;
    s->ready_step = -1;
    return LBW_OK;
}

// step whose turbine state lbw_alm_download_kinematics reports: the
// domain's step, unless the device kinematics have not reached it yet
static int64_t kin_view_step(const lbw_domain* d) {
    return std::min<int64_t>(d->step, d->alm->kin_state_step);
}

// parity of the most recent step's actuator outputs
static int last_parity(const lbw_domain* d) { return d->step > 0 ? (int)((d->step - 1) & 1) : 0; }

int lbw_alm_download_kinematics(lbw_domain* d, double* kin, double* spin, double* comp_state) {
    LBW_REQ(d, "null domain");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    if (s->kin_stream) LBW_CK(cudaStreamSynchronize(s->kin_stream));
    if (kin)
        LBW_CK(cudaMemcpy(kin, s->kin + (size_t)(d->step > 0 ? (d->step - 1) % 3 : 0) * s->n * kKin,
                          (size_t)s->n * kKin * 8, cudaMemcpyDeviceToHost));
    // the turbine state of step d->step (what the host objects hold after
    // d->step advances), even when the next step's kinematics already ran
    const int64_t v = kin_view_step(d);
    const bool hist = s->kin_valid[v % 3] == v;
    if (spin && s->kin_device)
        LBW_CK(cudaMemcpy(spin, hist ? s->k_spin_hist + (size_t)(v % 3) * s->nc * 9 : s->k_spin,
                          (size_t)s->nc * 72, cudaMemcpyDeviceToHost));
    if (comp_state && s->kin_device)
        LBW_CK(cudaMemcpy(comp_state,
                          hist ? s->k_cs_hist + (size_t)(v % 3) * s->nc * kCS : s->k_cs,
                          (size_t)s->nc * kCS * 8, cudaMemcpyDeviceToHost));
    return LBW_OK;
}

int64_t lbw_alm_kinematics_step(lbw_domain* d) {
    if (!d || !alm_active(d) || !d->alm->kin_device) return -1;
    return kin_view_step(d);
}

int lbw_alm_set_kinematics(lbw_domain* d, const double* kin) {
    LBW_REQ(d && kin, "null argument");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_REQ(!s->kin_device, "kinematics are computed on the device for this domain");
    LBW_CK(cudaSetDevice(d->device));
    const int slot = s->ring_pos;
    s->ring_pos = (s->ring_pos + 1) % kRing;
    LBW_CK(cudaEventSynchronize(s->ring_ev[slot]));
    double* h = s->h_ring + (size_t)slot * s->n * kKin;
    std::memcpy(h, kin, (size_t)s->n * kKin * 8);
    const int64_t m = d->step;
    LBW_CK(cudaMemcpyAsync(s->kin + (size_t)(m % 3) * s->n * kKin, h, (size_t)s->n * kKin * 8,
                           cudaMemcpyHostToDevice, d->alm_stream));
    LBW_CK(cudaEventRecord(s->ring_ev[slot], d->alm_stream));
    s->kin_queued_step = m;
    s->ready_step = -1;
    return LBW_OK;
}

int lbw_alm_get(lbw_domain* d, double* rho, double* u, double* blade_force) {
    LBW_REQ(d, "null domain");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    const int par = last_parity(d);
    std::vector<double> smp((size_t)s->n * 4);
    LBW_CK(cudaMemcpy(smp.data(), s->samples + (size_t)par * s->n * 4, smp.size() * 8,
                      cudaMemcpyDeviceToHost));
    if (blade_force)
        LBW_CK(cudaMemcpy(blade_force, s->blade + (size_t)par * s->n * 3, (size_t)s->n * 24,
                          cudaMemcpyDeviceToHost));
    int32_t err = 0;
    LBW_CK(cudaMemcpy(&err, s->error_flags, 4, cudaMemcpyDeviceToHost));
    for (int p = 0; p < s->n; ++p) {
        if (rho) rho[p] = smp[p * 4];
        if (u)
            for (int c = 0; c < 3; ++c) u[p * 3 + c] = smp[p * 4 + 1 + c];
    }
    if (err & 2) {
        set_error("actuator point outside the non-periodic domain");
        return LBW_EINVAL;
    }
    if (err & 4) {
        set_error("an actuator disk spans more than three x-slabs (its ring averages need "
                  "samples from beyond the neighbouring slabs)");
        return LBW_EINVAL;
    }
    if (err & 1) {
        set_error("density must be positive at an actuator point");
        return LBW_EINVAL;
    }
    return LBW_OK;
}

int lbw_alm_record_loads(lbw_domain* d, int64_t capacity) {
    LBW_REQ(d && capacity >= 0, "bad argument");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    if (s->h_loads) cudaFreeHost(s->h_loads);
    s->h_loads = nullptr;
    s->loads_cap = 0;
    if (capacity > 0) {
        LBW_REQ(capacity >= 2, "capacity must be >= 2");
        LBW_CK(cudaMallocHost(&s->h_loads, (size_t)capacity * s->n * 3 * sizeof(double)));
        s->loads_cap = capacity;
    }
    s->loads_from = d->step;
    // a chain already queued for the next step has not recorded its loads
    s->ready_step = -1;
    return LBW_OK;
}

int lbw_alm_read_loads(lbw_domain* d, double* out, int64_t max_steps, int64_t* first_step,
                       int64_t* n) {
    LBW_REQ(d && out && first_step && n && max_steps >= 0, "null argument");
    LBW_REQ(alm_active(d) && d->alm->loads_cap > 0, "load recording is not enabled");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    const int64_t avail = d->step - s->loads_from;
    LBW_REQ(avail < s->loads_cap || avail == 0,
            "load ring overflow: read the loads at least every capacity-1 steps");
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    const int64_t k = std::min(avail, max_steps);
    const size_t row = (size_t)s->n * 3;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t st = s->loads_from + i;
        std::memcpy(out + (size_t)i * row, s->h_loads + (size_t)(st % s->loads_cap) * row,
                    row * sizeof(double));
    }
    *first_step = s->loads_from;
    *n = k;
    s->loads_from += k;
    return LBW_OK;
}

int lbw_alm_clamp_flags(lbw_domain* d, int32_t* per_polar) {
    LBW_REQ(d && per_polar, "null argument");
    if (!alm_active(d) || d->alm->n_polars == 0) return LBW_OK;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaMemcpy(per_polar, d->alm->clamp_flags, d->alm->n_polars * 4,
                      cudaMemcpyDeviceToHost));
    return LBW_OK;
}

}  // extern "C"

LBW_TRACE_EXPORT(alm)
