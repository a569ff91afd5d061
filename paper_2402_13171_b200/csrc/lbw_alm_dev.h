// lbw_alm_dev.h — plain-data views of the actuator state shared by the host
// driver (lbw_alm.cu) and the kernels that run the actuator chain (the
// standalone chain kernels and the fused step kernel, lbw_fused.cuh).
#pragma once
#include <cstdint>

#include "lbw_internal.h"

namespace lbw {

constexpr int kKin = 18;
// per-step actuator data computed ahead of the step that uses it
// (kinematics, spin / component history, deposit geometry, row keys) live
// in slots j % kSlots: the flag-ordered chain computes them four steps
// ahead, and slot j is last read by the sweep of step j (and its row keys by
// the sweep of step j-1), so kSlots = 6 leaves one step of margin
constexpr int kSlots = 6;  // pos_lat(3) vel(3) e_chord(3) e_normal(3) e_span(3) pos_m(3)
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
    double* loads_row;        // (P,3) this step's row of the device loads ring, or nullptr
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
    double* spin_hist;   // (kSlots, nc, 9): spin state of step j in slot j % kSlots
    double* cs_hist;     // (kSlots, nc, kCS)
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
    // the constant part of the CTA's shared-memory image, packed once by the
    // host in the exact layout (kinematics_cta): the parameter block (spin
    // slots excepted) and the tail from the point block / walk schedule on;
    // staged with independent 8-byte loads (one round trip, not one per
    // field and loop iteration)
    const long long* img_prm;    // (nc * kKP) doubles
    const long long* img_tail;   // img_tail_words 8-byte words
    int32_t img_tail_words;
};

// parameters per component in the kinematics CTA's shared memory:
// rel_p 3, rel_T 9, axis 3, rate 1, rstep 9, spin 9, parent 1, first 1, is_disk 1, disk p 3, T 9
constexpr int kKP = 49;
constexpr int kMaxKw = 13;   // eps <= 2 -> at most floor(6 eps * 2) + 1 cells
constexpr int kOnTheFlyMaxPoints = 64;
// corner-force lists (flag-ordered chain): at most this many deposit terms
// per sampling corner; beyond it the sampling scans the points itself
constexpr int kCornerTerms = 24;
enum { MA_REMOTE = 0, MA_OWNED = 1, MA_CONST = 2 };


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

struct CubeArgs {
    double* local;   // (P,8,4) of this step's parity
    double* peer[2];
    // per cube cell: epoch of the launch that wrote it (same allocation,
    // after the values), so a reader knows which cells are this step's
    int32_t* tag_local;  // (P,8)
    int32_t* tag_peer[2];
    int32_t epoch;
};

// ---------------------------------------------------------------- fused step
// Per-step actuator data of the fused step kernel live in three slots
// (step j in slot j % 3): KK(j) writes them two steps ahead, K4(j) and
// sweep j read them, nothing of step j is overwritten before sweep j+1.

// Geometry of step j, written by KK(j): deposit cells / weights, the force
// rows it tags (tag j+1, read by sweep j), and the rows holding its
// sampling cubes (sample keys, tag j+1, slot = point*4 + corner row: sweep
// j-1 stores the macro of those rows into the sample pool for K4(j)).
struct FsGeom {
    int32_t* dep_cell;     // (P,3,kw)
    double* dep_w;         // (P,3,kw)
    uint64_t* frow_key;    // (nxl*ny)
    uint64_t* skey;        // (nxl*ny)
    uint32_t tag;          // j+1
    int32_t inflow;        // velocity_inflow_outflow x faces
};

// Sampling of step j from the pool sweep j-1 filled.
struct FsPool {
    const uint64_t* skey;  // sample row keys of step j
    const double* spool;   // (4P, 4, zp): rho, ux, uy, uz of each keyed row
    uint32_t tag;          // j+1
    int32_t inflow;
    double u_in[3];
    int32_t* error_flags;  // bit 3: a sampled row without a pool entry
    // raw != 0 (flag-ordered chain): the pool holds the force-free sums
    // (rho, sum f c) the sweep of step j-1 stored before its force was
    // known; the macro is completed here with that sweep's force at the
    // cell, u = (sum f c + F dt / 2) / rho -- moments_exact's arithmetic
    int32_t raw;
    ForceView fv;          // the force of sweep j-1
    // optional: for each (point, corner) of step j the deposit terms of step
    // j-1 that reach the corner cell -- (point, weight (wx wy) wz) in the
    // order actuator_force_k adds them -- built by the geometry kernel of
    // step j; count < 0: not listed (the sampling scans fv)
    const int32_t* cf_n;   // (P, 8)
    const int16_t* cf_p;   // (P, 8, kCornerTerms)
    const double* cf_w;    // (P, 8, kCornerTerms)
};

// One launch of the fused step kernel (lbw_fused.cuh): sweep m, the point
// forces of step m (K4, claimed as tasks by helper CTAs and by any sweep CTA
// that needs them) and the kinematics + geometry of step m+2 (KK, one CTA).
struct FusedArgs {
    SweepArgs sw;          // sweep m; sw.fv = the on-the-fly force view of step m
    AlmDev a;              // K4(m): kin slot m%3, flat = fused slot, outputs by parity
    MacroDev md;           // general sampling source (use_pool == 0)
    int32_t use_pool;
    FsPool pool;           // use_pool: the cube values from the pool of step m
    uint32_t* ctr;         // [task, done] of this launch (zeroed by the previous launch)
    uint32_t* ctr_next;    // zeroed here for the next launch
    const uint64_t* skey_next;  // sample keys of step m+1 (tag store_tag)
    double* spool_next;         // its pool, filled by this sweep
    uint32_t store_tag;         // m+2
    int32_t kk_on;              // KK(m+2) runs in CTA 0
    KinDev k;
    AlmDev a_kk;                // kin slot (m+2)%3
    FsGeom geo;                 // geometry of step m+2
    int32_t per_x;
    int32_t n_kk, n_help;       // leading CTAs: KK, point-task helpers
    uint32_t tiles_x, tiles_y;  // sweep tiles per plane (z blocks, y blocks)
    // optional timeline (LBW_FUSED_PROF): %globaltimer of this launch's
    // [first CTA start, KK start, KK end, last point task done, last
    // force-tile wait end, last CTA end]; nullptr = off.  prof_next: the
    // next launch's row, reset here
    unsigned long long* prof;
    unsigned long long* prof_next;
};

// one fused step launch (lbw_fused.cuh), per arithmetic flavour
cudaError_t launch_fused_exact(int op, bool pull, const FusedArgs& a, size_t smem,
                               cudaStream_t s);
cudaError_t launch_fused_fast(int op, bool pull, const FusedArgs& a, size_t smem, cudaStream_t s);

}  // namespace lbw
