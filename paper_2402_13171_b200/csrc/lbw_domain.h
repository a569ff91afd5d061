// lbw_domain.h — host-side state of one device-resident x-slab.
#pragma once
#include <string>
#include <vector>

#include "../../include/lbw.h"
#include "lbw_internal.h"

namespace lbw {

void set_error(const std::string& msg);

#define LBW_CK(call)                                                                    \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::lbw::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));       \
            return LBW_ECUDA;                                                           \
        }                                                                               \
    } while (0)

#define LBW_REQ(cond, msg)                  \
    do {                                    \
        if (!(cond)) {                      \
            ::lbw::set_error(msg);          \
            return LBW_EINVAL;              \
        }                                   \
    } while (0)

struct MacroSource {
    int kind = MS_UNIFORM;
    double uniform[4] = {1.0, 0.0, 0.0, 0.0};
    int buf = 0;          // MS_GATHER: population buffer
    bool pull = false;    //            stream from it (post-collision data)
    ForceView fv{nullptr, nullptr};
};

struct AlmState;  // lbw_alm.cu

}  // namespace lbw

struct lbw_domain {
    lbw_domain_desc desc{};
    lbw::Geom g{};
    lbw::Relax relax{};
    int device = 0;
    cudaStream_t stream = nullptr;
    void* buf[2] = {nullptr, nullptr};   // populations, storage type per g.single
    int cur = 0;             // buffer holding the current state
    bool state_pre = true;   // buf[cur] holds pre-collision populations
    int64_t step = 0;
    // force
    lbw::ForceSet user;      // dense body force set by the caller
    bool user_active = false;
    lbw::ForceView last_fv{nullptr, nullptr};  // force of the most recent collide
    lbw::ForceView shown_fv{nullptr, nullptr}; // what download_force reports
    // ALM sampling source for the next step
    lbw::MacroSource msrc;
    double* macro_dense = nullptr;
    // non-finite flag
    unsigned long long* d_nan = nullptr;
    unsigned long long* h_nan = nullptr;
    cudaEvent_t nan_event = nullptr;
    bool nan_pending = false;
    // staging for AoS transfers
    double* stage = nullptr;
    size_t stage_bytes = 0;
    int64_t bytes = 0;
    lbw::AlmState* alm = nullptr;
    // actuator work runs on its own stream so the next step's sampling /
    // forces / spreading overlap the current sweep (see lbw_domain_step)
    cudaStream_t alm_stream = nullptr;
    // optional SM partition (lbw_green.cu): green contexts of the sweep /
    // actuator-chain streams (CUgreenCtx), SMs given to the chain
    void* green_sweep = nullptr;
    void* green_alm = nullptr;
    int alm_sms = 0;
    cudaEvent_t ev_main = nullptr, ev_alm_done = nullptr;
    int64_t steps_done = 0;   // sweeps executed in this domain's lifetime
    bool prelaunch = true;
    cudaEvent_t ev_ready = nullptr;   // main stream passed the neighbour waits of a step
    cudaEvent_t ev_ready_prev = nullptr;  // ... of the step before
    bool touched = true;              // state changed by a call since the last step
    bool sweep_alt = true;            // alternate the interior plane order (LBW_SWEEP_ALT)
    bool fused = false;               // one fused launch per actuator step when eligible (LBW_FUSED=1)
    bool chainb = true;               // flag-ordered actuator chain when eligible (LBW_CHAIN_FLAGS)
    bool chainb_forced = false;       // LBW_CHAIN_FLAGS=1: regardless of the slab size
    bool chain_loop = false;          // LBW_CHAIN_LOOP=1: resident chain kernel per call
    // x-slab neighbours (lbw_peer.cu): side 0 = lo (x-1), side 1 = hi (x+1)
    bool linked = false;
    int nb_rank[2] = {-1, -1};
    int32_t nb_nxl[2] = {0, 0};
    void* nb_buf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [side][buffer]
    double* nb_cube[2] = {nullptr, nullptr};
    uint32_t* nb_flags[2] = {nullptr, nullptr};
    // my flags, written by the neighbours: [0] sweeps done by lo, [1] by hi,
    // [2] cube launches done by lo, [3] by hi
    uint32_t* flags = nullptr;
    unsigned long long* edge_counter = nullptr;  // edge-CTA arrivals (in the flags allocation)
    int64_t alm_launches = 0;
    // optional sweep timing (lbw_domain_sweep_timing)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    // multi-GPU halo targets (peer ghost planes) per buffer
    lbw::HaloOut halo[2] = {{nullptr, nullptr}, {nullptr, nullptr}};
    std::vector<void*> peer_mapped;
};

namespace lbw {
// lbw_alm.cu
// Launch the actuator chain of step m on d->alm_stream (clear set m&1,
// kinematics, sample/force/mark, fill); records d->ev_alm_done.
int alm_launch(lbw_domain* d, int64_t m);
// Step m's chain already queued and still valid?
bool alm_ready(const lbw_domain* d, int64_t m);
bool alm_can_prelaunch(const lbw_domain* d);
// LBW_ECUDA when a gated sweep's bounded wait expired (after a sync)
int alm_check_gate(lbw_domain* d);
// Sweep m may start before the chain of step m finishes: CTAs of planes in
// the chain's x range wait in-kernel for its completion flag (single slab,
// device kinematics, chain on its own SMs).  Fills the gate arguments.
bool alm_gate(lbw_domain* d, int64_t m, const uint32_t** flag, uint32_t* value,
              const int32_t** box, cudaEvent_t* kin_event);
ForceView alm_force_view(const lbw_domain* d, int64_t m);
// Fused step (lbw_fused.cuh): one launch per step -- sweep m, point forces
// of step m, kinematics + geometry of step m+2 -- on a single slab with
// device kinematics and <= 64 points (no disks, no caller body force).
bool alm_fused_eligible(const lbw_domain* d);
int alm_fused_launch(lbw_domain* d, bool pull, ForceView* fv_out);
// the previous step was a fused launch (its point forces are written inside
// that launch: a standalone chain must wait for all of it)
bool alm_after_fused(const lbw_domain* d);
// Flag-ordered actuator chain ("chain B", lbw_alm.cu): single slab, device
// kinematics, <= 64 points without disks.  Fills the chain fields of the
// sweep of step m (and its force view), queues what the chain needs first,
// and after the sweep (alm_chainb_after) the chain of the next step.
bool alm_chainb_eligible(const lbw_domain* d);
int alm_chainb_before(lbw_domain* d, SweepArgs* a);
int alm_chainb_after(lbw_domain* d, int64_t m, int32_t remaining);
bool alm_after_chainb(const lbw_domain* d);
// Wait for queued actuator work and forget any prelaunched step (the
// caller is about to change state it reads).
int alm_invalidate(lbw_domain* d);
void alm_destroy(lbw_domain* d);
bool alm_active(const lbw_domain* d);
// wait for the kinematics stream of the actuator chain
cudaError_t alm_sync_side(const lbw_domain* d);
int alm_support_halo(const lbw_domain* d);   // spreading support half-width in x (cells)
// device cube buffer (2, P, 8, 4) of the actuator sampling, or nullptr
double* alm_cube(const lbw_domain* d);

// lbw_peer.cu: cross-process GPU-side ordering with the slab neighbours
// (stream memory operations on flags in peer memory; no host round trip)
int peer_wait(lbw_domain* d, cudaStream_t s, int which, uint32_t value);    // which 0: sweeps, 1: cube
int peer_signal(lbw_domain* d, cudaStream_t s, int which, uint32_t value);
int stream_write32(cudaStream_t s, uint32_t* ptr, uint32_t value);   // GPU front-end write
void peer_close(lbw_domain* d);
int ensure_stage(lbw_domain* d, size_t bytes);

// lbw_green.cu: SM partition between the sweep and the actuator chain
int alm_sm_count(const lbw_domain* d);
// a profiler / sanitizer that serialises kernels is injected in the process
bool tool_injected();
int green_partition(lbw_domain* d, int alm_sms);
cudaStream_t green_alm_stream(lbw_domain* d);   // nullptr without a partition
void green_release(lbw_domain* d);
}  // namespace lbw
