// lbw_peer.cu — x-slab neighbours on other GPUs of the node.
//
// Data path: the sweep kernel stores the nine outgoing direction planes of
// its first / last x plane straight into the neighbour's ghost plane (CUDA
// IPC mapping, NVLink stores from inside K1, see HaloOut in k_sweep); the
// actuator cube values of cells near a slab face are stored into the
// neighbour's cube buffer the same way.
//
// Ordering: monotonically increasing 32-bit counters in each domain's
// memory, written by the neighbours with a stream write (preceded by a
// memory barrier, so the peer stores of the work before it are visible)
// and awaited with a stream wait (GEQ).  Both are executed by the GPU front
// end: no host round trip, no spinning kernel.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "lbw_domain.h"

namespace lbw {
namespace {

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitFn g_wait = nullptr;
WriteFn g_write = nullptr;

int driver_entry_points() {
    if (g_wait && g_write) return LBW_OK;
    cudaDriverEntryPointQueryResult q1, q2;
    void *w = nullptr, *r = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &r, cudaEnableDefault, &q2) != cudaSuccess ||
        !w || !r) {
        cudaGetLastError();
        set_error("driver stream memory operations unavailable");
        return LBW_ECOMM;
    }
    g_wait = (WaitFn)w;
    g_write = (WriteFn)r;
    return LBW_OK;
}

constexpr uint32_t kMagic = 0x4c425750;  // "LBWP"

struct PeerBlob {
    uint32_t magic;
    int32_t rank, nranks, nxl, ny, zp, n_points, has_cube, single;
    int64_t plane_stride;
    cudaIpcMemHandle_t buf[2];
    cudaIpcMemHandle_t cube;
    cudaIpcMemHandle_t flags;
};

}  // namespace

int peer_wait(lbw_domain* d, cudaStream_t s, int which, uint32_t value) {
    if (!d->linked) return LBW_OK;
    for (int side = 0; side < 2; ++side) {
        if (d->nb_rank[side] < 0) continue;
        const CUresult r = g_wait((CUstream)s, (CUdeviceptr)(d->flags + which * 2 + side), value,
                                  CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) {
            set_error("cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
            return LBW_ECOMM;
        }
    }
    return LBW_OK;
}

int stream_write32(cudaStream_t s, uint32_t* ptr, uint32_t value) {
    int rc = driver_entry_points();
    if (rc) return rc;
    const CUresult r = g_write((CUstream)s, (CUdeviceptr)ptr, value, 0);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
        return LBW_ECOMM;
    }
    return LBW_OK;
}

int peer_signal(lbw_domain* d, cudaStream_t s, int which, uint32_t value) {
    if (!d->linked) return LBW_OK;
    for (int side = 0; side < 2; ++side) {
        if (d->nb_rank[side] < 0) continue;
        // I am the hi neighbour of my lo neighbour (its slot 1) and the lo
        // neighbour of my hi neighbour (its slot 0)
        uint32_t* target = d->nb_flags[side] + which * 2 + (1 - side);
        const CUresult r = g_write((CUstream)s, (CUdeviceptr)target, value, 0);
        if (r != CUDA_SUCCESS) {
            set_error("cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
            return LBW_ECOMM;
        }
    }
    return LBW_OK;
}

void peer_close(lbw_domain* d) {
    for (void* p : d->peer_mapped) cudaIpcCloseMemHandle(p);
    d->peer_mapped.clear();
    if (d->flags) cudaFree(d->flags);
    d->flags = nullptr;
    d->edge_counter = nullptr;
    d->linked = false;
}

}  // namespace lbw

using namespace lbw;

extern "C" {

int64_t lbw_peer_blob_bytes(void) { return (int64_t)sizeof(PeerBlob); }

int lbw_domain_export_handle(lbw_domain* d, void* blob, int64_t* blob_bytes) {
    LBW_REQ(d && blob && blob_bytes, "null argument");
    LBW_REQ(*blob_bytes >= (int64_t)sizeof(PeerBlob), "blob buffer too small");
    LBW_CK(cudaSetDevice(d->device));
    int rc = driver_entry_points();
    if (rc) return rc;
    if (!d->flags) {
        if (cudaMalloc(&d->flags, 64) != cudaSuccess) {
            cudaGetLastError();
            set_error("flag allocation failed");
            return LBW_ENOMEM;
        }
        LBW_CK(cudaMemset(d->flags, 0, 64));
        d->bytes += 64;
        d->edge_counter = reinterpret_cast<unsigned long long*>(d->flags + 8);
    }
    PeerBlob b;
    std::memset(&b, 0, sizeof b);
    b.magic = kMagic;
    b.rank = d->desc.rank;
    b.nranks = d->desc.nranks;
    b.nxl = d->g.nxl;
    b.ny = d->g.ny;
    b.zp = d->g.zp;
    b.plane_stride = d->g.plane_stride;
    b.single = d->g.single;
    for (int k = 0; k < 2; ++k) LBW_CK(cudaIpcGetMemHandle(&b.buf[k], d->buf[k]));
    LBW_CK(cudaIpcGetMemHandle(&b.flags, d->flags));
    double* cube = alm_cube(d);
    b.has_cube = cube ? 1 : 0;
    b.n_points = alm_active(d) ? -1 : 0;
    if (cube) LBW_CK(cudaIpcGetMemHandle(&b.cube, cube));
    std::memcpy(blob, &b, sizeof b);
    *blob_bytes = (int64_t)sizeof b;
    return LBW_OK;
}

int lbw_domain_import_peers(lbw_domain* d, const void* lo_blob, const void* hi_blob) {
    LBW_REQ(d, "null domain");
    LBW_REQ(d->flags, "export this domain's handle before importing its peers");
    // a point's sampling cube and spreading support reach halo (+1) x cells:
    // with slabs that wide they never reach beyond the immediate neighbours
    LBW_REQ(!alm_active(d) || d->g.nxl >= std::max(3, alm_support_halo(d) + 2),
            "actuator runs need slabs of >= 3 x planes (support half-width + 2 with a "
            "Gaussian spreading kernel)");
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    const void* blobs[2] = {lo_blob, hi_blob};
    PeerBlob pb[2];
    int open_rank[2] = {-1, -1};
    void* open_ptr[2][4] = {};
    for (int side = 0; side < 2; ++side) {
        d->nb_rank[side] = -1;
        if (!blobs[side]) continue;
        std::memcpy(&pb[side], blobs[side], sizeof(PeerBlob));
        const PeerBlob& b = pb[side];
        LBW_REQ(b.magic == kMagic, "bad peer handle blob");
        LBW_REQ(b.ny == d->g.ny && b.zp == d->g.zp && b.plane_stride == d->g.plane_stride &&
                    b.single == d->g.single,
                "neighbour slab has a different y/z layout or storage precision");
        LBW_REQ(b.rank != d->desc.rank, "a slab cannot be its own neighbour");
        LBW_REQ((b.has_cube != 0) == (alm_cube(d) != nullptr),
                "neighbours disagree about actuator points");
        void* ptrs[4] = {};
        if (side == 1 && open_rank[0] == b.rank) {
            for (int k = 0; k < 4; ++k) ptrs[k] = open_ptr[0][k];
        } else {
            const cudaIpcMemHandle_t* hs[4] = {&b.buf[0], &b.buf[1], &b.flags, &b.cube};
            for (int k = 0; k < 4; ++k) {
                if (k == 3 && !b.has_cube) continue;
                LBW_CK(cudaIpcOpenMemHandle(&ptrs[k], *hs[k], cudaIpcMemLazyEnablePeerAccess));
                d->peer_mapped.push_back(ptrs[k]);
            }
            open_rank[side] = b.rank;
            for (int k = 0; k < 4; ++k) open_ptr[side][k] = ptrs[k];
        }
        d->nb_rank[side] = b.rank;
        d->nb_nxl[side] = b.nxl;
        d->nb_buf[side][0] = ptrs[0];
        d->nb_buf[side][1] = ptrs[1];
        d->nb_flags[side] = (uint32_t*)ptrs[2];
        d->nb_cube[side] = (double*)ptrs[3];
    }
    // edge planes go straight into the neighbours' ghost planes
    const int64_t eb = (int64_t)elem_bytes(d->g);
    for (int k = 0; k < 2; ++k) {
        d->halo[k].lo = d->nb_rank[0] >= 0
                            ? (char*)d->nb_buf[0][k] +
                                  (int64_t)(d->nb_nxl[0] + 1) * d->g.plane_stride * eb
                            : nullptr;
        d->halo[k].hi = d->nb_rank[1] >= 0
                            ? (char*)d->nb_buf[1][k] + 18 * d->g.dir_stride * eb
                            : nullptr;
    }
    LBW_REQ((d->g.lo_src == XS_GHOST) == (d->nb_rank[0] >= 0) &&
                (d->g.hi_src == XS_GHOST) == (d->nb_rank[1] >= 0),
            "neighbour set does not match the slab's x faces");
    d->linked = true;
    return LBW_OK;
}

}  // extern "C"
