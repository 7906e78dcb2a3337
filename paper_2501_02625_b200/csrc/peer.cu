// peer.cu — HQ-FSDP over NVLink peer memory, sm_100a.
//
// The reference gathers every rank's quantized weight rows into a full
// (WH)_Q before each GEMM (quantized_all_gather / backward_regather,
// hqfsdp.hpp:204-266) after an all-reduce of the per-rank absmax
// (hqfsdp.hpp:172-196).  Here the rows never move: each rank quantizes its
// shard into a buffer exported by CUDA IPC, and the GEMMs' TMA reads the
// peers' shards in place over NVLink (halo_linear_set_qweight_sharded).  What
// is left of the collectives is this file: a mailbox per rank, one kernel
// that posts the local absmax into every peer's mailbox, raises the caller's
// flag there (release, system scope) and spins on its own mailbox until all
// ranks have posted the same epoch (acquire) -- the scale all-reduce and the
// "shards written" / "shards no longer read" barriers, stream-ordered, with
// no host round trip.
//
// Mailbox layout (u32): [0, world) flags, [world, 3 world) absmax words in
// two banks by epoch parity.  A rank can run at most one epoch ahead of a
// peer's read of its box (posting epoch e + 2 needs that peer's e + 1 flag,
// raised only after its epoch-e kernel has read the box), so two banks keep
// a fast rank from overwriting a value a slow one has not read yet.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/halo_b200.h"
#include "common.cuh"
#include "halo_internal.h"

#include <cstring>

namespace halo_b200 {

struct PeerBoxes {
    unsigned* box[HALO_PEER_MAX];
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_peer_sync(PeerBoxes boxes, int world, int rank, unsigned epoch, const float* amax_in,
                            float* amax_out) {
    const int j = threadIdx.x;
    if (j < world) {
        unsigned* peer = boxes.box[j];
        const int bank = world + (int)(epoch & 1u) * world;
        if (amax_in) peer[bank + rank] = __float_as_uint(fabsf(*amax_in));
        st_release_sys(peer + rank, epoch);  // orders the absmax word before the flag
        const unsigned* mine = boxes.box[rank];
        // flags grow monotonically; (int) difference tolerates wrap-around
        while ((int)(ld_acquire_sys(mine + j) - epoch) < 0) __nanosleep(64);
    }
    __syncwarp();
    if (amax_out && j == 0) {
        const unsigned* mine = boxes.box[rank];
        unsigned m = 0;
        const int bank = world + (int)(epoch & 1u) * world;
        for (int i = 0; i < world; ++i) {
            const unsigned v = ld_acquire_sys(mine + bank + i);
            m = v > m ? v : m;  // non-negative floats order like their bits
        }
        *amax_out = __uint_as_float(m);
    }
}

}  // namespace halo_b200

using namespace halo_b200;

namespace {
halo_status peer_fail(const char* msg) {
    set_last_error(msg);
    return HALO_ERR_CUDA;
}
}  // namespace

extern "C" halo_status halo_peer_alloc(int64_t bytes, void** ptr) {
    if (!ptr || bytes <= 0) return HALO_ERR_INVALID_ARGUMENT;
    *ptr = nullptr;
    if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return peer_fail("peer_alloc: cudaMalloc failed");
    if (cudaMemset(*ptr, 0, (size_t)bytes) != cudaSuccess) return peer_fail("peer_alloc: cudaMemset failed");
    return HALO_OK;
}

extern "C" halo_status halo_peer_free(void* ptr) {
    if (ptr && cudaFree(ptr) != cudaSuccess) return peer_fail("peer_free: cudaFree failed");
    return HALO_OK;
}

extern "C" halo_status halo_ipc_handle(const void* ptr, void* handle) {
    if (!ptr || !handle) return HALO_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)) != cudaSuccess)
        return peer_fail("ipc_handle: cudaIpcGetMemHandle failed (pointer must come from halo_peer_alloc)");
    static_assert(sizeof(h) == HALO_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return HALO_OK;
}

extern "C" halo_status halo_ipc_open(const void* handle, void** ptr) {
    if (!handle || !ptr) return HALO_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    *ptr = nullptr;
    if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return peer_fail("ipc_open: cudaIpcOpenMemHandle failed");
    return HALO_OK;
}

extern "C" halo_status halo_ipc_close(void* ptr) {
    if (ptr && cudaIpcCloseMemHandle(ptr) != cudaSuccess) return peer_fail("ipc_close: cudaIpcCloseMemHandle failed");
    return HALO_OK;
}

extern "C" halo_status halo_peer_sync(void* const* mailboxes, int32_t world, int32_t rank, uint32_t epoch,
                                      const float* amax_in, float* amax_out, halo_stream_t stream) {
    if (!mailboxes || world < 1 || world > HALO_PEER_MAX || rank < 0 || rank >= world || epoch == 0)
        return HALO_ERR_INVALID_ARGUMENT;
    PeerBoxes b{};
    for (int i = 0; i < world; ++i) {
        if (!mailboxes[i]) return HALO_ERR_INVALID_ARGUMENT;
        b.box[i] = static_cast<unsigned*>(mailboxes[i]);
    }
    k_peer_sync<<<1, 32, 0, (cudaStream_t)stream>>>(b, world, rank, epoch, amax_in, amax_out);
    if (cudaGetLastError() != cudaSuccess) return peer_fail("peer_sync: launch failed");
    return HALO_OK;
}
