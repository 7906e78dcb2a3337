// hqfsdp_nccl.cpp — the HQ-FSDP weight protocol's data plane in C++ over
// NCCL (hqfsdp.hpp:172-300), one communicator per rank, everything
// stream-ordered (no host synchronisation):
//
//   quantized_all_gather (:204-237)  K1 phase A on the local shard (absmax of
//       the rotated rows) -> ncclAllReduce(max) of that one float -> K1 phase
//       B under compute_scales(max) (the kernel derives the scale,
//       quantize.hpp:234) straight into this rank's slice of the gathered
//       buffer -> ncclAllGather in place.  The codes equal a single-process
//       quantize of the rotated padded weight bit for bit (per-tensor scale).
//   backward_regather (:243-266)     the same codes under the SAVED scale (no
//       scale traffic); optional stale check on the device: the shard's
//       current absmax vs the one saved at the forward gather, OR-ed into a
//       flag word the caller tests once (:256-259).
//   reduce_scatter_grads (:271-300)  ncclReduceScatter(sum) of the full dW,
//       then * 1/world (NCCL's reduction order replaces the reference's
//       rank-order double sum: tolerance parity).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process that is torch's already-loaded NCCL, in a plain C++ process the
// system library; libhalo_b200.so itself links no NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../../include/halo_b200.h"

namespace halo_b200 {
void set_last_error(const char* msg);
void run_flag_neq(const float* a, const float* b, unsigned* flag, cudaStream_t st);
void run_scale_mul(void* buf, int dtype, int64_t n, float k, cudaStream_t st);
void run_fp6_pack(const uint8_t* codes, uint8_t* packed, int64_t n, cudaStream_t st);
void run_fp6_unpack(const uint8_t* packed, uint8_t* codes, int64_t n, cudaStream_t st);
}

namespace {

struct Nccl {
    void* h = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclReduceScatter) reduceScatter = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    decltype(&ncclGetVersion) getVersion = nullptr;
};

Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
        n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
        n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
        n.reduceScatter = (decltype(n.reduceScatter))dlsym(h, "ncclReduceScatter");
        n.errorString = (decltype(n.errorString))dlsym(h, "ncclGetErrorString");
        n.getVersion = (decltype(n.getVersion))dlsym(h, "ncclGetVersion");
        if (n.getUniqueId && n.commInitRank && n.commDestroy && n.allReduce && n.allGather && n.reduceScatter &&
            n.errorString)
            n.h = h;
    });
    return n.h ? &n : nullptr;
}

halo_status nfail(const std::string& m) {
    halo_b200::set_last_error(m.c_str());
    return HALO_ERR_NCCL;
}
halo_status afail(const std::string& m) {
    halo_b200::set_last_error(m.c_str());
    return HALO_ERR_INVALID_ARGUMENT;
}
halo_status ncheck(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return HALO_OK;
    Nccl* n = nccl();
    return nfail(std::string(what) + ": " + (n ? n->errorString(r) : "nccl"));
}

}  // namespace

struct halo_fsdp {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
    float* amax = nullptr;  // device: [0] local absmax, [1] reduced max
    uint8_t* wire = nullptr;  // FP6: packed gather buffer (grow-only)
    size_t wire_bytes = 0;
};

extern "C" halo_status halo_fsdp_get_unique_id(void* id) {
    Nccl* n = nccl();
    if (!n) return nfail("hqfsdp: libnccl.so.2 could not be loaded");
    if (!id) return afail("hqfsdp: null id");
    ncclUniqueId u;
    const halo_status s = ncheck(n->getUniqueId(&u), "ncclGetUniqueId");
    if (s == HALO_OK) std::memcpy(id, &u, sizeof(u));
    return s;
}

extern "C" halo_status halo_fsdp_create(const void* id, int32_t world, int32_t rank, halo_fsdp** out) {
    Nccl* n = nccl();
    if (!n) return nfail("hqfsdp: libnccl.so.2 could not be loaded");
    if (!id || !out || world < 1 || rank < 0 || rank >= world) return afail("hqfsdp: bad world / rank");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto* f = new halo_fsdp;
    f->world = world;
    f->rank = rank;
    halo_status s = ncheck(n->commInitRank(&f->comm, world, u, rank), "ncclCommInitRank");
    if (s == HALO_OK && cudaMalloc(&f->amax, 2 * sizeof(float)) != cudaSuccess) {
        halo_b200::set_last_error("hqfsdp: cudaMalloc failed");
        s = HALO_ERR_CUDA;
    }
    if (s != HALO_OK) {
        if (f->comm) n->commDestroy(f->comm);
        delete f;
        return s;
    }
    *out = f;
    return HALO_OK;
}

extern "C" halo_status halo_fsdp_destroy(halo_fsdp* f) {
    if (!f) return HALO_OK;
    Nccl* n = nccl();
    if (f->comm && n) n->commDestroy(f->comm);
    if (f->amax) cudaFree(f->amax);
    if (f->wire) cudaFree(f->wire);
    delete f;
    return HALO_OK;
}

extern "C" halo_status halo_fsdp_world(const halo_fsdp* f, int32_t* world, int32_t* rank) {
    if (!f) return afail("hqfsdp: null handle");
    if (world) *world = f->world;
    if (rank) *rank = f->rank;
    return HALO_OK;
}

static halo_status gather_codes(halo_fsdp* f, uint8_t* gathered, int64_t shard_bytes, int32_t format,
                                cudaStream_t st) {
    if (f->world == 1) return HALO_OK;
    if (format == HALO_FMT_FP6_E3M2 && shard_bytes % 4 == 0) {
        // the FP6 wire format: 3 bytes per 4 codes on the wire (hqfsdp.hpp:41-43)
        const int64_t pk = shard_bytes / 4 * 3;
        const size_t need = (size_t)pk * (size_t)f->world;
        if (f->wire_bytes < need) {
            if (f->wire) cudaFree(f->wire);
            f->wire = nullptr;
            f->wire_bytes = 0;
            if (cudaMalloc(&f->wire, need) != cudaSuccess) {
                halo_b200::set_last_error("hqfsdp: cudaMalloc failed");
                return HALO_ERR_CUDA;
            }
            f->wire_bytes = need;
        }
        halo_b200::run_fp6_pack(gathered + (int64_t)f->rank * shard_bytes, f->wire + (int64_t)f->rank * pk,
                                shard_bytes, st);
        const halo_status s = ncheck(nccl()->allGather(f->wire + (int64_t)f->rank * pk, f->wire, (size_t)pk,
                                                       ncclUint8, f->comm, st),
                                     "ncclAllGather (fp6 wire)");
        if (s != HALO_OK) return s;
        halo_b200::run_fp6_unpack(f->wire, gathered, shard_bytes * f->world, st);
        return HALO_OK;
    }
    // in place: this rank's slice already holds its codes
    return ncheck(nccl()->allGather(gathered + (int64_t)f->rank * shard_bytes, gathered, (size_t)shard_bytes,
                                    ncclUint8, f->comm, st),
                  "ncclAllGather (codes)");
}

extern "C" halo_status halo_fsdp_quantized_all_gather(halo_fsdp* f, const void* shard, int32_t dtype,
                                                      int64_t shard_rows, int64_t cols, int64_t had_block,
                                                      int32_t format, uint8_t* gathered, float* scale_out,
                                                      float* local_absmax_out, halo_stream_t stream) {
    if (!f || !shard || !gathered || !scale_out) return afail("hqfsdp: null argument");
    if (shard_rows <= 0 || cols <= 0) return afail("hqfsdp: empty shard");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t shard_bytes = shard_rows * cols;
    // hqfsdp.hpp:216-225 -- the per-rank absmax of the rotated shard
    halo_status s = halo_rotate_absmax(shard, dtype, shard_rows, cols, had_block, &f->amax[0], stream);
    if (s != HALO_OK) return s;
    if (local_absmax_out && cudaMemcpyAsync(local_absmax_out, &f->amax[0], 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return afail("hqfsdp: absmax copy failed");
    // :172-196 -- the max over ranks (order-insensitive), then the shared scale
    if (f->world > 1) {
        s = ncheck(nccl()->allReduce(&f->amax[0], &f->amax[1], 1, ncclFloat32, ncclMax, f->comm, st),
                   "ncclAllReduce (absmax)");
        if (s != HALO_OK) return s;
    } else if (cudaMemcpyAsync(&f->amax[1], &f->amax[0], 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
        return afail("hqfsdp: absmax copy failed");
    }
    s = halo_rotate_quantize_amax(shard, dtype, shard_rows, cols, had_block, format, &f->amax[1],
                                  gathered + (int64_t)f->rank * shard_bytes, scale_out, stream);
    if (s != HALO_OK) return s;
    return gather_codes(f, gathered, shard_bytes, format, st);
}

extern "C" halo_status halo_fsdp_backward_regather(halo_fsdp* f, const void* shard, int32_t dtype,
                                                   int64_t shard_rows, int64_t cols, int64_t had_block,
                                                   int32_t format, const float* scale,
                                                   const float* saved_local_absmax, uint32_t* stale_flag,
                                                   uint8_t* gathered, halo_stream_t stream) {
    if (!f || !shard || !gathered || !scale) return afail("hqfsdp: null argument (no saved forward scale)");
    if (shard_rows <= 0 || cols <= 0) return afail("hqfsdp: empty shard");
    cudaStream_t st = (cudaStream_t)stream;
    if (saved_local_absmax && stale_flag) {
        const halo_status s = halo_rotate_absmax(shard, dtype, shard_rows, cols, had_block, &f->amax[0], stream);
        if (s != HALO_OK) return s;
        halo_b200::run_flag_neq(&f->amax[0], saved_local_absmax, stale_flag, st);
    }
    const int64_t shard_bytes = shard_rows * cols;
    const halo_status s = halo_rotate_quantize(shard, dtype, shard_rows, cols, had_block, format, scale,
                                               gathered + (int64_t)f->rank * shard_bytes, nullptr, stream);
    if (s != HALO_OK) return s;
    return gather_codes(f, gathered, shard_bytes, format, st);
}

extern "C" halo_status halo_fsdp_reduce_scatter(halo_fsdp* f, const void* grad, int32_t dtype, int64_t shard_rows,
                                                int64_t cols, void* shard_out, halo_stream_t stream) {
    if (!f || !grad || !shard_out) return afail("hqfsdp: null argument");
    if (dtype != HALO_DTYPE_F32 && dtype != HALO_DTYPE_BF16) return afail("hqfsdp: gradient dtype f32 / bf16");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = shard_rows * cols;
    const ncclDataType_t t = dtype == HALO_DTYPE_F32 ? ncclFloat32 : ncclBfloat16;
    if (f->world == 1) {
        if (grad != shard_out &&
            cudaMemcpyAsync(shard_out, grad, (size_t)n * (dtype == HALO_DTYPE_F32 ? 4 : 2), cudaMemcpyDeviceToDevice,
                            st) != cudaSuccess)
            return afail("hqfsdp: copy failed");
        return HALO_OK;
    }
    const halo_status s = ncheck(nccl()->reduceScatter(grad, shard_out, (size_t)n, t, ncclSum, f->comm, st),
                                 "ncclReduceScatter (dW)");
    if (s != HALO_OK) return s;
    halo_b200::run_scale_mul(shard_out, dtype, n, 1.0f / (float)f->world, st);  // the mean, :288-292
    return HALO_OK;
}

extern "C" halo_status halo_fsdp_all_reduce_mean(halo_fsdp* f, void* buf, int32_t dtype, int64_t n,
                                                 halo_stream_t stream) {
    if (!f || !buf) return afail("hqfsdp: null argument");
    if (dtype != HALO_DTYPE_F32 && dtype != HALO_DTYPE_BF16) return afail("hqfsdp: dtype f32 / bf16");
    if (f->world == 1) return HALO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const ncclDataType_t t = dtype == HALO_DTYPE_F32 ? ncclFloat32 : ncclBfloat16;
    const halo_status s = ncheck(nccl()->allReduce(buf, buf, (size_t)n, t, ncclSum, f->comm, st), "ncclAllReduce");
    if (s != HALO_OK) return s;
    halo_b200::run_scale_mul(buf, dtype, n, 1.0f / (float)f->world, st);
    return HALO_OK;
}
