// sharded.cpp -- one huge transform split along the contraction axis over G GPUs
// (BASELINE.json configs[4]; SURVEY.md §8(b),(e)), with the collective inside the library.
//
//   rank g:  K1 on its column slice -> partial slab (p x r complex128)     pft_execute_partial
//            ncclReduce(slab, sum, root) over NVLink / NVSwitch            (this file)
//   root:    K2: remaining FFT pass + Eq. (7) on the reduced slab          pft_finalize
//
// All three steps are enqueued on the caller's stream (graph-capturable; NCCL supports stream
// capture), so a step is one asynchronous call per rank.  Both K1 and K2 are linear in the
// slab, so the sum over ranks of the partial slabs is the unsharded slab: results equal the
// single-GPU transform up to the order of the NCCL sum ("internal parallelism must
// not change results" -- here within 1e-16 relative; deterministic for a fixed G).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", the copy already in the process if
// there is one, e.g. PyTorch's), so the library still loads on a host without NCCL and the
// communicator a caller created with its own NCCL is driven by that same NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "api_guard.hpp"
#include "internal.hpp"

using namespace pft::detail;

namespace {

struct NcclApi {
    void* handle = nullptr;
    std::string error;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
    decltype(&ncclCommCuDevice) CommCuDevice = nullptr;
    decltype(&ncclReduce) Reduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            api.handle = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. torch's)
            if (api.handle) break;
        }
        if (!api.handle)
            for (const char* n : names) {
                api.handle = dlopen(n, RTLD_NOW | RTLD_LOCAL);
                if (api.handle) break;
            }
        if (!api.handle) {
            api.error = "NCCL (libnccl.so.2) not found";
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.handle, name));
            if (!fn) ok = false;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.CommCuDevice, "ncclCommCuDevice");
        sym(api.Reduce, "ncclReduce");
        sym(api.GetErrorString, "ncclGetErrorString");
        if (!ok) api.error = "NCCL library lacks a required entry point";
    });
    if (!api.error.empty()) fail(PFT_ERR_UNSUPPORTED, api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(PFT_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

void st_check(pft_status s) {
    if (s != PFT_OK) fail(s, pft_last_error());
}

}  // namespace

static_assert(PFT_NCCL_UNIQUE_ID_BYTES == NCCL_UNIQUE_ID_BYTES, "NCCL unique id size");

extern "C" {

pft_status pft_nccl_available(int* available) {
    PFT_API_BEGIN
    PFT_REQUIRE(available != nullptr, "available is null");
    try {
        nccl();
        *available = 1;
    } catch (const Error&) {
        *available = 0;
    }
    PFT_API_END
}

pft_status pft_nccl_get_unique_id(unsigned char* id) {
    PFT_API_BEGIN
    PFT_REQUIRE(id != nullptr, "id is null");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    PFT_API_END
}

pft_status pft_nccl_comm_init(int world, int rank, const unsigned char* id, int device, struct ncclComm** comm) {
    PFT_API_BEGIN
    PFT_REQUIRE(id != nullptr && comm != nullptr, "nccl_comm_init: bad arguments");
    PFT_REQUIRE(world >= 1 && rank >= 0 && rank < world, "nccl_comm_init: rank out of [0, world)");
    const NcclApi& api = nccl();
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        fail(PFT_ERR_NO_DEVICE, "nccl_comm_init: cannot select device " + std::to_string(device));
    }
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    const ncclResult_t r = api.CommInitRank(&c, world, u, rank);
    if (prev >= 0) cudaSetDevice(prev);
    nccl_check(r, "ncclCommInitRank");
    *comm = c;
    PFT_API_END
}

pft_status pft_nccl_comm_destroy(struct ncclComm* comm) {
    PFT_API_BEGIN
    if (comm) nccl_check(nccl().CommDestroy(comm), "ncclCommDestroy");
    PFT_API_END
}

pft_status pft_execute_sharded(pft_dplan_t d, const pft_c128* d_in_local, uint64_t row_stride, struct ncclComm* comm,
                               int root, pft_c128* d_slab, pft_c128* d_out, void* stream) {
    PFT_API_BEGIN
    PFT_REQUIRE(d != nullptr && d_in_local != nullptr && d_slab != nullptr && comm != nullptr,
                "execute_sharded: bad arguments");
    const NcclApi& api = nccl();
    int world = 0, rank = 0, cudev = -1;
    nccl_check(api.CommCount(comm, &world), "ncclCommCount");
    nccl_check(api.CommUserRank(comm, &rank), "ncclCommUserRank");
    nccl_check(api.CommCuDevice(comm, &cudev), "ncclCommCuDevice");
    PFT_REQUIRE(root >= 0 && root < world, "execute_sharded: root out of [0, world)");
    PFT_REQUIRE(rank != root || d_out != nullptr, "execute_sharded: the root needs d_out");
    int ddev = -1;
    st_check(pft_dplan_device(d, &ddev));
    PFT_REQUIRE(ddev == cudev, "execute_sharded: the device plan and the communicator are on different devices");
    size_t slab_bytes = 0;
    st_check(pft_partial_bytes(d, 1, &slab_bytes));
    // K1 on this rank's column slice -> partial slab
    st_check(pft_execute_partial(d, d_in_local, world, rank, row_stride, d_slab, stream));
    // sum of the partial slabs onto the root, in place (2 p r doubles)
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(cudev);
    const ncclResult_t r = api.Reduce(d_slab, d_slab, slab_bytes / sizeof(double), ncclDouble, ncclSum, root, comm,
                                      static_cast<cudaStream_t>(stream));
    if (prev >= 0) cudaSetDevice(prev);
    nccl_check(r, "ncclReduce");
    // the remaining FFT pass + Eq. (7) on the root
    if (rank == root) st_check(pft_finalize(d, d_slab, 1, d_out, stream));
    PFT_API_END
}

}  // extern "C"
