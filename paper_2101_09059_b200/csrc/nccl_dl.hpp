// nccl_dl.hpp -- NCCL point-to-point entry points resolved at run time.
//
// The halo exchange must run on the communicator torch's ProcessGroupNCCL created
// (ProcessGroupNCCL._comm_ptr()), i.e. on the libnccl.so.2 torch already loaded (2.28,
// site-packages/nvidia/nccl), not the older system copy.  dlopen(RTLD_NOLOAD) finds that
// in-process copy; the library therefore has no link-time NCCL dependency and loads on
// machines without NCCL (CPU tests).
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime_api.h>

namespace ens {

struct Nccl {
    using Comm = void*;
    enum { kSuccess = 0, kDouble = 8 };   // ncclSuccess, ncclFloat64 (nccl.h 2.28)
    int (*send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    const char* (*error_string)(int) = nullptr;
    int (*comm_count)(Comm, int*) = nullptr;       // ncclCommCount
    int (*comm_user_rank)(Comm, int*) = nullptr;   // ncclCommUserRank
    bool ok() const { return send && recv && group_start && group_end; }
};

// Resolve the entry points once; returns nullptr (and sets *err) if libnccl.so.2 is absent.
const Nccl* nccl_load(std::string* err);

}  // namespace ens
