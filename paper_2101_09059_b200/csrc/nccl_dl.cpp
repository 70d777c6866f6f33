// nccl_dl.cpp -- see nccl_dl.hpp.
#include "nccl_dl.hpp"

#include <dlfcn.h>

namespace ens {

const Nccl* nccl_load(std::string* err) {
    static Nccl nccl;
    static bool tried = false;
    static std::string why;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's in-process copy
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            why = std::string("libnccl.so.2 not found: ") + dlerror();
        } else {
            nccl.send = reinterpret_cast<decltype(nccl.send)>(dlsym(h, "ncclSend"));
            nccl.recv = reinterpret_cast<decltype(nccl.recv)>(dlsym(h, "ncclRecv"));
            nccl.group_start = reinterpret_cast<decltype(nccl.group_start)>(dlsym(h, "ncclGroupStart"));
            nccl.group_end = reinterpret_cast<decltype(nccl.group_end)>(dlsym(h, "ncclGroupEnd"));
            nccl.error_string = reinterpret_cast<decltype(nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
            nccl.comm_count = reinterpret_cast<decltype(nccl.comm_count)>(dlsym(h, "ncclCommCount"));
            nccl.comm_user_rank = reinterpret_cast<decltype(nccl.comm_user_rank)>(dlsym(h, "ncclCommUserRank"));
            if (!nccl.ok()) why = "libnccl.so.2 lacks ncclSend/ncclRecv/ncclGroupStart/ncclGroupEnd";
        }
    }
    if (!nccl.ok()) {
        if (err) *err = why;
        return nullptr;
    }
    return &nccl;
}

}  // namespace ens
