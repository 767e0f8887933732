// nccl_api.cu -- run-time binding of NCCL (see nccl_api.h).
#include <dlfcn.h>

#include <mutex>

#include "nccl_api.h"

namespace idk {

namespace {

template <class F>
bool bind(void* lib, const char* name, F* slot, std::string* missing) {
    *slot = reinterpret_cast<F>(dlsym(lib, name));
    if (!*slot) *missing += std::string(missing->empty() ? "" : ", ") + name;
    return *slot != nullptr;
}

}  // namespace

const NcclApi* nccl_api(std::string* err) {
    static NcclApi api;
    static std::string load_err;
    static bool ok = false;
    static std::once_flag once;
    std::call_once(once, [] {
        // an already-loaded NCCL first (torch's, or the caller's), then the loader's search path
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            const char* e = dlerror();
            load_err = std::string("libnccl.so.2 not found: ") + (e ? e : "dlopen failed");
            return;
        }
        std::string missing;
        bool all = true;
        all &= bind(lib, "ncclGetUniqueId", &api.GetUniqueId, &missing);
        all &= bind(lib, "ncclCommInitRank", &api.CommInitRank, &missing);
        all &= bind(lib, "ncclCommDestroy", &api.CommDestroy, &missing);
        all &= bind(lib, "ncclCommCount", &api.CommCount, &missing);
        all &= bind(lib, "ncclCommUserRank", &api.CommUserRank, &missing);
        all &= bind(lib, "ncclAllGather", &api.AllGather, &missing);
        all &= bind(lib, "ncclBroadcast", &api.Broadcast, &missing);
        all &= bind(lib, "ncclAllReduce", &api.AllReduce, &missing);
        all &= bind(lib, "ncclGroupStart", &api.GroupStart, &missing);
        all &= bind(lib, "ncclGroupEnd", &api.GroupEnd, &missing);
        all &= bind(lib, "ncclGetErrorString", &api.GetErrorString, &missing);
        all &= bind(lib, "ncclGetVersion", &api.GetVersion, &missing);
        if (!all) {
            load_err = "libnccl.so.2 lacks " + missing;
            return;
        }
        ok = true;
    });
    if (!ok) {
        if (err) *err = load_err;
        return nullptr;
    }
    return &api;
}

}  // namespace idk
