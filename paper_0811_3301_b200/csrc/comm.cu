// comm.cu -- the database-sharded search's threshold exchange inside the library (SURVEY 8(b)
// "nccl_comm", 8(e)): an NCCL communicator created through dtwlb_get_unique_id /
// dtwlb_comm_init and, when nn_opts.nccl_comm is set, ONE ncclAllReduce(MIN) of the query
// block's thresholds, stream-ordered on the call's stream, at each exchange point -- no host
// callback, no Python in the loop.  NCCL is loaded at run time (dlopen of libnccl.so.2: the one
// the process already has, e.g. torch's) so the library itself does not depend on it.
#include <dlfcn.h>

#include <cstring>

#include "kernels.cuh"

namespace dtwlb {

namespace {

// the few NCCL entry points used (C ABI of nccl.h; ncclUniqueId is 128 bytes)
typedef struct { char internal[128]; } UniqueId;
typedef void *Comm;
enum { kNcclFloat32 = 7, kNcclMin = 3 };  // ncclFloat32, ncclMin (nccl.h enum values)
using GetUniqueIdFn = int (*)(UniqueId *);
using CommInitRankFn = int (*)(Comm *, int, UniqueId, int);
using AllReduceFn = int (*)(const void *, void *, size_t, int, int, Comm, cudaStream_t);
using CommDestroyFn = int (*)(Comm);
using GetErrorStringFn = const char *(*)(int);

struct Nccl {
    bool ok = false;
    GetUniqueIdFn get_unique_id = nullptr;
    CommInitRankFn comm_init_rank = nullptr;
    AllReduceFn all_reduce = nullptr;
    CommDestroyFn comm_destroy = nullptr;
    GetErrorStringFn error_string = nullptr;
};

const Nccl &nccl() {
    static Nccl n = [] {
        Nccl r;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.get_unique_id = reinterpret_cast<GetUniqueIdFn>(dlsym(h, "ncclGetUniqueId"));
        r.comm_init_rank = reinterpret_cast<CommInitRankFn>(dlsym(h, "ncclCommInitRank"));
        r.all_reduce = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
        r.comm_destroy = reinterpret_cast<CommDestroyFn>(dlsym(h, "ncclCommDestroy"));
        r.error_string = reinterpret_cast<GetErrorStringFn>(dlsym(h, "ncclGetErrorString"));
        r.ok = r.get_unique_id && r.comm_init_rank && r.all_reduce && r.comm_destroy;
        return r;
    }();
    return n;
}

int nccl_fail(int rc, const char *what) {
    const Nccl &n = nccl();
    set_error(DTWLB_ENCCL, "%s: NCCL error %d (%s)", what, rc, n.error_string ? n.error_string(rc) : "?");
    return DTWLB_ENCCL;
}

int nccl_missing(const char *what) {
    set_error(DTWLB_ENCCL, "%s: NCCL (libnccl.so.2) not loadable", what);
    return DTWLB_ENCCL;
}

}  // namespace

// all-reduce MIN of count floats in place (device pointer), stream-ordered (search.cu)
int comm_allreduce_min(void *comm, float *thr, int64_t count, cudaStream_t st) {
    const Nccl &n = nccl();
    if (!n.ok) return nccl_missing("threshold exchange");
    const int rc = n.all_reduce(thr, thr, (size_t)count, kNcclFloat32, kNcclMin, comm, st);
    if (rc != 0) return nccl_fail(rc, "threshold exchange (ncclAllReduce)");
    return DTWLB_OK;
}

}  // namespace dtwlb

extern "C" {

int dtwlb_get_unique_id(void *out128) {
    using namespace dtwlb;
    if (!out128) {
        set_error(DTWLB_EINVAL, "dtwlb_get_unique_id: NULL output");
        return DTWLB_EINVAL;
    }
    const Nccl &n = nccl();
    if (!n.ok) return nccl_missing("dtwlb_get_unique_id");
    UniqueId id;
    const int rc = n.get_unique_id(&id);
    if (rc != 0) return nccl_fail(rc, "dtwlb_get_unique_id");
    std::memcpy(out128, &id, sizeof(id));
    return DTWLB_OK;
}

int dtwlb_comm_init(const void *id128, int32_t nranks, int32_t rank, void **comm) {
    using namespace dtwlb;
    if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error(DTWLB_EINVAL, "dtwlb_comm_init: bad arguments (nranks %d, rank %d)", nranks, rank);
        return DTWLB_EINVAL;
    }
    *comm = nullptr;
    const int dev_rc = require_device();
    if (dev_rc != DTWLB_OK) return dev_rc;
    const Nccl &n = nccl();
    if (!n.ok) return nccl_missing("dtwlb_comm_init");
    UniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    Comm c = nullptr;
    const int rc = n.comm_init_rank(&c, nranks, id, rank);
    if (rc != 0) return nccl_fail(rc, "dtwlb_comm_init (ncclCommInitRank)");
    *comm = c;
    return DTWLB_OK;
}

int dtwlb_comm_destroy(void *comm) {
    using namespace dtwlb;
    if (!comm) return DTWLB_OK;
    const Nccl &n = nccl();
    if (!n.ok) return nccl_missing("dtwlb_comm_destroy");
    const int rc = n.comm_destroy(comm);
    if (rc != 0) return nccl_fail(rc, "dtwlb_comm_destroy");
    return DTWLB_OK;
}

}  // extern "C"
