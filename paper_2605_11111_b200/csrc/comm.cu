// Communicators and the exchange patterns of the domain-parallel path over
// NCCL (NVLink 5 / NVSwitch inside a B200 node): the C-ABI data plane behind
// mesh.py's NativeTransport, replacing domainpar/mesh.py:252-403 (per-pair
// queues + np.concatenate).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 — normally the copy
// torch already loaded), so the library loads and every compute entry point
// works on hosts without NCCL; the dp_comm_* calls then return
// DP_ERR_UNSUPPORTED.  Every exchange is ONE ncclGroupStart/End of
// ncclSend/ncclRecv enqueued on the caller's stream (byte payloads: the
// wire format is the buffer's memory order).  Errors never throw: NCCL
// codes map to DP_ERR_COMM with ncclGetErrorString / ncclGetLastError in
// dp_last_error(), and dp_comm_wait() is the watchdog — it polls the stream
// and ncclCommGetAsyncError, aborts the communicator on an async error or a
// timeout, and reports DP_ERR_COMM / DP_ERR_TIMEOUT.
#include <dlfcn.h>
#include <nccl.h>
#include <time.h>

#include "common.cuh"

namespace dp {
namespace {

struct NcclApi {
    void *lib = nullptr;
    ncclResult_t (*GetVersion)(int *);
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommAbort)(ncclComm_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    const char *(*GetErrorString)(ncclResult_t);
    const char *(*GetLastError)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t);
};

NcclApi g_nccl;

template <typename F>
bool sym(void *lib, const char *name, F &out) {
    out = reinterpret_cast<F>(dlsym(lib, name));
    return out != nullptr;
}

int load_nccl(const char *path) {
    if (g_nccl.lib) return DP_OK;
    void *lib = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    DP_REQUIRE(lib, DP_ERR_UNSUPPORTED, "dp_comm: cannot load NCCL (%s): %s",
               path && path[0] ? path : "libnccl.so.2", dlerror());
    NcclApi a;
    a.lib = lib;
    bool ok = sym(lib, "ncclGetVersion", a.GetVersion) && sym(lib, "ncclGetUniqueId", a.GetUniqueId) &&
              sym(lib, "ncclCommInitRank", a.CommInitRank) && sym(lib, "ncclCommSplit", a.CommSplit) &&
              sym(lib, "ncclCommDestroy", a.CommDestroy) && sym(lib, "ncclCommAbort", a.CommAbort) &&
              sym(lib, "ncclCommGetAsyncError", a.CommGetAsyncError) &&
              sym(lib, "ncclGetErrorString", a.GetErrorString) &&
              sym(lib, "ncclGetLastError", a.GetLastError) && sym(lib, "ncclGroupStart", a.GroupStart) &&
              sym(lib, "ncclGroupEnd", a.GroupEnd) && sym(lib, "ncclSend", a.Send) &&
              sym(lib, "ncclRecv", a.Recv) && sym(lib, "ncclAllReduce", a.AllReduce);
    DP_REQUIRE(ok, DP_ERR_UNSUPPORTED, "dp_comm: NCCL at %s lacks a required symbol (need >= 2.18)",
               path ? path : "libnccl.so.2");
    g_nccl = a;
    return DP_OK;
}

struct Comm {
    ncclComm_t nc;
    int rank, size;
};

int nccl_err(ncclResult_t r, const char *what, ncclComm_t c) {
    const char *last = (c && g_nccl.GetLastError) ? g_nccl.GetLastError(c) : "";
    set_error("%s: NCCL error %d (%s) %s", what, (int)r, g_nccl.GetErrorString(r), last ? last : "");
    return DP_ERR_COMM;
}

#define DP_NCCL(expr, what, comm)                            \
    do {                                                     \
        ncclResult_t _r = (expr);                            \
        if (_r != ncclSuccess) return nccl_err(_r, what, comm); \
    } while (0)

#define DP_NEED_COMM(c)                                                                \
    do {                                                                               \
        DP_REQUIRE(g_nccl.lib, DP_ERR_UNSUPPORTED, "dp_comm: NCCL not loaded");        \
        DP_REQUIRE((c) != nullptr, DP_ERR_INVALID, "dp_comm: null communicator");      \
        DP_REQUIRE((c)->nc != nullptr, DP_ERR_COMM, "dp_comm: communicator was aborted"); \
    } while (0)

// One grouped exchange: ops[i] = (peer, is_recv, buf, bytes); zero-byte ops
// are dropped (NCCL would accept them, but they still cost a handshake).
int grouped(Comm *c, int n, const int *peer, const int *is_recv, void *const *buf,
            const int64_t *bytes, cudaStream_t st, const char *what) {
    for (int i = 0; i < n; ++i) {
        DP_REQUIRE(peer[i] >= 0 && peer[i] < c->size, DP_ERR_INVALID, "%s: peer %d outside [0, %d)",
                   what, peer[i], c->size);
        DP_REQUIRE(bytes[i] >= 0, DP_ERR_INVALID, "%s: negative byte count", what);
        DP_REQUIRE(bytes[i] == 0 || buf[i], DP_ERR_INVALID, "%s: null buffer", what);
    }
    DP_NCCL(g_nccl.GroupStart(), what, c->nc);
    ncclResult_t r = ncclSuccess;
    for (int i = 0; i < n && r == ncclSuccess; ++i) {
        if (bytes[i] == 0) continue;
        r = is_recv[i] ? g_nccl.Recv(buf[i], (size_t)bytes[i], ncclUint8, peer[i], c->nc, st)
                       : g_nccl.Send(buf[i], (size_t)bytes[i], ncclUint8, peer[i], c->nc, st);
    }
    ncclResult_t e = g_nccl.GroupEnd();
    if (r != ncclSuccess) return nccl_err(r, what, c->nc);
    if (e != ncclSuccess) return nccl_err(e, what, c->nc);
    return DP_OK;
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int dp_comm_load(const char *nccl_path) { return load_nccl(nccl_path); }

extern "C" int dp_comm_version(int *version) {
    DP_REQUIRE(g_nccl.lib, DP_ERR_UNSUPPORTED, "dp_comm: NCCL not loaded");
    DP_NCCL(g_nccl.GetVersion(version), "ncclGetVersion", nullptr);
    return DP_OK;
}

extern "C" int dp_comm_unique_id(void *id_out) {
    int rc = load_nccl(nullptr);
    if (rc) return rc;
    DP_REQUIRE(id_out, DP_ERR_INVALID, "dp_comm_unique_id: null output");
    ncclUniqueId id;
    DP_NCCL(g_nccl.GetUniqueId(&id), "ncclGetUniqueId", nullptr);
    memcpy(id_out, &id, sizeof(id));
    return DP_OK;
}

extern "C" int dp_comm_init(void **comm_out, int world, int rank, const void *unique_id) {
    int rc = load_nccl(nullptr);
    if (rc) return rc;
    DP_REQUIRE(comm_out && unique_id, DP_ERR_INVALID, "dp_comm_init: null argument");
    DP_REQUIRE(world >= 1 && rank >= 0 && rank < world, DP_ERR_INVALID,
               "dp_comm_init: rank %d of %d", rank, world);
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    ncclComm_t nc = nullptr;
    DP_NCCL(g_nccl.CommInitRank(&nc, world, id, rank), "ncclCommInitRank", nullptr);
    Comm *c = new Comm{nc, rank, world};
    *comm_out = c;
    return DP_OK;
}

extern "C" int dp_comm_split(void *parent, int color, int key, void **comm_out) {
    Comm *p = (Comm *)parent;
    DP_NEED_COMM(p);
    DP_REQUIRE(comm_out, DP_ERR_INVALID, "dp_comm_split: null output");
    ncclComm_t nc = nullptr;
    DP_NCCL(g_nccl.CommSplit(p->nc, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &nc, nullptr),
            "ncclCommSplit", p->nc);
    if (!nc) {   // this rank passed no color: no communicator
        *comm_out = nullptr;
        return DP_OK;
    }
    int rank = 0, size = 0;
    // rank / size of the new communicator: key order within the color
    void *ur = dlsym(g_nccl.lib, "ncclCommUserRank");
    void *cc = dlsym(g_nccl.lib, "ncclCommCount");
    DP_REQUIRE(ur && cc, DP_ERR_UNSUPPORTED, "dp_comm_split: NCCL lacks ncclCommUserRank/Count");
    DP_NCCL(((ncclResult_t(*)(const ncclComm_t, int *))ur)(nc, &rank), "ncclCommUserRank", nc);
    DP_NCCL(((ncclResult_t(*)(const ncclComm_t, int *))cc)(nc, &size), "ncclCommCount", nc);
    *comm_out = new Comm{nc, rank, size};
    return DP_OK;
}

extern "C" int dp_comm_info(void *comm, int *rank, int *size) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    if (rank) *rank = c->rank;
    if (size) *size = c->size;
    return DP_OK;
}

extern "C" int dp_comm_destroy(void *comm) {
    Comm *c = (Comm *)comm;
    if (!c) return DP_OK;
    ncclResult_t r = c->nc ? g_nccl.CommDestroy(c->nc) : ncclSuccess;
    delete c;
    if (r != ncclSuccess) return nccl_err(r, "ncclCommDestroy", nullptr);
    return DP_OK;
}

extern "C" int dp_comm_abort(void *comm) {
    Comm *c = (Comm *)comm;
    if (!c) return DP_OK;
    ncclResult_t r = c->nc ? g_nccl.CommAbort(c->nc) : ncclSuccess;
    delete c;
    if (r != ncclSuccess) return nccl_err(r, "ncclCommAbort", nullptr);
    return DP_OK;
}

extern "C" int dp_comm_exchange(void *comm, int n, const int *peers, const int *is_recv,
                                void *const *bufs, const int64_t *bytes, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    DP_REQUIRE(n >= 0 && (n == 0 || (peers && is_recv && bufs && bytes)), DP_ERR_INVALID,
               "dp_comm_exchange: bad op list");
    if (n == 0) return DP_OK;
    return grouped(c, n, peers, is_recv, bufs, bytes, (cudaStream_t)stream, "dp_comm_exchange");
}

extern "C" int dp_halo_sendrecv(void *comm, int left, int right, const void *send_left,
                                int64_t send_left_bytes, const void *send_right,
                                int64_t send_right_bytes, void *recv_left, int64_t recv_left_bytes,
                                void *recv_right, int64_t recv_right_bytes, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    int peer[4], rv[4];
    void *buf[4];
    int64_t nb[4];
    int n = 0;
    auto add = [&](int p, int r, const void *b, int64_t bytes) {
        if (p < 0 || bytes <= 0) return;
        peer[n] = p;
        rv[n] = r;
        buf[n] = const_cast<void *>(b);
        nb[n] = bytes;
        ++n;
    };
    add(left, 0, send_left, send_left_bytes);
    add(right, 0, send_right, send_right_bytes);
    add(left, 1, recv_left, recv_left_bytes);
    add(right, 1, recv_right, recv_right_bytes);
    if (n == 0) return DP_OK;
    return grouped(c, n, peer, rv, buf, nb, (cudaStream_t)stream, "dp_halo_sendrecv");
}

extern "C" int dp_ring_step(void *comm, const void *send, int64_t send_bytes, void *recv,
                            int64_t recv_bytes, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    if (c->size == 1) return DP_OK;
    int peer[2] = {(c->rank + 1) % c->size, (c->rank + c->size - 1) % c->size};
    int rv[2] = {0, 1};
    void *buf[2] = {const_cast<void *>(send), recv};
    int64_t nb[2] = {send_bytes, recv_bytes};
    return grouped(c, 2, peer, rv, buf, nb, (cudaStream_t)stream, "dp_ring_step");
}

extern "C" int dp_varlen_allgather(void *comm, const void *local, int64_t local_bytes, void *out,
                                   const int64_t *offsets, const int64_t *bytes, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    DP_REQUIRE(offsets && bytes, DP_ERR_INVALID, "dp_varlen_allgather: null extents");
    DP_REQUIRE(bytes[c->rank] == local_bytes, DP_ERR_INVALID,
               "dp_varlen_allgather: local %lld bytes but extents say %lld",
               (long long)local_bytes, (long long)bytes[c->rank]);
    const int n = 2 * (c->size - 1);
    if (n == 0) return DP_OK;
    int *peer = new int[n], *rv = new int[n];
    void **buf = new void *[n];
    int64_t *nb = new int64_t[n];
    int k = 0;
    for (int j = 0; j < c->size; ++j) {
        if (j == c->rank) continue;
        peer[k] = j; rv[k] = 0; buf[k] = const_cast<void *>(local); nb[k] = local_bytes; ++k;
        peer[k] = j; rv[k] = 1; buf[k] = (char *)out + offsets[j]; nb[k] = bytes[j]; ++k;
    }
    int rc = grouped(c, n, peer, rv, buf, nb, (cudaStream_t)stream, "dp_varlen_allgather");
    delete[] peer; delete[] rv; delete[] buf; delete[] nb;
    return rc;
}

extern "C" int dp_varlen_alltoall(void *comm, const void *const *send, const int64_t *send_bytes,
                                  void *const *recv, const int64_t *recv_bytes, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    DP_REQUIRE(send && send_bytes && recv && recv_bytes, DP_ERR_INVALID,
               "dp_varlen_alltoall: null argument");
    const int n = 2 * (c->size - 1);
    if (n == 0) return DP_OK;
    int *peer = new int[n], *rv = new int[n];
    void **buf = new void *[n];
    int64_t *nb = new int64_t[n];
    int k = 0;
    for (int j = 0; j < c->size; ++j) {
        if (j == c->rank) continue;
        peer[k] = j; rv[k] = 0; buf[k] = const_cast<void *>(send[j]); nb[k] = send_bytes[j]; ++k;
        peer[k] = j; rv[k] = 1; buf[k] = recv[j]; nb[k] = recv_bytes[j]; ++k;
    }
    int rc = grouped(c, n, peer, rv, buf, nb, (cudaStream_t)stream, "dp_varlen_alltoall");
    delete[] peer; delete[] rv; delete[] buf; delete[] nb;
    return rc;
}

extern "C" int dp_allreduce(void *comm, const void *send, void *recv, int64_t count, int dtype,
                            int op, void *stream) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    DP_REQUIRE(count >= 0, DP_ERR_INVALID, "dp_allreduce: negative count");
    DP_REQUIRE(op == DP_REDUCE_SUM || op == DP_REDUCE_MAX, DP_ERR_INVALID, "dp_allreduce: op %d", op);
    ncclDataType_t t;
    switch (dtype) {
        case DP_F32: t = ncclFloat32; break;
        case DP_F64: t = ncclFloat64; break;
        case DP_BF16: t = ncclBfloat16; break;
        default: set_error("dp_allreduce: dtype %d", dtype); return DP_ERR_INVALID;
    }
    if (count == 0) return DP_OK;
    DP_NCCL(g_nccl.AllReduce(send, recv, (size_t)count, t, op == DP_REDUCE_SUM ? ncclSum : ncclMax,
                             c->nc, (cudaStream_t)stream),
            "ncclAllReduce", c->nc);
    return DP_OK;
}

extern "C" int dp_comm_wait(void *comm, void *stream, double timeout_s) {
    Comm *c = (Comm *)comm;
    DP_NEED_COMM(c);
    cudaStream_t st = (cudaStream_t)stream;
    timespec t0;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (;;) {
        cudaError_t q = cudaStreamQuery(st);
        if (q == cudaSuccess) return DP_OK;
        if (q != cudaErrorNotReady) {
            set_error("dp_comm_wait: stream error %s", cudaGetErrorString(q));
            return DP_ERR_CUDA;
        }
        ncclResult_t ae = ncclSuccess;
        DP_NCCL(g_nccl.CommGetAsyncError(c->nc, &ae), "ncclCommGetAsyncError", c->nc);
        if (ae != ncclSuccess && ae != ncclInProgress) {
            int rc = nccl_err(ae, "dp_comm_wait: asynchronous NCCL error (communicator aborted)",
                              c->nc);
            g_nccl.CommAbort(c->nc);
            c->nc = nullptr;
            return rc;
        }
        timespec t1;
        clock_gettime(CLOCK_MONOTONIC, &t1);
        double dt = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
        if (timeout_s > 0 && dt > timeout_s) {
            set_error("dp_comm_wait: timed out after %.3gs (rank %d of %d); communicator aborted",
                      timeout_s, c->rank, c->size);
            g_nccl.CommAbort(c->nc);
            c->nc = nullptr;
            return DP_ERR_TIMEOUT;
        }
        timespec nap = {0, 200000};
        nanosleep(&nap, nullptr);
    }
}
