// sisph_comm.cuh — the data-path collectives of the slab-decomposed SISPH
// step: a face exchange with the two slab neighbours
// (halo refresh, migration) and a small fp64 allreduce (Lambda, the two
// residual sums of eq:convergence, the skin).
//
// Two transports implement the same interface:
//   * NcclTransport — production: one process per GPU, NCCL (dlopen'ed at
//     run time: the library torch loads, or the one named by the caller)
//     over NVLink/NVSwitch, every call stream-ordered on the handle's stream
//     (no host synchronisation except where a count must reach the host);
//   * LocalTransport — R ranks in ONE process on one GPU, for tests: every
//     call synchronises its rank's stream, meets the other ranks at a host
//     barrier and copies device to device.  No kernel ever waits on another
//     rank, so the ranks can share a GPU (B200_PROFILING.md: kernels that
//     wait on each other must not share one).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace sb {

struct Transport {
    int rank = 0, nranks = 1;
    int nb[2] = {-1, -1};   // neighbour rank across the low (0) / high (1) face, -1 if none
    std::string err;
    virtual ~Transport() {}
    // send sbuf[f] (sn[f] bytes) to nb[f] and receive rn[f] bytes from nb[f]
    // into rbuf[f], f = 0, 1.  Device buffers.  Sends go out high face first
    // and receives are posted low face first, so that with two ranks on a
    // periodic axis (both neighbours the same rank) face f's message lands in
    // the peer's face 1 - f.
    virtual int sendrecv(const void* const sbuf[2], const size_t sn[2], void* const rbuf[2], const size_t rn[2],
                         cudaStream_t st) = 0;
    // in-place allreduce of count doubles (device buffer): op 0 = sum, 1 = max
    virtual int allreduce(double* buf, int count, int op, cudaStream_t st) = 0;
};

// ---------------------------------------------------------------- NCCL
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    // path NULL or "" -> "libnccl.so.2" from the loader's search path (or the
    // copy already loaded into the process, e.g. by torch)
    bool load(const char* path, std::string& err)
    {
        if (h) return true;
        const char* p = (path && *path) ? path : "libnccl.so.2";
        h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("dlopen ") + p + ": " + dlerror();
            return false;
        }
#define SB_NCCL_SYM(f, name)                                          \
    f = reinterpret_cast<decltype(f)>(dlsym(h, name));                \
    if (!f) {                                                         \
        err = std::string("missing NCCL symbol ") + name;             \
        return false;                                                 \
    }
        SB_NCCL_SYM(GetUniqueId, "ncclGetUniqueId")
        SB_NCCL_SYM(CommInitRank, "ncclCommInitRank")
        SB_NCCL_SYM(CommDestroy, "ncclCommDestroy")
        SB_NCCL_SYM(Send, "ncclSend")
        SB_NCCL_SYM(Recv, "ncclRecv")
        SB_NCCL_SYM(AllReduce, "ncclAllReduce")
        SB_NCCL_SYM(GroupStart, "ncclGroupStart")
        SB_NCCL_SYM(GroupEnd, "ncclGroupEnd")
        SB_NCCL_SYM(GetErrorString, "ncclGetErrorString")
#undef SB_NCCL_SYM
        return true;
    }
};

inline NcclApi& nccl_api()
{
    static NcclApi a;
    return a;
}

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    NcclApi* api = nullptr;

    int init(const char* lib, const uint8_t id[128], int nranks_, int rank_)
    {
        api = &nccl_api();
        if (!api->load(lib, err)) return 1;
        ncclUniqueId u;
        memcpy(u.internal, id, sizeof(u.internal));
        rank = rank_;
        nranks = nranks_;
        ncclResult_t r = api->CommInitRank(&comm, nranks, u, rank);
        if (r != ncclSuccess) {
            err = std::string("ncclCommInitRank: ") + api->GetErrorString(r);
            return 1;
        }
        return 0;
    }
    ~NcclTransport() override
    {
        if (comm) api->CommDestroy(comm);
    }
    int check(ncclResult_t r, const char* what)
    {
        if (r == ncclSuccess) return 0;
        err = std::string(what) + ": " + api->GetErrorString(r);
        return 1;
    }
    int sendrecv(const void* const sbuf[2], const size_t sn[2], void* const rbuf[2], const size_t rn[2],
                 cudaStream_t st) override
    {
        if (check(api->GroupStart(), "ncclGroupStart")) return 1;
        // a failed Send / Recv inside the group still closes the group (keeping the first
        // error): an open group would leave this thread's later collectives undefined
        int bad = 0;
        for (int f = 1; f >= 0 && !bad; f--)
            if (nb[f] >= 0 && sn[f] > 0 && check(api->Send(sbuf[f], sn[f], ncclChar, nb[f], comm, st), "ncclSend"))
                bad = 1;
        for (int f = 0; f < 2 && !bad; f++)
            if (nb[f] >= 0 && rn[f] > 0 && check(api->Recv(rbuf[f], rn[f], ncclChar, nb[f], comm, st), "ncclRecv"))
                bad = 1;
        const ncclResult_t ge = api->GroupEnd();
        if (bad) return 1;
        return check(ge, "ncclGroupEnd");
    }
    int allreduce(double* buf, int count, int op, cudaStream_t st) override
    {
        // also with one rank (the slab path forced on one GPU): the same NCCL call runs
        return check(api->AllReduce(buf, buf, (size_t)count, ncclDouble, op == 0 ? ncclSum : ncclMax, comm, st),
                     "ncclAllReduce");
    }
};

// ---------------------------------------------------------------- in-process hub
struct LocalHub {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    bool aborted = false;   // a rank gave up waiting: every later barrier fails at once
    // per rank, per face: posted send buffer / size
    std::vector<const void*> sptr;
    std::vector<size_t> ssz;
    std::vector<double*> rptr;
    explicit LocalHub(int n) : nranks(n), sptr(2 * n), ssz(2 * n), rptr(n) {}
    // false if a rank did not arrive within the timeout (it failed: its
    // caller reports the error instead of hanging) or the hub was aborted
    bool barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) return false;
        long g = generation;
        if (++arrived == nranks) {
            arrived = 0;
            generation++;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != g || aborted; }) || aborted) {
            aborted = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

struct LocalTransport : Transport {
    LocalHub* hub = nullptr;
    int fail_barrier()
    {
        err = "local transport: another rank did not reach the exchange (it failed or hung)";
        return 1;
    }
    int sync(cudaStream_t st)
    {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            err = std::string("cudaStreamSynchronize: ") + cudaGetErrorString(e);
            return 1;
        }
        return 0;
    }
    int sendrecv(const void* const sbuf[2], const size_t sn[2], void* const rbuf[2], const size_t rn[2],
                 cudaStream_t st) override
    {
        if (sync(st)) return 1;
        for (int f = 0; f < 2; f++) {
            hub->sptr[2 * rank + f] = nb[f] >= 0 ? sbuf[f] : nullptr;
            hub->ssz[2 * rank + f] = nb[f] >= 0 ? sn[f] : 0;
        }
        if (!hub->barrier()) return fail_barrier();
        int rc = 0;
        for (int f = 0; f < 2 && !rc; f++) {
            if (nb[f] < 0 || rn[f] == 0) continue;
            // my face f borders the neighbour's face 1 - f
            const int src = 2 * nb[f] + (1 - f);
            if (hub->ssz[src] != rn[f]) {
                err = "local transport: message size mismatch";
                rc = 1;
                break;
            }
            cudaError_t e = cudaMemcpyAsync(rbuf[f], hub->sptr[src], rn[f], cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) {
                err = std::string("cudaMemcpyAsync: ") + cudaGetErrorString(e);
                rc = 1;
            }
        }
        if (!rc) rc = sync(st);
        if (!hub->barrier()) return fail_barrier();   // senders' buffers stay valid until every copy is done
        return rc;
    }
    int allreduce(double* buf, int count, int op, cudaStream_t st) override
    {
        if (nranks == 1) return 0;
        if (sync(st)) return 1;
        hub->rptr[rank] = buf;
        if (!hub->barrier()) return fail_barrier();
        // every rank reduces all ranks' values in rank order (identical bits everywhere)
        std::vector<double> acc(count), tmp(count);
        int rc = 0;
        for (int r = 0; r < nranks && !rc; r++) {
            if (cudaMemcpy(tmp.data(), hub->rptr[r], count * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
                err = "local transport: allreduce copy failed";
                rc = 1;
            }
            for (int q = 0; q < count; q++)
                acc[q] = r == 0 ? tmp[q] : (op == 0 ? acc[q] + tmp[q] : (tmp[q] > acc[q] ? tmp[q] : acc[q]));
        }
        if (!hub->barrier()) return fail_barrier();   // all reads done before anyone overwrites its buffer
        if (!rc && cudaMemcpy(buf, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
            err = "local transport: allreduce write-back failed";
            rc = 1;
        }
        return rc;
    }
};

}  // namespace sb
