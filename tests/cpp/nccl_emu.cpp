// nccl_emu.cpp -- TEST INFRASTRUCTURE: an in-process stand-in for the five NCCL
// entry points libfkde_b200.so uses (ncclGetUniqueId, ncclCommInitRank,
// ncclCommInitAll, ncclAllGather, ncclCommDestroy, ncclGetErrorString), loaded
// through FKDE_NCCL_LIB.  Ranks are host threads of one process and may share a
// device, so the engine's multi-rank code (row shards of the score pass, the
// x^SD allgather layout, query shards, the density gather) runs on one GPU.
// ncclAllGather: host barrier -> every rank's stream waits for every rank's
// "send ready" event -> device-to-device copies of the other ranks' slices ->
// second barrier on "copies done" events, so no rank overwrites its slice while
// a peer still reads it.  Driver API only (the engine links the CUDA runtime
// statically; the streams it passes are driver streams of the primary context).
// Build: g++ -std=c++17 -O2 -shared -fPIC -I/usr/local/cuda/include nccl_emu.cpp
//        -L/usr/local/cuda/lib64/stubs -lcuda -o libnccl_emu.so
#include <cuda.h>
#include <cuda_runtime_api.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <string>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace {

struct Group {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const void*> send;
    std::vector<CUevent> ev_in, ev_out;
    explicit Group(int w) : world(w), send(w), ev_in(w, nullptr), ev_out(w, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

std::mutex g_reg_mu;
std::map<std::string, Group*> g_groups;
long g_next_id = 1;

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

}  // namespace

struct ncclComm {
    Group* g;
    int rank;
};

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    std::memset(id->internal, 0, sizeof(id->internal));
    std::snprintf(id->internal, sizeof(id->internal), "emu-%ld", g_next_id++);
    return ncclSuccess;
}

// the calling thread has the rank's device current (the engine calls
// cudaSetDevice first)
static ncclResult_t make_comm(ncclComm_t* comm, Group* g, int rank) {
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->ev_in[rank] && (cuEventCreate(&g->ev_in[rank], CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS ||
                            cuEventCreate(&g->ev_out[rank], CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS))
        return ncclUnhandledCudaError;
    *comm = new ncclComm{g, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    Group* g;
    {
        std::lock_guard<std::mutex> lk(g_reg_mu);
        std::string key(id.internal);
        auto it = g_groups.find(key);
        if (it == g_groups.end()) it = g_groups.emplace(key, new Group(nranks)).first;
        g = it->second;
    }
    return make_comm(comm, g, rank);
}

// (single-process form: every rank's events are created in the caller's
// current context -- the emulated ranks must share one device)
ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
    for (int i = 1; i < ndev; ++i)
        if (devlist && devlist[i] != devlist[0]) return ncclInvalidUsage;
    Group* g = new Group(ndev);
    for (int i = 0; i < ndev; ++i)
        if (make_comm(&comms[i], g, i) != ncclSuccess) return ncclUnhandledCudaError;
    return ncclSuccess;
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t dt,
                           ncclComm_t comm, cudaStream_t stream) {
    Group* g = comm->g;
    const int r = comm->rank;
    const size_t bytes = count * type_size(dt);
    CUstream st = reinterpret_cast<CUstream>(stream);
    bool ok = true;
    g->send[r] = sendbuff;
    ok &= cuEventRecord(g->ev_in[r], st) == CUDA_SUCCESS;
    g->barrier();
    for (int q = 0; q < g->world; ++q) ok &= cuStreamWaitEvent(st, g->ev_in[q], 0) == CUDA_SUCCESS;
    char* dst = static_cast<char*>(recvbuff);
    for (int q = 0; q < g->world; ++q)
        if (static_cast<const void*>(dst + q * bytes) != g->send[q])
            ok &= cuMemcpyDtoDAsync(reinterpret_cast<CUdeviceptr>(dst + q * bytes),
                                    reinterpret_cast<CUdeviceptr>(g->send[q]), bytes, st) == CUDA_SUCCESS;
    ok &= cuEventRecord(g->ev_out[r], st) == CUDA_SUCCESS;
    g->barrier();
    for (int q = 0; q < g->world; ++q) ok &= cuStreamWaitEvent(st, g->ev_out[q], 0) == CUDA_SUCCESS;
    g->barrier();   // nobody re-records its events before every rank has enqueued these waits
    return ok ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "no error" : "nccl_emu error"; }

}  // extern "C"
