// Multi-GPU plumbing inside the library (SURVEY.md §8(b) cgh_multi_*): one
// process per GPU. NCCL communicators for the collectives the distributed
// modes need (all-to-all for the NCCL corner turn, all-reduce of error sums,
// all-gather of OSPR |R|^2 totals), CUDA IPC peer mappings of the slab
// buffers for the fused peer-store corner turn, and a device barrier on peer
// flag words that orders the peers' next reads after the turn.
//
// NCCL is resolved at run time (dlopen / dlsym of libnccl.so.2): when the
// process already has an NCCL loaded (torch's), that copy is used, so the
// library never brings a second NCCL into a process.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "runtime.cuh"

namespace {

using namespace cgh;

// ---- the NCCL entry points used here (nccl.h ABI, resolved at run time)
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
typedef int ncclResult_t;   // ncclSuccess == 0
enum { ncclInt8 = 0, ncclChar = 0, ncclFloat64 = 8 };
enum { ncclSum = 0 };

struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            n.lib = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);   // already in the process (torch)
            if (n.lib) break;
        }
        if (!n.lib)
            for (const char* nm : names) {
                n.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
                if (n.lib) break;
            }
        if (!n.lib) return;
#define CGH_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(n.lib, name))
        CGH_SYM(GetUniqueId, "ncclGetUniqueId");
        CGH_SYM(CommInitRank, "ncclCommInitRank");
        CGH_SYM(CommDestroy, "ncclCommDestroy");
        CGH_SYM(Send, "ncclSend");
        CGH_SYM(Recv, "ncclRecv");
        CGH_SYM(GroupStart, "ncclGroupStart");
        CGH_SYM(GroupEnd, "ncclGroupEnd");
        CGH_SYM(AllReduce, "ncclAllReduce");
        CGH_SYM(AllGather, "ncclAllGather");
        CGH_SYM(GetErrorString, "ncclGetErrorString");
#undef CGH_SYM
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.GroupStart && n.GroupEnd &&
               n.AllReduce && n.AllGather;
    });
    return n;
}

#define CGH_NCCL(call)                                                                                \
    do {                                                                                              \
        const ncclResult_t r_ = (call);                                                               \
        if (r_ != 0)                                                                                  \
            return fail(CGH_ERR_CUDA, "%s: NCCL error %d (%s)", #call, int(r_),                       \
                        nccl().GetErrorString ? nccl().GetErrorString(r_) : "?");                     \
    } while (0)

// Barrier over `world` flag words per rank: thread g stores `epoch` into rank
// g's flags[rank] (peer memory over NVLink, system-scope release), then every
// thread waits until its own flags[g] reached `epoch` (acquire). Each call
// uses a fresh epoch, so no reset is needed.
__global__ void device_barrier_kernel(unsigned* const* __restrict__ peer_flags, int world, int rank, unsigned epoch) {
    const int g = threadIdx.x;
    if (g < world) {
        unsigned* dst = peer_flags[g] + rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
        const unsigned* mine = peer_flags[rank] + g;
        unsigned v;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
        } while (int(v - epoch) < 0);
    }
}

}  // namespace

struct cgh_multi {
    int dev = 0, world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    unsigned* flags = nullptr;          // this rank's flag words [world]
    unsigned epoch = 0;
    unsigned** peer_flags_d = nullptr;  // device array of every rank's flag pointer
    std::vector<void*> opened;          // IPC mappings to close
};

extern "C" {

int cgh_multi_available(void) { return nccl().ok ? 1 : 0; }

int cgh_multi_unique_id(uint8_t* out128) {
    if (!out128) return fail(CGH_ERR_VALUE, "null output");
    if (!nccl().ok) return fail(CGH_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
    ncclUniqueId id;
    CGH_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out128, id.internal, 128);
    return CGH_OK;
}

int cgh_multi_create(int32_t device, int32_t world, int32_t rank, const uint8_t* id128, void* stream, cgh_multi** out) {
    if (!out || !id128 || world < 1 || rank < 0 || rank >= world) return fail(CGH_ERR_VALUE, "bad arguments");
    *out = nullptr;
    if (!nccl().ok) return fail(CGH_ERR_NO_DEVICE, "NCCL (libnccl.so.2) not available");
    CGH_CUDA(cudaSetDevice(device));
    cgh_multi* m = new cgh_multi();
    m->dev = device;
    m->world = world;
    m->rank = rank;
    if (stream) {
        m->st = static_cast<cudaStream_t>(stream);
    } else {
        cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking);
        m->own_stream = true;
    }
    ncclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    const ncclResult_t r = nccl().CommInitRank(&m->comm, world, id, rank);
    if (r != 0) {
        if (m->own_stream) cudaStreamDestroy(m->st);
        delete m;
        return fail(CGH_ERR_CUDA, "ncclCommInitRank: NCCL error %d", int(r));
    }
    cudaError_t e = cudaMalloc(&m->flags, sizeof(unsigned) * world);
    if (e == cudaSuccess) e = cudaMemset(m->flags, 0, sizeof(unsigned) * world);
    if (e == cudaSuccess) e = cudaMalloc(&m->peer_flags_d, sizeof(unsigned*) * world);
    if (e != cudaSuccess) {
        nccl().CommDestroy(m->comm);
        delete m;
        return fail(CGH_ERR_MEMORY, "barrier flags: %s", cudaGetErrorString(e));
    }
    *out = m;
    return CGH_OK;
}

int cgh_multi_destroy(cgh_multi* m) {
    if (!m) return CGH_OK;
    cudaSetDevice(m->dev);
    cudaStreamSynchronize(m->st);
    for (void* p : m->opened) cudaIpcCloseMemHandle(p);
    if (m->comm) nccl().CommDestroy(m->comm);
    if (m->flags) cudaFree(m->flags);
    if (m->peer_flags_d) cudaFree(m->peer_flags_d);
    if (m->own_stream) cudaStreamDestroy(m->st);
    delete m;
    return CGH_OK;
}

static cudaStream_t pick(cgh_multi* m, void* stream) { return stream ? static_cast<cudaStream_t>(stream) : m->st; }

// Block g (bytes_per_peer) of send goes to rank g; block g of recv comes from rank g.
int cgh_multi_all_to_all(cgh_multi* m, const void* send, void* recv, int64_t bytes_per_peer, void* stream) {
    if (!m || !send || !recv || bytes_per_peer < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    const cudaStream_t st = pick(m, stream);
    CGH_NCCL(nccl().GroupStart());
    for (int g = 0; g < m->world; ++g) {
        CGH_NCCL(nccl().Send(static_cast<const char*>(send) + size_t(g) * bytes_per_peer, size_t(bytes_per_peer),
                             ncclChar, g, m->comm, st));
        CGH_NCCL(nccl().Recv(static_cast<char*>(recv) + size_t(g) * bytes_per_peer, size_t(bytes_per_peer), ncclChar,
                             g, m->comm, st));
    }
    CGH_NCCL(nccl().GroupEnd());
    return CGH_OK;
}

int cgh_multi_all_reduce_sum_f64(cgh_multi* m, double* buf, int64_t count, void* stream) {
    if (!m || !buf || count < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    CGH_NCCL(nccl().AllReduce(buf, buf, size_t(count), ncclFloat64, ncclSum, m->comm, pick(m, stream)));
    return CGH_OK;
}

// recv = [rank 0's send | rank 1's send | ...], bytes each
int cgh_multi_all_gather(cgh_multi* m, const void* send, void* recv, int64_t bytes, void* stream) {
    if (!m || !send || !recv || bytes < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    CGH_NCCL(nccl().AllGather(send, recv, size_t(bytes), ncclChar, m->comm, pick(m, stream)));
    return CGH_OK;
}

// ---- peer mappings (CUDA IPC): export a device allocation, open a peer's
int cgh_multi_ipc_handle(cgh_multi* m, void* ptr, uint8_t* out64) {
    if (!m || !ptr || !out64) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    cudaIpcMemHandle_t h;
    CGH_CUDA(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(out64, &h, 64);
    return CGH_OK;
}

int cgh_multi_ipc_open(cgh_multi* m, const uint8_t* handle64, void** out) {
    if (!m || !handle64 || !out) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    void* p = nullptr;
    CGH_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    m->opened.push_back(p);
    *out = p;
    return CGH_OK;
}

// Plain device allocations (cudaMalloc: IPC-exportable allocation bases).
int cgh_device_alloc(int32_t device, int64_t bytes, void** out) {
    if (!out || bytes <= 0) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaMalloc(out, size_t(bytes));
    if (e != cudaSuccess) return fail(CGH_ERR_MEMORY, "cudaMalloc(%lld): %s", (long long)bytes, cudaGetErrorString(e));
    return CGH_OK;
}
int cgh_device_free(int32_t device, void* ptr) {
    if (!ptr) return CGH_OK;
    CGH_CUDA(cudaSetDevice(device));
    CGH_CUDA(cudaFree(ptr));
    return CGH_OK;
}

// This rank's barrier flag array (export it with cgh_multi_ipc_handle).
int cgh_multi_flags(cgh_multi* m, void** out) {
    if (!m || !out) return fail(CGH_ERR_VALUE, "bad arguments");
    *out = m->flags;
    return CGH_OK;
}

// Every rank's flag array as seen from this rank (index = rank; own entry =
// this rank's own array), set once after the handles are exchanged.
int cgh_multi_set_peer_flags(cgh_multi* m, void* const* flags) {
    if (!m || !flags) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(m->dev));
    std::vector<unsigned*> v(static_cast<size_t>(m->world));
    for (int g = 0; g < m->world; ++g) v[size_t(g)] = static_cast<unsigned*>(flags[g]);
    CGH_CUDA(cudaMemcpy(m->peer_flags_d, v.data(), sizeof(unsigned*) * m->world, cudaMemcpyHostToDevice));
    return CGH_OK;
}

// Device barrier over the peer flags on `stream`: work queued after it on any
// rank starts only when every rank has reached it (e.g. after a corner turn
// that stored into peer memory).
int cgh_multi_device_barrier(cgh_multi* m, void* stream) {
    if (!m) return fail(CGH_ERR_VALUE, "null communicator");
    CGH_CUDA(cudaSetDevice(m->dev));
    m->epoch += 1;
    device_barrier_kernel<<<1, 32 * ((m->world + 31) / 32), 0, pick(m, stream)>>>(m->peer_flags_d, m->world, m->rank,
                                                                                 m->epoch);
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

}  // extern "C"
