// fake_nccl.cpp — TEST INFRASTRUCTURE: a functional stand-in for the NCCL calls libattncache uses, so that the
// library's collective code (csrc/collective.cu: count exchanges, query all-gather, key max-all-reduce, grouped
// send/recv of routed rows and relocated request state) runs at world 2-4 with every rank on ONE GPU
// (tests/test_gpu_fake_nccl.py; real NCCL refuses two ranks on one device).  It is not a performance stand-in:
// every call synchronises the caller's stream and moves the bytes through a host file mapping shared by the
// ranks (collectives between host barriers; send / recv through per-pair mailboxes), so no rank's kernels ever
// wait on another rank's kernels.
// Loaded by the library through ATTNCACHE_NCCL_LIB.  Build: g++ -shared -fPIC -O2 fake_nccl.cpp -lcudart.
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

namespace {

constexpr int kMaxRanks = 16;
constexpr size_t kHeader = 8192;

struct Header {
    std::atomic<int> arrive;  // barrier (collectives: every rank takes part)
    std::atomic<int> gen;
    // point-to-point mailbox (src, dst): chunks posted by src and consumed by dst.  P2P needs no global step:
    // like NCCL, a rank with nothing to send or receive in a group does not take part.
    std::atomic<uint64_t> posted[kMaxRanks][kMaxRanks];
    std::atomic<uint64_t> consumed[kMaxRanks][kMaxRanks];
};

struct FakeComm {
    int rank = 0, world = 1;
    size_t slot = 0;  // bytes per rank slot (all-gather / all-reduce) and per (src, dst) mailbox
    uint8_t *base = nullptr;
    size_t bytes = 0;
    char path[160] = "";
    Header *hdr() const { return reinterpret_cast<Header *>(base); }
    uint8_t *slot_of(int r) const { return base + kHeader + (size_t)r * slot; }
    uint8_t *box(int src, int dst) const { return base + kHeader + (size_t)world * slot + ((size_t)src * world + dst) * slot; }
};

void barrier(FakeComm *c) {
    Header *h = c->hdr();
    const int g = h->gen.load(std::memory_order_acquire);
    if (h->arrive.fetch_add(1, std::memory_order_acq_rel) == c->world - 1) {
        h->arrive.store(0, std::memory_order_relaxed);
        h->gen.fetch_add(1, std::memory_order_release);
    } else {
        while (h->gen.load(std::memory_order_acquire) == g) sched_yield();
    }
}

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
        default: return 0;
    }
}

struct P2p {
    bool send;
    void *buf;
    size_t bytes;
    int peer;
    FakeComm *comm;
    cudaStream_t st;
};
int g_group = 0;
std::vector<P2p> g_ops;

ncclResult_t run_p2p(std::vector<P2p> &ops) {
    if (ops.empty()) return ncclSuccess;
    for (auto &o : ops)
        if (cudaStreamSynchronize(o.st) != cudaSuccess) return ncclUnhandledCudaError;
    // progress every send and receive of the group chunk by chunk (`slot` bytes per chunk) through its pair's
    // mailbox until all are done: a send posts a chunk once the receiver consumed the previous one
    std::vector<size_t> done(ops.size(), 0);
    bool left = true;
    while (left) {
        left = false;
        bool moved = false;
        for (size_t i = 0; i < ops.size(); ++i) {
            P2p &o = ops[i];
            if (done[i] >= o.bytes) continue;
            left = true;
            FakeComm *c = o.comm;
            Header *h = c->hdr();
            const int src = o.send ? c->rank : o.peer, dst = o.send ? o.peer : c->rank;
            const uint64_t posted = h->posted[src][dst].load(std::memory_order_acquire);
            const uint64_t consumed = h->consumed[src][dst].load(std::memory_order_acquire);
            const size_t n = o.bytes - done[i] < c->slot ? o.bytes - done[i] : c->slot;
            if (o.send && posted == consumed) {
                if (cudaMemcpy(c->box(src, dst), (const uint8_t *)o.buf + done[i], n, cudaMemcpyDeviceToHost) != cudaSuccess)
                    return ncclUnhandledCudaError;
                h->posted[src][dst].store(posted + 1, std::memory_order_release);
                done[i] += n;
                moved = true;
            } else if (!o.send && posted > consumed) {
                if (cudaMemcpy((uint8_t *)o.buf + done[i], c->box(src, dst), n, cudaMemcpyHostToDevice) != cudaSuccess)
                    return ncclUnhandledCudaError;
                h->consumed[src][dst].store(consumed + 1, std::memory_order_release);
                done[i] += n;
                moved = true;
            }
        }
        if (left && !moved) sched_yield();
    }
    // a receive is complete when its last chunk is consumed; a send when the receiver took its last chunk (the
    // caller may reuse the buffer, but the mailbox must be free before this rank's next send to the same peer:
    // the next post waits for that anyway)
    ops.clear();
    return ncclSuccess;
}

// FAKE_NCCL_HANG_ON=allgather: after the all-gather's work, the stream waits (cuStreamWaitValue32) on a
// host-mapped flag that only ncclCommAbort sets: the stream never finishes on its own, like a collective whose
// peer died.  The library's host waits must poll the async error, abort, and return.
volatile uint32_t *g_release = nullptr;
CUdeviceptr g_release_dev = 0;
ncclResult_t maybe_hang(cudaStream_t st, const char *op) {
    const char *h = getenv("FAKE_NCCL_HANG_ON");
    if (!h || strcmp(h, op) != 0) return ncclSuccess;
    if (!g_release) {
        void *p = nullptr, *d = nullptr;
        if (cudaHostAlloc(&p, 4, cudaHostAllocMapped) != cudaSuccess) return ncclUnhandledCudaError;
        if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) return ncclUnhandledCudaError;
        g_release = (volatile uint32_t *)p;
        g_release_dev = (CUdeviceptr)d;
    }
    *g_release = 0;
    return cuStreamWaitValue32((CUstream)st, g_release_dev, 1, CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
               ? ncclSuccess : ncclUnhandledCudaError;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetVersion(int *v) {
    *v = 22809;
    return ncclSuccess;
}
const char *ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "no error" : "fake_nccl error"; }
// FAKE_NCCL_ASYNC_ERROR=1 makes every communicator report an asynchronous error (the library's abort path)
ncclResult_t ncclCommGetAsyncError(ncclComm_t, ncclResult_t *e) {
    const char *f = getenv("FAKE_NCCL_ASYNC_ERROR");
    *e = (f && *f == '1') ? ncclRemoteError : ncclSuccess;
    return ncclSuccess;
}
int g_aborts = 0;  // read by the tests through fake_nccl_abort_count()
int fake_nccl_abort_count() { return g_aborts; }

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
    memset(id, 0, sizeof *id);
    snprintf(id->internal, sizeof id->internal, "/tmp/fake_nccl_%d_%ld", (int)getpid(), (long)clock());
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *out, int nranks, ncclUniqueId id, int rank) {
    if (nranks > kMaxRanks) return ncclInvalidArgument;
    FakeComm *c = new FakeComm();
    c->rank = rank;
    c->world = nranks;
    const char *mb = getenv("FAKE_NCCL_SLOT_MB");
    c->slot = (size_t)(mb ? atoi(mb) : 16) << 20;
    c->bytes = kHeader + (size_t)nranks * c->slot + (size_t)nranks * nranks * c->slot;
    static_assert(sizeof(Header) <= kHeader, "header");
    snprintf(c->path, sizeof c->path, "%s", id.internal);
    const int fd = open(c->path, O_RDWR | O_CREAT, 0600);
    if (fd < 0 || ftruncate(fd, (off_t)c->bytes) != 0) return ncclSystemError;  // zero-filled: the barrier starts at 0
    c->base = (uint8_t *)mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (c->base == MAP_FAILED) return ncclSystemError;
    barrier(c);
    *out = reinterpret_cast<ncclComm_t>(c);
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    FakeComm *c = reinterpret_cast<FakeComm *>(comm);
    barrier(c);
    munmap(c->base, c->bytes);
    if (c->rank == 0) unlink(c->path);
    delete c;
    return ncclSuccess;
}

// No barrier: the peers of an aborted communicator may be gone.
ncclResult_t ncclCommAbort(ncclComm_t comm) {
    if (g_release) *g_release = 1;  // releases a stream left waiting by FAKE_NCCL_HANG_ON
    FakeComm *c = reinterpret_cast<FakeComm *>(comm);
    munmap(c->base, c->bytes);
    delete c;
    ++g_aborts;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
    ++g_group;
    return ncclSuccess;
}
ncclResult_t ncclGroupEnd() {
    if (--g_group > 0) return ncclSuccess;
    return run_p2p(g_ops);
}

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
    g_ops.push_back({true, const_cast<void *>(buf), count * type_size(t), peer, reinterpret_cast<FakeComm *>(comm), st});
    return g_group ? ncclSuccess : run_p2p(g_ops);
}
ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
    g_ops.push_back({false, buf, count * type_size(t), peer, reinterpret_cast<FakeComm *>(comm), st});
    return g_group ? ncclSuccess : run_p2p(g_ops);
}

ncclResult_t ncclAllGather(const void *send, void *recv, size_t count, ncclDataType_t t, ncclComm_t comm,
                           cudaStream_t st) {
    FakeComm *c = reinterpret_cast<FakeComm *>(comm);
    const size_t b = count * type_size(t);
    if (b > c->slot) return ncclInvalidUsage;
    if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
    if (b && cudaMemcpy(c->slot_of(c->rank), send, b, cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
    barrier(c);
    for (int r = 0; r < c->world; ++r)
        if (b && cudaMemcpy((uint8_t *)recv + (size_t)r * b, c->slot_of(r), b, cudaMemcpyHostToDevice) != cudaSuccess)
            return ncclUnhandledCudaError;
    barrier(c);
    return maybe_hang(st, "allgather");
}

ncclResult_t ncclAllReduce(const void *send, void *recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
    FakeComm *c = reinterpret_cast<FakeComm *>(comm);
    if ((t != ncclUint64 && t != ncclInt64) || (op != ncclMax && op != ncclSum)) return ncclInvalidUsage;
    const size_t b = count * 8;
    if (b > c->slot) return ncclInvalidUsage;
    if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
    if (b && cudaMemcpy(c->slot_of(c->rank), send, b, cudaMemcpyDeviceToHost) != cudaSuccess) return ncclUnhandledCudaError;
    barrier(c);
    std::vector<uint64_t> acc(count);
    for (int r = 0; r < c->world; ++r) {
        const uint64_t *v = reinterpret_cast<const uint64_t *>(c->slot_of(r));
        for (size_t i = 0; i < count; ++i) {
            if (r == 0) acc[i] = v[i];
            else if (op == ncclSum) acc[i] += v[i];
            else if (t == ncclUint64) acc[i] = v[i] > acc[i] ? v[i] : acc[i];
            else acc[i] = (int64_t)v[i] > (int64_t)acc[i] ? v[i] : acc[i];
        }
    }
    barrier(c);
    if (b && cudaMemcpy(recv, acc.data(), b, cudaMemcpyHostToDevice) != cudaSuccess) return ncclUnhandledCudaError;
    return ncclSuccess;
}

}  // extern "C"
