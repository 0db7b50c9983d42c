// The once-per-generation exchange of a row-sharded run: every rank contributes the fitness of its
// partition_rows block (modes.cpp:506-516) and receives everybody else's.  This is the GPU form of the reference's
// Channel<T> (include/gapa/channel.hpp:12-35), which ships with the library — so does this: C and C++ hosts get a
// multi-GPU run without bringing a communication layer of their own.
//
// Two transports behind one object:
//   * PEER  — mailboxes in HBM written directly by the peers over NVLink / NVSwitch.  Rank r stores its block into every
//     peer's mailbox and then a sequence number (release, system scope); it spins (acquire) until the peers' numbers
//     have arrived in its own mailbox and copies their blocks out.  One kernel per exchange, no host involvement, no
//     rendezvous protocol: a 4 KB all-gather is pure latency, and this is one NVLink store + one flag per peer.
//     Mailboxes are double-buffered by the sequence parity (a rank can be at most one exchange ahead of a peer that
//     has not consumed yet: it cannot pass exchange q+1 before that peer has pushed q+1, which the peer does after its
//     exchange-q kernel, pull included, has completed).  Ranks in one process exchange raw pointers (peer access is
//     enabled between their devices); ranks in different processes exchange CUDA IPC handles.
//   * NCCL  — ncclAllGather on the caller's stream, loaded at run time from libnccl.so.2 (the one PyTorch ships is
//     already in the process when the host is Python; a C++ host uses the system library).
// gapa_cuda_comm_allgather has the gapa_cuda_allgather_fn signature: pass it, with the comm as `user`, to
// gapa_cuda_run / gapa_cuda_ga_create.
#include <dlfcn.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <thread>

#include "internal.cuh"

namespace gapa_b200 {

static constexpr int kMaxWorld = 16;
static constexpr int kCtrlBytes = GAPA_CUDA_COMM_CTRL_BYTES;
static constexpr uint32_t kHandleMagic = 0x47415041u;  // "GAPA"

struct CommHandle {  // what a rank publishes; fits GAPA_CUDA_COMM_HANDLE_BYTES
    uint32_t magic;
    int32_t device;
    int64_t pid;
    uint64_t local_ptr;
    uint64_t capacity;
    cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(CommHandle) <= GAPA_CUDA_COMM_HANDLE_BYTES, "handle does not fit its ABI size");

struct CommPeers {
    char* base[kMaxWorld];
};

// layout of every rank's allocation
__host__ __device__ inline size_t comm_flags_off(size_t cap) { return (2 * cap * sizeof(double) + 127) & ~size_t{127}; }
__host__ __device__ inline size_t comm_ctrl_flags_off(size_t cap) { return comm_flags_off(cap) + 128; }
__host__ __device__ inline size_t comm_ctrl_off(size_t cap) { return comm_ctrl_flags_off(cap) + 128; }
__host__ __device__ inline size_t comm_status_off(size_t cap) { return comm_ctrl_off(cap) + 2 * static_cast<size_t>(kMaxWorld) * kCtrlBytes; }
__host__ __device__ inline size_t comm_bytes(size_t cap) { return comm_status_off(cap) + 128; }

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// thread 0 of the CTA waits for `flag` to reach `seq`; a peer that never arrives turns into a status, not a hang
__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t seq, unsigned long long timeout_ns, int* status) {
    const unsigned long long t0 = global_ns();
    while (static_cast<int32_t>(ld_acquire_sys(flag) - seq) < 0) {
        if (global_ns() - t0 > timeout_ns) {
            atomicExch(status, GAPA_CUDA_E_CUDA);
            break;
        }
        __nanosleep(64);
    }
}

// CTA p of rank r: push r's block into p's mailbox, raise r's flag there, wait for p's flag here, pull p's block.
// phases: kPush | kPull in one launch is the exchange; the two halves are launched separately (with the ranks meeting on
// the host in between) only when ranks share a device inside one process, where a spinning kernel could wait for a
// kernel queued behind it in the same hardware queue.
enum { kPush = 1, kPull = 2 };
__global__ void __launch_bounds__(256) k_comm_allgather(CommPeers peers, int rank, size_t cap, uint32_t seq, double* fit_full,
                                                        int block, int* run_status, unsigned long long timeout_ns, int phases) {
    griddep_launch();
    griddep_wait();
    const int p = blockIdx.x;
    if (p == rank) return;
    const size_t parity = seq & 1u;
    const int lo = rank * block;
    if (phases & kPush) {
        double* theirs = reinterpret_cast<double*>(peers.base[p]) + parity * cap;
        for (int i = threadIdx.x; i < block; i += blockDim.x) theirs[lo + i] = fit_full[lo + i];
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(reinterpret_cast<uint32_t*>(peers.base[p] + comm_flags_off(cap)) + rank, seq);
    }
    if (!(phases & kPull)) return;
    if (threadIdx.x == 0) {
        int* status = reinterpret_cast<int*>(peers.base[rank] + comm_status_off(cap));
        wait_flag(reinterpret_cast<const uint32_t*>(peers.base[rank] + comm_flags_off(cap)) + p, seq, timeout_ns, status);
        if (*reinterpret_cast<volatile int*>(status) && run_status) atomicExch(run_status, GAPA_CUDA_E_CUDA);
    }
    __syncthreads();
    const double* mine = reinterpret_cast<const double*>(peers.base[rank]) + parity * cap;
    for (int i = threadIdx.x; i < block; i += blockDim.x) fit_full[p * block + i] = __ldcv(mine + p * block + i);
}

// the same exchange for a few bytes per rank (bootstrap data: IPC handles of the population stores)
__global__ void __launch_bounds__(kCtrlBytes) k_comm_ctrl(CommPeers peers, int rank, int world, size_t cap, uint32_t seq, const char* mine,
                                                           int bytes, char* all_out, unsigned long long timeout_ns, int phases) {
    griddep_launch();
    griddep_wait();
    const int p = blockIdx.x;
    const size_t parity = seq & 1u;
    if (p == rank) {
        if ((phases & kPush) && threadIdx.x < bytes) all_out[static_cast<size_t>(rank) * kCtrlBytes + threadIdx.x] = mine[threadIdx.x];
        return;
    }
    if (phases & kPush) {
        char* theirs = peers.base[p] + comm_ctrl_off(cap) + (parity * kMaxWorld + rank) * kCtrlBytes;
        if (threadIdx.x < bytes) theirs[threadIdx.x] = mine[threadIdx.x];
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(reinterpret_cast<uint32_t*>(peers.base[p] + comm_ctrl_flags_off(cap)) + rank, seq);
    }
    if (!(phases & kPull)) return;
    if (threadIdx.x == 0) {
        wait_flag(reinterpret_cast<const uint32_t*>(peers.base[rank] + comm_ctrl_flags_off(cap)) + p, seq, timeout_ns,
                  reinterpret_cast<int*>(peers.base[rank] + comm_status_off(cap)));
    }
    __syncthreads();
    const char* box = peers.base[rank] + comm_ctrl_off(cap) + (parity * kMaxWorld + p) * kCtrlBytes;
    if (threadIdx.x < bytes) all_out[static_cast<size_t>(p) * kCtrlBytes + threadIdx.x] = *reinterpret_cast<const volatile char*>(box + threadIdx.x);
    (void)world;
}

// Ranks that share ONE device inside ONE process (development boxes, the single-GPU tests): a spinning exchange kernel
// of one rank would deadlock against anything device-wide the other rank's host thread still has to do before ITS
// exchange (lazy module loading, cudaFree, cudaMalloc of scratch that grows).  There the ranks first meet on the host,
// so every exchange kernel is launched only when all of them are about to be.  Ranks on separate GPUs never wait here.
struct HostBarrier {
    std::mutex mu;
    std::condition_variable cv;
    int world = 0, waiting = 0;
    uint64_t generation = 0;
    bool arrive_and_wait(unsigned long long timeout_ns) {
        std::unique_lock<std::mutex> lock(mu);
        const uint64_t mine = generation;
        if (++waiting == world) {
            waiting = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        return cv.wait_for(lock, std::chrono::nanoseconds(timeout_ns), [&] { return generation != mine; });
    }
};
static std::shared_ptr<HostBarrier> host_barrier_for(uint64_t key, int world) {
    static std::mutex mu;
    static std::map<uint64_t, std::weak_ptr<HostBarrier>> registry;
    std::lock_guard<std::mutex> lock(mu);
    std::shared_ptr<HostBarrier> b = registry[key].lock();
    if (!b) {
        b = std::make_shared<HostBarrier>();
        b->world = world;
        registry[key] = b;
    }
    return b;
}

// ---- NCCL, resolved at run time -----------------------------------------------------------------------------
struct NcclId {
    char internal[128];
};
struct NcclApi {
    void* lib = nullptr;
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    std::string error;
};
static NcclApi* nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (!api.lib) {
            api.error = "libnccl.so.2 could not be loaded";
            return;
        }
        api.GetUniqueId = reinterpret_cast<int (*)(NcclId*)>(dlsym(api.lib, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<int (*)(void**, int, NcclId, int)>(dlsym(api.lib, "ncclCommInitRank"));
        api.AllGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(dlsym(api.lib, "ncclAllGather"));
        api.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(api.lib, "ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(api.lib, "ncclGetErrorString"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy) api.error = "libnccl.so.2 lacks the expected symbols";
    });
    return &api;
}
static constexpr int kNcclFloat64 = 8, kNcclChar = 0;  // ncclDataType_t

}  // namespace gapa_b200

using namespace gapa_b200;

struct gapa_cuda_comm {
    int kind = GAPA_COMM_PEER;
    int rank = 0, world = 1, device = 0;
    size_t cap = 0;  // doubles per mailbox parity
    char* local = nullptr;
    CommPeers peers{};
    bool opened[kMaxWorld] = {};
    bool connected = false;
    uint32_t seq = 0, ctrl_seq = 0;
    unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
    DevBuf ctrl_stage;  // mine [kCtrlBytes] + all [world x kCtrlBytes]
    void* nccl = nullptr;
    std::shared_ptr<HostBarrier> host_barrier;  // only when ranks of this process share a device
    std::mutex mu;
};

static unsigned long long comm_timeout_ns() {
    const char* raw = std::getenv("GAPA_COMM_TIMEOUT_MS");
    const long ms = raw && *raw ? std::strtol(raw, nullptr, 10) : 20000;
    return static_cast<unsigned long long>(std::max(1L, ms)) * 1000ull * 1000ull;
}

extern "C" {

int gapa_cuda_comm_create(gapa_cuda_ctx* ctx, int rank, int world, int pop_size, gapa_cuda_comm** out, void* handle_out) {
    if (!ctx || !out || !handle_out) return fail(GAPA_CUDA_E_INVALID, "comm_create: null argument");
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return fail(GAPA_CUDA_E_INVALID, "comm_create: rank / world outside 1..%d", kMaxWorld);
    if (pop_size < 1) return fail(GAPA_CUDA_E_INVALID, "comm_create: pop_size must be >= 1");
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));
    gapa_cuda_comm* c = new gapa_cuda_comm();
    c->kind = GAPA_COMM_PEER;
    c->rank = rank;
    c->world = world;
    c->device = ctx->device;
    c->cap = static_cast<size_t>((pop_size + world - 1) / world) * world;
    c->timeout_ns = comm_timeout_ns();
    if (cudaMalloc(reinterpret_cast<void**>(&c->local), comm_bytes(c->cap)) != cudaSuccess) {
        delete c;
        return fail(GAPA_CUDA_E_NOMEM, "comm_create: cudaMalloc of the mailbox failed");
    }
    cudaMemset(c->local, 0, comm_bytes(c->cap));
    CommHandle h{};
    h.magic = kHandleMagic;
    h.device = ctx->device;
    h.pid = static_cast<int64_t>(getpid());
    h.local_ptr = reinterpret_cast<uint64_t>(c->local);
    h.capacity = c->cap;
    if (cudaIpcGetMemHandle(&h.ipc, c->local) != cudaSuccess) (void)cudaGetLastError();  // same-process peers do not need it
    std::memset(handle_out, 0, GAPA_CUDA_COMM_HANDLE_BYTES);
    std::memcpy(handle_out, &h, sizeof(h));
    *out = c;
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_connect(gapa_cuda_comm* c, const void* all_handles) {
    if (!c || !all_handles) return fail(GAPA_CUDA_E_INVALID, "comm_connect: null argument");
    if (c->kind != GAPA_COMM_PEER) return fail(GAPA_CUDA_E_INVALID, "comm_connect: not a peer-mailbox communicator");
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    const char* raw = static_cast<const char*>(all_handles);
    for (int r = 0; r < c->world; ++r) {
        CommHandle h;
        std::memcpy(&h, raw + static_cast<size_t>(r) * GAPA_CUDA_COMM_HANDLE_BYTES, sizeof(h));
        if (h.magic != kHandleMagic || h.capacity != c->cap) return fail(GAPA_CUDA_E_INVALID, "comm_connect: handle of rank %d does not match this communicator", r);
        if (r == c->rank) {
            c->peers.base[r] = c->local;
            continue;
        }
        if (h.device != c->device) {
            int can = 0;
            GAPA_CUDA_TRY(cudaDeviceCanAccessPeer(&can, c->device, h.device));
            if (!can) return fail(GAPA_CUDA_E_CUDA, "comm_connect: device %d cannot access device %d (no NVLink / PCIe peer path); use the NCCL transport", c->device, h.device);
        }
        if (h.pid == static_cast<int64_t>(getpid())) {
            if (h.device != c->device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GAPA_CUDA_TRY(e);
                (void)cudaGetLastError();
            }
            c->peers.base[r] = reinterpret_cast<char*>(h.local_ptr);
        } else {
            void* mapped = nullptr;
            GAPA_CUDA_TRY(cudaIpcOpenMemHandle(&mapped, h.ipc, cudaIpcMemLazyEnablePeerAccess));
            c->peers.base[r] = static_cast<char*>(mapped);
            c->opened[r] = true;
        }
    }
    GAPA_TRY(c->ctrl_stage.ensure(static_cast<size_t>(kCtrlBytes) * (c->world + 1)));
    cudaMemset(c->ctrl_stage.ptr, 0, c->ctrl_stage.cap);  // slots are copied back whole; only `bytes` of each are written (initcheck)
    {   // ranks of this process that share a device meet on the host before every exchange (see HostBarrier)
        bool shared_device = false, one_process = true;
        CommHandle first{};
        std::memcpy(&first, raw, sizeof(first));
        for (int r = 0; r < c->world; ++r) {
            CommHandle h;
            std::memcpy(&h, raw + static_cast<size_t>(r) * GAPA_CUDA_COMM_HANDLE_BYTES, sizeof(h));
            one_process = one_process && h.pid == static_cast<int64_t>(getpid());
            for (int q = 0; q < r; ++q) {
                CommHandle o;
                std::memcpy(&o, raw + static_cast<size_t>(q) * GAPA_CUDA_COMM_HANDLE_BYTES, sizeof(o));
                shared_device = shared_device || (o.device == h.device && o.pid == h.pid);
            }
        }
        if (shared_device && one_process) c->host_barrier = host_barrier_for(first.local_ptr, c->world);
    }
    c->connected = true;
    return GAPA_CUDA_OK;
}

int gapa_cuda_nccl_unique_id(void* id128_out) {
    if (!id128_out) return fail(GAPA_CUDA_E_INVALID, "nccl_unique_id: null argument");
    NcclApi* api = nccl_api();
    if (!api->error.empty()) return fail(GAPA_CUDA_E_CUDA, "NCCL: %s", api->error.c_str());
    NcclId id{};
    const int rc = api->GetUniqueId(&id);
    if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "ncclGetUniqueId: %s", api->GetErrorString ? api->GetErrorString(rc) : "failed");
    std::memcpy(id128_out, &id, sizeof(id));
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_create_nccl(gapa_cuda_ctx* ctx, const void* unique_id128, int rank, int world, gapa_cuda_comm** out) {
    if (!ctx || !unique_id128 || !out) return fail(GAPA_CUDA_E_INVALID, "comm_create_nccl: null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(GAPA_CUDA_E_INVALID, "comm_create_nccl: rank outside world");
    NcclApi* api = nccl_api();
    if (!api->error.empty()) return fail(GAPA_CUDA_E_CUDA, "NCCL: %s", api->error.c_str());
    GAPA_CUDA_TRY(cudaSetDevice(ctx->device));
    NcclId id;
    std::memcpy(&id, unique_id128, sizeof(id));
    gapa_cuda_comm* c = new gapa_cuda_comm();
    c->kind = GAPA_COMM_NCCL;
    c->rank = rank;
    c->world = world;
    c->device = ctx->device;
    const int rc = api->CommInitRank(&c->nccl, world, id, rank);
    if (rc != 0) {
        delete c;
        return fail(GAPA_CUDA_E_CUDA, "ncclCommInitRank: %s", api->GetErrorString ? api->GetErrorString(rc) : "failed");
    }
    if (c->ctrl_stage.ensure(static_cast<size_t>(kCtrlBytes) * (world + 1)) != GAPA_CUDA_OK) {
        api->CommDestroy(c->nccl);
        delete c;
        return GAPA_CUDA_E_NOMEM;
    }
    cudaMemset(c->ctrl_stage.ptr, 0, c->ctrl_stage.cap);
    c->connected = true;
    *out = c;
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_allgather(void* user, double* fit_full_dev, int s, int padded_block, void* stream) {
    gapa_cuda_comm* c = static_cast<gapa_cuda_comm*>(user);
    if (!c || !fit_full_dev) return fail(GAPA_CUDA_E_INVALID, "comm_allgather: null argument");
    if (!c->connected) return fail(GAPA_CUDA_E_INVALID, "comm_allgather: communicator is not connected");
    if (c->world == 1 && c->kind == GAPA_COMM_PEER) return GAPA_CUDA_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (c->kind == GAPA_COMM_NCCL) {
        NcclApi* api = nccl_api();
        const int rc = api->AllGather(fit_full_dev + static_cast<size_t>(c->rank) * padded_block, fit_full_dev,
                                      static_cast<size_t>(padded_block), kNcclFloat64, c->nccl, st);
        if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "ncclAllGather: %s", api->GetErrorString ? api->GetErrorString(rc) : "failed");
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return GAPA_CUDA_OK;
    }
    if (static_cast<size_t>(padded_block) * c->world > c->cap || padded_block * c->world < s)
        return fail(GAPA_CUDA_E_INVALID, "comm_allgather: %d x %d doubles do not fit the communicator's population size", c->world, padded_block);
    std::lock_guard<std::mutex> lock(c->mu);
    const uint32_t seq = ++c->seq;
    if (c->host_barrier) {  // ranks sharing a device in one process: push, meet on the host, pull (see HostBarrier)
        GAPA_LAUNCH(k_comm_allgather, c->world, 256, 0, st, c->peers, c->rank, c->cap, seq, fit_full_dev, padded_block,
                    static_cast<int*>(nullptr), c->timeout_ns, static_cast<int>(kPush));
        GAPA_CUDA_TRY(cudaStreamSynchronize(st));
        if (!c->host_barrier->arrive_and_wait(c->timeout_ns))
            return fail(GAPA_CUDA_E_CUDA, "comm: a rank of this process did not reach the exchange within the timeout (GAPA_COMM_TIMEOUT_MS)");
        GAPA_LAUNCH(k_comm_allgather, c->world, 256, 0, st, c->peers, c->rank, c->cap, seq, fit_full_dev, padded_block,
                    static_cast<int*>(nullptr), c->timeout_ns, static_cast<int>(kPull));
        return GAPA_CUDA_OK;
    }
    GAPA_LAUNCH(k_comm_allgather, c->world, 256, 0, st, c->peers, c->rank, c->cap, seq, fit_full_dev, padded_block,
                static_cast<int*>(nullptr), c->timeout_ns, kPush | kPull);
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_allgather_bytes(gapa_cuda_comm* c, const void* mine_host, int bytes, void* all_host) {
    if (!c || !mine_host || !all_host) return fail(GAPA_CUDA_E_INVALID, "comm_allgather_bytes: null argument");
    if (bytes < 1 || bytes > kCtrlBytes) return fail(GAPA_CUDA_E_INVALID, "comm_allgather_bytes: 1..%d bytes per rank", kCtrlBytes);
    if (!c->connected) return fail(GAPA_CUDA_E_INVALID, "comm_allgather_bytes: communicator is not connected");
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    std::lock_guard<std::mutex> lock(c->mu);
    char* mine_dev = c->ctrl_stage.as<char>();
    char* all_dev = mine_dev + kCtrlBytes;
    GAPA_CUDA_TRY(cudaMemcpy(mine_dev, mine_host, static_cast<size_t>(bytes), cudaMemcpyHostToDevice));
    if (c->kind == GAPA_COMM_NCCL) {
        NcclApi* api = nccl_api();
        GAPA_CUDA_TRY(cudaMemcpy(all_dev + static_cast<size_t>(c->rank) * kCtrlBytes, mine_dev, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice));
        const int rc = api->AllGather(all_dev + static_cast<size_t>(c->rank) * kCtrlBytes, all_dev, kCtrlBytes, kNcclChar, c->nccl, nullptr);
        if (rc != 0) return fail(GAPA_CUDA_E_CUDA, "ncclAllGather: %s", api->GetErrorString ? api->GetErrorString(rc) : "failed");
    } else {
        const uint32_t seq = ++c->ctrl_seq;
        if (c->host_barrier) {
            GAPA_LAUNCH(k_comm_ctrl, c->world, kCtrlBytes, 0, nullptr, c->peers, c->rank, c->world, c->cap, seq, mine_dev, bytes, all_dev,
                        c->timeout_ns, static_cast<int>(kPush));
            GAPA_CUDA_TRY(cudaDeviceSynchronize());
            if (!c->host_barrier->arrive_and_wait(c->timeout_ns))
                return fail(GAPA_CUDA_E_CUDA, "comm: a rank of this process did not reach the exchange within the timeout (GAPA_COMM_TIMEOUT_MS)");
            GAPA_LAUNCH(k_comm_ctrl, c->world, kCtrlBytes, 0, nullptr, c->peers, c->rank, c->world, c->cap, seq, mine_dev, bytes, all_dev,
                        c->timeout_ns, static_cast<int>(kPull));
        } else {
            GAPA_LAUNCH(k_comm_ctrl, c->world, kCtrlBytes, 0, nullptr, c->peers, c->rank, c->world, c->cap, seq, mine_dev, bytes, all_dev,
                        c->timeout_ns, kPush | kPull);
        }
    }
    GAPA_CUDA_TRY(cudaDeviceSynchronize());
    std::vector<char> all(static_cast<size_t>(c->world) * kCtrlBytes);
    GAPA_CUDA_TRY(cudaMemcpy(all.data(), all_dev, all.size(), cudaMemcpyDeviceToHost));
    for (int r = 0; r < c->world; ++r) std::memcpy(static_cast<char*>(all_host) + static_cast<size_t>(r) * bytes, all.data() + static_cast<size_t>(r) * kCtrlBytes, static_cast<size_t>(bytes));
    if (c->kind == GAPA_COMM_PEER) {
        int status = 0;
        GAPA_CUDA_TRY(cudaMemcpy(&status, c->local + comm_status_off(c->cap), sizeof(int), cudaMemcpyDeviceToHost));
        if (status) return fail(GAPA_CUDA_E_CUDA, "comm: a peer did not arrive within the timeout (GAPA_COMM_TIMEOUT_MS)");
    }
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_status(gapa_cuda_comm* c) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "comm_status: null argument");
    if (c->kind != GAPA_COMM_PEER || !c->local) return GAPA_CUDA_OK;
    GAPA_CUDA_TRY(cudaSetDevice(c->device));
    int status = 0;
    GAPA_CUDA_TRY(cudaMemcpy(&status, c->local + comm_status_off(c->cap), sizeof(int), cudaMemcpyDeviceToHost));
    if (status) return fail(GAPA_CUDA_E_CUDA, "comm: a peer did not arrive within the timeout (GAPA_COMM_TIMEOUT_MS)");
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_info(const gapa_cuda_comm* c, int* kind, int* rank, int* world) {
    if (!c) return fail(GAPA_CUDA_E_INVALID, "comm_info: null argument");
    if (kind) *kind = c->kind;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return GAPA_CUDA_OK;
}

int gapa_cuda_comm_destroy(gapa_cuda_comm* c) {
    if (!c) return GAPA_CUDA_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < c->world; ++r)
        if (c->opened[r]) cudaIpcCloseMemHandle(c->peers.base[r]);
    if (c->nccl) nccl_api()->CommDestroy(c->nccl);
    if (c->local) cudaFree(c->local);
    c->ctrl_stage.release();
    delete c;
    return GAPA_CUDA_OK;
}

// run_mode_m's shape for C / C++ hosts (modes.cpp:190-349): one process, one host thread per context (normally one per
// GPU), row blocks by partition_rows, the exchange built in.  results[r] is rank r's result (identical histories and
// populations on every rank — test_parallel.cpp:86-104; pass null output pointers where they are not wanted).
int gapa_cuda_run_multi(gapa_cuda_ctx* const* ctxs, int world, const gapa_cuda_run_params* params, int transport,
                        gapa_cuda_run_result* results) {
    if (!ctxs || !params || !results) return fail(GAPA_CUDA_E_INVALID, "run_multi: null argument");
    if (world < 1 || world > kMaxWorld) return fail(GAPA_CUDA_E_INVALID, "run_multi: world outside 1..%d", kMaxWorld);
    for (int r = 0; r < world; ++r)
        if (!ctxs[r]) return fail(GAPA_CUDA_E_INVALID, "run_multi: null context for rank %d", r);
    if (transport != GAPA_COMM_PEER && transport != GAPA_COMM_NCCL) return fail(GAPA_CUDA_E_INVALID, "run_multi: unknown transport %d", transport);
    std::vector<gapa_cuda_comm*> comms(static_cast<size_t>(world), nullptr);
    std::vector<int> status(static_cast<size_t>(world), GAPA_CUDA_OK);
    std::vector<std::string> message(static_cast<size_t>(world));
    auto cleanup = [&]() {
        for (gapa_cuda_comm* c : comms) gapa_cuda_comm_destroy(c);
    };
    NcclId id{};
    if (transport == GAPA_COMM_PEER) {
        std::vector<char> handles(static_cast<size_t>(world) * GAPA_CUDA_COMM_HANDLE_BYTES);
        for (int r = 0; r < world; ++r) {
            const int rc = gapa_cuda_comm_create(ctxs[r], r, world, params->pop_size, &comms[static_cast<size_t>(r)],
                                                 handles.data() + static_cast<size_t>(r) * GAPA_CUDA_COMM_HANDLE_BYTES);
            if (rc != GAPA_CUDA_OK) {
                cleanup();
                return rc;
            }
        }
        for (int r = 0; r < world; ++r) {
            const int rc = gapa_cuda_comm_connect(comms[static_cast<size_t>(r)], handles.data());
            if (rc != GAPA_CUDA_OK) {
                cleanup();
                return rc;
            }
        }
    } else {
        const int rc = gapa_cuda_nccl_unique_id(&id);
        if (rc != GAPA_CUDA_OK) return rc;
    }
    std::vector<std::thread> threads;
    for (int r = 0; r < world; ++r)
        threads.emplace_back([&, r] {
            int rc = GAPA_CUDA_OK;
            if (transport == GAPA_COMM_NCCL) rc = gapa_cuda_comm_create_nccl(ctxs[r], &id, r, world, &comms[static_cast<size_t>(r)]);
            if (rc == GAPA_CUDA_OK) {
                gapa_cuda_run_params p = *params;
                p.rank = r;
                p.world = world;
                rc = gapa_cuda_run(ctxs[r], &p, world > 1 ? gapa_cuda_comm_allgather : nullptr, comms[static_cast<size_t>(r)], &results[r]);
                if (rc == GAPA_CUDA_OK && world > 1) rc = gapa_cuda_comm_status(comms[static_cast<size_t>(r)]);
            }
            status[static_cast<size_t>(r)] = rc;
            if (rc != GAPA_CUDA_OK) message[static_cast<size_t>(r)] = gapa_cuda_last_error();
        });
    for (std::thread& t : threads) t.join();
    cleanup();
    for (int r = 0; r < world; ++r)
        if (status[static_cast<size_t>(r)] != GAPA_CUDA_OK) return fail(status[static_cast<size_t>(r)], "run_multi: rank %d: %s", r, message[static_cast<size_t>(r)].c_str());
    return GAPA_CUDA_OK;
}

}  // extern "C"
