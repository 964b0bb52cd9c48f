// dist.cu -- multi-GPU plumbing over NCCL (NVLink 5 / NVSwitch).
//
// One process per GPU.  libnccl.so.2 is loaded at run time (dlopen) so the
// library binds to the SAME NCCL the process's PyTorch uses (the binding sets
// AMBER_NCCL_LIB to torch's bundled copy); the communicator is our own,
// created from a unique id that rank 0 makes (amber_nccl_unique_id) and the
// caller broadcasts (e.g. torch.distributed.broadcast_object_list).
//
// Wealth sharding: agents are split in contiguous id
// ranges; each step the scatter kernel buckets cross-shard receivers per
// destination rank, this file exchanges the bucket sizes (all-to-all of one
// count per peer) and then the ids (grouped ncclSend/ncclRecv), and the
// receive kernel adds them to the owner's counters.
#include <dlfcn.h>

#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <set>

#include "internal.cuh"
#include "nccl.h"

namespace amber {

namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
    std::string error;
};

// communicators aborted by Runtime::sync (never ncclCommDestroy'd afterwards)
std::mutex& aborted_mu()
{
    static std::mutex m;
    return m;
}
std::set<void*>& aborted()
{
    static std::set<void*> s;
    return s;
}

NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* path = getenv("AMBER_NCCL_LIB");
        api.handle = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.handle) {
            api.error = std::string("dlopen NCCL failed: ") + dlerror();
            return;
        }
#define AMBER_SYM(field, sym)                                                      \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.handle, #sym));    \
    if (!api.field) api.error = "NCCL symbol missing: " #sym;
        AMBER_SYM(GetUniqueId, ncclGetUniqueId)
        AMBER_SYM(CommInitRank, ncclCommInitRank)
        AMBER_SYM(CommDestroy, ncclCommDestroy)
        AMBER_SYM(GetErrorString, ncclGetErrorString)
        AMBER_SYM(AllReduce, ncclAllReduce)
        AMBER_SYM(AllGather, ncclAllGather)
        AMBER_SYM(Send, ncclSend)
        AMBER_SYM(Recv, ncclRecv)
        AMBER_SYM(GroupStart, ncclGroupStart)
        AMBER_SYM(GroupEnd, ncclGroupEnd)
        AMBER_SYM(CommGetAsyncError, ncclCommGetAsyncError)
        AMBER_SYM(CommAbort, ncclCommAbort)
#undef AMBER_SYM
        if (api.error.empty()) {
            // Runtime::sync polls these while it waits on a stream with collectives
            g_nccl_async_error = [](void* comm, std::string* msg) -> int {
                ncclResult_t e = ncclSuccess;
                if (api.CommGetAsyncError(static_cast<ncclComm_t>(comm), &e) != ncclSuccess) return 0;
                if (e == ncclSuccess || e == ncclInProgress) return 0;
                if (msg) *msg = api.GetErrorString(e);
                return 1;
            };
            g_nccl_abort = [](void* comm) {
                api.CommAbort(static_cast<ncclComm_t>(comm));
                std::lock_guard<std::mutex> g(aborted_mu());
                aborted().insert(comm);
            };
        }
    });
    if (!api.error.empty()) fail(AMBER_E_NCCL, api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess) fail(AMBER_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

// ------------------------------------------------------------- communicator
struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
};

Comm* make_comm(const amber_runtime* r)
{
    AMBER_REQUIRE(r && r->nccl_unique_id, "a communicator needs amber_runtime.nccl_unique_id");
    const int world = r->world > 1 ? r->world : 1;
    NcclApi& api = nccl();
    ncclUniqueId id;
    std::memcpy(&id, r->nccl_unique_id, sizeof(id));
    auto* c = new Comm;
    c->rank = r->rank;
    c->world = world;
    AMBER_CUDA(cudaSetDevice(r->device));
    ncclResult_t res = api.CommInitRank(&c->comm, world, id, r->rank);
    if (res != ncclSuccess) {
        delete c;
        nccl_check(res, "ncclCommInitRank");
    }
    return c;
}

void destroy_comm(Comm* c)
{
    if (!c) return;
    bool was_aborted = false;
    {
        std::lock_guard<std::mutex> g(aborted_mu());
        was_aborted = aborted().erase(c->comm) > 0;
    }
    if (c->comm && !was_aborted) nccl().CommDestroy(c->comm);
    delete c;
}

void comm_allreduce_u64(Comm* c, cudaStream_t s, unsigned long long* d, size_t n)
{
    nccl_check(nccl().AllReduce(d, d, n, ncclUint64, ncclSum, c->comm, s), "ncclAllReduce");
}

void comm_allgather_f64(Comm* c, cudaStream_t s, const double* send, double* recv, size_t n_per_rank)
{
    nccl_check(nccl().AllGather(send, recv, n_per_rank, ncclFloat64, c->comm, s), "ncclAllGather");
}

// ---------------------------------------------------------------- loopback transport
// In-process stand-in for NCCL: `world` virtual shards of one model on ONE
// device, each driven from its own host thread.  Exchanges are host barriers
// plus device-to-device copies; no kernel ever waits on another, so it is safe
// on a single GPU.  Used by the tests to run the sharded algorithm end to end.
static const char kLoopbackMagic[8] = {'A', 'M', 'B', 'E', 'R', 'L', 'B', 0};

struct LoopbackHub {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    std::vector<std::vector<unsigned>> counts;       // [rank][peer]
    std::vector<const uint32_t*> send_ids;           // [rank]
    std::vector<uint64_t> send_cap;                  // [rank]
    std::vector<std::vector<unsigned long long>> vals;  // [rank][k]

    explicit LoopbackHub(int w) : world(w), counts(w), send_ids(w, nullptr), send_cap(w, 0), vals(w) {}

    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

std::shared_ptr<LoopbackHub> loopback_hub(const char* id, int world)
{
    static std::mutex reg_mu;
    static std::map<std::string, std::weak_ptr<LoopbackHub>> reg;
    std::lock_guard<std::mutex> g(reg_mu);
    std::string key(id, 128);
    auto it = reg.find(key);
    if (it != reg.end())
        if (auto h = it->second.lock()) {
            AMBER_REQUIRE(h->world == world, "loopback group world size mismatch");
            return h;
        }
    auto h = std::make_shared<LoopbackHub>(world);
    reg[key] = h;
    return h;
}

// Loopback all-gather of equal-size double blocks (sweep results); false if
// `r` does not name a loopback group.
bool loopback_allgather_f64(const amber_runtime* r, const std::vector<double>& mine, std::vector<double>& all)
{
    if (!r || !r->nccl_unique_id || std::memcmp(r->nccl_unique_id, kLoopbackMagic, sizeof(kLoopbackMagic)) != 0)
        return false;
    auto hub = loopback_hub(static_cast<const char*>(r->nccl_unique_id), r->world);
    std::vector<unsigned long long> bits(mine.size());
    std::memcpy(bits.data(), mine.data(), mine.size() * 8);
    hub->vals[r->rank] = bits;
    hub->barrier();
    all.assign(mine.size() * r->world, 0.0);
    for (int p = 0; p < r->world; ++p) std::memcpy(all.data() + p * mine.size(), hub->vals[p].data(), mine.size() * 8);
    hub->barrier();
    return true;
}

// ---------------------------------------------------------------- host collectives
// The caller's own host transport (amber_runtime.host_allgather / host_barrier,
// e.g. a gloo process group): used by the sharded wealth model's P2P exchange
// when no NCCL id is given -- IPC handles all-gathered on the host, one host
// barrier per step after the stream drains.
struct HostColl {
    int (*allgather)(const void*, void*, size_t, void*) = nullptr;
    int (*barrier)(void*) = nullptr;
    void* ctx = nullptr;
    bool on() const { return allgather && barrier; }
    void gather(const void* send, void* recv, size_t bytes) const
    {
        if (allgather(send, recv, bytes, ctx) != 0) fail(AMBER_E_NCCL, "host_allgather failed");
    }
    void sync() const
    {
        if (barrier(ctx) != 0) fail(AMBER_E_NCCL, "host_barrier failed");
    }
};

// ---------------------------------------------------------------- wealth exchange
struct WealthExchange {
    Comm* comm = nullptr;                 // NCCL transport
    std::shared_ptr<LoopbackHub> hub;     // or the loopback transport
    HostColl hc;                          // or the caller's host collectives (P2P exchange only)
    int rank = 0, world = 1;
    DevBuf<unsigned int> send_counts_copy, recv_counts;
    std::vector<unsigned int> h_send, h_recv;
    DevBuf<unsigned long long> flag;
};

WealthExchange* make_wealth_exchange_rt(Runtime& rt, const amber_runtime* r)
{
    auto* x = new WealthExchange;
    x->rank = rt.rank;
    x->world = rt.world;
    if (r && !r->nccl_unique_id && r->host_allgather && r->host_barrier) {
        x->hc.allgather = r->host_allgather;
        x->hc.barrier = r->host_barrier;
        x->hc.ctx = r->host_ctx;
    } else {
        if (!(r && r->nccl_unique_id)) {
            delete x;
            fail(AMBER_E_INVALID_ARG, "world > 1 needs amber_runtime.nccl_unique_id (or host collectives)");
        }
        if (std::memcmp(r->nccl_unique_id, kLoopbackMagic, sizeof(kLoopbackMagic)) == 0)
            x->hub = loopback_hub(static_cast<const char*>(r->nccl_unique_id), rt.world);
        else {
            x->comm = make_comm(r);
            rt.nccl_comms.push_back(x->comm->comm);
        }
    }
    x->send_counts_copy.allocate(&rt, rt.world);
    x->recv_counts.allocate(&rt, rt.world);
    x->flag.allocate(&rt, 1);
    x->h_send.assign(rt.world, 0);
    x->h_recv.assign(rt.world, 0);
    return x;
}

void wealth_p2p_close(WealthExchange* x);

void destroy_wealth_exchange(WealthExchange* x)
{
    if (!x) return;
    wealth_p2p_close(x);
    if (x->comm) destroy_comm(x->comm);
    x->hub.reset();
    x->send_counts_copy.reset();
    x->recv_counts.reset();
    x->flag.reset();
    delete x;
}

// Ship bucketed receivers to their owner ranks.  d_recv_total receives the
// number of ids written contiguously into d_recv_ids.
bool wealth_exchange_any(WealthExchange* x, Runtime& rt, bool local_flag);

void wealth_exchange_run(WealthExchange* x, Runtime& rt, const unsigned int* d_send_counts,
                         const uint32_t* d_send_ids, uint64_t send_cap, uint32_t* d_recv_ids,
                         unsigned long long* d_recv_total)
{
    if (x->hub) {  // loopback: post, barrier, pull the peers' buckets addressed to me, barrier
        LoopbackHub& h = *x->hub;
        const int W = x->world, me = x->rank;
        AMBER_CUDA(cudaMemcpyAsync(x->h_send.data(), d_send_counts, W * sizeof(unsigned), cudaMemcpyDeviceToHost,
                                   rt.stream));
        rt.sync();  // send buckets complete
        h.counts[me].assign(x->h_send.begin(), x->h_send.end());
        h.send_ids[me] = d_send_ids;
        h.send_cap[me] = send_cap;
        h.barrier();
        unsigned long long total = 0;
        for (int p = 0; p < W; ++p) {
            if (p == me) continue;
            const unsigned long long c = h.counts[p][me];
            if (c > h.send_cap[p]) fail(AMBER_E_CUDA, "wealth exchange: send bucket overflow");
            if (c)
                AMBER_CUDA(cudaMemcpyAsync(d_recv_ids + total, h.send_ids[p] + static_cast<uint64_t>(me) * h.send_cap[p],
                                           c * sizeof(uint32_t), cudaMemcpyDeviceToDevice, rt.stream));
            total += c;
        }
        AMBER_CUDA(cudaMemcpyAsync(d_recv_total, &total, sizeof(total), cudaMemcpyHostToDevice, rt.stream));
        rt.sync();
        h.barrier();  // peers may now reuse their send buckets
        return;
    }
    if (x->hc.on()) fail(AMBER_E_UNSUPPORTED, "host collectives carry the P2P wealth exchange only "
                                             "(AMBER_WEALTH_EXCHANGE=nccl needs an NCCL id)");
    NcclApi& api = nccl();
    const int W = x->comm->world, me = x->comm->rank;
    // 1) sizes: one count to each peer
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < W; ++p) {
        nccl_check(api.Send(d_send_counts + p, 1, ncclUint32, p, x->comm->comm, rt.stream), "ncclSend(count)");
        nccl_check(api.Recv(x->recv_counts.p + p, 1, ncclUint32, p, x->comm->comm, rt.stream), "ncclRecv(count)");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    AMBER_CUDA(cudaMemcpyAsync(x->h_send.data(), d_send_counts, W * sizeof(unsigned), cudaMemcpyDeviceToHost,
                               rt.stream));
    AMBER_CUDA(cudaMemcpyAsync(x->h_recv.data(), x->recv_counts.p, W * sizeof(unsigned), cudaMemcpyDeviceToHost,
                               rt.stream));
    rt.sync();
    // overflow is agreed on by every rank BEFORE any payload send/recv is
    // posted, so no rank throws with a group open while its peers block in
    // their matching grouped calls
    bool over = false;
    for (int p = 0; p < W; ++p)
        if (p != me && (x->h_send[p] > send_cap || x->h_recv[p] > send_cap)) over = true;
    if (wealth_exchange_any(x, rt, over)) fail(AMBER_E_CUDA, "wealth exchange: send bucket overflow (some rank)");
    // 2) payload: grouped point-to-point, received contiguously in peer order
    unsigned long long total = 0;
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < W; ++p) {
        if (p == me) continue;
        const unsigned long long ns = x->h_send[p];
        if (ns) nccl_check(api.Send(d_send_ids + p * send_cap, ns, ncclUint32, p, x->comm->comm, rt.stream), "ncclSend");
        if (x->h_recv[p])
            nccl_check(api.Recv(d_recv_ids + total, x->h_recv[p], ncclUint32, p, x->comm->comm, rt.stream), "ncclRecv");
        total += x->h_recv[p];
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    AMBER_CUDA(cudaMemcpyAsync(d_recv_total, &total, sizeof(total), cudaMemcpyHostToDevice, rt.stream));
    rt.sync();  // `total` lives on this host stack frame
}

// ---------------------------------------------------------------- wealth P2P exchange
// The fused compute + transfer path: every rank keeps its send
// buckets (both step parities, one cudaMalloc) mapped into its peers' address
// spaces; after a stream-ordered barrier the owner's receive kernel reads the
// buckets addressed to it straight out of the peers' memory over NVLink and
// applies them as counter atomics -- no counts round trip through the host,
// no staging copies.  Mapping: CUDA IPC handles all-gathered over NCCL
// (multi-process) or raw pointers through the hub (loopback, one process).
struct P2PMap {
    std::vector<void*> peers;   // [world] base of each rank's bucket block (mine included)
    std::vector<bool> opened;   // IPC-opened (to close)
    DevBuf<unsigned int> token; // 1-element barrier all-reduce
};

// Registry of the open mappings.  Ranks of a loopback group open and close
// theirs from their own host threads, so every access holds p2p_mu.
static std::mutex p2p_mu;
static std::map<WealthExchange*, std::unique_ptr<P2PMap>>& p2p_maps()
{
    static std::map<WealthExchange*, std::unique_ptr<P2PMap>> m;
    return m;
}

// Maps my bucket block into every peer; false (on every rank) if any rank cannot.
bool wealth_p2p_open(WealthExchange* x, Runtime& rt, void* my_base, std::vector<void*>& peers)
{
    auto map = std::make_unique<P2PMap>();
    const int W = x->world, me = x->rank;
    map->peers.assign(W, nullptr);
    map->opened.assign(W, false);
    if (x->hub) {
        LoopbackHub& h = *x->hub;
        h.send_ids[me] = static_cast<const uint32_t*>(my_base);
        h.barrier();
        for (int p = 0; p < W; ++p) map->peers[p] = const_cast<uint32_t*>(h.send_ids[p]);
        h.barrier();
    } else if (x->hc.on()) {
        // cross-process mapping: CUDA IPC handles all-gathered over the host transport
        bool ok = true;
        std::string why;
        cudaIpcMemHandle_t mine;
        std::memset(&mine, 0, sizeof(mine));
        cudaError_t e = cudaIpcGetMemHandle(&mine, my_base);
        if (e != cudaSuccess) {
            ok = false;
            why = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
        }
        cudaGetLastError();
        std::vector<cudaIpcMemHandle_t> hs(W);
        x->hc.gather(&mine, hs.data(), sizeof(mine));
        map->peers[me] = my_base;
        for (int p = 0; p < W && ok; ++p) {
            if (p == me) continue;
            void* ptr = nullptr;
            e = cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                ok = false;
                why = std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(p) + "): " + cudaGetErrorString(e);
                break;
            }
            map->peers[p] = ptr;
            map->opened[p] = true;
        }
        const int bad = ok ? 0 : 1;
        std::vector<int> all(W);
        x->hc.gather(&bad, all.data(), sizeof(int));  // every rank takes the same path
        for (int v : all)
            if (v) ok = false;
        if (!ok) {
            for (int p = 0; p < W; ++p)
                if (map->opened[p]) cudaIpcCloseMemHandle(map->peers[p]);
            fail(AMBER_E_CUDA, "host-collective P2P exchange: a rank could not map its peers' buckets" +
                                   (why.empty() ? std::string(" (another rank failed)") : ": " + why));
        }
    } else {
        bool ok = true;
        cudaIpcMemHandle_t mine;
        if (cudaIpcGetMemHandle(&mine, my_base) != cudaSuccess) ok = false;
        cudaGetLastError();
        DevBuf<char> all;
        all.allocate(&rt, static_cast<size_t>(W) * sizeof(mine));
        DevBuf<char> one;
        one.allocate(&rt, sizeof(mine));
        AMBER_CUDA(cudaMemcpyAsync(one.p, &mine, sizeof(mine), cudaMemcpyHostToDevice, rt.stream));
        nccl_check(nccl().AllGather(one.p, all.p, sizeof(mine), ncclChar, x->comm->comm, rt.stream), "ncclAllGather(ipc)");
        std::vector<cudaIpcMemHandle_t> hs(W);
        AMBER_CUDA(cudaMemcpyAsync(hs.data(), all.p, W * sizeof(mine), cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        map->peers[me] = my_base;
        for (int p = 0; p < W && ok; ++p) {
            if (p == me) continue;
            void* ptr = nullptr;
            if (cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                ok = false;
                break;
            }
            map->peers[p] = ptr;
            map->opened[p] = true;
        }
        // every rank must take the same path
        DevBuf<unsigned long long> flag;
        flag.allocate(&rt, 1);
        unsigned long long bad = ok ? 0ull : 1ull;
        AMBER_CUDA(cudaMemcpyAsync(flag.p, &bad, 8, cudaMemcpyHostToDevice, rt.stream));
        comm_allreduce_u64(x->comm, rt.stream, flag.p, 1);
        AMBER_CUDA(cudaMemcpyAsync(&bad, flag.p, 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        if (bad) {
            for (int p = 0; p < W; ++p)
                if (map->opened[p]) cudaIpcCloseMemHandle(map->peers[p]);
            return false;
        }
        map->token.allocate(&rt, 1);
        map->token.zero_async(rt.stream);
    }
    peers = map->peers;
    std::lock_guard<std::mutex> g(p2p_mu);
    p2p_maps()[x] = std::move(map);
    return true;
}

void wealth_p2p_close(WealthExchange* x)
{
    std::lock_guard<std::mutex> g(p2p_mu);
    auto it = p2p_maps().find(x);
    if (it == p2p_maps().end()) return;
    for (size_t p = 0; p < it->second->peers.size(); ++p)
        if (it->second->opened[p]) cudaIpcCloseMemHandle(it->second->peers[p]);
    p2p_maps().erase(it);
}

// Every rank's buckets of this step are complete before anyone reads them:
// a one-element all-reduce on the stream (NCCL; no host round trip), or a
// host barrier after the stream drains (loopback).
void wealth_p2p_barrier(WealthExchange* x, Runtime& rt)
{
    if (x->hub) {
        rt.sync();
        x->hub->barrier();
        return;
    }
    if (x->hc.on()) {
        rt.sync();
        x->hc.sync();
        return;
    }
    P2PMap* mp;
    {
        std::lock_guard<std::mutex> g(p2p_mu);
        mp = p2p_maps().at(x).get();
    }
    P2PMap& m = *mp;
    nccl_check(nccl().AllReduce(m.token.p, m.token.p, 1, ncclUint32, ncclSum, x->comm->comm, rt.stream),
               "ncclAllReduce(barrier)");
}

// loopback all-reduce (sum) of n host values
static std::vector<unsigned long long> loopback_sum(WealthExchange* x, const std::vector<unsigned long long>& mine)
{
    LoopbackHub& h = *x->hub;
    h.vals[x->rank] = mine;
    h.barrier();
    std::vector<unsigned long long> out(mine.size(), 0ull);
    for (int p = 0; p < x->world; ++p)
        for (size_t k = 0; k < out.size(); ++k) out[k] += h.vals[p][k];
    h.barrier();
    return out;
}

// host-collective all-reduce (sum) of n host values
static std::vector<unsigned long long> host_sum(WealthExchange* x, const std::vector<unsigned long long>& mine)
{
    std::vector<unsigned long long> all(mine.size() * x->world), out(mine.size(), 0ull);
    x->hc.gather(mine.data(), all.data(), mine.size() * 8);
    for (int p = 0; p < x->world; ++p)
        for (size_t k = 0; k < out.size(); ++k) out[k] += all[p * mine.size() + k];
    return out;
}

bool wealth_exchange_any(WealthExchange* x, Runtime& rt, bool local_flag)
{
    if (x->hub) return loopback_sum(x, {local_flag ? 1ull : 0ull})[0] != 0;
    if (x->hc.on()) return host_sum(x, {local_flag ? 1ull : 0ull})[0] != 0;
    unsigned long long v = local_flag ? 1ull : 0ull;
    AMBER_CUDA(cudaMemcpyAsync(x->flag.p, &v, 8, cudaMemcpyHostToDevice, rt.stream));
    comm_allreduce_u64(x->comm, rt.stream, x->flag.p, 1);
    AMBER_CUDA(cudaMemcpyAsync(&v, x->flag.p, 8, cudaMemcpyDeviceToHost, rt.stream));
    rt.sync();
    return v != 0;
}

void wealth_exchange_allreduce_u64(WealthExchange* x, Runtime& rt, unsigned long long* d_vals, int n)
{
    if (x->hub || x->hc.on()) {
        std::vector<unsigned long long> h(n);
        AMBER_CUDA(cudaMemcpyAsync(h.data(), d_vals, n * 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        h = x->hub ? loopback_sum(x, h) : host_sum(x, h);
        AMBER_CUDA(cudaMemcpyAsync(d_vals, h.data(), n * 8, cudaMemcpyHostToDevice, rt.stream));
        rt.sync();
        return;
    }
    comm_allreduce_u64(x->comm, rt.stream, d_vals, static_cast<size_t>(n));
}

// ---------------------------------------------------------------- generic shard communicator
// All-gather / all-reduce for the sharded models other than wealth (SIR:
// per-step all-gather of the I bitmap), over NCCL or the loopback transport.
struct ShardComm {
    Comm* comm = nullptr;
    std::shared_ptr<LoopbackHub> hub;
    int rank = 0, world = 1;
    std::vector<const void*> peers;  // loopback: posted send buffers
};

ShardComm* make_shard_comm(Runtime& rt, const amber_runtime* r)
{
    AMBER_REQUIRE(r && r->nccl_unique_id, "world > 1 needs amber_runtime.nccl_unique_id");
    auto* c = new ShardComm;
    c->rank = rt.rank;
    c->world = rt.world;
    if (std::memcmp(r->nccl_unique_id, kLoopbackMagic, sizeof(kLoopbackMagic)) == 0)
        c->hub = loopback_hub(static_cast<const char*>(r->nccl_unique_id), rt.world);
    else {
        c->comm = make_comm(r);
        rt.nccl_comms.push_back(c->comm->comm);
    }
    return c;
}

void destroy_shard_comm(ShardComm* c)
{
    if (!c) return;
    if (c->comm) destroy_comm(c->comm);
    c->hub.reset();
    delete c;
}

// recv[p * count + k] = send of rank p, k < count (device buffers, stream-ordered).
void shard_allgather_u32(ShardComm* c, Runtime& rt, const uint32_t* send, uint32_t* recv, size_t count)
{
    if (c->hub) {
        LoopbackHub& h = *c->hub;
        rt.sync();  // my send block is complete
        {
            std::lock_guard<std::mutex> g(h.mu);
            if (h.vals[c->rank].size() < 1) h.vals[c->rank].resize(1);
            h.vals[c->rank][0] = reinterpret_cast<unsigned long long>(send);
        }
        h.barrier();
        for (int p = 0; p < c->world; ++p) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(h.vals[p][0]);
            AMBER_CUDA(cudaMemcpyAsync(recv + p * count, src, count * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                       rt.stream));
        }
        rt.sync();
        h.barrier();  // peers may now overwrite their send blocks
        return;
    }
    nccl_check(nccl().AllGather(send, recv, count, ncclUint32, c->comm->comm, rt.stream), "ncclAllGather");
}

// Variable all-to-all of fixed-size elements.  send holds `world` blocks of
// `cap` elements (block p for rank p), d_counts[p] elements of block p are
// valid.  The received elements are stored contiguously in peer order in recv
// (capacity recv_cap elements); returns their number.  Synchronising.
uint64_t shard_alltoallv(ShardComm* c, Runtime& rt, const void* send, const uint32_t* d_counts, size_t cap,
                         size_t elem, void* recv, size_t recv_cap)
{
    const int W = c->world, me = c->rank;
    std::vector<uint32_t> hs(W);
    AMBER_CUDA(cudaMemcpyAsync(hs.data(), d_counts, W * sizeof(uint32_t), cudaMemcpyDeviceToHost, rt.stream));
    rt.sync();  // counts and send blocks complete
    for (int p = 0; p < W; ++p)
        if (hs[p] > cap) fail(AMBER_E_CUDA, "shard exchange: send bucket overflow (capacity " + std::to_string(cap) + ")");
    const char* sb = static_cast<const char*>(send);
    char* rb = static_cast<char*>(recv);
    if (c->hub) {
        LoopbackHub& h = *c->hub;
        h.counts[me].assign(hs.begin(), hs.end());
        h.send_ids[me] = static_cast<const uint32_t*>(send);
        h.send_cap[me] = cap;
        h.barrier();
        uint64_t total = 0;
        for (int p = 0; p < W; ++p) {
            const uint64_t k = h.counts[p][me];
            if (total + k > recv_cap) fail(AMBER_E_CUDA, "shard exchange: receive buffer overflow");
            if (k)
                AMBER_CUDA(cudaMemcpyAsync(rb + total * elem,
                                           reinterpret_cast<const char*>(h.send_ids[p]) + static_cast<uint64_t>(me) * cap * elem,
                                           k * elem, cudaMemcpyDeviceToDevice, rt.stream));
            total += k;
        }
        rt.sync();
        h.barrier();  // peers may now reuse their send blocks
        return total;
    }
    NcclApi& api = nccl();
    DevBuf<uint32_t> rc;
    rc.allocate(&rt, W);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < W; ++p) {
        nccl_check(api.Send(d_counts + p, 1, ncclUint32, p, c->comm->comm, rt.stream), "ncclSend(count)");
        nccl_check(api.Recv(rc.p + p, 1, ncclUint32, p, c->comm->comm, rt.stream), "ncclRecv(count)");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    std::vector<uint32_t> hr(W);
    AMBER_CUDA(cudaMemcpyAsync(hr.data(), rc.p, W * sizeof(uint32_t), cudaMemcpyDeviceToHost, rt.stream));
    rt.sync();
    uint64_t total = 0;
    for (int p = 0; p < W; ++p) total += hr[p];
    if (total > recv_cap) fail(AMBER_E_CUDA, "shard exchange: receive buffer overflow");
    uint64_t off = 0;
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < W; ++p) {
        if (hs[p])
            nccl_check(api.Send(sb + static_cast<uint64_t>(p) * cap * elem, hs[p] * elem, ncclChar, p, c->comm->comm,
                                rt.stream), "ncclSend");
        if (hr[p]) nccl_check(api.Recv(rb + off * elem, hr[p] * elem, ncclChar, p, c->comm->comm, rt.stream), "ncclRecv");
        off += hr[p];
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    rt.sync();
    return total;
}

// In-place sum over ranks of n device values.
void shard_allreduce_u64(ShardComm* c, Runtime& rt, unsigned long long* d, size_t n)
{
    if (c->hub) {
        LoopbackHub& h = *c->hub;
        std::vector<unsigned long long> mine(n);
        AMBER_CUDA(cudaMemcpyAsync(mine.data(), d, n * 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        h.vals[c->rank] = mine;
        h.barrier();
        std::vector<unsigned long long> out(n, 0ull);
        for (int p = 0; p < c->world; ++p)
            for (size_t k = 0; k < n; ++k) out[k] += h.vals[p][k];
        h.barrier();
        AMBER_CUDA(cudaMemcpyAsync(d, out.data(), n * 8, cudaMemcpyHostToDevice, rt.stream));
        rt.sync();
        return;
    }
    comm_allreduce_u64(c->comm, rt.stream, d, n);
}

}  // namespace amber

extern "C" int amber_loopback_id_impl(void* out, size_t out_bytes)
{
    using namespace amber;
    AMBER_REQUIRE(out && out_bytes >= 128, "amber_loopback_id needs a 128-byte buffer");
    static std::atomic<unsigned long long> counter{1};
    char id[128] = {0};
    std::memcpy(id, kLoopbackMagic, sizeof(kLoopbackMagic));
    const unsigned long long k = counter.fetch_add(1);
    std::memcpy(id + 8, &k, sizeof(k));
    std::memcpy(out, id, 128);
    return 0;
}

extern "C" int amber_nccl_unique_id_impl(void* out, size_t out_bytes)
{
    using namespace amber;
    AMBER_REQUIRE(out && out_bytes >= sizeof(ncclUniqueId), "amber_nccl_unique_id needs a 128-byte buffer");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
    return 0;
}
