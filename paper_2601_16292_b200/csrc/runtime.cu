// runtime.cu -- runtime binding, allocator hooks, profiler, column/metric
// copies and the generic digest reduction (product path).
#include <chrono>
#include <cstdlib>
#include <thread>

#include "internal.cuh"

namespace amber {

void Runtime::init(const amber_runtime* r)
{
    device = r ? r->device : 0;
    AMBER_CUDA(cudaSetDevice(device));
    if (r && r->stream) {
        stream = static_cast<cudaStream_t>(r->stream);
        own_stream = false;
    } else {
        AMBER_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        own_stream = true;
    }
    if (r && r->alloc) {
        AMBER_REQUIRE(r->free != nullptr, "amber_runtime.alloc set without .free");
        alloc = r->alloc;
        release = r->free;
        ctx = r->alloc_ctx;
    }
    rank = r ? r->rank : 0;
    world = (r && r->world > 1) ? r->world : 1;
    AMBER_REQUIRE(rank >= 0 && rank < world, "amber_runtime.rank out of [0, world)");
    AMBER_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
}

int (*g_nccl_async_error)(void* comm, std::string* msg) = nullptr;
void (*g_nccl_abort)(void* comm) = nullptr;

void Runtime::sync()
{
    if (nccl_comms.empty() || !g_nccl_async_error) {
        AMBER_CUDA(cudaStreamSynchronize(stream));
        return;
    }
    static const double limit = [] {
        const char* v = std::getenv("AMBER_NCCL_TIMEOUT_S");
        return v && *v ? std::atof(v) : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (long it = 0;; ++it) {
        const cudaError_t q = cudaStreamQuery(stream);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) AMBER_CUDA(q);
        std::string msg;
        for (void* c : nccl_comms)
            if (g_nccl_async_error(c, &msg)) {
                for (void* d : nccl_comms) g_nccl_abort(d);
                nccl_comms.clear();
                fail(AMBER_E_NCCL, "NCCL asynchronous error: " + msg);
            }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit) {
            for (void* d : nccl_comms) g_nccl_abort(d);
            nccl_comms.clear();
            fail(AMBER_E_NCCL, "NCCL wait exceeded AMBER_NCCL_TIMEOUT_S (a peer rank stopped?); communicators aborted");
        }
        if (it > 2000) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

void Runtime::destroy()
{
    if (own_stream && stream) cudaStreamDestroy(stream);
    stream = nullptr;
}

void* Runtime::alloc_bytes(size_t bytes)
{
    void* p = nullptr;
    if (alloc) {
        p = alloc(bytes, stream, ctx);
        if (!p) fail(AMBER_E_OOM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes");
    } else {
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(AMBER_E_OOM, "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
        }
    }
    return p;
}

void Runtime::free_bytes(void* p, size_t bytes)
{
    if (!p) return;
    if (release)
        release(p, bytes, stream, ctx);
    else
        cudaFree(p);
}

// ---------------------------------------------------------------- profiler
cudaEvent_t Profiler::get_event()
{
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    AMBER_CUDA(cudaEventCreate(&e));
    return e;
}

void Profiler::clear()
{
    for (auto& k : kernels)
        for (auto& pr : k.ev) {
            pool.push_back(pr.first);
            pool.push_back(pr.second);
        }
    kernels.clear();
}

bool Profiler::query(int idx, std::string* name, int64_t* launches, double* total_ms)
{
    if (idx < 0 || idx >= static_cast<int>(kernels.size())) return false;
    auto& k = kernels[idx];
    double ms = 0;
    for (auto& pr : k.ev) {
        AMBER_CUDA(cudaEventSynchronize(pr.second));
        float f = 0;
        AMBER_CUDA(cudaEventElapsedTime(&f, pr.first, pr.second));
        ms += f;
    }
    *name = k.name;
    *launches = static_cast<int64_t>(k.ev.size());
    *total_ms = ms;
    return true;
}

Profiler::~Profiler()
{
    clear();
    for (auto e : pool) cudaEventDestroy(e);
}

// ---------------------------------------------------------------- options
bool Model::set_option(const char* key, int64_t v)
{
    std::string k(key);
    if (k == "block") {
        AMBER_REQUIRE(v == 0 || (v >= 32 && v <= 1024 && v % 32 == 0), "block must be 0 or a multiple of 32 in [32,1024]");
        block = v;
    } else if (k == "grid") {
        AMBER_REQUIRE(v >= 0, "grid must be >= 0");
        grid = v;
    } else if (k == "persistent") {
        persistent = v ? 1 : 0;
    } else if (k == "digest") {
        digest_on = v ? 1 : 0;
    } else {
        return false;
    }
    return true;
}

bool Model::get_option(const char* key, int64_t* v)
{
    std::string k(key);
    if (k == "block") *v = block;
    else if (k == "grid") *v = grid;
    else if (k == "persistent") *v = persistent;
    else if (k == "digest") *v = digest_on;
    else if (k == "metrics_capacity") *v = metrics_cap;
    else return false;
    return true;
}

// ---------------------------------------------------------------- copies
void copy_out(Runtime& rt, void* dst, const void* src, size_t bytes, bool dst_on_dev)
{
    if (!bytes) return;
    AMBER_CUDA(cudaMemcpyAsync(dst, src, bytes, dst_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               rt.stream));
    rt.sync();
}

void copy_in(Runtime& rt, void* dst, const void* src, size_t bytes, bool src_on_dev)
{
    if (!bytes) return;
    AMBER_CUDA(cudaMemcpyAsync(dst, src, bytes, src_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               rt.stream));
    rt.sync();
}

template <class T>
void read_ring(Runtime& rt, const T* ring, int64_t cap, int64_t first, int64_t end, void* dst, size_t bytes,
               int64_t* n_out)
{
    int64_t lo = first > end - cap ? first : end - cap;
    int64_t n = end > lo ? end - lo : 0;
    if (bytes < static_cast<size_t>(n) * sizeof(T))
        fail(AMBER_E_BUFFER_TOO_SMALL, "metrics buffer too small: need " + std::to_string(n * sizeof(T)) + " bytes");
    std::vector<T> host(cap);
    AMBER_CUDA(cudaMemcpyAsync(host.data(), ring, cap * sizeof(T), cudaMemcpyDeviceToHost, rt.stream));
    rt.sync();
    T* out = static_cast<T*>(dst);
    for (int64_t s = lo; s < end; ++s) out[s - lo] = host[s % cap];
    if (n_out) *n_out = n;
}

template void read_ring<int64_t>(Runtime&, const int64_t*, int64_t, int64_t, int64_t, void*, size_t, int64_t*);
template void read_ring<uint64_t>(Runtime&, const uint64_t*, int64_t, int64_t, int64_t, void*, size_t, int64_t*);
template void read_ring<double>(Runtime&, const double*, int64_t, int64_t, int64_t, void*, size_t, int64_t*);

// ---------------------------------------------------------------- digest
template <class T>
__global__ void digest_kernel(const T* __restrict__ col, int64_t n, int64_t id0, unsigned long long* out)
{
    unsigned long long acc[1] = {0ull};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t bits;
        if constexpr (sizeof(T) == 1)
            bits = static_cast<uint32_t>(col[i]);
        else
            bits = static_cast<uint32_t>(col[i]);
        acc[0] += digest_term(static_cast<unsigned long long>(id0 + i), bits);
    }
    unsigned long long* const outs[1] = {out};
    block_sum_atomic<1>(acc, outs);
}

template <class T>
static uint64_t device_digest(Runtime& rt, const T* col, int64_t n, int64_t id0)
{
    DevBuf<unsigned long long> acc;
    acc.allocate(&rt, 1);
    acc.zero_async(rt.stream);
    int grid = static_cast<int>(std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1), 256), rt.num_sms * 8));
    digest_kernel<T><<<grid, 256, 0, rt.stream>>>(col, n, id0, acc.p);
    check_launch("digest_kernel");
    unsigned long long h = 0;
    AMBER_CUDA(cudaMemcpyAsync(&h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, rt.stream));
    rt.sync();
    return h;
}

uint64_t device_digest_u32(Runtime& rt, const uint32_t* col, int64_t n, int64_t id0)
{
    return device_digest<uint32_t>(rt, col, n, id0);
}

uint64_t device_digest_u8(Runtime& rt, const uint8_t* col, int64_t n, int64_t id0)
{
    return device_digest<uint8_t>(rt, col, n, id0);
}

}  // namespace amber
