// population.cu -- generic device Population: the paper's
// columnar API (Sec. 3.1.2 lines 85-96, Listing 1; Sec. 3.3;
// Sec. 6.2) with SPEC's semantics (columnar-core module): typed
// columns, tombstone alive mask, stable never-reused ids (rows stay sorted by
// id, so id -> row is a binary search), order-preserving compaction, and
// population-wide updates / aggregates given as postfix expression programs
// that one kernel evaluates per row (a tiny vectorised expression engine:
// Listing 1's `wealth + 10` is [COL wealth][CONST 10][ADD]).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cub/cub.cuh>
#include <map>
#include <mutex>

#include "internal.cuh"
#include "philox.cuh"

namespace amber {

namespace {

constexpr int kMaxProg = 64, kMaxStack = 8, kMaxCols = 32;
constexpr int kThreads = 256, kRPT = 4, kTile = kThreads * kRPT;   // rows per tile
constexpr size_t kStackBytes = kMaxStack * kTile * sizeof(double);   // 64 KB per block

struct Prog {
    int n;
    int uses_id;    // program reads the agent id (ID / RAND): load the id column
    int max_depth;  // deepest stack the program reaches (sizes the shared stack tile)
    amber_instr ins[kMaxProg];
};

struct ColView {
    void* p;
    int dtype;
};

struct Cols {
    ColView c[kMaxCols];
    int n;
};

__device__ __forceinline__ double load_col(const ColView& c, int64_t row)
{
    switch (c.dtype) {
        case AMBER_I32: return static_cast<double>(static_cast<const int32_t*>(c.p)[row]);
        case AMBER_I64: return static_cast<double>(static_cast<const int64_t*>(c.p)[row]);
        case AMBER_F32: return static_cast<double>(static_cast<const float*>(c.p)[row]);
        case AMBER_F64: return static_cast<const double*>(c.p)[row];
        default: return static_cast<double>(static_cast<const uint8_t*>(c.p)[row]);
    }
}

__device__ __forceinline__ void store_col(const ColView& c, int64_t row, double v)
{
    switch (c.dtype) {
        case AMBER_I32: static_cast<int32_t*>(c.p)[row] = static_cast<int32_t>(v); break;
        case AMBER_I64: static_cast<int64_t*>(c.p)[row] = static_cast<int64_t>(v); break;
        case AMBER_F32: static_cast<float*>(c.p)[row] = static_cast<float>(v); break;
        case AMBER_F64: static_cast<double*>(c.p)[row] = v; break;
        default: static_cast<uint8_t*>(c.p)[row] = static_cast<uint8_t>(v); break;
    }
}

// Columnar stack machine: every instruction is applied to a whole tile of
// kTile rows before the next one (as a column engine would), so the dispatch
// is amortised over the tile.  Thread tid owns rows tid, tid+256, ... of the
// tile (coalesced column loads) and only ever touches its own rows' stack
// slots, so no barrier is needed between instructions.  stk[slot*kTile + j].
__device__ void eval_tile(const Prog& P, const Cols& C, int64_t row0, int64_t rows, const int64_t* __restrict__ ids,
                          uint32_t step, const PhiloxKey& key, double* stk)
{
    const int tid = threadIdx.x;
    int sp = 0;
    for (int k = 0; k < P.n; ++k) {
        const amber_instr in = P.ins[k];
        switch (in.op) {
            case AMBER_OP_CONST:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) stk[sp * kTile + m * kThreads + tid] = in.value;
                ++sp;
                break;
            case AMBER_OP_COL: {
                double v[kRPT];
#pragma unroll
                for (int m = 0; m < kRPT; ++m) {
                    const int64_t r = row0 + m * kThreads + tid;
                    v[m] = r < rows ? load_col(C.c[in.arg], r) : 0.0;
                }
#pragma unroll
                for (int m = 0; m < kRPT; ++m) stk[sp * kTile + m * kThreads + tid] = v[m];
                ++sp;
                break;
            }
            case AMBER_OP_ID:
            case AMBER_OP_RAND:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) {
                    const int64_t r = row0 + m * kThreads + tid;
                    const int64_t id = r < rows ? ids[r] : 0;
                    double v = static_cast<double>(id);
                    if (in.op == AMBER_OP_RAND) {
                        const uint4 w = stream_block(key, static_cast<uint32_t>(in.arg),
                                                     static_cast<unsigned long long>(id) >> 2, step);
                        const uint32_t q = static_cast<uint32_t>(id & 3);
                        v = static_cast<double>(u01(q == 0 ? w.x : (q == 1 ? w.y : (q == 2 ? w.z : w.w))));
                    }
                    stk[sp * kTile + m * kThreads + tid] = v;
                }
                ++sp;
                break;
            case AMBER_OP_STEP:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) stk[sp * kTile + m * kThreads + tid] = static_cast<double>(step);
                ++sp;
                break;
            case AMBER_OP_NEG:
            case AMBER_OP_ABS:
            case AMBER_OP_FLOOR:
            case AMBER_OP_SQRT:
            case AMBER_OP_NOT:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) {
                    double& a = stk[(sp - 1) * kTile + m * kThreads + tid];
                    switch (in.op) {
                        case AMBER_OP_NEG: a = -a; break;
                        case AMBER_OP_ABS: a = fabs(a); break;
                        case AMBER_OP_FLOOR: a = floor(a); break;
                        case AMBER_OP_SQRT: a = sqrt(a); break;
                        default: a = a == 0.0 ? 1.0 : 0.0; break;
                    }
                }
                break;
            case AMBER_OP_SELECT:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) {
                    const int j = m * kThreads + tid;
                    const double b = stk[(sp - 1) * kTile + j], a = stk[(sp - 2) * kTile + j],
                                 c = stk[(sp - 3) * kTile + j];
                    stk[(sp - 3) * kTile + j] = c != 0.0 ? a : b;
                }
                sp -= 2;
                break;
            default:
#pragma unroll
                for (int m = 0; m < kRPT; ++m) {
                    const int j = m * kThreads + tid;
                    const double b = stk[(sp - 1) * kTile + j], a = stk[(sp - 2) * kTile + j];
                    double r = 0.0;
                    switch (in.op) {
                        case AMBER_OP_ADD: r = a + b; break;
                        case AMBER_OP_SUB: r = a - b; break;
                        case AMBER_OP_MUL: r = a * b; break;
                        case AMBER_OP_DIV: r = a / b; break;
                        case AMBER_OP_MIN: r = fmin(a, b); break;
                        case AMBER_OP_MAX: r = fmax(a, b); break;
                        case AMBER_OP_LT: r = a < b; break;
                        case AMBER_OP_LE: r = a <= b; break;
                        case AMBER_OP_GT: r = a > b; break;
                        case AMBER_OP_GE: r = a >= b; break;
                        case AMBER_OP_EQ: r = a == b; break;
                        case AMBER_OP_NE: r = a != b; break;
                        case AMBER_OP_AND: r = (a != 0.0) && (b != 0.0); break;
                        case AMBER_OP_OR: r = (a != 0.0) || (b != 0.0); break;
                        default: break;
                    }
                    stk[(sp - 2) * kTile + j] = r;
                }
                --sp;
        }
    }
}

__global__ void __launch_bounds__(kThreads) pop_update_kernel(Prog expr, Prog where, Cols C, int target,
                                                              const int64_t* __restrict__ ids,
                                                              const uint8_t* __restrict__ alive, int64_t rows,
                                                              uint32_t step, PhiloxKey key,
                                                              unsigned long long* n_updated)
{
    extern __shared__ double stk[];
    unsigned long long cnt = 0;
    const int tid = threadIdx.x;
    for (int64_t row0 = static_cast<int64_t>(blockIdx.x) * kTile; row0 < rows; row0 += static_cast<int64_t>(gridDim.x) * kTile) {
        bool sel[kRPT];
#pragma unroll
        for (int m = 0; m < kRPT; ++m) {
            const int64_t r = row0 + m * kThreads + tid;
            sel[m] = r < rows && alive[r];
        }
        if (where.n) {
            eval_tile(where, C, row0, rows, ids, step, key, stk);
#pragma unroll
            for (int m = 0; m < kRPT; ++m) sel[m] = sel[m] && stk[m * kThreads + tid] != 0.0;
        }
        eval_tile(expr, C, row0, rows, ids, step, key, stk);  // all reads of a row happen before its write
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
            if (sel[m]) {
                store_col(C.c[target], row0 + m * kThreads + tid, stk[m * kThreads + tid]);
                ++cnt;
            }
    }
    unsigned long long vals[1] = {cnt};
    unsigned long long* const outs[1] = {n_updated};
    block_sum_atomic<1>(vals, outs);
}

// Per-block partials (sum, min, max, count), reduced on the host in block order.
__global__ void __launch_bounds__(kThreads) pop_aggregate_kernel(Prog expr, Prog where, Cols C,
                                                                 const int64_t* __restrict__ ids,
                                                                 const uint8_t* __restrict__ alive, int64_t rows,
                                                                 uint32_t step, PhiloxKey key, double* partial)
{
    extern __shared__ double stk[];
    double s = 0.0, mn = INFINITY, mx = -INFINITY, c = 0.0;
    const int tid = threadIdx.x;
    for (int64_t row0 = static_cast<int64_t>(blockIdx.x) * kTile; row0 < rows; row0 += static_cast<int64_t>(gridDim.x) * kTile) {
        bool sel[kRPT];
#pragma unroll
        for (int m = 0; m < kRPT; ++m) {
            const int64_t r = row0 + m * kThreads + tid;
            sel[m] = r < rows && alive[r];
        }
        if (where.n) {
            eval_tile(where, C, row0, rows, ids, step, key, stk);
#pragma unroll
            for (int m = 0; m < kRPT; ++m) sel[m] = sel[m] && stk[m * kThreads + tid] != 0.0;
        }
        if (expr.n) eval_tile(expr, C, row0, rows, ids, step, key, stk);
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
            if (sel[m]) {
                const double v = expr.n ? stk[m * kThreads + tid] : 0.0;
                s += v;
                mn = fmin(mn, v);
                mx = fmax(mx, v);
                c += 1.0;
            }
    }
    __shared__ double red[4][32];
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
        red[0][wid] = s;
        red[1][wid] = mn;
        red[2][wid] = mx;
        red[3][wid] = c;
    }
    __syncthreads();
    if (tid == 0) {
        double S = 0, MN = INFINITY, MX = -INFINITY, CC = 0;
        for (int w = 0; w < nw; ++w) {
            S += red[0][w];
            MN = fmin(MN, red[1][w]);
            MX = fmax(MX, red[2][w]);
            CC += red[3][w];
        }
        partial[4 * blockIdx.x + 0] = S;
        partial[4 * blockIdx.x + 1] = MN;
        partial[4 * blockIdx.x + 2] = MX;
        partial[4 * blockIdx.x + 3] = CC;
    }
}

// Fast path for the most common update shape (Listing 1):
// target = col[a] OP (constant | col[b]), no filter.  8 rows per thread with
// every load issued before the first use (memory-level parallelism); same
// double arithmetic and store conversion as the interpreter.
constexpr int kBinRows = 8;

__global__ void __launch_bounds__(256) pop_binop_kernel(ColView tgt, ColView a, ColView b, int b_is_const, double k,
                                                        int op, const uint8_t* __restrict__ alive, int64_t rows,
                                                        unsigned long long* n_updated)
{
    unsigned long long cnt = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * kBinRows; base < rows;
         base += stride * kBinRows) {
        double va[kBinRows], vb[kBinRows];
        bool live[kBinRows];
#pragma unroll
        for (int m = 0; m < kBinRows; ++m) {
            const int64_t r = base + static_cast<int64_t>(m) * blockDim.x + threadIdx.x;
            live[m] = r < rows && alive[r];
            va[m] = r < rows ? load_col(a, r) : 0.0;
            vb[m] = b_is_const ? k : (r < rows ? load_col(b, r) : 0.0);
        }
#pragma unroll
        for (int m = 0; m < kBinRows; ++m) {
            if (!live[m]) continue;
            const double x = va[m], y = vb[m];
            double v;
            switch (op) {
                case AMBER_OP_ADD: v = x + y; break;
                case AMBER_OP_SUB: v = x - y; break;
                case AMBER_OP_MUL: v = x * y; break;
                case AMBER_OP_DIV: v = x / y; break;
                case AMBER_OP_MIN: v = fmin(x, y); break;
                default: v = fmax(x, y); break;
            }
            store_col(tgt, base + static_cast<int64_t>(m) * blockDim.x + threadIdx.x, v);
            ++cnt;
        }
    }
    unsigned long long vals[1] = {cnt};
    unsigned long long* const outs[1] = {n_updated};
    block_sum_atomic<1>(vals, outs);
}

// Same fast path when target and operand columns share one element type:
// typed loads (no per-element dtype dispatch), all 8 rows' loads in flight.
template <class T>
__global__ void __launch_bounds__(256) pop_binop_typed_kernel(T* __restrict__ tgt, const T* __restrict__ a,
                                                              const T* __restrict__ b, int b_is_const, double k, int op,
                                                              const uint8_t* __restrict__ alive, int64_t rows,
                                                              unsigned long long* n_updated)
{
    unsigned long long cnt = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * kBinRows; base < rows;
         base += stride * kBinRows) {
        T va[kBinRows], vb[kBinRows];
        uint8_t live[kBinRows];
#pragma unroll
        for (int m = 0; m < kBinRows; ++m) {
            const int64_t r = base + static_cast<int64_t>(m) * blockDim.x + threadIdx.x;
            const bool in = r < rows;
            live[m] = in ? alive[r] : 0;
            va[m] = in ? a[r] : T(0);
            vb[m] = (!b_is_const && in) ? b[r] : T(0);
        }
#pragma unroll
        for (int m = 0; m < kBinRows; ++m) {
            if (!live[m]) continue;
            const double x = static_cast<double>(va[m]), y = b_is_const ? k : static_cast<double>(vb[m]);
            double v;
            switch (op) {
                case AMBER_OP_ADD: v = x + y; break;
                case AMBER_OP_SUB: v = x - y; break;
                case AMBER_OP_MUL: v = x * y; break;
                case AMBER_OP_DIV: v = x / y; break;
                case AMBER_OP_MIN: v = fmin(x, y); break;
                default: v = fmax(x, y); break;
            }
            tgt[base + static_cast<int64_t>(m) * blockDim.x + threadIdx.x] = static_cast<T>(v);
            ++cnt;
        }
    }
    unsigned long long vals[1] = {cnt};
    unsigned long long* const outs[1] = {n_updated};
    block_sum_atomic<1>(vals, outs);
}

// 4-byte columns: thread g owns rows [8g, 8g+8) -> two 128-bit loads per
// operand column, one 64-bit load of the alive mask, two 128-bit stores.
template <class T>
__device__ __forceinline__ double binop(int op, double x, double y)
{
    switch (op) {
        case AMBER_OP_ADD: return x + y;
        case AMBER_OP_SUB: return x - y;
        case AMBER_OP_MUL: return x * y;
        case AMBER_OP_DIV: return x / y;
        case AMBER_OP_MIN: return fmin(x, y);
        default: return fmax(x, y);
    }
}

template <class T>
__global__ void __launch_bounds__(256) pop_binop_vec4_kernel(T* __restrict__ tgt, const T* __restrict__ a,
                                                             const T* __restrict__ b, int b_is_const, double k, int op,
                                                             const uint8_t* __restrict__ alive, int64_t rows,
                                                             unsigned long long* n_updated)
{
    static_assert(sizeof(T) == 4, "4-byte element types only");
    unsigned long long cnt = 0;
    const int64_t groups = rows / 8;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint2 lv = __ldcs(reinterpret_cast<const uint2*>(alive) + g);
        const uint4 a0 = __ldcs(reinterpret_cast<const uint4*>(a) + 2 * g);
        const uint4 a1 = __ldcs(reinterpret_cast<const uint4*>(a) + 2 * g + 1);
        uint4 b0 = make_uint4(0u, 0u, 0u, 0u), b1 = b0;
        if (!b_is_const) {
            b0 = __ldcs(reinterpret_cast<const uint4*>(b) + 2 * g);
            b1 = __ldcs(reinterpret_cast<const uint4*>(b) + 2 * g + 1);
        }
        uint4 o0 = a0, o1 = a1;
        if (lv.x == 0x01010101u && lv.y == 0x01010101u) {  // all eight rows live (the common case)
            const uint32_t ai[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const uint32_t bi[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            uint32_t oi[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                T x, y;
                memcpy(&x, &ai[m], 4);
                memcpy(&y, &bi[m], 4);
                const T v = static_cast<T>(binop<T>(op, static_cast<double>(x), b_is_const ? k : static_cast<double>(y)));
                memcpy(&oi[m], &v, 4);
            }
            o0 = make_uint4(oi[0], oi[1], oi[2], oi[3]);
            o1 = make_uint4(oi[4], oi[5], oi[6], oi[7]);
            __stcs(reinterpret_cast<uint4*>(tgt) + 2 * g, o0);
            __stcs(reinterpret_cast<uint4*>(tgt) + 2 * g + 1, o1);
            cnt += 8;
        } else {
            for (int m = 0; m < 8; ++m) {
                const int64_t r = 8 * g + m;
                if (!alive[r]) continue;
                const double y = b_is_const ? k : static_cast<double>(b[r]);
                tgt[r] = static_cast<T>(binop<T>(op, static_cast<double>(a[r]), y));
                ++cnt;
            }
        }
    }
    if (blockIdx.x == 0) {  // tail rows
        for (int64_t r = groups * 8 + threadIdx.x; r < rows; r += blockDim.x) {
            if (!alive[r]) continue;
            const double y = b_is_const ? k : static_cast<double>(b[r]);
            tgt[r] = static_cast<T>(binop<T>(op, static_cast<double>(a[r]), y));
            ++cnt;
        }
    }
    unsigned long long vals[1] = {cnt};
    unsigned long long* const outs[1] = {n_updated};
    block_sum_atomic<1>(vals, outs);
}

__global__ void pop_fill_kernel(ColView c, int64_t r0, int64_t r1, double v)
{
    for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x)
        store_col(c, r, v);
}

__global__ void pop_new_rows_kernel(int64_t* ids, uint8_t* alive, int64_t r0, int64_t r1, int64_t id0)
{
    for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x) {
        ids[r] = id0 + (r - r0);
        alive[r] = 1;
    }
}

// rows are sorted by id: binary search; row index or -1 (unknown) / -2 (dead)
__global__ void pop_find_kernel(const int64_t* __restrict__ ids, const uint8_t* __restrict__ alive, int64_t rows,
                                const int64_t* __restrict__ q, int64_t n, int64_t* __restrict__ row_out, int* bad)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = rows - 1, found = -1;
        while (lo <= hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ids[mid] == q[k]) {
                found = mid;
                break;
            }
            if (ids[mid] < q[k]) lo = mid + 1;
            else hi = mid - 1;
        }
        if (found >= 0 && !alive[found]) found = -2;
        row_out[k] = found;
        if (found < 0) atomicExch(bad, 1);
    }
}

__global__ void pop_kill_kernel(uint8_t* alive, const int64_t* rows, int64_t n, int* dup)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        alive[rows[k]] = 0;
}

__global__ void pop_scatter_kernel(ColView c, const int64_t* rows, const double* vals, int64_t n)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        store_col(c, rows[k], vals[k]);
}

size_t dtype_size(int dt)
{
    switch (dt) {
        case AMBER_I32: case AMBER_F32: return 4;
        case AMBER_I64: case AMBER_F64: return 8;
        case AMBER_U8: return 1;
        default: fail(AMBER_E_INVALID_ARG, "population columns must be I32, I64, F32, F64 or U8");
    }
}

}  // namespace

// ---------------------------------------------------------------- expression JIT
// General update programs are compiled at run time (NVRTC, sm_100a) into a
// straight-line kernel: every referenced column of a row is loaded with its
// own type, the postfix program becomes a chain of double expressions (the
// interpreter's exact semantics: same ops, --fmad=false, IEEE div/sqrt, C store
// conversion), the filter selects the store.  4 rows per thread, branch-free
// loads, one count atomic per block.  Kernels are cached by source text;
// without NVRTC (or if a compile fails) the interpreter runs instead.
struct JitArgs {
    void* col[kMaxCols];
    const int64_t* ids;
    const uint8_t* alive;
    long long rows;
    unsigned step;
    unsigned k0[10], k1[10];
    unsigned long long* count;
    double* partial;
};

struct NvrtcApi {
    void* h = nullptr;
    int (*create)(void**, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    int (*compile)(void*, int, const char* const*) = nullptr;
    int (*cubin_size)(void*, size_t*) = nullptr;
    int (*cubin)(void*, char*) = nullptr;
    int (*log_size)(void*, size_t*) = nullptr;
    int (*log)(void*, char*) = nullptr;
    int (*destroy)(void**) = nullptr;
    std::string csrc;  // include dir (this library's csrc/)
    bool ok = false;
};

static NvrtcApi& nvrtc()
{
    static NvrtcApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.create = reinterpret_cast<decltype(api.create)>(dlsym(api.h, "nvrtcCreateProgram"));
        api.compile = reinterpret_cast<decltype(api.compile)>(dlsym(api.h, "nvrtcCompileProgram"));
        api.cubin_size = reinterpret_cast<decltype(api.cubin_size)>(dlsym(api.h, "nvrtcGetCUBINSize"));
        api.cubin = reinterpret_cast<decltype(api.cubin)>(dlsym(api.h, "nvrtcGetCUBIN"));
        api.log_size = reinterpret_cast<decltype(api.log_size)>(dlsym(api.h, "nvrtcGetProgramLogSize"));
        api.log = reinterpret_cast<decltype(api.log)>(dlsym(api.h, "nvrtcGetProgramLog"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.h, "nvrtcDestroyProgram"));
        Dl_info info{};
        if (!dladdr(reinterpret_cast<void*>(&nvrtc), &info) || !info.dli_fname) return;
        std::string so(info.dli_fname);
        api.csrc = so.substr(0, so.rfind('/') + 1) + "csrc";
        FILE* f = fopen((api.csrc + "/philox.cuh").c_str(), "r");
        if (!f) return;
        fclose(f);
        api.ok = api.create && api.compile && api.cubin_size && api.cubin && api.log_size && api.log && api.destroy;
    });
    return api;
}

static const char* jit_ctype(int dt)
{
    switch (dt) {
        case AMBER_I32: return "int";
        case AMBER_I64: return "long long";
        case AMBER_F32: return "float";
        case AMBER_F64: return "double";
        default: return "unsigned char";
    }
}

// Postfix program -> C expression statements; returns the result variable.
static std::string jit_emit(const Prog& P, const Cols& C, const std::string& pfx, std::string& body)
{
    std::vector<std::string> st;
    char buf[256];
    for (int k = 0; k < P.n; ++k) {
        const amber_instr& in = P.ins[k];
        const std::string v = pfx + std::to_string(k);
        auto pop1 = [&] { std::string x = st.back(); st.pop_back(); return x; };
        switch (in.op) {
            case AMBER_OP_CONST: {  // exact bit pattern (also inf / nan)
                unsigned long long bits;
                std::memcpy(&bits, &in.value, 8);
                snprintf(buf, sizeof buf, "__longlong_as_double((long long)0x%llxULL)", bits);
                body += "const double " + v + " = " + buf + ";\n";
                break;
            }
            case AMBER_OP_COL:  // component of the column's 4-row vector (loaded once per group)
                body += "const double " + v + " = (double)c" + std::to_string(in.arg) + "[j];\n";
                break;
            case AMBER_OP_ID: body += "const double " + v + " = (double)id;\n"; break;
            case AMBER_OP_RAND: body += "const double " + v + " = rnd(K, " + std::to_string(in.arg) + "u, id, a.step);\n"; break;
            case AMBER_OP_STEP: body += "const double " + v + " = (double)a.step;\n"; break;
            case AMBER_OP_NEG: body += "const double " + v + " = -" + pop1() + ";\n"; break;
            case AMBER_OP_ABS: body += "const double " + v + " = fabs(" + pop1() + ");\n"; break;
            case AMBER_OP_FLOOR: body += "const double " + v + " = floor(" + pop1() + ");\n"; break;
            case AMBER_OP_SQRT: body += "const double " + v + " = sqrt(" + pop1() + ");\n"; break;
            case AMBER_OP_NOT: { const std::string x = pop1(); body += "const double " + v + " = " + x + " == 0.0 ? 1.0 : 0.0;\n"; break; }
            case AMBER_OP_SELECT: {
                const std::string b = pop1(), x = pop1(), c = pop1();
                body += "const double " + v + " = " + c + " != 0.0 ? " + x + " : " + b + ";\n";
                break;
            }
            default: {
                const std::string b = pop1(), x = pop1();
                std::string e;
                switch (in.op) {
                    case AMBER_OP_ADD: e = x + " + " + b; break;
                    case AMBER_OP_SUB: e = x + " - " + b; break;
                    case AMBER_OP_MUL: e = x + " * " + b; break;
                    case AMBER_OP_DIV: e = x + " / " + b; break;
                    case AMBER_OP_MIN: e = "fmin(" + x + ", " + b + ")"; break;
                    case AMBER_OP_MAX: e = "fmax(" + x + ", " + b + ")"; break;
                    case AMBER_OP_LT: e = "(" + x + " < " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_LE: e = "(" + x + " <= " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_GT: e = "(" + x + " > " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_GE: e = "(" + x + " >= " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_EQ: e = "(" + x + " == " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_NE: e = "(" + x + " != " + b + ") ? 1.0 : 0.0"; break;
                    case AMBER_OP_AND: e = "(" + x + " != 0.0 && " + b + " != 0.0) ? 1.0 : 0.0"; break;
                    case AMBER_OP_OR: e = "(" + x + " != 0.0 || " + b + " != 0.0) ? 1.0 : 0.0"; break;
                    default: e = "0.0"; break;
                }
                body += "const double " + v + " = " + e + ";\n";
            }
        }
        st.push_back(v);
    }
    return st.empty() ? std::string("1.0") : st.back();
}

static const char* kJitPrelude =
    "#include \"philox.cuh\"\n"
    "struct JitArgs { void* col[32]; const long long* ids; const unsigned char* alive; long long rows; unsigned step; "
    "unsigned k0[10], k1[10]; unsigned long long* count; double* partial; };\n"
    "__device__ __forceinline__ double rnd(const amber::PhiloxKey& K, unsigned tag, long long id, unsigned step) {\n"
    "  const uint4 w = amber::stream_block(K, tag, (unsigned long long)id >> 2, step);\n"
    "  const unsigned q = (unsigned)(id & 3);\n"
    "  return (double)amber::u01(q == 0 ? w.x : (q == 1 ? w.y : (q == 2 ? w.z : w.w)));\n}\n"
    "template <class T> __device__ __forceinline__ void ld4(const void* p, long long r0, T (&v)[4]) {\n"
    "  if (sizeof(T) == 1) { const uchar4 x = *(const uchar4*)((const T*)p + r0); v[0] = (T)x.x; v[1] = (T)x.y; v[2] = (T)x.z; v[3] = (T)x.w; }\n"
    "  else if (sizeof(T) == 4) { const uint4 x = *(const uint4*)((const T*)p + r0);\n"
    "    const unsigned u[4] = {x.x, x.y, x.z, x.w}; for (int j = 0; j < 4; ++j) v[j] = *(const T*)&u[j]; }\n"
    "  else { const ulonglong2 x = *(const ulonglong2*)((const T*)p + r0), y = *(const ulonglong2*)((const T*)p + r0 + 2);\n"
    "    const unsigned long long u[4] = {x.x, x.y, y.x, y.y}; for (int j = 0; j < 4; ++j) v[j] = *(const T*)&u[j]; }\n}\n";

static void jit_cols(const Prog& P, std::vector<int>& used)
{
    for (int k = 0; k < P.n; ++k)
        if (P.ins[k].op == AMBER_OP_COL && std::find(used.begin(), used.end(), P.ins[k].arg) == used.end())
            used.push_back(P.ins[k].arg);
}

static std::string jit_aggregate_source(const Prog& pe, const Prog& pw, const Cols& C)
{
    std::string body;
    const std::string rw = pw.n ? jit_emit(pw, C, "w", body) : std::string("1.0");
    const std::string re = pe.n ? jit_emit(pe, C, "e", body) : std::string("0.0");
    const bool uses_id = pe.uses_id || pw.uses_id;
    std::vector<int> used;
    jit_cols(pw, used);
    jit_cols(pe, used);
    std::string s = kJitPrelude;
    s += "extern \"C\" __global__ void __launch_bounds__(256) amber_jit_aggregate(const JitArgs a) {\n"
         "  amber::PhiloxKey K;\n  for (int i = 0; i < 10; ++i) { K.k0[i] = a.k0[i]; K.k1[i] = a.k1[i]; }\n"
         "  double S = 0.0, MN = __longlong_as_double(0x7ff0000000000000LL), MX = -MN, CC = 0.0;\n"
         "  const long long stride = (long long)gridDim.x * 256;\n"
         "  for (long long g = (long long)blockIdx.x * 256 + threadIdx.x; 4 * g < a.rows; g += stride) {\n"
         "    const long long r0 = 4 * g;\n"
         "    unsigned char al[4]; ld4(a.alive, r0, al);\n";
    for (int k : used)
        s += "    " + std::string(jit_ctype(C.c[k].dtype)) + " c" + std::to_string(k) + "[4]; ld4(a.col[" +
             std::to_string(k) + "], r0, c" + std::to_string(k) + ");\n";
    if (uses_id) s += "    long long idv[4]; ld4(a.ids, r0, idv);\n";
    s += "#pragma unroll\n    for (int j = 0; j < 4; ++j) {\n";
    if (uses_id) s += "      const long long id = idv[j];\n";
    s += body;
    s += "      if (r0 + j < a.rows && al[j] && (" + rw + ") != 0.0) {\n"
         "        const double v = " + re + ";\n"
         "        S += v; MN = fmin(MN, v); MX = fmax(MX, v); CC += 1.0;\n      }\n    }\n  }\n"
         "  __shared__ double red[4][8];\n"
         "  for (int o = 16; o > 0; o >>= 1) { S += __shfl_xor_sync(0xffffffffu, S, o);\n"
         "    MN = fmin(MN, __shfl_xor_sync(0xffffffffu, MN, o)); MX = fmax(MX, __shfl_xor_sync(0xffffffffu, MX, o));\n"
         "    CC += __shfl_xor_sync(0xffffffffu, CC, o); }\n"
         "  const int w = threadIdx.x >> 5;\n"
         "  if ((threadIdx.x & 31) == 0) { red[0][w] = S; red[1][w] = MN; red[2][w] = MX; red[3][w] = CC; }\n"
         "  __syncthreads();\n"
         "  if (threadIdx.x == 0) { double s0 = 0.0, s1 = red[1][0], s2 = red[2][0], s3 = 0.0;\n"
         "    for (int k = 0; k < 8; ++k) { s0 += red[0][k]; s1 = fmin(s1, red[1][k]); s2 = fmax(s2, red[2][k]); s3 += red[3][k]; }\n"
         "    a.partial[4 * blockIdx.x] = s0; a.partial[4 * blockIdx.x + 1] = s1; a.partial[4 * blockIdx.x + 2] = s2;\n"
         "    a.partial[4 * blockIdx.x + 3] = s3; }\n}\n";
    return s;
}

// tgt >= 0: update kernel (merged vector store of the target column);
// tgt < 0: aggregate kernel (per-block sum / min / max / count partials).
static std::string jit_update_source(const Prog& pe, const Prog& pw, const Cols& C, int tgt)
{
    if (tgt < 0) return jit_aggregate_source(pe, pw, C);
    std::string body;
    const std::string rw = pw.n ? jit_emit(pw, C, "w", body) : std::string("1.0");
    const std::string re = jit_emit(pe, C, "e", body);
    const bool uses_id = pe.uses_id || pw.uses_id;
    std::vector<int> used;
    jit_cols(pw, used);
    jit_cols(pe, used);
    if (std::find(used.begin(), used.end(), tgt) == used.end()) used.push_back(tgt);  // merged store reads it
    const std::string tt = jit_ctype(C.c[tgt].dtype);
    std::string s = kJitPrelude;
    s += "template <class T> __device__ __forceinline__ void st4(void* p, long long r0, const T (&v)[4]) {\n"
         "  if (sizeof(T) == 1) { *(uchar4*)((T*)p + r0) = make_uchar4((unsigned char)v[0], (unsigned char)v[1], (unsigned char)v[2], (unsigned char)v[3]); }\n"
         "  else if (sizeof(T) == 4) { unsigned u[4]; for (int j = 0; j < 4; ++j) u[j] = *(const unsigned*)&v[j];\n"
         "    *(uint4*)((T*)p + r0) = make_uint4(u[0], u[1], u[2], u[3]); }\n"
         "  else { unsigned long long u[4]; for (int j = 0; j < 4; ++j) u[j] = *(const unsigned long long*)&v[j];\n"
         "    *(ulonglong2*)((T*)p + r0) = make_ulonglong2(u[0], u[1]); *(ulonglong2*)((T*)p + r0 + 2) = make_ulonglong2(u[2], u[3]); }\n}\n";
    s += "extern \"C\" __global__ void __launch_bounds__(256) amber_jit_update(const JitArgs a) {\n"
         "  amber::PhiloxKey K;\n  for (int i = 0; i < 10; ++i) { K.k0[i] = a.k0[i]; K.k1[i] = a.k1[i]; }\n"
         "  unsigned long long cnt = 0;\n"
         "  const long long stride = (long long)gridDim.x * 256;\n"
         "  for (long long g = (long long)blockIdx.x * 256 + threadIdx.x; 4 * g < a.rows; g += stride) {\n"
         "    const long long r0 = 4 * g;\n"
         "    unsigned char al[4]; ld4(a.alive, r0, al);\n";
    for (int k : used)
        s += "    " + std::string(jit_ctype(C.c[k].dtype)) + " c" + std::to_string(k) + "[4]; ld4(a.col[" +
             std::to_string(k) + "], r0, c" + std::to_string(k) + ");\n";
    if (uses_id) s += "    long long idv[4]; ld4(a.ids, r0, idv);\n";
    s += "    " + tt + " out[4];\n";
    s += "#pragma unroll\n    for (int j = 0; j < 4; ++j) {\n";
    if (uses_id) s += "      const long long id = idv[j];\n";
    s += body;
    s += "      const bool sel = r0 + j < a.rows && al[j] && (" + rw + ") != 0.0;\n"
         "      out[j] = sel ? (" + tt + ")(" + re + ") : c" + std::to_string(tgt) + "[j];\n"
         "      cnt += sel;\n    }\n"
         "    st4(a.col[" + std::to_string(tgt) + "], r0, out);\n  }\n"
         "  if (a.count) {\n"
         "    __shared__ unsigned long long red[8];\n"
         "    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);\n"
         "    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;\n"
         "    __syncthreads();\n"
         "    if (threadIdx.x == 0) { unsigned long long t = 0; for (int w = 0; w < 8; ++w) t += red[w];\n"
         "      if (t) atomicAdd(a.count, t); }\n  }\n}\n";
    return s;
}

struct JitCache {
    std::mutex mu;
    std::map<std::string, cudaKernel_t> kernels;
    std::vector<cudaLibrary_t> libs;
};

static JitCache& jit_cache()
{
    static JitCache c;
    return c;
}

// Compiled kernel for this source, or nullptr (no NVRTC / compile error: interpret instead).
static cudaKernel_t jit_kernel(const std::string& src, const char* name = "amber_jit_update")
{
    NvrtcApi& api = nvrtc();
    if (!api.ok) return nullptr;
    JitCache& jc = jit_cache();
    std::lock_guard<std::mutex> g(jc.mu);
    auto it = jc.kernels.find(src);
    if (it != jc.kernels.end()) return it->second;
    cudaKernel_t kern = nullptr;
    void* prog = nullptr;
    if (api.create(&prog, src.c_str(), "amber_jit_update.cu", 0, nullptr, nullptr) == 0) {
        const std::string inc = "-I" + api.csrc;
        const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--prec-div=true", "--prec-sqrt=true",
                              "--std=c++17", inc.c_str()};
        if (api.compile(prog, 6, opts) == 0) {
            size_t n = 0;
            api.cubin_size(prog, &n);
            std::vector<char> cubin(n);
            api.cubin(prog, cubin.data());
            cudaLibrary_t lib = nullptr;
            if (cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) == cudaSuccess &&
                cudaLibraryGetKernel(&kern, lib, name) == cudaSuccess) {
                jc.libs.push_back(lib);
            } else {
                cudaGetLastError();
                kern = nullptr;
            }
        }
        api.destroy(&prog);
    }
    jc.kernels[src] = kern;  // failures cached too (interpreted from then on)
    return kern;
}

struct Population {
    Runtime rt;
    bool jit = true;                      // AMBER_POP_JIT=0 at creation: interpreter only
    int64_t n_jit = 0, n_interp = 0;      // general-program updates by path
    PhiloxKey key{};
    struct Column {
        std::string name;
        int dtype;
        DevBuf<char> data;
    };
    std::vector<std::unique_ptr<Column>> cols;
    DevBuf<int64_t> ids;
    DevBuf<uint8_t> alive;
    int64_t cap = 0, rows = 0, live = 0, next_id = 0, step = 0;

    Population(const amber_column_spec* specs, int n, int64_t capacity, uint64_t seed, const amber_runtime* r)
    {
        if (const char* e = getenv("AMBER_POP_JIT")) jit = e[0] != '0';
        rt.init(r);
        key = philox_key(seed);
        AMBER_REQUIRE(n >= 1 && n <= kMaxCols, "population needs 1..32 columns");
        for (int k = 0; k < n; ++k) {
            AMBER_REQUIRE(specs[k].name && *specs[k].name, "empty column name");
            std::string nm(specs[k].name);
            AMBER_REQUIRE(nm != "id", "column name 'id' is reserved");
            for (auto& c : cols) AMBER_REQUIRE(c->name != nm, "duplicate column name " + nm);
            dtype_size(specs[k].dtype);
            auto c = std::make_unique<Column>();
            c->name = nm;
            c->dtype = specs[k].dtype;
            cols.push_back(std::move(c));
        }
        reserve(std::max<int64_t>(capacity, 16));
        AMBER_CUDA(cudaFuncSetAttribute(pop_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStackBytes)));
        AMBER_CUDA(cudaFuncSetAttribute(pop_aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kStackBytes)));
    }

    ~Population()
    {
        if (rt.stream) cudaStreamSynchronize(rt.stream);
        cols.clear();
        cnt.reset();
        ids.reset();
        alive.reset();
        rt.destroy();
    }

    Cols views() const
    {
        Cols C{};
        C.n = static_cast<int>(cols.size());
        for (int k = 0; k < C.n; ++k) C.c[k] = ColView{cols[k]->data.p, cols[k]->dtype};
        return C;
    }

    int col_index(const std::string& nm) const
    {
        for (size_t k = 0; k < cols.size(); ++k)
            if (cols[k]->name == nm) return static_cast<int>(k);
        return -1;
    }

    void reserve(int64_t want)
    {
        if (want <= cap) return;
        const int64_t nc = (std::max<int64_t>(want, cap * 2) + 3) & ~3ll;  // JIT kernels move 4 rows per vector
        auto grow = [&](DevBuf<char>& b, size_t esz) {
            DevBuf<char> nb;
            nb.allocate(&rt, nc * esz);
            if (rows) AMBER_CUDA(cudaMemcpyAsync(nb.p, b.p, rows * esz, cudaMemcpyDeviceToDevice, rt.stream));
            std::swap(b.p, nb.p);
            std::swap(b.n, nb.n);
            b.rt = &rt;
        };
        for (auto& c : cols) grow(c->data, dtype_size(c->dtype));
        DevBuf<int64_t> ni;
        ni.allocate(&rt, nc);
        DevBuf<uint8_t> na;
        na.allocate(&rt, nc);
        if (rows) {
            AMBER_CUDA(cudaMemcpyAsync(ni.p, ids.p, rows * 8, cudaMemcpyDeviceToDevice, rt.stream));
            AMBER_CUDA(cudaMemcpyAsync(na.p, alive.p, rows, cudaMemcpyDeviceToDevice, rt.stream));
        }
        std::swap(ids.p, ni.p);
        std::swap(ids.n, ni.n);
        ids.rt = &rt;
        std::swap(alive.p, na.p);
        std::swap(alive.n, na.n);
        alive.rt = &rt;
        rt.sync();
        cap = nc;
    }

    static size_t stack_bytes(const Prog& a, const Prog& b)
    {
        return static_cast<size_t>(std::max(1, std::max(a.max_depth, b.max_depth))) * kTile * sizeof(double);
    }

    int tiles_grid(size_t smem = kStackBytes) const
    {
        const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(2048 / kThreads, (220u << 10) / smem)));
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(rows, 1), kTile),
                                                                        static_cast<int64_t>(rt.num_sms) * per_sm)));
    }

    int grid_for(int64_t n) const
    {
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), rt.num_sms * 8)));
    }

    int64_t add(int64_t n, const double* defaults)
    {
        AMBER_REQUIRE(n >= 0, "add_agents needs n >= 0");
        reserve(rows + n);
        const int64_t first = next_id;
        if (n) {
            for (size_t k = 0; k < cols.size(); ++k) {
                pop_fill_kernel<<<grid_for(n), 256, 0, rt.stream>>>(ColView{cols[k]->data.p, cols[k]->dtype}, rows,
                                                                    rows + n, defaults ? defaults[k] : 0.0);
                check_launch("pop_fill_kernel");
            }
            pop_new_rows_kernel<<<grid_for(n), 256, 0, rt.stream>>>(ids.p, alive.p, rows, rows + n, next_id);
            check_launch("pop_new_rows_kernel");
            rt.sync();
        }
        rows += n;
        live += n;
        next_id += n;
        return first;
    }

    // validated id -> row lookup on the device (throws if any id is unknown/dead)
    void find_rows(const int64_t* h_ids, int64_t n, DevBuf<int64_t>& d_rows)
    {
        DevBuf<int64_t> q;
        DevBuf<int> bad;
        q.allocate(&rt, n);
        d_rows.allocate(&rt, n);
        bad.allocate(&rt, 1);
        bad.zero_async(rt.stream);
        AMBER_CUDA(cudaMemcpyAsync(q.p, h_ids, n * 8, cudaMemcpyHostToDevice, rt.stream));
        pop_find_kernel<<<grid_for(n), 256, 0, rt.stream>>>(ids.p, alive.p, rows, q.p, n, d_rows.p, bad.p);
        check_launch("pop_find_kernel");
        int hb = 0;
        AMBER_CUDA(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        if (hb) fail(AMBER_E_INVALID_ARG, "unknown or dead agent id");
    }

    void remove(const int64_t* h_ids, int64_t n)
    {
        if (!n) return;
        std::vector<int64_t> u(h_ids, h_ids + n);
        std::sort(u.begin(), u.end());
        AMBER_REQUIRE(std::adjacent_find(u.begin(), u.end()) == u.end(), "duplicate id in remove_agents");
        DevBuf<int64_t> d_rows;
        find_rows(u.data(), n, d_rows);
        pop_kill_kernel<<<grid_for(n), 256, 0, rt.stream>>>(alive.p, d_rows.p, n, nullptr);
        check_launch("pop_kill_kernel");
        rt.sync();
        live -= n;
    }

    void compact()
    {
        if (live == rows) return;
        DevBuf<int> n_sel;
        n_sel.allocate(&rt, 1);
        auto select = [&](void* data, size_t esz) {
            DevBuf<char> out;
            out.allocate(&rt, std::max<int64_t>(cap, 1) * esz);
            size_t tmp = 0;
            // flagged selection of fixed-size records via 1/2/4/8-byte element types
            auto run = [&](auto* in, auto* o) {
                cub::DeviceSelect::Flagged(nullptr, tmp, in, alive.p, o, n_sel.p, rows, rt.stream);
                DevBuf<char> t;
                t.allocate(&rt, tmp + 16);
                AMBER_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, in, alive.p, o, n_sel.p, rows, rt.stream));
                rt.sync();
            };
            if (esz == 1) run(static_cast<uint8_t*>(data), reinterpret_cast<uint8_t*>(out.p));
            else if (esz == 4) run(static_cast<uint32_t*>(data), reinterpret_cast<uint32_t*>(out.p));
            else run(static_cast<unsigned long long*>(data), reinterpret_cast<unsigned long long*>(out.p));
            AMBER_CUDA(cudaMemcpyAsync(data, out.p, live * esz, cudaMemcpyDeviceToDevice, rt.stream));
            rt.sync();
        };
        for (auto& c : cols) select(c->data.p, dtype_size(c->dtype));
        select(ids.p, 8);
        AMBER_CUDA(cudaMemsetAsync(alive.p, 1, live, rt.stream));
        rt.sync();
        rows = live;
    }

    Prog prog(const amber_instr* ins, int n, bool allow_empty) const
    {
        Prog P{};
        AMBER_REQUIRE(n >= 0 && n <= kMaxProg, "expression longer than 64 instructions");
        AMBER_REQUIRE(allow_empty || n > 0, "empty expression");
        AMBER_REQUIRE(n == 0 || ins, "NULL expression");
        int depth = 0;
        for (int k = 0; k < n; ++k) {
            const int op = ins[k].op;
            int pop = 0, push = 1;
            if (op == AMBER_OP_CONST || op == AMBER_OP_ID || op == AMBER_OP_STEP || op == AMBER_OP_RAND) {
                pop = 0;
                if (op == AMBER_OP_ID || op == AMBER_OP_RAND) P.uses_id = 1;
            } else if (op == AMBER_OP_COL) {
                AMBER_REQUIRE(ins[k].arg >= 0 && ins[k].arg < static_cast<int>(cols.size()), "column index out of range");
            } else if (op >= AMBER_OP_NEG && op <= AMBER_OP_SQRT) {
                pop = 1;
            } else if (op == AMBER_OP_NOT) {
                pop = 1;
            } else if ((op >= AMBER_OP_ADD && op <= AMBER_OP_MAX) || (op >= AMBER_OP_LT && op <= AMBER_OP_NE) ||
                       op == AMBER_OP_AND || op == AMBER_OP_OR) {
                pop = 2;
            } else if (op == AMBER_OP_SELECT) {
                pop = 3;
            } else {
                fail(AMBER_E_INVALID_ARG, "unknown expression op " + std::to_string(op));
            }
            AMBER_REQUIRE(depth >= pop, "expression stack underflow");
            depth += push - pop;
            AMBER_REQUIRE(depth <= kMaxStack, "expression stack deeper than 8");
            P.max_depth = std::max(P.max_depth, depth);
            P.ins[k] = ins[k];
        }
        AMBER_REQUIRE(n == 0 || depth == 1, "expression must leave exactly one value");
        P.n = n;
        return P;
    }

    DevBuf<unsigned long long> cnt;  // persistent update counter (one per population)

    int64_t update(const std::string& target, const amber_instr* e, int ne, const amber_instr* w, int nw, bool want_count)
    {
        const int tgt = col_index(target);
        if (tgt < 0) fail(AMBER_E_UNKNOWN_NAME, "no column " + target);
        const Prog pe = prog(e, ne, false), pw = prog(w, nw, true);
        if (!cnt.p) cnt.allocate(&rt, 1);
        unsigned long long* cnt_p = want_count ? cnt.p : nullptr;
        if (want_count) cnt.zero_async(rt.stream);
        const bool fast = pw.n == 0 && pe.n == 3 && pe.ins[0].op == AMBER_OP_COL &&
                          (pe.ins[1].op == AMBER_OP_CONST || pe.ins[1].op == AMBER_OP_COL) &&
                          pe.ins[2].op >= AMBER_OP_ADD && pe.ins[2].op <= AMBER_OP_MAX;
        const Cols C = views();
        cudaKernel_t jk = nullptr;
        const int bcol = (fast && pe.ins[1].op == AMBER_OP_COL) ? pe.ins[1].arg : -1;
        const bool same_type = fast && C.c[pe.ins[0].arg].dtype == C.c[tgt].dtype &&
                               (bcol < 0 || C.c[bcol].dtype == C.c[tgt].dtype);
        const int gfast = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(ceil_div(std::max<int64_t>(rows, 1), 256 * kBinRows), rt.num_sms * 8)));
        if (rows && same_type) {
            const int isc = bcol < 0;
            const double kk = pe.ins[1].value;
            const int op = pe.ins[2].op;
            void* tp = C.c[tgt].p;
            const void* ap = C.c[pe.ins[0].arg].p;
            const void* bp = bcol >= 0 ? C.c[bcol].p : ap;
            auto go4 = [&](auto tag) {
                using T = decltype(tag);
                const int g4 = static_cast<int>(std::max<int64_t>(
                    1, std::min<int64_t>(ceil_div(std::max<int64_t>(rows / 8, 1), 256), rt.num_sms * 8)));
                pop_binop_vec4_kernel<T><<<g4, 256, 0, rt.stream>>>(static_cast<T*>(tp), static_cast<const T*>(ap),
                                                                    static_cast<const T*>(bp), isc, kk, op, alive.p,
                                                                    rows, cnt_p);
            };
            auto go = [&](auto tag) {
                using T = decltype(tag);
                pop_binop_typed_kernel<T><<<gfast, 256, 0, rt.stream>>>(static_cast<T*>(tp), static_cast<const T*>(ap),
                                                                         static_cast<const T*>(bp), isc, kk, op, alive.p,
                                                                         rows, cnt_p);
            };
            switch (C.c[tgt].dtype) {
                case AMBER_I32: go4(int32_t{}); break;
                case AMBER_I64: go(int64_t{}); break;
                case AMBER_F32: go4(float{}); break;
                case AMBER_F64: go(double{}); break;
                default: go(uint8_t{}); break;
            }
            check_launch("pop_binop_typed_kernel");
        } else if (rows && fast) {
            const int g = gfast;
            pop_binop_kernel<<<g, 256, 0, rt.stream>>>(C.c[tgt], C.c[pe.ins[0].arg],
                                                       C.c[pe.ins[1].op == AMBER_OP_COL ? pe.ins[1].arg : 0],
                                                       pe.ins[1].op == AMBER_OP_CONST, pe.ins[1].value, pe.ins[2].op,
                                                       alive.p, rows, cnt_p);
            check_launch("pop_binop_kernel");
        } else if (rows && jit && (jk = jit_kernel(jit_update_source(pe, pw, C, tgt)))) {
            ++n_jit;
            JitArgs ja{};
            for (int k = 0; k < C.n; ++k) ja.col[k] = C.c[k].p;
            ja.ids = ids.p;
            ja.alive = alive.p;
            ja.rows = rows;
            ja.step = static_cast<uint32_t>(step);
            for (int i = 0; i < 10; ++i) {
                ja.k0[i] = key.k0[i];
                ja.k1[i] = key.k1[i];
            }
            ja.count = cnt_p;
            void* kargs[] = {&ja};
            const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 1024), rt.num_sms * 16)));
            AMBER_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(jk), dim3(g), dim3(256), kargs, 0, rt.stream));
            check_launch("amber_jit_update");
        } else if (rows) {
            // the shared stack tile only needs the programs' deepest stack: shallow
            // programs (the common case) run more blocks per SM, so more column
            // loads are in flight (measured: depth 3 -> 64 KB -> 24 KB per block)
            ++n_interp;
            const size_t smem = stack_bytes(pe, pw);
            pop_update_kernel<<<tiles_grid(smem), kThreads, smem, rt.stream>>>(pe, pw, views(), tgt, ids.p, alive.p, rows,
                                                                     static_cast<uint32_t>(step), key, cnt_p);
            check_launch("pop_update_kernel");
        }
        if (!want_count) return -1;  // asynchronous: nothing to wait for
        unsigned long long h = 0;
        AMBER_CUDA(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, rt.stream));
        rt.sync();
        return static_cast<int64_t>(h);
    }

    double aggregate(int agg, const amber_instr* e, int ne, const amber_instr* w, int nw)
    {
        AMBER_REQUIRE(agg >= AMBER_AGG_SUM && agg <= AMBER_AGG_COUNT, "unknown aggregate");
        const Prog pe = prog(e, ne, agg == AMBER_AGG_COUNT), pw = prog(w, nw, true);
        const size_t smem = stack_bytes(pe, pw);
        const int g = tiles_grid(smem);
        DevBuf<double> part;
        part.allocate(&rt, 4 * g);
        std::vector<double> h(4 * g, 0.0);
        cudaKernel_t jk = nullptr;
        const Cols C = views();
        if (rows && jit && (jk = jit_kernel(jit_update_source(pe, pw, C, -1), "amber_jit_aggregate"))) {
            ++n_jit;
            JitArgs ja{};
            for (int k = 0; k < C.n; ++k) ja.col[k] = C.c[k].p;
            ja.ids = ids.p;
            ja.alive = alive.p;
            ja.rows = rows;
            ja.step = static_cast<uint32_t>(step);
            for (int i = 0; i < 10; ++i) {
                ja.k0[i] = key.k0[i];
                ja.k1[i] = key.k1[i];
            }
            ja.partial = part.p;
            void* kargs[] = {&ja};
            AMBER_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(jk), dim3(g), dim3(256), kargs, 0, rt.stream));
            check_launch("amber_jit_aggregate");
            AMBER_CUDA(cudaMemcpyAsync(h.data(), part.p, h.size() * 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
        } else if (rows) {
            ++n_interp;
            pop_aggregate_kernel<<<g, kThreads, smem, rt.stream>>>(pe, pw, views(), ids.p, alive.p, rows,
                                                           static_cast<uint32_t>(step), key, part.p);
            check_launch("pop_aggregate_kernel");
            AMBER_CUDA(cudaMemcpyAsync(h.data(), part.p, h.size() * 8, cudaMemcpyDeviceToHost, rt.stream));
            rt.sync();
        } else {
            for (int b = 0; b < g; ++b) {
                h[4 * b + 1] = INFINITY;
                h[4 * b + 2] = -INFINITY;
            }
        }
        double S = 0, MN = INFINITY, MX = -INFINITY, CC = 0;
        for (int b = 0; b < g; ++b) {
            S += h[4 * b];
            MN = std::fmin(MN, h[4 * b + 1]);
            MX = std::fmax(MX, h[4 * b + 2]);
            CC += h[4 * b + 3];
        }
        if (agg == AMBER_AGG_COUNT) return CC;
        if (agg == AMBER_AGG_SUM) return S;
        AMBER_REQUIRE(CC > 0, "mean/min/max of an empty selection");
        if (agg == AMBER_AGG_MEAN) return S / CC;
        return agg == AMBER_AGG_MIN ? MN : MX;
    }

    void read(const std::string& nm, void* dst, size_t bytes, bool on_dev)
    {
        void* data;
        size_t esz;
        if (nm == "id") {
            data = ids.p;
            esz = 8;
        } else {
            const int k = col_index(nm);
            if (k < 0) fail(AMBER_E_UNKNOWN_NAME, "no column " + nm);
            data = cols[k]->data.p;
            esz = dtype_size(cols[k]->dtype);
        }
        if (bytes < static_cast<size_t>(live) * esz) fail(AMBER_E_BUFFER_TOO_SMALL, "dst too small for column " + nm);
        if (!live) return;
        DevBuf<char> out;
        out.allocate(&rt, live * esz);
        DevBuf<int> n_sel;
        n_sel.allocate(&rt, 1);
        size_t tmp = 0;
        auto run = [&](auto* in, auto* o) {
            cub::DeviceSelect::Flagged(nullptr, tmp, in, alive.p, o, n_sel.p, rows, rt.stream);
            DevBuf<char> t;
            t.allocate(&rt, tmp + 16);
            AMBER_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, in, alive.p, o, n_sel.p, rows, rt.stream));
            rt.sync();
        };
        if (esz == 1) run(static_cast<uint8_t*>(data), reinterpret_cast<uint8_t*>(out.p));
        else if (esz == 4) run(static_cast<uint32_t*>(data), reinterpret_cast<uint32_t*>(out.p));
        else run(static_cast<unsigned long long*>(data), reinterpret_cast<unsigned long long*>(out.p));
        copy_out(rt, dst, out.p, live * esz, on_dev);
    }

    void batch_set(const std::string& nm, const int64_t* h_ids, const double* vals, int64_t n)
    {
        const int k = col_index(nm);
        if (k < 0) fail(AMBER_E_UNKNOWN_NAME, "no column " + nm);
        if (!n) return;
        // last staged write wins: keep the last occurrence of every id
        std::map<int64_t, double> last;
        for (int64_t i = 0; i < n; ++i) last[h_ids[i]] = vals[i];
        std::vector<int64_t> u;
        std::vector<double> v;
        for (auto& kv : last) {
            u.push_back(kv.first);
            v.push_back(kv.second);
        }
        DevBuf<int64_t> d_rows;
        find_rows(u.data(), static_cast<int64_t>(u.size()), d_rows);  // validates all before writing
        DevBuf<double> d_vals;
        d_vals.allocate(&rt, v.size());
        AMBER_CUDA(cudaMemcpyAsync(d_vals.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, rt.stream));
        pop_scatter_kernel<<<grid_for(v.size()), 256, 0, rt.stream>>>(ColView{cols[k]->data.p, cols[k]->dtype}, d_rows.p,
                                                                      d_vals.p, static_cast<int64_t>(v.size()));
        check_launch("pop_scatter_kernel");
        rt.sync();
    }
};

Population* make_population(const amber_column_spec* cols, int n, int64_t cap, uint64_t seed, const amber_runtime* rt)
{
    return new Population(cols, n, cap, seed, rt);
}
void destroy_population(Population* p) { delete p; }
int64_t population_add(Population* p, int64_t n, const double* d) { return p->add(n, d); }
void population_remove(Population* p, const int64_t* ids, int64_t n) { p->remove(ids, n); }
void population_compact(Population* p) { p->compact(); }
void population_update_paths(Population* p, int64_t* jit, int64_t* interp)
{
    if (jit) *jit = p->n_jit;
    if (interp) *interp = p->n_interp;
}

void population_size(Population* p, int64_t* live, int64_t* rows)
{
    if (live) *live = p->live;
    if (rows) *rows = p->rows;
}
int64_t population_update(Population* p, const char* t, const amber_instr* e, int ne, const amber_instr* w, int nw,
                          bool want_count)
{
    return p->update(t, e, ne, w, nw, want_count);
}
void population_synchronize(Population* p) { AMBER_CUDA(cudaStreamSynchronize(p->rt.stream)); }
double population_aggregate(Population* p, int agg, const amber_instr* e, int ne, const amber_instr* w, int nw)
{
    return p->aggregate(agg, e, ne, w, nw);
}
void population_read(Population* p, const char* nm, void* dst, size_t bytes, bool on_dev) { p->read(nm, dst, bytes, on_dev); }
void population_batch_set(Population* p, const char* nm, const int64_t* ids, const double* v, int64_t n)
{
    p->batch_set(nm, ids, v, n);
}
void population_set_step(Population* p, int64_t s)
{
    AMBER_REQUIRE(s >= 0 && s < (1ll << 32), "step out of range");
    p->step = s;
}

}  // namespace amber
