// capi.cu -- the extern "C" boundary declared in include/amber.h.
// Every entry point converts internal exceptions into AMBER_E_* codes and a
// thread-local message; no C++ exception crosses the ABI.
#include <new>

#include "internal.cuh"

extern "C" int amber_nccl_unique_id_impl(void* out, size_t out_bytes);
extern "C" int amber_loopback_id_impl(void* out, size_t out_bytes);

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f)
{
    try {
        g_last_error.clear();
        return f();
    } catch (const amber::Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return AMBER_E_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return AMBER_E_INVALID_ARG;
    } catch (...) {
        g_last_error = "unknown internal error";
        return AMBER_E_INVALID_ARG;
    }
}

amber::Model* impl(amber_model* m)
{
    if (!m || !m->impl) amber::fail(AMBER_E_INVALID_ARG, "NULL model");
    return m->impl;
}

void need(const void* p, const char* what)
{
    if (!p) amber::fail(AMBER_E_INVALID_ARG, std::string("NULL ") + what);
}

}  // namespace

extern "C" {

int amber_version(void) { return AMBER_ABI_VERSION; }

const char* amber_last_error(void) { return g_last_error.c_str(); }

int amber_model_create(amber_kind kind, int64_t n_agents, const void* params, size_t params_size, uint64_t seed,
                       const amber_runtime* rt, amber_model** out)
{
    return guarded([&] {
        amber::NvtxRange nv("amber_model_create");
        need(out, "out");
        *out = nullptr;
        need(params, "params");
        AMBER_REQUIRE(n_agents >= 1, "n_agents must be >= 1");
        if (rt && rt->world > 1 && kind != AMBER_WEALTH && kind != AMBER_SIR_GRAPH && kind != AMBER_BOIDS)
            amber::fail(AMBER_E_UNSUPPORTED, "only AMBER_WEALTH, AMBER_SIR_GRAPH and AMBER_BOIDS are sharded across "
                                             "ranks (others: replicas / amber_sweep)");
        amber::Model* m = nullptr;
        switch (kind) {
            case AMBER_WEALTH:
                AMBER_REQUIRE(params_size >= sizeof(amber_wealth_params), "params_size < sizeof(amber_wealth_params)");
                m = amber::make_wealth(n_agents, *static_cast<const amber_wealth_params*>(params), seed, rt);
                break;
            case AMBER_SIR_GRAPH:
                AMBER_REQUIRE(params_size >= sizeof(amber_sir_params), "params_size < sizeof(amber_sir_params)");
                m = amber::make_sir(n_agents, *static_cast<const amber_sir_params*>(params), seed, rt);
                break;
            case AMBER_BOIDS:
                AMBER_REQUIRE(params_size >= sizeof(amber_boids_params), "params_size < sizeof(amber_boids_params)");
                m = amber::make_boids(n_agents, *static_cast<const amber_boids_params*>(params), seed, rt);
                break;
            case AMBER_SIR_SPACE:
                AMBER_REQUIRE(params_size >= sizeof(amber_sir_space_params),
                              "params_size < sizeof(amber_sir_space_params)");
                m = amber::make_sir_space(n_agents, *static_cast<const amber_sir_space_params*>(params), seed, rt);
                break;
            case AMBER_WALK:
                AMBER_REQUIRE(params_size >= sizeof(amber_walk_params), "params_size < sizeof(amber_walk_params)");
                m = amber::make_walk(n_agents, *static_cast<const amber_walk_params*>(params), seed, rt);
                break;
            default:
                amber::fail(AMBER_E_UNKNOWN_KIND, "unknown amber_kind " + std::to_string(static_cast<int>(kind)));
        }
        *out = new amber_model{m};
        return 0;
    });
}

int amber_model_destroy(amber_model* m)
{
    return guarded([&] {
        if (!m) return 0;
        delete m->impl;
        delete m;
        return 0;
    });
}

int amber_step(amber_model* m, int64_t n_steps)
{
    return guarded([&] {
        amber::NvtxRange nv("amber_step");
        impl(m)->step(n_steps);
        return 0;
    });
}

int amber_synchronize(amber_model* m)
{
    return guarded([&] {
        impl(m)->synchronize();
        return 0;
    });
}

int amber_step_count(amber_model* m, int64_t* out)
{
    return guarded([&] {
        need(out, "out");
        *out = impl(m)->t;
        return 0;
    });
}

int amber_set_step(amber_model* m, int64_t step)
{
    return guarded([&] {
        impl(m)->set_step(step);
        return 0;
    });
}

int amber_column_info(amber_model* m, const char* name, amber_dtype* dtype, int64_t* global_len, int64_t* local_off,
                      int64_t* local_len)
{
    return guarded([&] {
        need(name, "name");
        if (!impl(m)->column_info(name, dtype, global_len, local_off, local_len))
            amber::fail(AMBER_E_UNKNOWN_NAME, std::string("no column ") + name);
        return 0;
    });
}

int amber_read_column(amber_model* m, const char* name, void* dst, size_t dst_bytes, int dst_on_device)
{
    return guarded([&] {
        amber::NvtxRange nv("amber_read_column");
        need(name, "name");
        need(dst, "dst");
        impl(m)->read_column(name, dst, dst_bytes, dst_on_device != 0);
        return 0;
    });
}

int amber_write_column(amber_model* m, const char* name, const void* src, size_t src_bytes, int src_on_device)
{
    return guarded([&] {
        amber::NvtxRange nv("amber_write_column");
        need(name, "name");
        need(src, "src");
        impl(m)->write_column(name, src, src_bytes, src_on_device != 0);
        return 0;
    });
}

int amber_read_metrics(amber_model* m, const char* name, void* dst, size_t dst_bytes, int64_t* n_out)
{
    return guarded([&] {
        need(name, "name");
        need(dst, "dst");
        impl(m)->read_metrics(name, dst, dst_bytes, n_out);
        return 0;
    });
}

int amber_reset_metrics(amber_model* m)
{
    return guarded([&] {
        impl(m)->reset_metrics();
        return 0;
    });
}

int amber_digest(amber_model* m, const char* name, uint64_t* out)
{
    return guarded([&] {
        need(name, "name");
        need(out, "out");
        *out = impl(m)->digest(name);
        return 0;
    });
}

int amber_set_option(amber_model* m, const char* key, int64_t value)
{
    return guarded([&] {
        need(key, "key");
        if (!impl(m)->set_option(key, value)) amber::fail(AMBER_E_UNKNOWN_NAME, std::string("no option ") + key);
        return 0;
    });
}

int amber_get_option(amber_model* m, const char* key, int64_t* value)
{
    return guarded([&] {
        need(key, "key");
        need(value, "value");
        if (!impl(m)->get_option(key, value)) amber::fail(AMBER_E_UNKNOWN_NAME, std::string("no option ") + key);
        return 0;
    });
}

int amber_profile_enable(amber_model* m, int enable)
{
    return guarded([&] {
        amber::Model* x = impl(m);
        AMBER_CUDA(cudaStreamSynchronize(x->rt.stream));
        x->prof.enable(enable != 0);
        return 0;
    });
}

int amber_profile_query(amber_model* m, int idx, char* name, size_t name_cap, int64_t* launches, double* total_ms)
{
    return guarded([&] {
        need(launches, "launches");
        need(total_ms, "total_ms");
        std::string nm;
        if (!impl(m)->prof.query(idx, &nm, launches, total_ms))
            amber::fail(AMBER_E_INVALID_ARG, "profile index out of range");
        if (name && name_cap) {
            std::strncpy(name, nm.c_str(), name_cap - 1);
            name[name_cap - 1] = 0;
        }
        return 0;
    });
}

int amber_sweep(amber_kind kind, int64_t n_agents, const void* base_params, size_t params_size,
                const amber_replicate* reps, int64_t n_reps, int64_t n_steps, const amber_runtime* rt,
                double* out_final_r_frac, amber_sweep_stats* stats)
{
    return guarded([&] {
        amber::NvtxRange nv("amber_sweep");
        if (kind != AMBER_SIR_GRAPH) amber::fail(AMBER_E_UNKNOWN_KIND, "amber_sweep supports AMBER_SIR_GRAPH only");
        need(base_params, "base_params");
        AMBER_REQUIRE(params_size >= sizeof(amber_sir_params), "params_size < sizeof(amber_sir_params)");
        AMBER_REQUIRE(n_reps >= 0 && n_steps >= 0 && n_agents >= 2, "bad sweep sizes");
        if (n_reps) {
            need(reps, "reps");
            need(out_final_r_frac, "out_final_r_frac");
        }
        amber::run_sweep(n_agents, *static_cast<const amber_sir_params*>(base_params), reps, n_reps, n_steps, rt,
                         out_final_r_frac, stats);
        return 0;
    });
}

int amber_shard_range(int64_t n_agents, int world, int rank, int64_t* lo, int64_t* hi)
{
    return guarded([&] {
        need(lo, "lo");
        need(hi, "hi");
        AMBER_REQUIRE(n_agents >= 1 && world >= 1 && rank >= 0 && rank < world, "bad shard request");
        amber::shard_range(n_agents, world, rank, lo, hi);
        return 0;
    });
}

int amber_sir_shard_range(int64_t n_agents, int world, int rank, int64_t* lo, int64_t* hi)
{
    return guarded([&] {
        need(lo, "lo");
        need(hi, "hi");
        AMBER_REQUIRE(n_agents >= 1 && world >= 1 && rank >= 0 && rank < world, "bad shard request");
        int64_t len = 0, shard = 0;
        amber::sir_shard_range(n_agents, world, rank, lo, &len, &shard);
        *hi = *lo + len;
        return 0;
    });
}

int amber_sweep_range(int64_t n_reps, int world, int rank, int64_t* r0, int64_t* r1)
{
    return guarded([&] {
        need(r0, "r0");
        need(r1, "r1");
        AMBER_REQUIRE(n_reps >= 0 && world >= 1 && rank >= 0 && rank < world, "bad sweep-range request");
        amber::sweep_range(n_reps, world, rank, r0, r1);
        return 0;
    });
}

static amber::Population* pimpl(amber_population* p)
{
    if (!p || !p->impl) amber::fail(AMBER_E_INVALID_ARG, "NULL population");
    return p->impl;
}

int amber_population_create(const amber_column_spec* cols, int n_cols, int64_t capacity, uint64_t seed,
                            const amber_runtime* rt, amber_population** out)
{
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        need(cols, "cols");
        *out = new amber_population{amber::make_population(cols, n_cols, capacity, seed, rt)};
        return 0;
    });
}

int amber_population_destroy(amber_population* p)
{
    return guarded([&] {
        if (!p) return 0;
        amber::destroy_population(p->impl);
        delete p;
        return 0;
    });
}

int amber_population_add_agents(amber_population* p, int64_t n, const double* defaults, int64_t* first_id)
{
    return guarded([&] {
        const int64_t f = amber::population_add(pimpl(p), n, defaults);
        if (first_id) *first_id = f;
        return 0;
    });
}

int amber_population_remove_agents(amber_population* p, const int64_t* ids, int64_t n)
{
    return guarded([&] {
        AMBER_REQUIRE(n >= 0 && (n == 0 || ids), "bad id list");
        amber::population_remove(pimpl(p), ids, n);
        return 0;
    });
}

int amber_population_compact(amber_population* p)
{
    return guarded([&] {
        amber::population_compact(pimpl(p));
        return 0;
    });
}

int amber_population_size(amber_population* p, int64_t* live, int64_t* rows)
{
    return guarded([&] {
        amber::population_size(pimpl(p), live, rows);
        return 0;
    });
}

int amber_population_update_paths(amber_population* p, int64_t* n_jit, int64_t* n_interp)
{
    return guarded([&] {
        amber::population_update_paths(pimpl(p), n_jit, n_interp);
        return 0;
    });
}

int amber_population_update(amber_population* p, const char* target, const amber_instr* expr, int n_expr,
                            const amber_instr* where, int n_where, int64_t* n_updated)
{
    return guarded([&] {
        need(target, "target");
        const int64_t k = amber::population_update(pimpl(p), target, expr, n_expr, where, n_where, n_updated != nullptr);
        if (n_updated) *n_updated = k;
        return 0;
    });
}

int amber_population_aggregate(amber_population* p, int agg, const amber_instr* expr, int n_expr,
                               const amber_instr* where, int n_where, double* out)
{
    return guarded([&] {
        need(out, "out");
        *out = amber::population_aggregate(pimpl(p), agg, expr, n_expr, where, n_where);
        return 0;
    });
}

int amber_population_read_column(amber_population* p, const char* name, void* dst, size_t dst_bytes,
                                 int dst_on_device)
{
    return guarded([&] {
        need(name, "name");
        need(dst, "dst");
        amber::population_read(pimpl(p), name, dst, dst_bytes, dst_on_device != 0);
        return 0;
    });
}

int amber_population_batch_set(amber_population* p, const char* name, const int64_t* ids, const double* values,
                               int64_t n)
{
    return guarded([&] {
        need(name, "name");
        AMBER_REQUIRE(n >= 0 && (n == 0 || (ids && values)), "bad batch");
        amber::population_batch_set(pimpl(p), name, ids, values, n);
        return 0;
    });
}

int amber_population_synchronize(amber_population* p)
{
    return guarded([&] {
        amber::population_synchronize(pimpl(p));
        return 0;
    });
}

int amber_population_set_step(amber_population* p, int64_t step)
{
    return guarded([&] {
        amber::population_set_step(pimpl(p), step);
        return 0;
    });
}

int amber_loopback_id(void* out, size_t out_bytes)
{
    return guarded([&] { return amber_loopback_id_impl(out, out_bytes); });
}

int amber_nccl_unique_id(void* out, size_t out_bytes)
{
    return guarded([&] { return amber_nccl_unique_id_impl(out, out_bytes); });
}

}  // extern "C"
