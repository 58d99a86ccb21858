// Timing driver for the CPU reference arm of bench.py (TEST/BENCH
// INFRASTRUCTURE ONLY). Links the UNMODIFIED reference library built by
// oracle/Makefile (namespace renamed synkpar -> synkpar_ref at preprocessing)
// and drives it through its own public API and stock code path:
//
//   gather: SharedInputArray [rows x cols] f32 -> ParallelFunction with a
//           no-op kernel (row count, Sum) called with an IndexList of
//           `batch` rows; CallReport.scatter_s isolates excerpt_rows ->
//           gather_rows.
//   sgd:    SyncSgd::train_step of the MLP (in-width-out, layers 2) on a
//           SharedInputArray dataset, indexed batches (C1).
//   collective: ReplicatedVariable::all_reduce(Mean) and broadcast(0) of a
//           `--bytes` f32 buffer at `--workers` ranks (C4).
//   slicing: ParallelFunction over an explicit scatter input [rows x cols]
//           f32 with num_slices slices; the kernel returns column sums (Sum),
//           column maxima (Max) and the shard itself (Gather) -- the
//           acceptance battery's columnwise kernels (acceptance_main.cpp:86-133)
//           written over spans (C3).
//
// Prints one JSON object on stdout.

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "synkpar/bench.hpp"
#include "synkpar/function.hpp"
#include "synkpar/mlp.hpp"
#include "synkpar/sgd.hpp"
#include "synkpar/shared_input.hpp"

using namespace synkpar;  // -> synkpar_ref
using Clock = std::chrono::steady_clock;

static std::uint64_t splitmix(std::uint64_t& s) {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static long arg(int argc, char** argv, const char* name, long dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], name)) return std::atol(argv[i + 1]);
    return dflt;
}

static std::string sarg(int argc, char** argv, const char* name, const char* dflt) {
    for (int i = 1; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], name)) return argv[i + 1];
    return dflt;
}

static int run_gather(int argc, char** argv) {
    const std::size_t rows = arg(argc, argv, "--rows", 10000000);
    const std::size_t cols = arg(argc, argv, "--cols", 256);
    const std::size_t batch = arg(argc, argv, "--batch", 4096);
    const long steps = arg(argc, argv, "--steps", 10);
    const long warmup = arg(argc, argv, "--warmup", 2);
    std::size_t workers = arg(argc, argv, "--workers", 0);
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());

    auto t_alloc = Clock::now();
    SharedInputArray data = SharedInputArray::alloc({rows, cols}, DType::Float32);
    {
        // Fill through the public write() in row blocks with a cheap seeded stream.
        const std::size_t block = 1u << 16;
        std::uint64_t s = 7;
        for (std::size_t r0 = 0; r0 < rows; r0 += block) {
            std::size_t n = std::min(block, rows - r0);
            NdBuffer b = NdBuffer::zeros({n, cols}, DType::Float32);
            auto v = b.as_mut<float>();
            for (std::size_t i = 0; i < v.size(); ++i)
                v[i] = float(double(splitmix(s) >> 11) * (2.0 / 9007199254740992.0) - 1.0);
            data.write(RowRange{r0, r0 + n}, b);
        }
    }
    double alloc_s = std::chrono::duration<double>(Clock::now() - t_alloc).count();

    WorkerPool pool = WorkerPool::fork(ForkOptions{.workers = workers, .pin_threads = true});
    Kernel k;
    k.name = "row_count";
    k.arity = 1;
    k.fn = [](const std::vector<NdBuffer>& in, const KernelContext&) {
        return KernelResult{{NdBuffer::scalar(double(in[0].rows()))}, {}};
    };
    ParallelFunction f = function(pool, k, {InputSpec{InputMode::Scatter}}, {OutputSpec{ReduceOp::Sum}});
    distribute(pool);

    std::mt19937_64 rng(1234);
    std::uniform_int_distribution<std::size_t> pick(0, rows - 1);
    double timed = 0.0, scatter = 0.0;
    for (long s = 0; s < warmup + steps; ++s) {
        IndexList idx(batch);
        for (auto& i : idx) i = pick(rng);
        CallOptions o;
        o.indexes = IndexSelection(std::move(idx));
        auto t0 = Clock::now();
        CallResult r = f.call({FunctionArg(data)}, o);
        double dt = std::chrono::duration<double>(Clock::now() - t0).count();
        if (r.outputs[0].get(0) != double(batch)) {
            std::fprintf(stderr, "row count mismatch\n");
            return 2;
        }
        if (s >= warmup) {
            timed += dt;
            scatter += r.report.scatter_s;
        }
    }
    const double bytes_per_row = 2.0 * cols * 4 + 8;  // read + write + u64 index
    const double gbs = double(batch) * steps * bytes_per_row / timed / 1e9;
    std::printf("{\"mode\": \"gather\", \"rows\": %zu, \"cols\": %zu, \"batch\": %zu, \"steps\": %ld, \"workers\": %zu,"
                " \"seconds\": %.6f, \"ms_per_step\": %.4f, \"gbs\": %.4f, \"scatter_s_mean\": %.6f,"
                " \"setup_s\": %.2f}\n",
                rows, cols, batch, steps, workers, timed, 1e3 * timed / steps, gbs, scatter / steps, alloc_s);
    return 0;
}

static int run_sgd(int argc, char** argv) {
    const std::size_t in_dim = arg(argc, argv, "--in", 784), width = arg(argc, argv, "--width", 512);
    const std::size_t out_dim = arg(argc, argv, "--out", 10), layers = arg(argc, argv, "--layers", 2);
    const std::size_t batch = arg(argc, argv, "--batch", 256), ds_rows = arg(argc, argv, "--rows", 65536);
    const long steps = arg(argc, argv, "--steps", 5), warmup = arg(argc, argv, "--warmup", 1);
    std::size_t workers = arg(argc, argv, "--workers", 0);
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    const std::string dt = sarg(argc, argv, "--dtype", "f32");
    const DType dtype = dt == "f64" ? DType::Float64 : DType::Float32;

    MlpConfig cfg{in_dim, width, out_dim, layers, 1};
    Dataset ds = mlp_make_dataset(ds_rows, cfg, 2, dtype);
    SharedInputArray sx = SharedInputArray::from_buffer(ds.x), sy = SharedInputArray::from_buffer(ds.y);
    WorkerPool pool = WorkerPool::fork(ForkOptions{.workers = workers, .pin_threads = true});
    FlatParamBlock block = FlatParamBlock::create(pool, mlp_init_params(cfg, dtype));
    ParallelFunction f = function(pool, mlp_grad_kernel(block), {InputSpec{InputMode::Scatter}, InputSpec{InputMode::Scatter}},
                                  {OutputSpec{ReduceOp::Mean}}, mlp_grad_updates(block));
    SyncSgd trainer(pool, block, SgdRule{}, 0.01);
    std::mt19937_64 rng(42);
    std::uniform_int_distribution<std::size_t> pick(0, ds_rows - 1);
    // Table-1 accounting of the reference's own bench (src/bench.cpp:186-198):
    // function = grad + step compute means, shuffle = index selection +
    // grad-call scatter, straggler = grad + step stragglers, all-reduce.
    double timed = 0.0, allreduce = 0.0, function_s = 0.0, shuffle = 0.0, straggler = 0.0, loss = 0.0;
    for (long s = 0; s < warmup + steps; ++s) {
        auto t0 = Clock::now();
        IndexList idx(batch);
        for (auto& i : idx) i = pick(rng);
        CallOptions o;
        o.indexes = IndexSelection(std::move(idx));
        const double select_s = std::chrono::duration<double>(Clock::now() - t0).count();
        loss = trainer.train_step(f, {FunctionArg(sx), FunctionArg(sy)}, o);
        double d = std::chrono::duration<double>(Clock::now() - t0).count();
        if (s >= warmup) {
            const StepReport& sr = trainer.last_report();
            timed += d;
            allreduce += sr.allreduce_s;
            function_s += sr.grad_call.compute_mean_s() + sr.step_call.compute_mean_s();
            shuffle += select_s + sr.grad_call.scatter_s;
            straggler += sr.grad_call.straggler_s + sr.step_call.straggler_s;
        }
    }
    std::printf("{\"mode\": \"sgd\", \"batch\": %zu, \"steps\": %ld, \"workers\": %zu, \"seconds\": %.6f,"
                " \"ms_per_step\": %.4f, \"samples_per_s\": %.3f, \"allreduce_s_mean\": %.6f, \"loss\": %.9g,"
                " \"table1\": {\"total_s\": %.6f, \"function_s\": %.6f, \"shuffle_s\": %.6f, \"straggler_s\": %.6f,"
                " \"allreduce_s\": %.6f}}\n",
                batch, steps, workers, timed, 1e3 * timed / steps, double(batch) * steps / timed, allreduce / steps,
                loss, timed, function_s, shuffle, straggler, allreduce);
    return 0;
}

// The reference's own trainer benchmark (src/bench.cpp run_bench): the loss
// of every step of every run, for trajectory comparisons with ours.
static int run_bench_mode(int argc, char** argv) {
    BenchConfig c;
    c.workers.clear();
    const std::string w = sarg(argc, argv, "--workers-list", "1,2");
    for (std::size_t at = 0; at < w.size();) {
        std::size_t comma = w.find(',', at);
        if (comma == std::string::npos) comma = w.size();
        c.workers.push_back(std::stoul(w.substr(at, comma - at)));
        at = comma + 1;
    }
    c.steps = arg(argc, argv, "--steps", 4);
    c.batch = arg(argc, argv, "--batch", 16);
    c.batch_mode = sarg(argc, argv, "--batch-mode", "scaled") == "fixed" ? BatchMode::Fixed : BatchMode::ScaledByWorkers;
    c.width = arg(argc, argv, "--width", 32);
    c.layers = arg(argc, argv, "--layers", 2);
    c.seed = arg(argc, argv, "--seed", 0);
    c.in_dim = arg(argc, argv, "--in", 16);
    c.out_dim = arg(argc, argv, "--out", 4);
    c.pin_threads = false;
    BenchReport rep = run_bench(c);
    std::printf("{\"mode\": \"bench\", \"runs\": [");
    for (std::size_t i = 0; i < rep.runs.size(); ++i) {
        std::printf("%s{\"workers\": %zu, \"losses\": [", i ? ", " : "", rep.runs[i].workers);
        for (std::size_t k = 0; k < rep.runs[i].losses.size(); ++k)
            std::printf("%s%.17g", k ? ", " : "", rep.runs[i].losses[k]);
        std::printf("]}");
    }
    std::printf("]}\n");
    return 0;
}

static int run_slicing(int argc, char** argv) {
    const std::size_t rows = arg(argc, argv, "--rows", 262144), cols = arg(argc, argv, "--cols", 1024);
    const std::size_t slices = arg(argc, argv, "--slices", 4);
    const long steps = arg(argc, argv, "--steps", 3), warmup = arg(argc, argv, "--warmup", 1);
    std::size_t workers = arg(argc, argv, "--workers", 0);
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    NdBuffer x = NdBuffer::zeros({rows, cols}, DType::Float32);
    {
        std::uint64_t s = 7;
        for (float& v : x.as_mut<float>()) v = float(double(splitmix(s) >> 11) * (2.0 / 9007199254740992.0) - 1.0);
    }
    WorkerPool pool = WorkerPool::fork(ForkOptions{.workers = workers, .pin_threads = true});
    Kernel k;
    k.name = "column_stats";
    k.arity = 1;
    k.fn = [](const std::vector<NdBuffer>& in, const KernelContext&) {
        const NdBuffer& a = in[0];
        const std::size_t c = a.row_size();
        NdBuffer sum = NdBuffer::zeros({c}, a.dtype());
        NdBuffer mx = NdBuffer::full({c}, -std::numeric_limits<double>::infinity(), a.dtype());
        auto v = a.as<float>();
        auto so = sum.as_mut<float>();
        auto mo = mx.as_mut<float>();
        for (std::size_t r = 0; r < a.rows(); ++r)
            for (std::size_t j = 0; j < c; ++j) {
                const float e = v[r * c + j];
                so[j] += e;
                mo[j] = e > mo[j] ? e : mo[j];
            }
        return KernelResult{{sum, mx, a}, {}};
    };
    ParallelFunction f = function(pool, k, {InputSpec{InputMode::Scatter}},
                                  {OutputSpec{ReduceOp::Sum}, OutputSpec{ReduceOp::Max}, OutputSpec{ReduceOp::Gather}});
    distribute(pool);
    double timed = 0.0;
    for (long s = 0; s < warmup + steps; ++s) {
        CallOptions o;
        o.num_slices = slices;
        auto t0 = Clock::now();
        CallResult r = f.call({FunctionArg(x)}, o);
        double d = std::chrono::duration<double>(Clock::now() - t0).count();
        if (r.outputs[2].rows() != rows) {
            std::fprintf(stderr, "gather rows mismatch\n");
            return 2;
        }
        if (s >= warmup) timed += d;
    }
    const double bytes = double(rows) * cols * 4;
    std::printf("{\"mode\": \"slicing\", \"rows\": %zu, \"cols\": %zu, \"slices\": %zu, \"steps\": %ld,"
                " \"workers\": %zu, \"seconds\": %.6f, \"ms_per_step\": %.4f, \"gbs\": %.4f}\n",
                rows, cols, slices, steps, workers, timed, 1e3 * timed / steps, bytes * steps / timed / 1e9);
    return 0;
}

static int run_collective(int argc, char** argv) {
    const std::size_t bytes = arg(argc, argv, "--bytes", 1 << 20);
    const long steps = arg(argc, argv, "--steps", 5), warmup = arg(argc, argv, "--warmup", 1);
    const std::size_t workers = std::max(2L, arg(argc, argv, "--workers", 2));
    const std::size_t n = std::max<std::size_t>(1, bytes / 4);
    WorkerPool pool = WorkerPool::fork(ForkOptions{.workers = workers, .pin_threads = true});
    ReplicatedVariable var = replicate(pool, NdBuffer::zeros({n}, DType::Float32));
    std::uint64_t seed = 1000;
    for (std::size_t r = 0; r < workers; ++r) {
        NdBuffer v = NdBuffer::zeros({n}, DType::Float32);
        for (float& e : v.as_mut<float>()) e = float(double(splitmix(seed) >> 11) * (2.0 / 9007199254740992.0) - 1.0);
        var.set_value(r, v);
    }
    double t_ar = 0.0, t_bc = 0.0;
    for (long s = 0; s < warmup + steps; ++s) {
        auto t0 = Clock::now();
        var.all_reduce(ReduceOp::Mean);
        auto t1 = Clock::now();
        var.broadcast(0);
        auto t2 = Clock::now();
        if (s >= warmup) {
            t_ar += std::chrono::duration<double>(t1 - t0).count();
            t_bc += std::chrono::duration<double>(t2 - t1).count();
        }
    }
    const double S = double(n) * 4, W = double(workers);
    t_ar /= double(steps);
    t_bc /= double(steps);
    std::printf("{\"mode\": \"collective\", \"bytes\": %.0f, \"workers\": %zu, \"steps\": %ld,"
                " \"allreduce_us\": %.3f, \"allreduce_busbw_gbs\": %.4f, \"broadcast_us\": %.3f,"
                " \"broadcast_busbw_gbs\": %.4f}\n",
                S, workers, steps, 1e6 * t_ar, S / t_ar * 2 * (W - 1) / W / 1e9, 1e6 * t_bc, S / t_bc / 1e9);
    return 0;
}

int main(int argc, char** argv) {
    std::string mode = sarg(argc, argv, "--mode", "gather");
    try {
        if (mode == "gather") return run_gather(argc, argv);
        if (mode == "sgd") return run_sgd(argc, argv);
        if (mode == "slicing") return run_slicing(argc, argv);
        if (mode == "bench") return run_bench_mode(argc, argv);
        if (mode == "collective") return run_collective(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_driver: %s\n", e.what());
        return 1;
    }
    std::fprintf(stderr, "unknown --mode %s\n", mode.c_str());
    return 1;
}
