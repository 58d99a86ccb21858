// Debug repro (not part of the build): run_bench with W in {1,2} + SIGSEGV backtrace.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cstdio>

#include "synkpar/bench.hpp"

static void on_segv(int sig) {
    void* frames[64];
    int n = backtrace(frames, 64);
    fprintf(stderr, "signal %d\n", sig);
    backtrace_symbols_fd(frames, n, 2);
    _exit(1);
}

int main() {
    signal(SIGSEGV, on_segv);
    synkpar::BenchConfig c;
    c.workers = {1, 2};
    c.steps = 2;
    c.batch = 8;
    c.width = 8;
    c.layers = 2;
    c.in_dim = 4;
    c.out_dim = 2;
    c.seed = 3;
    c.pin_threads = false;
    auto r = synkpar::run_bench(c);
    printf("%s", synkpar::report_to_json(r).c_str());
    return 0;
}
