/* Debug helper (not part of the build): LD_PRELOAD to print a native backtrace
 * on SIGSEGV, running on an alternate stack so stack overflows are caught too. */
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static void on_segv(int sig, siginfo_t* info, void* ctx) {
    (void)ctx;
    void* frames[64];
    char msg[128];
    int len = snprintf(msg, sizeof msg, "native signal %d at address %p\n", sig, info ? info->si_addr : 0);
    write(2, msg, len);
    int n = backtrace(frames, 64);
    backtrace_symbols_fd(frames, n, 2);
    _exit(1);
}

__attribute__((constructor)) void install(void) {
    static char altstack[1 << 16];
    stack_t ss;
    memset(&ss, 0, sizeof ss);
    ss.ss_sp = altstack;
    ss.ss_size = sizeof altstack;
    sigaltstack(&ss, 0);
    struct sigaction sa;
    memset(&sa, 0, sizeof sa);
    sa.sa_sigaction = on_segv;
    sa.sa_flags = SA_SIGINFO | SA_ONSTACK;
    sigaction(SIGSEGV, &sa, 0);
}
