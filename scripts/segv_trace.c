/* LD_PRELOAD debugging aid: on SIGSEGV print a backtrace (addresses + the mapping of
 * libbfly_b200.so) so the frames can be resolved with addr2line on the build machine. */
#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>
static void handler(int sig) {
    void* frames[64];
    int n = backtrace(frames, 64);
    fprintf(stderr, "segv_trace: signal %d, %d frames\n", sig, n);
    backtrace_symbols_fd(frames, n, 2);
    FILE* f = fopen("/proc/self/maps", "r");
    if (f) {
        char line[512];
        while (fgets(line, sizeof line, f))
            if (strstr(line, "libbfly_b200") && strstr(line, "r-xp")) fputs(line, stderr);
        fclose(f);
    }
    _exit(139);
}
__attribute__((constructor)) static void install(void) {
    struct sigaction sa;
    memset(&sa, 0, sizeof sa);
    sa.sa_handler = handler;
    sigaction(SIGSEGV, &sa, NULL);
    sigaction(SIGBUS, &sa, NULL);
    sigaction(SIGABRT, &sa, NULL);
}
