// LD_PRELOAD helper: print a native backtrace on SIGSEGV (no gdb in the image).
// gcc -shared -fPIC -o build/segv_bt.so tools/diag/segv_bt.c
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <unistd.h>
static void h(int s) {
    void* b[64];
    int n = backtrace(b, 64);
    fprintf(stderr, "=== signal %d backtrace\n", s);
    backtrace_symbols_fd(b, n, 2);
    _exit(139);
}
__attribute__((constructor)) static void init(void) { signal(SIGSEGV, h); }
