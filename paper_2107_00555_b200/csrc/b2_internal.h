// Internal helpers shared by the libb2 translation units.
#pragma once
#include <cuda_runtime.h>

int b2_fail(int code, const char *fmt, ...);
int b2_cuda_check(cudaError_t e, const char *what);
void b2_count_launch();

// Drop a stale error left by an earlier, already-reported failure so the
// check after our own launch sees only that launch.
#define B2_CLEAR_ERROR() ((void)cudaGetLastError())

#define B2_LAUNCH_CHECK(what)                                   \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return b2_cuda_check(_e, what);      \
    b2_count_launch();                                          \
  } while (0)
