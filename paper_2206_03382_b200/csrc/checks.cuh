// Device-side bounds / invariant checks (compute-sanitizer is unavailable on this pool). Built in
// with -DMOE_CHECKS (tools/checks_build.sh -> paper_2206_03382_b200/libmoe_b200_checks.so); the
// GPU test suite runs against that build (MOE_LIB_PATH) and a violated check traps the kernel,
// which the ABI reports as MOE_ECUDA. Compiled out of the product library.
#pragma once

#include <cstdio>

#ifdef MOE_CHECKS
#define MOE_CHECK(cond, what)                                                                   \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("MOE_CHECK failed: %s (%s) at %s:%d block %d thread %d\n", what, #cond, __FILE__, \
             __LINE__, blockIdx.x, threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define MOE_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif
