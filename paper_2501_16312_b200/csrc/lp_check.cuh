// lp_check.cuh -- LP_CHECK: device-side index invariants of checked builds.
#pragma once

// Device-side bounds checks (the compute-sanitizer stand-in; compute-sanitizer is closed on the GPU
// pool): a -DLP_CHECKED build (liblinprim_checked.so, _build.build(variant="checked")) traps on
// every violated index invariant below; the product build compiles them out.
#ifdef LP_CHECKED
#include <cstdio>
#define LP_CHECK(cond)                                                                                   \
  do {                                                                                                   \
    if (!(cond)) {                                                                                       \
      printf("LP_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, blockIdx.x, \
             threadIdx.x);                                                                               \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)
#else
#define LP_CHECK(cond) \
  do {                 \
  } while (0)
#endif

