/*
 * oracle.c -- plain single-threaded CPU oracle for FastPAM SWAP / BUILD.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle_impl.h).  Built by
 * __graft_entry__.build() / oracle/__init__.py into oracle/liboracle.so with
 * plain `gcc -O2` (no -ffast-math: IEEE fp64 semantics are required).
 *
 * Instantiates oracle_impl.h for the two input types of BASELINE.json:
 *   *_u32 : uint32 dissimilarities, exact int64 sums  (configs C1, C5)
 *   *_f32 : float32 dissimilarities, fp64 sums        (configs C2, C3, C4)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

/* Reading R5: relative acceptance margin of the float path. */
#define ORACLE_EPS_REL 1e-12

#define D_T uint32_t
#define ACC_T int64_t
#define SFX _u32
#define ORACLE_IS_FLOAT 0
#include "oracle_impl.h"
#undef D_T
#undef ACC_T
#undef SFX
#undef ORACLE_IS_FLOAT

#define D_T float
#define ACC_T double
#define SFX _f32
#define ORACLE_IS_FLOAT 1
#include "oracle_impl.h"
#undef D_T
#undef ACC_T
#undef SFX
#undef ORACLE_IS_FLOAT
