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

/* Dissimilarity matrix from points (NEXT-2 pin; "a dissimilarity
 * matrix ... computed in advance").  Plain definitions, fp64 / int64:
 *   oracle_dist_l2: D[i][j] = sqrt(sum_t (x_it - x_jt)^2)   (Euclidean)
 *   oracle_dist_l1: D[i][j] = sum_t |x_it - x_jt|           (Manhattan, integer)
 * Row i of X is X[i*d .. i*d+d); D is n x n row-major. */
void oracle_dist_l2(const float* X, int32_t n, int32_t d, double* D) {
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < n; ++j) {
            double s = 0;
            for (int32_t t = 0; t < d; ++t) {
                const double u = (double)X[(int64_t)i * d + t] - (double)X[(int64_t)j * d + t];
                s += u * u;
            }
            D[(int64_t)i * n + j] = sqrt(s);
        }
}

void oracle_dist_l1(const int32_t* X, int32_t n, int32_t d, int64_t* D) {
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < n; ++j) {
            int64_t s = 0;
            for (int32_t t = 0; t < d; ++t) {
                const int64_t u = (int64_t)X[(int64_t)i * d + t] - (int64_t)X[(int64_t)j * d + t];
                s += u < 0 ? -u : u;
            }
            D[(int64_t)i * n + j] = s;
        }
}
