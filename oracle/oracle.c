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

/* FastCLARA from points (NEXT-3; "the remaining objects are
 * assigned to their closest medoid"; reading C2 in DESIGN.md):
 * TD over ALL n objects of the medoids M (point indices) by the definition,
 * Eq. eqn:td, with the dissimilarity recomputed from the points.
 *   L2: d = (double)(float)sqrt(sum_t (x_ot - x_mt)^2)  (the f32 value of the
 *       Euclidean distance, as in the f32 dissimilarity matrices), fp64 sum
 *   L1: d = sum_t |x_ot - x_mt| in int64, int64 sum
 * mins (may be NULL) receives each object's distance to its closest medoid;
 * asg (may be NULL) the slot of that medoid (smallest slot on ties, R2). */
double oracle_td_points_l2(const float* X, int32_t n, int32_t d, const int32_t* M, int32_t k, double* mins,
                           int32_t* asg) {
    double td = 0;
    for (int32_t o = 0; o < n; ++o) {
        double best = 0;
        int32_t bj = -1;
        for (int32_t j = 0; j < k; ++j) {
            double s = 0;
            for (int32_t t = 0; t < d; ++t) {
                const double u = (double)X[(int64_t)o * d + t] - (double)X[(int64_t)M[j] * d + t];
                s += u * u;
            }
            const double v = (double)(float)sqrt(s);
            if (bj < 0 || v < best) { best = v; bj = j; }
        }
        if (mins) mins[o] = best;
        if (asg) asg[o] = bj;
        td += best;
    }
    return td;
}

int64_t oracle_td_points_l1(const int32_t* X, int32_t n, int32_t d, const int32_t* M, int32_t k, int64_t* mins,
                            int32_t* asg) {
    int64_t td = 0;
    for (int32_t o = 0; o < n; ++o) {
        int64_t best = 0;
        int32_t bj = -1;
        for (int32_t j = 0; j < k; ++j) {
            int64_t s = 0;
            for (int32_t t = 0; t < d; ++t) {
                const int64_t u = (int64_t)X[(int64_t)o * d + t] - (int64_t)X[(int64_t)M[j] * d + t];
                s += u < 0 ? -u : u;
            }
            if (bj < 0 || s < best) { best = s; bj = j; }
        }
        if (mins) mins[o] = best;
        if (asg) asg[o] = bj;
        td += best;
    }
    return td;
}
