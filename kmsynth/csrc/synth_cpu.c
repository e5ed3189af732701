/*
 * synth_cpu.c -- multi-threaded CPU materialisation of a config's
 * dissimilarity matrix (INPUT GENERATOR, no method arithmetic).
 *
 * Bit-identical to kmsynth.dist_numpy (and to the CUDA materialiser
 * synth_dist.cu): L1 = exact int64 sum of |x_ot - x_ct| over integer
 * coordinates, stored as uint32; L2 = f32(sqrt(acc)) with
 * acc = acc + diff * diff evaluated in fp64 in t order, every operation
 * rounded on its own (built with -ffp-contract=off, no fast-math).
 *
 * Used by scripts/make_goldens.py to produce the full-size inputs the oracle
 * runs on (C4: 10 GB, C5: 40 GB) in minutes instead of hours of numpy.
 */
#include <math.h>
#include <stdint.h>

void kmsynth_cpu_dist_l1(const int32_t* X, int64_t n, int32_t d, int64_t c0, int64_t c1, int64_t ld, uint32_t* out) {
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t o = 0; o < n; ++o) {
        const int32_t* xo = X + o * d;
        uint32_t* row = out + o * ld;
        for (int64_t c = c0; c < c1; ++c) {
            const int32_t* xc = X + c * d;
            int64_t s = 0;
            for (int32_t t = 0; t < d; ++t) {
                int64_t u = (int64_t)xo[t] - (int64_t)xc[t];
                s += u < 0 ? -u : u;
            }
            row[c - c0] = (uint32_t)s;
        }
    }
}

void kmsynth_cpu_dist_l2(const double* X, int64_t n, int32_t d, int64_t c0, int64_t c1, int64_t ld, float* out) {
    #pragma omp parallel for schedule(dynamic, 64)
    for (int64_t o = 0; o < n; ++o) {
        const double* xo = X + o * d;
        float* row = out + o * ld;
        for (int64_t c = c0; c < c1; ++c) {
            const double* xc = X + c * d;
            double acc = 0.0;
            for (int32_t t = 0; t < d; ++t) {
                double diff = xo[t] - xc[t];
                double sq = diff * diff;
                acc = acc + sq;
            }
            row[c - c0] = (float)sqrt(acc);
        }
    }
}
