/*
 * oracle_impl.h -- body of the CPU oracle, instantiated twice by oracle.c:
 *   D_T = uint32_t, ACC_T = int64_t   (suffix _u32: integer-quantised dissimilarities)
 *   D_T = float,    ACC_T = double    (suffix _f32: float32 dissimilarities, fp64 sums)
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this code.  It
 * shares nothing with the CUDA path (paper_2008_05171_b200/csrc).
 *
 * Everything here is a plain, single-threaded restatement of PAPER.md
 * (Schubert & Rousseeuw, "Fast and eager k-medoids clustering"); each
 * function cites the lines it follows.  Notation:
 *   d(x_o, x_c) := D[o*ld + c]   (row = the object o, column = the medoid /
 *   candidate c; reading R0).  Every D value is widened to ACC_T
 *   before any arithmetic (SURVEY 8(c) "Accumulation").
 *   Medoids live in slots 0..k-1; nearest(o)/second(o) are slot indices.
 *
 * Readings of the paper used here (all listed in DESIGN.md):
 *   R1 best-swap key is (dTD, slot i, candidate c) lexicographic  (c1)
 *   R2 nearest/second ties go to the smaller slot                  (c3)
 *   R3 BUILD includes the x_o = x_c term                          (c5)
 *   R4 BUILD ties: smallest point index; no early stop           (c6)
 *   R5 acceptance: int dTD < 0; float dTD < -EPS_REL*|TD|        (c7)
 *   R6 FastPAM2 per-iteration procedure                           (c10)
 *   F1-F5 FasterPAM scan order, termination, pass count, slot choice,
 *         swap target (oracle_fasterpam_run)                       (c12)
 */

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SFX)
#define DIST(o, c) ((ACC_T)D[(int64_t)(o) * ld + (c)])

/* R5: acceptance of a swap / convergence test (Alg.2, Alg.3 P:898:
 * "break loop if dTD* >= 0").  The float reading adds a relative margin so
 * fp64 rounding cannot produce +-eps cycles. */
static int FN(improving)(ACC_T v, ACC_T td) {
#if ORACLE_IS_FLOAT
    return v < -ORACLE_EPS_REL * fabs(td);
#else
    (void)td;
    return v < 0;
#endif
}

/* Eq. eqn:td: TD = sum over all objects of the dissimilarity to
 * the closest medoid. */
ACC_T FN(oracle_td)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k) {
    ACC_T td = 0;
    for (int32_t o = 0; o < n; ++o) {
        ACC_T best = DIST(o, M[0]);
        for (int32_t j = 1; j < k; ++j) {
            ACC_T d = DIST(o, M[j]);
            if (d < best) best = d;
        }
        td += best;
    }
    return td;
}

/* Alg.2 line P:347-348 / Alg.3: nearest(o), d_n(o), d_s(o) (and
 * the second-nearest slot).  Two plain passes: nearest is the
 * smallest (d, slot); second is the smallest (d, slot) over slots != nearest
 * (reading R2).  Needs k >= 2 (the second nearest must exist). */
int FN(oracle_assign)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k,
                      int32_t* nearest, int32_t* second, ACC_T* dn, ACC_T* ds) {
    if (k < 2) return -1;
    for (int32_t o = 0; o < n; ++o) {
        int32_t a = 0;
        for (int32_t j = 1; j < k; ++j)
            if (DIST(o, M[j]) < DIST(o, M[a])) a = j;
        int32_t b = (a == 0) ? 1 : 0;
        for (int32_t j = 0; j < k; ++j)
            if (j != a && DIST(o, M[j]) < DIST(o, M[b])) b = j;
        nearest[o] = a; second[o] = b;
        dn[o] = DIST(o, M[a]); ds[o] = DIST(o, M[b]);
    }
    return 0;
}

/* Removal loss dTD^{-m_i} = sum_{nearest(o)=i} d_s(o) - d_n(o)
 * (Alg.3 line P:875). */
void FN(oracle_removal_loss)(int32_t n, int32_t k, const int32_t* nearest, const ACC_T* dn,
                             const ACC_T* ds, ACC_T* R) {
    for (int32_t i = 0; i < k; ++i) R[i] = 0;
    for (int32_t o = 0; o < n; ++o) R[nearest[o]] += ds[o] - dn[o];
}

/* The four-case change function, Eq. eqn:change.  doc is
 * d(x_o, x_c); (a) and (c) apply when nearest(o) != i, (b1)/(b2) when
 * nearest(o) == i. */
ACC_T FN(oracle_change)(ACC_T doc, int32_t nearest_o, ACC_T dn_o, ACC_T ds_o, int32_t i) {
    if (nearest_o != i) {
        if (doc >= dn_o) return 0;            /* (a) */
        return doc - dn_o;                    /* (c) */
    }
    if (doc < ds_o) return doc - dn_o;        /* (b1) */
    return ds_o - dn_o;                       /* (b2) */
}

static int FN(is_medoid)(const int32_t* M, int32_t k, int32_t x) {
    for (int32_t j = 0; j < k; ++j)
        if (M[j] == x) return 1;
    return 0;
}

/* Original PAM SWAP search, Alg.2 lines P:351-364: for every medoid slot i
 * and every non-medoid x_c, dTD = sum over x_o not in M \ {m_i} of
 * change(x_o, m_i, x_c) (Eq. eqn:td2).  Best starts at
 * (0, null, null) and is replaced on strict "<" with the medoid loop
 * outermost, which is the (dTD, i, c) key of reading R1.
 * Returns 1 if a candidate with dTD < 0 was found. */
int FN(oracle_pam_best)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k,
                        const int32_t* nearest, const ACC_T* dn, const ACC_T* ds,
                        ACC_T* best_dtd, int32_t* best_i, int32_t* best_c) {
    ACC_T bd = 0; int32_t bi = -1, bc = -1;
    for (int32_t i = 0; i < k; ++i) {
        for (int32_t c = 0; c < n; ++c) {
            if (FN(is_medoid)(M, k, c)) continue;
            ACC_T dtd = 0;
            for (int32_t o = 0; o < n; ++o) {
                if (o != M[i] && FN(is_medoid)(M, k, o)) continue;
                dtd += FN(oracle_change)(DIST(o, c), nearest[o], dn[o], ds[o], i);
            }
            if (dtd < bd) { bd = dtd; bi = i; bc = c; }
        }
    }
    *best_dtd = bd; *best_i = bi; *best_c = bc;
    return bi >= 0;
}

/* FastPAM1 inner loop for one non-medoid candidate x_c, Alg.3 lines
 * P:879-891 (Eq. eqn:better-change3):
 *   dTD_i <- dTD^{-m_i};  dTD^{+x_c} <- 0
 *   for every x_o:  case (i)  d < d_n : plus += d - d_n ; dTD_nearest += d_n - d_s
 *                   case (ii) d < d_s : dTD_nearest += d - d_s
 * vec[i] receives dTD_i (without the shared accumulator); *plus receives
 * dTD^{+x_c}.  col[o] = d(x_o, x_c) for o = 0..n-1. */
void FN(oracle_fastpam1_candidate_col)(const D_T* col, int32_t n, int32_t k,
                                       const int32_t* nearest, const ACC_T* dn,
                                       const ACC_T* ds, const ACC_T* R,
                                       ACC_T* vec, ACC_T* plus) {
    for (int32_t i = 0; i < k; ++i) vec[i] = R[i];
    ACC_T p = 0;
    for (int32_t o = 0; o < n; ++o) {
        ACC_T doj = (ACC_T)col[o];
        if (doj < dn[o]) {
            p += doj - dn[o];
            vec[nearest[o]] += dn[o] - ds[o];
        } else if (doj < ds[o]) {
            vec[nearest[o]] += doj - ds[o];
        }
    }
    *plus = p;
}

/* Same, reading column c of D directly. */
void FN(oracle_fastpam1_candidate)(const D_T* D, int64_t ld, int32_t n, int32_t k, int32_t c,
                                   const int32_t* nearest, const ACC_T* dn, const ACC_T* ds,
                                   const ACC_T* R, ACC_T* vec, ACC_T* plus) {
    for (int32_t i = 0; i < k; ++i) vec[i] = R[i];
    ACC_T p = 0;
    for (int32_t o = 0; o < n; ++o) {
        ACC_T doj = DIST(o, c);
        if (doj < dn[o]) {
            p += doj - dn[o];
            vec[nearest[o]] += dn[o] - ds[o];
        } else if (doj < ds[o]) {
            vec[nearest[o]] += doj - ds[o];
        }
    }
    *plus = p;
}

/* Full FastPAM1 table: table[i*n + c] = dTD(m_i, x_c) = dTD_i + dTD^{+x_c}
 * (Alg.3 line P:893) for every non-medoid c; medoid columns are left
 * untouched.  Used for lockstep float checks. */
void FN(oracle_fastpam1_table)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k,
                               const int32_t* nearest, const ACC_T* dn, const ACC_T* ds,
                               const ACC_T* R, ACC_T* table) {
    ACC_T* vec = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    for (int32_t c = 0; c < n; ++c) {
        if (FN(is_medoid)(M, k, c)) continue;
        ACC_T plus;
        FN(oracle_fastpam1_candidate)(D, ld, n, k, c, nearest, dn, ds, R, vec, &plus);
        for (int32_t i = 0; i < k; ++i) table[(int64_t)i * n + c] = vec[i] + plus;
    }
    free(vec);
}

/* Alg.3 lines P:876-897: per candidate, i = argmin dTD_i (smaller slot on
 * ties), dTD_i += dTD^{+x_c}; keep the best over candidates.
 * Reading R1: a candidate replaces the best when (dTD, i) is strictly
 * smaller (candidates come in ascending c, so c breaks the remaining ties),
 * starting from (0, null, null). */
int FN(oracle_fastpam1_best)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k,
                             const int32_t* nearest, const ACC_T* dn, const ACC_T* ds,
                             const ACC_T* R, ACC_T* best_dtd, int32_t* best_i, int32_t* best_c) {
    ACC_T* vec = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    ACC_T bd = 0; int32_t bi = -1, bc = -1;
    for (int32_t c = 0; c < n; ++c) {
        if (FN(is_medoid)(M, k, c)) continue;
        ACC_T plus;
        FN(oracle_fastpam1_candidate)(D, ld, n, k, c, nearest, dn, ds, R, vec, &plus);
        int32_t i = 0;
        for (int32_t j = 1; j < k; ++j)
            if (vec[j] < vec[i]) i = j;
        ACC_T v = vec[i] + plus;
        if (v < bd || (bi >= 0 && v == bd && i < bi)) { bd = v; bi = i; bc = c; }
    }
    free(vec);
    *best_dtd = bd; *best_i = bi; *best_c = bc;
    return bi >= 0;
}

/* FastPAM2, steps 2-3 of reading R6 (from P:861-862 and
 * P:945-947): for every slot i the best candidate (sv[i], sc[i]) =
 * lexicographic min over non-medoid c of (dTD(m_i, x_c), c), with dTD the
 * FastPAM1 value of Alg.3 P:879-893 (candidates in ascending c, strict "<").
 * sc[i] = -1 if there is no non-medoid. */
void FN(oracle_fastpam2_slot_best)(const D_T* D, int64_t ld, int32_t n, const int32_t* M, int32_t k,
                                   const int32_t* nearest, const ACC_T* dn, const ACC_T* ds,
                                   const ACC_T* R, ACC_T* sv, int32_t* sc) {
    ACC_T* vec = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    for (int32_t i = 0; i < k; ++i) { sv[i] = 0; sc[i] = -1; }
    for (int32_t c = 0; c < n; ++c) {
        if (FN(is_medoid)(M, k, c)) continue;
        ACC_T plus;
        FN(oracle_fastpam1_candidate)(D, ld, n, k, c, nearest, dn, ds, R, vec, &plus);
        for (int32_t i = 0; i < k; ++i) {
            ACC_T v = vec[i] + plus;
            if (sc[i] < 0 || v < sv[i]) { sv[i] = v; sc[i] = c; }
        }
    }
    free(vec);
}

/* One SWAP run (Alg.2 P:347-372 for variant 0 = PAM, Alg.3 P:871-905 for
 * variant 1 = FastPAM1, reading R6 for variant 2 = FastPAM2).
 * M (in/out, k slots) is updated in place (slot semantics P:366).  The
 * cache is recomputed from scratch after every swap ("update").
 * trace_* receive (slot, candidate, dTD) of every executed swap, up to
 * trace_cap entries.  n_iter counts passes including the final non-improving
 * one.  Returns 0 converged, 1 max_iter reached, <0 error. */
int FN(oracle_swap_run)(const D_T* D, int64_t ld, int32_t n, int32_t* M, int32_t k,
                        int32_t variant, int32_t max_iter,
                        int32_t* trace_i, int32_t* trace_c, ACC_T* trace_dtd, int32_t trace_cap,
                        int32_t* n_iter, int32_t* n_swaps, ACC_T* td_out, int32_t* assignment) {
    if (k < 2 || k >= n) return -1;
    int32_t* nearest = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* second = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    ACC_T* dn = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    ACC_T* ds = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    ACC_T* R = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    ACC_T* vec = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    ACC_T* sv = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);   /* FastPAM2 per-slot best value */
    int32_t* sc = (int32_t*)malloc(sizeof(int32_t) * (size_t)k); /* FastPAM2 per-slot best c */
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    int32_t iters = 0, swaps = 0, status = 1;
    ACC_T td = FN(oracle_td)(D, ld, n, M, k);
    FN(oracle_assign)(D, ld, n, M, k, nearest, second, dn, ds);
    while (iters < max_iter) {
        iters++;
        FN(oracle_removal_loss)(n, k, nearest, dn, ds, R);
        if (variant == 0 || variant == 1) {
            ACC_T bd; int32_t bi, bc;
            if (variant == 0)
                FN(oracle_pam_best)(D, ld, n, M, k, nearest, dn, ds, &bd, &bi, &bc);
            else
                FN(oracle_fastpam1_best)(D, ld, n, M, k, nearest, dn, ds, R, &bd, &bi, &bc);
            if (bi < 0 || !FN(improving)(bd, td)) { status = 0; break; }
            if (swaps < trace_cap) { trace_i[swaps] = bi; trace_c[swaps] = bc; trace_dtd[swaps] = bd; }
            swaps++;
            M[bi] = bc;
            FN(oracle_assign)(D, ld, n, M, k, nearest, second, dn, ds);
            td += bd;
        } else {
            /* Reading R6:
             * 2-3. per slot i the best candidate (v_i, c_i) = lexicographic
             *      min over non-medoid c of (dTD(m_i, x_c), c). */
            FN(oracle_fastpam2_slot_best)(D, ld, n, M, k, nearest, dn, ds, R, sv, sc);
            /* 4. stop when no slot improves (same rule as PAM). */
            int32_t any = 0;
            for (int32_t i = 0; i < k; ++i)
                if (sc[i] >= 0 && FN(improving)(sv[i], td)) any = 1;
            if (!any) { status = 0; break; }
            /* 5. slots ordered by (v_i, i) ascending (insertion sort). */
            for (int32_t i = 0; i < k; ++i) order[i] = i;
            for (int32_t a = 1; a < k; ++a) {
                int32_t x = order[a], b = a - 1;
                while (b >= 0 && (sv[order[b]] > sv[x] || (sv[order[b]] == sv[x] && order[b] > x))) {
                    order[b + 1] = order[b]; b--;
                }
                order[b + 1] = x;
            }
            /* 6-7. the first swap is applied with its dTD; every later slot
             * with an improving v_i is re-evaluated exactly on the current
             * state (R recomputed) and applied only if still improving. */
            ACC_T td0 = td;   /* the slot set is fixed by the values at the start of the phase */
            for (int32_t r = 0; r < k; ++r) {
                int32_t i = order[r], c = sc[i];
                if (c < 0 || !FN(improving)(sv[i], td0)) continue;
                ACC_T v;
                if (r == 0) {
                    v = sv[i];
                } else {
                    if (FN(is_medoid)(M, k, c)) continue;
                    ACC_T plus;
                    FN(oracle_removal_loss)(n, k, nearest, dn, ds, R);
                    FN(oracle_fastpam1_candidate)(D, ld, n, k, c, nearest, dn, ds, R, vec, &plus);
                    v = vec[i] + plus;
                    if (!FN(improving)(v, td)) continue;
                }
                if (swaps < trace_cap) { trace_i[swaps] = i; trace_c[swaps] = c; trace_dtd[swaps] = v; }
                swaps++;
                M[i] = c;
                FN(oracle_assign)(D, ld, n, M, k, nearest, second, dn, ds);
                td += v;
            }
        }
    }
    if (status == 1) {
        /* max_iter reached without a non-improving pass */
    }
    *n_iter = iters; *n_swaps = swaps; *td_out = td;
    if (assignment)
        for (int32_t o = 0; o < n; ++o) assignment[o] = nearest[o];
    free(nearest); free(second); free(dn); free(ds); free(R); free(vec);
    free(sv); free(sc); free(order);
    return status;
}

/* FasterPAM: FastPAM1 with eager swapping, Alg.4 (section
 * "FasterPAM").  Readings (F1-F5):
 *   F1 candidates are visited in ascending point index, cyclically
 *      (c = t mod n for the scan position t = 0, 1, 2, ...); medoids are
 *      skipped ("x_c not in {m_1..m_k}").
 *   F2 "break outer loop if x_c = x_last" is tested at every
 *      position BEFORE the medoid skip (x_last is itself a medoid right
 *      after its swap); with x_last still invalid, the scan stops after one
 *      whole pass without a swap.  Both are "stop at the first position t
 *      with t - t_last = n", t_last = the position of the last swap (0
 *      before any swap).
 *   F3 iterations = passes begun = ceil(t_stop / n) ("multiple
 *      swaps per pass"); max_iter caps the passes begun.
 *   F4 i = argmin_i dTD_i, smaller slot on ties (as Alg.3),
 *      then dTD_i += dTD^{+x_c} (the garbled
 *      "dTD^{+nearest(o)}" accumulators of P:1008-1013 are read as
 *      dTD_{nearest(o)}).
 *   F5 acceptance as R5; the swap exchanges m_i with x_c (P:1019 and
 *      P:1022 write x_o); the nearest/second cache and the
 *      removal losses are then recomputed from scratch ("update").
 * trace_* as in oracle_swap_run; trace_pos (may be NULL) receives the scan
 * position t of every swap.  Returns 0 converged, 1 max_iter reached. */
int FN(oracle_fasterpam_run)(const D_T* D, int64_t ld, int32_t n, int32_t* M, int32_t k, int32_t max_iter,
                             int32_t* trace_i, int32_t* trace_c, ACC_T* trace_dtd, int64_t* trace_pos,
                             int32_t trace_cap, int32_t* n_iter, int32_t* n_swaps, ACC_T* td_out,
                             int32_t* assignment) {
    if (k < 2 || k >= n) return -1;
    int32_t* nearest = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* second = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    ACC_T* dn = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    ACC_T* ds = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    ACC_T* R = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    ACC_T* vec = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)k);
    int32_t swaps = 0, status = 0;
    int64_t t = 0, t_last = 0;
    ACC_T td = FN(oracle_td)(D, ld, n, M, k);
    FN(oracle_assign)(D, ld, n, M, k, nearest, second, dn, ds);
    FN(oracle_removal_loss)(n, k, nearest, dn, ds, R);
    for (;; ++t) {
        if (t - t_last == n) break;                                 /* F2 */
        if (t % n == 0 && t / n >= max_iter) { status = 1; break; } /* F3 cap */
        const int32_t c = (int32_t)(t % n);
        if (FN(is_medoid)(M, k, c)) continue;                       /* F1 */
        ACC_T plus;
        FN(oracle_fastpam1_candidate)(D, ld, n, k, c, nearest, dn, ds, R, vec, &plus);
        int32_t i = 0;
        for (int32_t j = 1; j < k; ++j)
            if (vec[j] < vec[i]) i = j;                             /* F4 */
        const ACC_T v = vec[i] + plus;
        if (!FN(improving)(v, td)) continue;                        /* F5 */
        if (swaps < trace_cap) {
            trace_i[swaps] = i; trace_c[swaps] = c; trace_dtd[swaps] = v;
            if (trace_pos) trace_pos[swaps] = t;
        }
        swaps++;
        M[i] = c;
        td += v;
        FN(oracle_assign)(D, ld, n, M, k, nearest, second, dn, ds);
        FN(oracle_removal_loss)(n, k, nearest, dn, ds, R);
        t_last = t;
    }
    *n_iter = (int32_t)((t + n - 1) / n);
    *n_swaps = swaps; *td_out = td;
    if (assignment)
        for (int32_t o = 0; o < n; ++o) assignment[o] = nearest[o];
    free(nearest); free(second); free(dn); free(ds); free(R); free(vec);
    return status;
}

/* PAM BUILD, Alg.1.
 * First medoid: smallest distance sum sum_{x_o != x_c} d(x_o, x_c)
 * (strict "<", so the smallest index wins ties).
 * d_nearest(o) <- d(x_o, m_1) (reading R0 orientation).
 * Each further medoid: dTD(x_c) = sum over x_o not in M of
 * min(d(x_o,x_c) - d_nearest(o), 0), including x_o = x_c (reading R3),
 * best on strict "<" (R4); TD <- TD + dTD* (P:312); d_nearest updated
 * (P:313-316).  gains[0] = TD of the first medoid, gains[i] = dTD* of step i.
 * Needs 1 <= k < n. */
int FN(oracle_build)(const D_T* D, int64_t ld, int32_t n, int32_t k, int32_t* M,
                     ACC_T* td_out, ACC_T* gains) {
    if (k < 1 || k >= n) return -1;
    ACC_T* dnear = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    int32_t* is_med = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    ACC_T td = 0; int32_t m1 = -1;
    for (int32_t c = 0; c < n; ++c) {
        ACC_T tdj = 0;
        for (int32_t o = 0; o < n; ++o)
            if (o != c) tdj += DIST(o, c);
        if (m1 < 0 || tdj < td) { td = tdj; m1 = c; }
    }
    M[0] = m1; is_med[m1] = 1; gains[0] = td;
    for (int32_t o = 0; o < n; ++o) dnear[o] = (o == m1) ? 0 : DIST(o, m1);
    for (int32_t i = 1; i < k; ++i) {
        ACC_T bd = 0; int32_t bx = -1;
        for (int32_t c = 0; c < n; ++c) {
            if (is_med[c]) continue;
            ACC_T dtd = 0;
            for (int32_t o = 0; o < n; ++o) {
                if (is_med[o]) continue;
                ACC_T delta = DIST(o, c) - dnear[o];
                if (delta < 0) dtd += delta;
            }
            if (bx < 0 || dtd < bd) { bd = dtd; bx = c; }
        }
        td += bd; M[i] = bx; is_med[bx] = 1; gains[i] = bd;
        for (int32_t o = 0; o < n; ++o) {
            if (is_med[o]) { if (o == bx) dnear[o] = 0; continue; }
            ACC_T d = DIST(o, bx);
            if (d < dnear[o]) dnear[o] = d;
        }
    }
    *td_out = td;
    free(dnear); free(is_med);
    return 0;
}

/* NEXT-4 initialisations.  Random numbers are INPUTS (drawn
 * by the caller, identical for the oracle and the GPU).
 *
 * Distance-weighted ("k-means++" adapted to arbitrary dissimilarities,
 * P:1046-1059; reading I1): the first seed is
 * min(n-1, floor(u[0] n)); seed i > 0 is the smallest index c whose running
 * sum of w(o) = min_j d(x_o, m_j) over o = 0..c exceeds u[i] * W, W = sum
 * of all w (sequential sums in index order, ACC_T); if W = 0 the smallest
 * non-medoid is taken.  d(x_o, m_j) = D[o][m_j] (reading R0). */
int FN(oracle_init_weighted)(const D_T* D, int64_t ld, int32_t n, int32_t k, const double* u, int32_t* M) {
    if (k < 1 || k > n) return -1;
    ACC_T* w = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    int32_t c = (int32_t)(u[0] * (double)n);
    if (c >= n) c = n - 1;
    M[0] = c;
    for (int32_t o = 0; o < n; ++o) w[o] = DIST(o, c);
    for (int32_t i = 1; i < k; ++i) {
        ACC_T W = 0;
        for (int32_t o = 0; o < n; ++o) W += w[o];
        int32_t pick = -1;
        if (W > 0) {
            const double r = u[i] * (double)W;
            ACC_T run = 0;
            for (int32_t o = 0; o < n; ++o) {
                run += w[o];
                if ((double)run > r) { pick = o; break; }
            }
        }
        if (pick < 0)                       /* W = 0 (or r rounded to W): smallest non-medoid */
            for (int32_t o = 0; o < n && pick < 0; ++o)
                if (!FN(is_medoid)(M, i, o)) pick = o;
        M[i] = pick;
        for (int32_t o = 0; o < n; ++o) {
            const ACC_T d = DIST(o, pick);
            if (d < w[o]) w[o] = d;
        }
    }
    free(w);
    return 0;
}

/* LAB, Linear Approximative BUILD (the SISAP'19 paper that
 * defines it is not in the container: reading I2).  Step i draws the
 * sample S_i = the first s entries of seq[i*(s+k) ...] that are not yet
 * medoids (the caller supplies distinct indices per row, -1 = padding); for each
 * candidate c in S_i (in order) g(c) = sum over o in S_i (in order) of
 * d(x_o, x_c) for i = 0 (BUILD's first step, Alg.1) and of
 * min(d(x_o, x_c) - d_nearest(o), 0) for i > 0 (Alg.1 P:300-310 restricted
 * to the subsample, self term included as reading R3); the smallest
 * (g, c) is the next medoid; d_nearest is then updated for all objects. */
int FN(oracle_init_lab)(const D_T* D, int64_t ld, int32_t n, int32_t k, int32_t s, const int32_t* seq, int32_t* M) {
    if (k < 1 || k > n || s < 1) return -1;
    ACC_T* dnear = (ACC_T*)malloc(sizeof(ACC_T) * (size_t)n);
    int32_t* S = (int32_t*)malloc(sizeof(int32_t) * (size_t)s);
    for (int32_t i = 0; i < k; ++i) {
        const int32_t* row = seq + (int64_t)i * (s + k);
        int32_t m = 0;
        for (int32_t j = 0; j < s + k && m < s; ++j)
            if (row[j] >= 0 && !FN(is_medoid)(M, i, row[j])) S[m++] = row[j];
        ACC_T bg = 0; int32_t bc = -1;
        for (int32_t a = 0; a < m; ++a) {
            const int32_t c = S[a];
            ACC_T g = 0;
            for (int32_t b = 0; b < m; ++b) {
                const int32_t o = S[b];
                if (i == 0) g += DIST(o, c);
                else {
                    const ACC_T delta = DIST(o, c) - dnear[o];
                    if (delta < 0) g += delta;
                }
            }
            if (bc < 0 || g < bg || (g == bg && c < bc)) { bg = g; bc = c; }
        }
        M[i] = bc;
        for (int32_t o = 0; o < n; ++o) {
            const ACC_T d = DIST(o, bc);
            if (i == 0 || d < dnear[o]) dnear[o] = d;
        }
    }
    free(dnear); free(S);
    return 0;
}

#undef DIST
#undef FN
#undef CAT
#undef CAT2
