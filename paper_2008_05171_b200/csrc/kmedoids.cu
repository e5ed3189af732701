// kmedoids.cu -- host driver and C ABI (include/kmedoids.h) of the B200
// FastPAM SWAP library.  Every step of the hot path runs in the kernels of
// km_kernels.cuh; this file only validates arguments, owns scratch buffers,
// enqueues kernels on the handle's stream and copies the per-iteration
// decision (one 32-byte record) back to the host for the convergence test.
#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <type_traits>
#include <vector>
#include <cudaTypedefs.h>
#include <thread>

#include "../../include/kmedoids.h"
#include "km_kernels.cuh"
#include "km_fasterpam.cuh"
#include "km_post.cuh"
#include "km_dist.cuh"
#include "km_init.cuh"
#include "km_build_delta.cuh"
#include "km_clara.cuh"
#include "km_fp2_owner.cuh"

namespace {

thread_local std::string g_err;

km_status fail(km_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define KM_CK(call)                                                                               \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(KM_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define KM_CKL()                                                                                  \
    do {                                                                                          \
        ++launches;                                                                               \
        cudaError_t e_ = cudaGetLastError();                                                      \
        if (e_ != cudaSuccess) return fail(KM_ECUDA, "kernel launch failed (kmedoids.cu:%d): %s", __LINE__, cudaGetErrorString(e_)); \
    } while (0)

#define KM_TRY(expr)                  \
    do {                              \
        km_status s_ = (expr);        \
        if (s_ != KM_OK) return s_;   \
    } while (0)

constexpr int NUM_SMS = 148;
constexpr int TARGET_WAVES = 3;
constexpr int MAX_K = 8192;
// SWAP / BUILD stream (k_swap_stream_seg2, k_build_tma): 7 consumer warps + 1
// producer, TMA ring of 5 stages x 4 rows (~72 KB shared memory), 3 CTAs = 24
// warps per SM (<= 80 registers).
constexpr int SG_NC = 7, SG_RB = 4, SG_S = 5, SG_MINB = 3;
constexpr int FP2_SPLIT = 8;
constexpr int FP2_SB_MIN_K = 256;   // k from which k_fp2_slot_best takes 4 slots per block   // column splits of the FastPAM2 per-slot reduction

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of row parts so the (column tiles x parts) grid fills the GPU.
int choose_parts(int64_t n, int64_t w, int cols_per_cta, int resident) {
    const int64_t ncb = cdiv(w, cols_per_cta);
    int64_t P = cdiv((int64_t)NUM_SMS * resident * TARGET_WAVES, ncb);
    P = std::min<int64_t>(P, std::max<int64_t>(1, n / 64));
    P = std::max<int64_t>(P, 1);
    return (int)P;
}


// Row parts of the segment stream (measured): at most
// ~1500 rows per part, at least 1.7 and at most 8 waves of resident CTAs (3
// per SM) -- more, shorter CTAs balance the Poisson-lumpy hit work across
// SMs; every part costs ring fill/drain and 36 bytes per column of part
// outputs that the post kernel folds.  Round 2 sweep of the step (stream +
// post): C3 P = 58 -> 33 (0.300 -> 0.290 ms), C4 P = 50 -> 34 (1.509 ->
// 1.500 ms); round 1's rule (n/1000 rows, >= 3 waves) predates the fused
// post kernel.
constexpr int PART_SKEW_DEFAULT = 15;  // 16ths; see km::part_lo (C4 stream 1.565 -> 1.478 ms)

int choose_parts_seg(int64_t n, int64_t w) {
    const int64_t ncb = cdiv(w, SG_NC * 128);
    const int64_t slots = (int64_t)NUM_SMS * SG_MINB;
    int64_t P = cdiv(n, 1500);
    P = std::max<int64_t>(P, cdiv(17 * slots, 10 * ncb));
    P = std::min<int64_t>(P, std::max<int64_t>(1, 8 * slots / ncb));
    P = std::min<int64_t>(P, std::max<int64_t>(1, n / 64));
    return (int)std::max<int64_t>(P, 1);
}

}  // namespace

struct ImplBase {
    virtual ~ImplBase() {}
    virtual km_status set_medoids(const int32_t* M) = 0;
    virtual km_status init_build(int32_t* M_out, void* td_out) = 0;
    virtual km_status swap_iter(km_variant v, int32_t* swaps, void* td_out) = 0;
    virtual km_status get_state(int32_t* M, int32_t* asg, void* td, int32_t* it, int32_t* sw) = 0;
    virtual km_status get_cache(int32_t* nr, int32_t* sc, void* dn, void* ds) = 0;
    virtual km_status eval_candidates(void* v, int32_t* s) = 0;
    virtual km_status shard_exchange(int32_t nranks, km_exchange* out) = 0;
    virtual km_status shard_set_medoids(const int32_t* M, const void* cols) = 0;
    virtual km_status shard_eval() = 0;
    virtual km_status shard_select(const int64_t* rcb, int32_t* found, int32_t* slot, int32_t* cand,
                                   int32_t* owner, void* dtd) = 0;
    virtual km_status shard_pack_column(int32_t cand) = 0;
    virtual km_status shard_apply() = 0;
    virtual km_status shard_decide() = 0;
    virtual km_status shard_apply_async() = 0;
    virtual km_status shard_status(int32_t wait, int32_t* conv, int32_t* iters, int32_t* swaps, void* td) = 0;
    virtual km_status shard_resync(int32_t* calls) = 0;
    virtual km_status shard_trace(int32_t* slots, int32_t* cands, void* dtds, int32_t cap, int32_t* count) = 0;
    virtual km_status build_eval(int32_t step) = 0;
    virtual km_status build_select(const int64_t* rcb, int32_t* cand, int32_t* owner, void* gain) = 0;
    virtual km_status build_apply(int32_t step) = 0;
    virtual km_status build_decide(int32_t step) = 0;
    virtual km_status build_apply_async(int32_t step) = 0;
    virtual km_status last_swaps_out(int32_t* slots, int32_t* cands, void* dtds, int32_t cap, int32_t* count) = 0;
    virtual km_status fp2_last_plan(void* v, int32_t* c, int32_t* order, int32_t* m) = 0;
    virtual km_status fp2_shard_exchange(int32_t nranks, km_fp2_exchange* out) = 0;
    virtual km_status fp2_shard_eval() = 0;
    virtual km_status fp2_shard_plan(const int64_t* rcb, int32_t* m_out, int32_t* maxcnt_out) = 0;
    virtual km_status fp2_shard_apply(int32_t* swaps_out, void* td_out) = 0;
    virtual km_status fp2_round_buffers(void** send, void** recv, size_t* stride) = 0;
    virtual km_status fp2_round_eval() = 0;
    virtual km_status fp2_round_apply(int32_t* more_out, int32_t* swaps_out, void* td_out) = 0;
    virtual km_status init_weighted(const double* u, int32_t* M_out, void* td_out) = 0;
    virtual km_status init_lab(int32_t s, const int32_t* seq, int32_t* M_out, void* td_out) = 0;
    virtual km_status clara(int32_t ns, int32_t s, const int32_t* samples, km_variant v, int32_t* M_out,
                            void* td_out, int32_t* best_out) = 0;
    virtual km_status inc_iters(int32_t max_iters, int32_t* swaps, void* td_out, int32_t* iters_done,
                                bool* converged) = 0;
    virtual km_status fp1_run_pipelined(int32_t max_iter, int32_t* iters_out, int32_t* swaps_out, bool* converged) = 0;
    virtual km_status fp2_run_pipelined(int32_t max_iter, int32_t* iters_out, int32_t* swaps_out, bool* converged) = 0;
    virtual km_status check_diagonal() = 0;
    virtual km_status set_symmetric(int32_t on) = 0;
    bool profiling = false;
    double prof_ms = 0.0;
    int64_t prof_launches = 0;
    virtual km_status prof_harvest() { return KM_OK; }   // pending stream timings (async sharded mode)
    virtual const char* stream_kernel_name() const = 0;
    int64_t launches = 0;
    int k = 0;
    int64_t n = 0;
    bool sharded = false;
};

struct km_handle {
    std::unique_ptr<ImplBase> impl;
};

namespace {

template <typename T>
struct Impl : ImplBase {
    using A = typename km::Acc<T>::type;
    using RI = km::RowInfo<T>;
    using Rec = km::Rec<A>;
    using Dec = km::Decision<A>;

    const T* D = nullptr;
    int64_t ld = 0, c0 = 0, c1 = 0;
    int w = 0;
    cudaStream_t st = nullptr;
    int P = 1, Pbt = 1, B = 1, ncomb = 1, ntd = 1, sort_chunk = 256;
    int nranks = 1;
    int wpad = 0;
    bool ready = false;     // medoids + cache valid
    int* bad_count = nullptr;       // input validation counter (k_validate_*)

    std::vector<void*> bufs;        // every device allocation, freed in the destructor
    int *M = nullptr, *point_slot = nullptr, *near = nullptr, *sec = nullptr;
    T *MC = nullptr, *dn = nullptr, *ds = nullptr, *colbuf = nullptr;
    T* fp2_cols = nullptr;          // FastPAM2: columns of a speculative batch [FP2_B][n]
    int *rescan = nullptr, *rescan_count = nullptr;   // objects whose nearest/second slot was swapped
    RI* ri = nullptr;
    double2* rowd = nullptr;        // float path: (double dn, double ds) in sorted order
    int *seg_start = nullptr, *empty_slot = nullptr, *slot_tot = nullptr;
    int *head_slot = nullptr, *tail_slot = nullptr;
    A *R = nullptr, *o_plus = nullptr, *o_head = nullptr, *o_tail = nullptr, *o_imin = nullptr;
    int* o_islot = nullptr;
    A* b_out = nullptr;
    A* cand_v = nullptr;
    int* cand_slot = nullptr;
    Rec *partials = nullptr, *rec_local = nullptr, *rec_recv = nullptr;
    unsigned* counters = nullptr;   // [0] combine, [1] td
    A *td = nullptr, *td_partials = nullptr;
    Dec* dec = nullptr;
    Dec* h_dec = nullptr;           // pinned mirror
    A* h_td = nullptr;              // pinned mirror of TD (FastPAM1 iteration)
    // FastPAM2 state (allocated on first use)
    A* fp2_acc = nullptr;           // [k][w] complete acc_c[i]
    A* fp2_plus = nullptr;          // [w]    dTD^{+x_c}
    Rec* fp2_best = nullptr;        // [k]    per-slot (v_i, i, c_i)
    Rec* fp2_part = nullptr;        // [k][FP2_SPLIT] partial per-slot bests
    int* fp2_order = nullptr;       // [k]
    A* fp2_partials = nullptr;      // cooperative-kernel block partials
    int fp2_blocks = 0;
    std::vector<Rec> h_best;
    // swaps of the last iteration (slot, c, dTD)
    Rec* trace = nullptr;
    int trace_cap = 0;
    std::vector<Rec> last_swaps;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    ~Impl() override {
        for (auto& sl : clara_slots) {
            sl.sub.reset();
            if (sl.stream) cudaStreamDestroy(sl.stream);
            if (sl.fin) cudaEventDestroy(sl.fin);
            if (sl.h_med) cudaFreeHost(sl.h_med);
            if (sl.h_td) cudaFreeHost(sl.h_td);
        }
        for (auto& g : fp1_g) if (g) cudaGraphExecDestroy(g);
        for (auto& p : g_ev) for (auto e : p) if (e) cudaEventDestroy(e);
        for (auto e : g_done) if (e) cudaEventDestroy(e);
        if (h_ring) cudaFreeHost(h_ring);
        if (build_exec) cudaGraphExecDestroy(build_exec);
        if (cap_st) cudaStreamDestroy(cap_st);
        if (side_st) cudaStreamDestroy(side_st);
        for (auto& e : fork_ev) if (e) cudaEventDestroy(e);
        for (void* p : bufs) cudaFree(p);
        if (h_dec) cudaFreeHost(h_dec);
        if (h_td) cudaFreeHost(h_td);
        if (h_f2out) cudaFreeHost(h_f2out);
        if (h_f2dec) cudaFreeHost(h_f2dec);
        if (h_f2td) cudaFreeHost(h_f2td);
        for (auto e : f2_done) if (e) cudaEventDestroy(e);
        for (auto e : sp_ev) if (e) cudaEventDestroy(e);
        for (auto e : f2_ev) if (e) cudaEventDestroy(e);
        for (auto e : sh_ev) if (e) cudaEventDestroy(e);
        for (auto& p : pr_ev) for (auto e : p) if (e) cudaEventDestroy(e);
        if (sh_mirror) cudaFreeHost(sh_mirror);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }

    void dealloc(void* p) {
        if (!p) return;
        for (auto& b : bufs)
            if (b == p) { cudaFree(p); b = nullptr; }
    }

    template <typename X>
    km_status alloc(X** out, size_t count) {
        void* p = nullptr;
        size_t bytes = std::max<size_t>(count, 1) * sizeof(X);
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(KM_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        }
        bufs.push_back(p);
        *out = (X*)p;
        return KM_OK;
    }

    km_status init(const void* Dp, int64_t n_, int64_t ld_, int64_t c0_, int64_t c1_, int k_, cudaStream_t s) {
        D = (const T*)Dp; n = n_; ld = ld_; c0 = c0_; c1 = c1_; k = k_; st = s;
        w = (int)(c1 - c0);
        sharded = !(c0 == 0 && c1 == n);
        const char* eg = getenv("KM_GRAPH");
        use_graph = !(eg && eg[0] == '0');
        P = choose_parts_seg(n, w);
        const char* ep = getenv("KM_PARTS");          // measurement override of the stream's row parts
        // (<= 4096: km::part_lo's int64 products stay in range for any n < 2^31)
        if (ep && atoi(ep) > 0) P = std::min<int>(std::min(atoi(ep), 4096), (int)std::max<int64_t>(1, n / 64));
        {
            // part-size tilt of the streams (km_common.cuh part_lo); one value
            // per process (a __constant__ of this device), KM_PART_SKEW in 16ths
            int skew = PART_SKEW_DEFAULT;
            if (const char* es = getenv("KM_PART_SKEW")) skew = std::min(64, std::max(0, atoi(es)));
            KM_CK(cudaMemcpyToSymbol(km::c_part_skew, &skew, sizeof(int)));
        }
        Pbt = choose_parts(n, w, SG_NC * 128, SG_MINB);
        wpad = (int)((w + 3) / 4 * 4);
        // counting-sort chunk: >= 256 objects and at most 128 chunks (keeps the
        // k x B count matrix of the one-block scan small)
        sort_chunk = (int)std::max<int64_t>(km::SORT_CHUNK_MIN, cdiv(cdiv(n, 128), 32) * 32);
        if (const char* ec = getenv("KM_SORT_CHUNKS"))   // measurement override: target number of chunks
            if (atoi(ec) > 0) sort_chunk = (int)std::max<int64_t>(32, cdiv(cdiv(n, atoi(ec)), 32) * 32);
        B = (int)cdiv(n, sort_chunk);
        ncomb = (int)cdiv(w, 128);
        ntd = (int)std::min<int64_t>(cdiv(n, 256), 1024);
        KM_TRY(alloc(&M, k));
        KM_TRY(alloc(&point_slot, n));
        KM_TRY(alloc(&near, n));
        KM_TRY(alloc(&sec, n));
        KM_TRY(alloc(&MC, (size_t)k * n));
        KM_TRY(alloc(&dn, n));
        KM_TRY(alloc(&ds, n));
        KM_TRY(alloc(&colbuf, n));
        KM_TRY(alloc(&rescan, n));
        KM_TRY(alloc(&rescan_count, 1));
        KM_TRY(alloc(&ri, n));
        if (km::Acc<T>::is_float) KM_TRY(alloc(&rowd, n));
        KM_TRY(alloc(&seg_start, k + 1));
        KM_TRY(alloc(&slot_tot, k));
        KM_TRY(alloc(&empty_slot, 1));
        KM_TRY(alloc(&head_slot, P));
        KM_TRY(alloc(&tail_slot, P));
        KM_TRY(alloc(&R, k));
        const size_t pw = (size_t)std::max(P, Pbt) * w;
        KM_TRY(alloc(&o_plus, pw));
        KM_TRY(alloc(&o_head, pw));
        KM_TRY(alloc(&o_tail, pw));
        KM_TRY(alloc(&o_imin, pw));
        KM_TRY(alloc(&o_islot, pw));
        b_out = o_plus;   // BUILD partial sums reuse the plus buffer (sized for max(P, Pbt))
        KM_TRY(alloc(&cand_v, w));
        KM_TRY(alloc(&cand_slot, w));
        KM_TRY(alloc(&partials, std::max<int64_t>(cdiv(w, 32), 1)));
        KM_TRY(alloc(&rec_local, 1));
        KM_TRY(alloc(&counters, 2));
        KM_TRY(alloc(&td, 1));
        KM_TRY(alloc(&td_partials, ntd));
        KM_TRY(alloc(&dec, 1));
        KM_CK(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned), st));
        KM_CK(cudaMemsetAsync(dec, 0, sizeof(Dec), st));
        KM_CK(cudaMemsetAsync(point_slot, 0xff, n * sizeof(int), st));
        KM_CK(cudaMallocHost((void**)&h_dec, sizeof(Dec)));
        memset(h_dec, 0, sizeof(Dec));
        KM_CK(cudaMallocHost((void**)&h_td, sizeof(A)));
        KM_CK(cudaEventCreate(&ev0));
        KM_CK(cudaEventCreate(&ev1));
        KM_TRY(alloc(&bad_count, 1));
        KM_TRY(check_diagonal());
        if (const char* es = getenv("KM_STEP_PROF")) step_prof = es[0] == '1';
        if (step_prof)
            for (auto& e : sp_ev) KM_CK(cudaEventCreate(&e));
        KM_CK(cudaStreamSynchronize(st));
        return KM_OK;
    }

    // ---- pieces of the hot path -------------------------------------------
    // inside a graph capture the event must be an external record node
    bool capturing = false;
    cudaError_t record_ev(cudaEvent_t e) {
        return capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
    }

    km_status sync_dec() {
        KM_CK(cudaMemcpyAsync(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        if (profiling && pending_prof) {
            float ms = 0.f;
            KM_CK(cudaEventElapsedTime(&ms, ev0, ev1));
            prof_ms += ms;
            prof_launches += 1;
            pending_prof = false;
        }
        return KM_OK;
    }
    bool pending_prof = false;
    bool step_prof = false;
    cudaEvent_t sp_ev[5] = {};
    // KM_STEP_PROF, FastPAM2: prep | stream | combine | slot best | plan | sequential | host copies
    cudaEvent_t f2_ev[8] = {};
    double f2_sum[7] = {};
    int f2_n = 0;
    void f2_mark(int i) {
        if (!step_prof) return;
        if (!f2_ev[0]) for (auto& e : f2_ev) cudaEventCreate(&e);
        cudaEventRecord(f2_ev[i], st);
    }
    void f2_take() {
        if (!step_prof || !f2_ev[0]) return;
        cudaEventSynchronize(f2_ev[7]);
        for (int i = 0; i < 7; ++i) {
            float t = 0.f;
            cudaEventElapsedTime(&t, f2_ev[i], f2_ev[i + 1]);
            f2_sum[i] += t;
        }
        if (++f2_n % 10 == 0)
            fprintf(stderr, "[kmedoids] FastPAM2 phases over %d iterations (us): prep %.1f stream %.1f combine %.1f "
                    "slot_best %.1f plan %.1f sequential %.1f copies %.1f\n", f2_n, 1e3 * f2_sum[0] / f2_n,
                    1e3 * f2_sum[1] / f2_n, 1e3 * f2_sum[2] / f2_n, 1e3 * f2_sum[3] / f2_n, 1e3 * f2_sum[4] / f2_n,
                    1e3 * f2_sum[5] / f2_n, 1e3 * f2_sum[6] / f2_n);
    }
    double sp_sum[5] = {};
    int sp_n = 0;
    // CUDA graph of the FastPAM1 iteration (KM_GRAPH=0 disables)
    bool use_graph = true;
    cudaStream_t cap_st = nullptr;
    int64_t fp1_graph_kernels = 0;
    int64_t fp1_iters = 0;

    km_status assign_full_and_td() {
        const int nb = (int)cdiv(n, 256);
        km::k_assign_full<T><<<nb, 256, 0, st>>>(MC, (int)n, k, near, sec, dn, ds);
        KM_CKL();
        km::k_td_from_dn<T, A><<<ntd, 256, 0, st>>>(dn, (int)n, td_partials, counters + 1, td);
        KM_CKL();
        return KM_OK;
    }

    km_status set_point_slots(const int32_t* Mh) {
        std::vector<int32_t> ps((size_t)n, -1);
        for (int j = 0; j < k; ++j) {
            if (Mh[j] < 0 || Mh[j] >= n) return fail(KM_EINVAL, "medoid %d out of range [0,%lld)", Mh[j], (long long)n);
            if (ps[Mh[j]] >= 0) return fail(KM_EINVAL, "duplicate medoid %d", Mh[j]);
            ps[Mh[j]] = j;
        }
        KM_CK(cudaMemcpyAsync(M, Mh, k * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        KM_CK(cudaMemcpyAsync(point_slot, ps.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        KM_CK(cudaStreamSynchronize(st));   // ps goes out of scope
        return KM_OK;
    }

    // D declared exactly symmetric (kmedoids_set_symmetric): verified by one
    // tiled pass; the FastPAM2 re-evaluations then read candidate rows
    bool symmetric = false;
    km_status set_symmetric(int32_t on) override {
        if (!on) { symmetric = false; return KM_OK; }
        if (sharded) return fail(KM_EINVAL, "set_symmetric on a sharded handle (a slab holds no whole rows)");
        KM_CK(cudaMemsetAsync(bad_count, 0, sizeof(int), st));
        const unsigned nb = (unsigned)cdiv(n, 32);
        if (nb > 65535) return fail(KM_EINVAL, "set_symmetric: n too large for the check grid");
        km::k_check_symmetric<T><<<dim3(nb, nb), 256, 0, st>>>(D, ld, (int)n, bad_count);
        KM_CKL();
        int nbad = 0;
        KM_CK(cudaMemcpyAsync(&nbad, bad_count, sizeof(int), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        if (nbad) return fail(KM_EINVAL, "D is not symmetric (%d mismatching entries)", nbad);
        symmetric = true;
        return KM_OK;
    }

    // the slab's diagonal entries must be exactly 0 (O(n) device pass; synchronises)
    km_status check_diagonal() override {
        if (c1 <= c0) return KM_OK;
        KM_CK(cudaMemsetAsync(bad_count, 0, sizeof(int), st));
        km::k_validate_diag<T><<<(unsigned)cdiv(c1 - c0, 256), 256, 0, st>>>(D, ld, c0, c1, bad_count);
        KM_CKL();
        int nbad = 0;
        KM_CK(cudaMemcpyAsync(&nbad, bad_count, sizeof(int), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        if (nbad) return fail(KM_EINVAL, "D has %d nonzero (or NaN) diagonal entries; d(x_o, x_o) must be 0", nbad);
        return KM_OK;
    }

    // float path: the gathered medoid columns (every d(x_o, m_j)) must be
    // >= 0 and not NaN (KM_EINVAL otherwise; synchronises)
    km_status validate_mc() {
        if constexpr (!km::Acc<T>::is_float) {
            return KM_OK;
        } else {
            KM_CK(cudaMemsetAsync(bad_count, 0, sizeof(int), st));
            km::k_validate_cols<T><<<NUM_SMS * 2, 256, 0, st>>>(MC, (int64_t)k * n, bad_count);
            KM_CKL();
            int nbad = 0;
            KM_CK(cudaMemcpyAsync(&nbad, bad_count, sizeof(int), cudaMemcpyDeviceToHost, st));
            KM_CK(cudaStreamSynchronize(st));
            if (nbad) return fail(KM_EINVAL, "a medoid column of D holds a negative or NaN dissimilarity");
            return KM_OK;
        }
    }

    km_status reset_counters() {
        KM_CK(cudaMemsetAsync(dec, 0, sizeof(Dec), st));
        return KM_OK;
    }

    km_status set_medoids(const int32_t* Mh) override {
        if (sharded) return fail(KM_EINVAL, "set_medoids on a sharded handle; use kmedoids_shard_set_medoids");
        if (k < 2) return fail(KM_EINVAL, "SWAP needs k >= 2");
        KM_TRY(set_point_slots(Mh));
        dim3 g((unsigned)cdiv(n, 256), k);
        km::k_gather_medoid_cols<T><<<g, 256, 0, st>>>(D, ld, (int)n, c0, c1, M, MC);
        KM_CKL();
        KM_TRY(validate_mc());
        KM_TRY(assign_full_and_td());
        KM_TRY(reset_counters());
        KM_CK(cudaStreamSynchronize(st));
        ready = true;
        fp3_reset();
        fp1_prepped = false;
        inc_valid = false;
        return KM_OK;
    }

    // a2: sort rows by nearest slot, removal loss, part metadata: phases 3-7
    // of the cooperative k_fp1_post, launched alone.
    km_status prep() {
        KM_TRY(post_alloc());
        return launch_post(true);
    }

    // a3 + a4 (local): stream the slab, combine into the local best record.
    // Stream timing of the device-decided sharded protocol: iterations are
    // enqueued without host round trips, so each launch gets its own event
    // pair from a ring, harvested when a pair is reused (16 launches later:
    // long complete) or at kmedoids_stream_time.
    static constexpr int PROF_RING = 16;
    bool prof_ring_mode = false;
    cudaEvent_t pr_ev[PROF_RING][2] = {};
    int64_t pr_next = 0, pr_done = 0;
    km_status prof_ring_pair(cudaEvent_t** pair) {
        const int slot = (int)(pr_next % PROF_RING);
        if (!pr_ev[slot][0])
            for (auto& e : pr_ev[slot]) KM_CK(cudaEventCreate(&e));
        if (pr_next - pr_done >= PROF_RING) KM_TRY(prof_take(pr_done));
        *pair = pr_ev[slot];
        ++pr_next;
        return KM_OK;
    }
    km_status prof_take(int64_t idx) {
        cudaEvent_t* p = pr_ev[idx % PROF_RING];
        KM_CK(cudaEventSynchronize(p[1]));
        float ms = 0.f;
        KM_CK(cudaEventElapsedTime(&ms, p[0], p[1]));
        prof_ms += ms; prof_launches += 1;
        pr_done = idx + 1;
        return KM_OK;
    }
    km_status prof_harvest() override {
        while (pr_done < pr_next) KM_TRY(prof_take(pr_done));
        return KM_OK;
    }

    bool fp1_mode = false;          // eval_local is enqueueing a FastPAM1 iteration (sticky convergence applies)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;   // stream-kernel events of the graph being captured
    km_status eval_local(bool do_prep = true) {
        if (do_prep) KM_TRY(prep());
        cudaEvent_t* pair = nullptr;
        if (profiling && prof_ring_mode) KM_TRY(prof_ring_pair(&pair));
        if (pair) KM_CK(cudaEventRecord(pair[0], st));
        else if (profiling) KM_CK(record_ev(ev_a ? ev_a : ev0));
        KM_TRY((launch_seg2<SG_NC, SG_RB, SG_S, SG_MINB>(D, w, wpad, P, o_plus, o_head, o_tail, o_imin, o_islot,
                                                          nullptr, fp1_mode ? &dec->done : nullptr)));
        KM_CKL();
        if (pair) KM_CK(cudaEventRecord(pair[1], st));
        else if (profiling) { KM_CK(record_ev(ev_b ? ev_b : ev1)); pending_prof = true; }
        // FastPAM1 iterations fold the part outputs in the post kernel's phase 0
        if (!(fp1_mode && post_fuse))
            KM_TRY(launch_combine(w, c0, P, o_plus, o_head, o_tail, o_imin, o_islot, head_slot, tail_slot, cand_v,
                                  cand_slot, nullptr, nullptr));
        return KM_OK;
    }

    // a4: per-candidate combine of the stream's part outputs, one thread per
    // column.  Measured slower and removed: folding part groups in parallel
    // warps (round 1: +10-30 us per step at C4/C5), 2/4/8 threads per column
    // merging range states by shuffles (round 2: +3-10 us at C4), and the
    // fold in the stream's tail by the last CTA of each tile (round 2: the
    // stream +90 us at C4: the fold of the last wave is latency-bound).  The
    // combine reads the part outputs (36 B per part and column: ~0.4 us per
    // part at C4), so its cost follows the part count P.
    km_status launch_combine(int ww, int64_t colb, int Pw, const A* pl, const A* hd, const A* tl, const A* im,
                             const int* isl, const int* hsl, const int* tsl, A* cv, int* cs, A* acc_o, A* plus_o) {
        constexpr int TPB = 128;   // 32 / 64 threads per block measured slower, 256 equal
        const size_t sm = (size_t)k * sizeof(A) + 2 * (size_t)Pw * sizeof(int);
        const bool stage = sm <= 32 * 1024;
        // 8 parts loaded ahead per thread (measured: 4 equal, 16 +15 us at C4: registers)
        km::k_swap_combine<A, 8><<<(unsigned)cdiv(ww, TPB), TPB, stage ? sm : 0, st>>>(
            ww, colb, Pw, pl, hd, tl, im, isl, hsl, tsl, R, empty_slot, point_slot, cv, cs, partials, counters,
            rec_local, acc_o, plus_o, k, stage);
        KM_CKL();
        return KM_OK;
    }

    template <int NC, int RB, int S, int MINB = 2>
    km_status launch_seg(A* acc_out) {
        return launch_seg2<NC, RB, S, MINB>(D, w, wpad, P, o_plus, o_head, o_tail, o_imin, o_islot, acc_out, f2_skip);
    }
    const int* f2_skip = nullptr;   // queued FastPAM2 iterations: the stream returns once Decision::done is set

    // The stream over the column window [Dw, Dw + ww) of the slab (Dw 16-byte
    // aligned) with Pw row parts; outputs indexed [part][column of window].
    template <int NC, int RB, int S, int MINB = 2>
    km_status launch_seg_win(const T* Dw, int ww, int wpadw, int Pw, A* plus_o, A* head_o, A* tail_o, A* imin_o,
                             int* islot_o, A* acc_out) {
        return launch_seg2<NC, RB, S, MINB>(Dw, ww, wpadw, Pw, plus_o, head_o, tail_o, imin_o, islot_o, acc_out);
    }

    bool seg2_attr_set = false;
    const char* stream_kernel_name() const override { return "k_swap_stream_seg2"; }
    template <int NC, int RB, int S, int MINB = 2>
    km_status launch_seg2(const T* Dw, int ww, int wpadw, int Pw, A* plus_o, A* head_o, A* tail_o, A* imin_o,
                          int* islot_o, A* acc_out, const int* skip_if = nullptr) {
        using C = km::SegCfg<T, NC, RB, S>;
        auto kern = km::k_swap_stream_seg2<T, A, NC, RB, S, MINB>;
        if (!seg2_attr_set) {
            KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            seg2_attr_set = true;
        }
        dim3 g((unsigned)cdiv(ww, C::COLS), Pw);
        // FastPAM2 / window k-vectors kept in L2 for the per-slot reduction
        // that follows when they fit comfortably (C3: 16 MB), else streamed
        const bool acc_keep = acc_out && (size_t)k * ww * sizeof(A) <= ((size_t)48 << 20);
        kern<<<g, C::THREADS, C::SMEM, st>>>(Dw, ld, ww, wpadw, (int)n, Pw, ri, R, plus_o, head_o, tail_o, imin_o,
                                              islot_o, acc_out, rowd, acc_keep, skip_if);
        return KM_OK;
    }

    km_status assign_incremental() {
        const int nb = (int)cdiv(n, 256);
        km::k_assign_incremental<T, A><<<nb, 256, 0, st>>>(MC, (int)n, k, dec, near, sec, dn, ds, rescan,
                                                            rescan_count);
        KM_CKL();
        km::k_assign_rescan<T, A><<<NUM_SMS, 256, 0, st>>>(MC, (int)n, k, dec, rescan, rescan_count, near, sec, dn,
                                                           ds);
        KM_CKL();
        return KM_OK;
    }

    km_status apply_local() {
        const int nb = (int)cdiv(n, 256);
        km::k_gather_decided_col<T, A><<<nb, 256, 0, st>>>(D, ld, (int)n, c0, c1, dec, MC, nullptr);
        KM_CKL();
        KM_TRY(assign_incremental());
        return KM_OK;
    }

    void copy_td(void* td_out) {
        if (!td_out) return;
        A v;
        cudaMemcpy(&v, td, sizeof(A), cudaMemcpyDeviceToHost);
        memcpy(td_out, &v, sizeof(A));
    }

    // ---- fused post-stream kernel (km_post.cuh) --------------------------------
    bool fp1_prepped = false;       // slot sort / R / part metadata valid for the current cache
    int post_blocks = 0;
    int *post_counts = nullptr, *post_offsets = nullptr;
    A* post_rpart = nullptr;
    unsigned long long* post_tph = nullptr;   // KM_STEP_PROF: phase stamps of k_fp1_post
    double post_ph_sum[8] = {};
    Rec* post_recs = nullptr;                  // [post_blocks] phase-0 block records
    // k_fp1_post phase 0 (the combine folded into the post kernel; KM_POST_FUSE=0:
    // the separate k_swap_combine, measurement override)
    bool post_fuse = true;
    size_t post_smem_base() const { return ((size_t)k * sizeof(int) + 15) / 16 * 16 + (size_t)k * sizeof(A); }
    size_t post_stage_bytes() const { return (size_t)k * sizeof(A) + 2 * (size_t)P * sizeof(int); }
    bool post_stage0() const { return post_smem_base() + post_stage_bytes() <= 24 * 1024; }
    // fused: the staging area (when R and the part slots fit), then the range states
    size_t post_smem() const {
        return post_fuse ? km::post_rs_offset<A>(k, P, post_stage0()) + km::post_rs_bytes<A>() : post_smem_base();
    }

    km_status post_alloc() {
        if (post_counts) return KM_OK;
        auto kern = km::k_fp1_post<T, A>;
        if (const char* e = getenv("KM_POST_FUSE")) post_fuse = e[0] != '0';
        const size_t sm = post_smem();
        if (sm > 48 * 1024) KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int dev = 0, per_sm = 0, nsm = 0;
        KM_CK(cudaGetDevice(&dev));
        KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        KM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, km::POST_THREADS, sm));
        if (per_sm < 1) return fail(KM_ECUDA, "k_fp1_post cannot be resident");
        int bps = 3;                                    // blocks per SM (KM_POST_BPS: measurement override)
        if (const char* e = getenv("KM_POST_BPS")) bps = std::max(1, std::min(8, atoi(e)));
        post_blocks = std::min(nsm * std::min(per_sm, bps), km::POST_MAX_BLOCKS);
        post_blocks = (int)std::min<int64_t>(post_blocks, std::max<int64_t>(1, cdiv(n, 64)));
        KM_TRY(alloc(&post_counts, (size_t)k * post_blocks));
        KM_TRY(alloc(&post_offsets, (size_t)k * post_blocks));
        KM_TRY(alloc(&post_rpart, (size_t)k * post_blocks));
        KM_TRY(alloc(&post_recs, post_blocks));
        if (step_prof) KM_TRY(alloc(&post_tph, 16));
        return KM_OK;
    }

    int post_reg = -1;
    km_status launch_post(bool prep_only = false) {
        km::PostArgs<T, A> g;
        g.D = D; g.ld = ld; g.n = (int)n; g.k = k; g.c0 = c0; g.c1 = c1; g.recs = rec_local; g.nrec = 1;
        g.td = td; g.M = M; g.point_slot = point_slot; g.dec = dec; g.MC = MC; g.near = near; g.sec = sec;
        g.dn = dn; g.ds = ds; g.rescan = rescan; g.rescan_count = rescan_count; g.counts = post_counts;
        g.offsets = post_offsets; g.rpart = post_rpart; g.slot_tot = slot_tot; g.seg_start = seg_start; g.empty_slot = empty_slot;
        g.ri = ri; g.rowd = rowd; g.R = R; g.P = P; g.head_slot = head_slot; g.tail_slot = tail_slot;
        g.tph = post_tph;
        g.prep_only = prep_only ? 1 : 0;
        if (post_reg < 0) {                 // KM_POST_REG=0: the chunk-loop path (large-n path, for tests)
            const char* e = getenv("KM_POST_REG");
            post_reg = (e && e[0] == '0') ? 0 : 1;
        }
        g.allow_reg = post_reg;
        g.sym = symmetric ? 1 : 0;
        g.h_ring = h_ring; g.ring = RING; g.seq = post_seq;
        g.fuse = (post_fuse && !prep_only) ? 1 : 0;
        g.w = w; g.stage0 = post_stage0() ? 1 : 0;
        g.pp_plus = o_plus; g.pp_head = o_head; g.pp_tail = o_tail; g.pp_imin = o_imin; g.pp_islot = o_islot;
        g.cand_v = cand_v; g.cand_slot = cand_slot; g.blk_recs = post_recs;
        void* args[] = {&g};
        KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp1_post<T, A>, dim3(post_blocks), dim3(km::POST_THREADS), args,
                                          post_smem(), st));
        ++launches;
        return KM_OK;
    }

    // One FastPAM1 iteration, enqueued on st (graph-capturable: fixed pointers,
    // no host-side memory other than the pinned decision mirror).  With the
    // post kernel the slot sort of this iteration was done by the previous
    // one (or by swap_iter before the first).
    km_status enqueue_fp1_iteration() {
        const bool prof_save = profiling;
        if (use_graph) profiling = graph_events() == 1;   // inline stream events (mode 2: fp1_capture adds them)
        fp1_mode = true;
        km_status s = eval_local(false);
        fp1_mode = false;
        profiling = prof_save;
        if (s != KM_OK) return s;
        if (step_prof) KM_CK(record_ev(sp_ev[2]));
        KM_TRY(launch_post());          // writes the pinned h_dec / h_td mirrors itself
        if (step_prof) KM_CK(record_ev(sp_ev[3]));
        if (step_prof) KM_CK(record_ev(sp_ev[4]));
        return KM_OK;
    }

    // the iteration with its stream-kernel events on a side branch of the
    // graph: start event as a root beside the stream kernel, end event after
    // it, the post kernel depending on the stream kernel only
    km_status enqueue_fp1_iteration_side(int gi) {
        if (!side_st) {
            KM_CK(cudaStreamCreateWithFlags(&side_st, cudaStreamNonBlocking));
            for (auto& e : fork_ev) KM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        KM_CK(cudaEventRecord(fork_ev[0], st));
        KM_CK(cudaStreamWaitEvent(side_st, fork_ev[0], 0));
        KM_CK(cudaEventRecordWithFlags(g_ev[gi][0], side_st, cudaEventRecordExternal));
        const bool prof_save = profiling;
        profiling = false;
        fp1_mode = true;
        km_status s = eval_local(false);
        fp1_mode = false;
        profiling = prof_save;
        if (s != KM_OK) return s;
        KM_CK(cudaEventRecord(fork_ev[1], st));
        KM_CK(cudaStreamWaitEvent(side_st, fork_ev[1], 0));
        KM_CK(cudaEventRecordWithFlags(g_ev[gi][1], side_st, cudaEventRecordExternal));
        KM_TRY(launch_post());
        KM_CK(cudaEventRecord(fork_ev[2], side_st));
        KM_CK(cudaStreamWaitEvent(st, fork_ev[2], 0));
        return KM_OK;
    }

    km_status swap_iter(km_variant v, int32_t* swaps, void* td_out) override {
        if (sharded) return fail(KM_EINVAL, "swap_iter on a sharded handle; use the kmedoids_shard_* phases");
        if (!ready) return fail(KM_EINVAL, "no medoids: call kmedoids_set_medoids or kmedoids_init_build first");
        if (v != KM_FASTPAM1 && v != KM_FASTPAM2 && v != KM_FASTERPAM && v != KM_FASTPAM1_INC)
            return fail(KM_EINVAL, "unknown variant %d", (int)v);
        if (v != KM_FASTPAM1) KM_TRY(clear_fp1_done());
        if (v == KM_FASTPAM2) return swap_iter_fp2(swaps, td_out);
        if (v == KM_FASTERPAM) return swap_iter_fp3(swaps, td_out);
        if (v == KM_FASTPAM1_INC) return inc_iters(1, swaps, td_out, nullptr, nullptr);
        KM_TRY(fp1_launch());
        KM_TRY(fp1_collect(fp1_seq - 1, true));
        return fp1_result(swaps, td_out);
    }

    // ---- FastPAM1 iterations: launch / collect ---------------------------------
    // Each iteration (stream + post kernel) is one CUDA graph launch; its
    // outcome reaches the host through the pinned ring h_ring (slot = launch
    // sequence number % RING, written by the post kernel), so the host can
    // keep the next iteration queued while it reads the current one
    // (fp1_run_pipelined).  A pass that finds no improving swap sets the
    // sticky Decision::done: iterations queued behind it are no-ops.  Two
    // graphs alternate so that each queued iteration has its own stream-kernel
    // events (profiling) while the previous one is collected.
    static constexpr int RING = 8;
    static constexpr int NGRAPH = 2;
    km::IterMirror<A>* h_ring = nullptr;
    int* post_seq = nullptr;            // device launch counter of the FastPAM1 post kernel
    int64_t fp1_seq = 0;                // host copy: FastPAM1 iterations launched
    cudaGraphExec_t fp1_g[NGRAPH] = {};
    cudaEvent_t g_ev[NGRAPH][2] = {};   // stream kernel start / end inside graph g
    cudaEvent_t g_done[NGRAPH] = {};    // recorded after each launch of graph g
    bool gev_ok[NGRAPH] = {};           // the last launch of slot g recorded its stream events
    bool fp1_any_done = false;          // a FastPAM1 pass may have set Decision::done

    km_status fp1_ring_alloc() {
        if (h_ring) return KM_OK;
        KM_CK(cudaMallocHost((void**)&h_ring, RING * sizeof(km::IterMirror<A>)));
        memset((void*)h_ring, 0xff, RING * sizeof(km::IterMirror<A>));   // seq = -1: nothing written yet
        KM_TRY(alloc(&post_seq, 1));
        KM_CK(cudaMemsetAsync(post_seq, 0, sizeof(int), st));
        for (int g = 0; g < NGRAPH; ++g) {
            KM_CK(cudaEventCreate(&g_ev[g][0]));
            KM_CK(cudaEventCreate(&g_ev[g][1]));
            KM_CK(cudaEventCreateWithFlags(&g_done[g], cudaEventDisableTiming));
        }
        return KM_OK;
    }

    // (other entry points that change the state clear the sticky flag)
    km_status clear_fp1_done() {
        if (!fp1_any_done) return KM_OK;
        KM_CK(cudaMemsetAsync(&dec->done, 0, sizeof(int32_t), st));
        fp1_any_done = false;
        return KM_OK;
    }

    // stream-kernel events of the iteration graph (measurement override
    // KM_GRAPH_EVENTS): 1 = on the path (event -> stream -> event -> post),
    // 2 = on a side branch (the post depends on the stream kernel only),
    // 0 = none.  Measured (scratch/evcost.py, K queued iterations): every
    // event record node on the path cost ~3 us of step time; on the side
    // branch the step equals the event-free graph (C2 82 -> 75 us, C3 291 ->
    // 285 us, C4 -5 us) and the stream kernel is still timed.
    int graph_events_mode = -1;
    int graph_events() {
        if (graph_events_mode < 0) {
            const char* e = getenv("KM_GRAPH_EVENTS");
            graph_events_mode = e ? std::max(0, std::min(2, atoi(e))) : 2;
            if (step_prof) graph_events_mode = 1;         // KM_STEP_PROF stamps the path itself
        }
        return graph_events_mode;
    }
    cudaStream_t side_st = nullptr;
    cudaEvent_t fork_ev[3] = {};

    km_status fp1_capture(int gi) {
        const int64_t l0 = launches;
        // capture on a private stream (the caller's may be the legacy default
        // stream, which cannot capture); launch on the caller's
        if (!cap_st) KM_CK(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
        cudaStream_t user_st = st;
        st = cap_st;
        cudaError_t be = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        if (be != cudaSuccess) { st = user_st; return fail(KM_ECUDA, "begin capture: %s", cudaGetErrorString(be)); }
        capturing = true;
        ev_a = g_ev[gi][0]; ev_b = g_ev[gi][1];
        km_status cs;
        if (graph_events() == 2) cs = enqueue_fp1_iteration_side(gi);
        else cs = enqueue_fp1_iteration();
        ev_a = ev_b = nullptr;
        capturing = false;
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &g);
        st = user_st;
        if (cs == KM_OK && ce == cudaSuccess) {
            ce = cudaGraphInstantiate(&fp1_g[gi], g, 0);
            if (ce != cudaSuccess) fp1_g[gi] = nullptr;
        }
        if (g) cudaGraphDestroy(g);
        fp1_graph_kernels = launches - l0;
        launches = l0;
        if (cs != KM_OK) return cs;
        if (!fp1_g[gi]) return fail(KM_ECUDA, "FastPAM1 iteration graph: %s", cudaGetErrorString(ce));
        return KM_OK;
    }

    // Enqueue FastPAM1 iteration number fp1_seq (no host wait).
    km_status fp1_launch() {
        KM_TRY(fp1_ring_alloc());
        inc_valid = false;
        KM_TRY(post_alloc());
        if (!fp1_prepped) {
            KM_TRY(prep());
            KM_CK(cudaMemsetAsync(rescan_count, 0, sizeof(int), st));
            fp1_prepped = true;
        }
        const int gi = (int)(fp1_seq % NGRAPH);
        const bool graph = use_graph && fp1_iters >= 1;   // the first iteration runs directly (allocations)
        if (graph && !fp1_g[gi])
            for (int g = 0; g < NGRAPH; ++g)               // both graphs at once: no capture inside later steps
                if (!fp1_g[g]) KM_TRY(fp1_capture(g));
        if (step_prof) KM_CK(cudaEventRecord(sp_ev[0], st));
        gev_ok[gi] = !graph || graph_events() != 0;
        if (graph) {
            KM_CK(cudaGraphLaunch(fp1_g[gi], st));
            launches += fp1_graph_kernels;
        } else {
            ev_a = g_ev[gi][0]; ev_b = g_ev[gi][1];
            const bool prof_save = profiling;
            profiling = true;
            km_status s2 = enqueue_fp1_iteration();
            profiling = prof_save;
            ev_a = ev_b = nullptr;
            KM_TRY(s2);
        }
        if (!fp1_ring_polled) KM_CK(cudaEventRecord(g_done[gi], st));
        ++fp1_seq;
        ++fp1_iters;
        fp1_any_done = true;
        return KM_OK;
    }

    // Wait for iteration `seq` and take its outcome into h_dec / h_td.
    km_status fp1_collect(int64_t seq, bool single) {
        const int gi = (int)(seq % NGRAPH);
        KM_CK(cudaEventSynchronize(g_done[gi]));
        const km::IterMirror<A>& m = h_ring[seq % RING];
        if (m.seq != (int32_t)seq) return fail(KM_ECUDA, "iteration ring out of step (%d vs %lld)", m.seq, (long long)seq);
        *h_dec = m.d;
        *h_td = m.td;
        if (profiling && !m.noop && gev_ok[gi]) {
            float ms = 0.f;
            KM_CK(cudaEventSynchronize(g_ev[gi][1]));
            KM_CK(cudaEventElapsedTime(&ms, g_ev[gi][0], g_ev[gi][1]));
            prof_ms += ms; prof_launches += 1;
        }
        pending_prof = false;
        if (single && step_prof) KM_TRY(step_prof_take(gi));
        return KM_OK;
    }

    km_status fp1_result(int32_t* swaps, void* td_out) {
        last_swaps.clear();
        if (h_dec->apply) {
            Rec r; r.v = h_dec->dtd; r.slot = h_dec->slot; r.c = h_dec->c;
            last_swaps.push_back(r);
        }
        if (swaps) *swaps = h_dec->apply;
        if (td_out) memcpy(td_out, h_td, sizeof(A));
        return h_dec->apply ? KM_OK : KM_CONVERGED;
    }

    // Up to max_iter FastPAM1 iterations with one queued ahead of the one
    // being read (no host round trip between iterations).  Stops at the first
    // pass without an improving swap (counted).
    km_status fp1_run_pipelined(int32_t max_iter, int32_t* iters_out, int32_t* swaps_out, bool* converged) override {
        if (sharded) return fail(KM_EINVAL, "swap iterations on a sharded handle; use the kmedoids_shard_* phases");
        if (!ready) return fail(KM_EINVAL, "no medoids: call kmedoids_set_medoids or kmedoids_init_build first");
        int32_t done_it = 0, sw = 0;
        bool conv = false;
        int64_t next = fp1_seq;             // next iteration to collect
        int64_t launched = 0;
        while (done_it < max_iter && !conv) {
            while (launched < max_iter && fp1_seq - next < 2) {
                KM_TRY(fp1_launch());
                ++launched;
            }
            KM_TRY(fp1_collect(next, false));
            ++next;
            ++done_it;
            if (h_dec->apply) ++sw; else conv = true;
        }
        fp1_result(nullptr, nullptr);      // last_swaps of the last collected pass (KM_CONVERGED is not an error)
        if (fp1_seq > next) KM_CK(cudaEventSynchronize(g_done[(fp1_seq - 1) % NGRAPH]));   // queued no-ops
        if (iters_out) *iters_out = done_it;
        if (swaps_out) *swaps_out = sw;
        if (converged) *converged = conv;
        return KM_OK;
    }

    // The same loop split for a host thread that drives several handles at
    // once (FastCLARA samples, one stream each): fp1_async_begin queues the
    // first two iterations, fp1_async_poll collects every finished one
    // without blocking (cudaEventQuery on its completion event) and queues
    // the next; *finished once a pass without an improving swap (or
    // max_iter passes) has been collected.  Work enqueued on the handle's
    // stream afterwards is ordered behind the queued no-op iteration.
    // Completion is seen in the pinned ring itself (the post kernel writes
    // the entry's seq last, behind a system fence): no event record per
    // launch, no event query per poll.
    struct Fp1Async { int64_t next = 0, launched = 0; int32_t max_iter = 0, done_it = 0, sw = 0; bool conv = false;
                      int misses = 0; };
    Fp1Async fa;
    bool fp1_ring_polled = false;           // launches record no g_done event (fp1_async_*)
    km_status fp1_async_begin(int32_t max_iter) {
        if (sharded) return fail(KM_EINVAL, "swap iterations on a sharded handle; use the kmedoids_shard_* phases");
        if (!ready) return fail(KM_EINVAL, "no medoids: call kmedoids_set_medoids or kmedoids_init_build first");
        KM_TRY(fp1_ring_alloc());
        fp1_ring_polled = true;
        fa = Fp1Async();
        fa.next = fp1_seq;
        fa.max_iter = max_iter;
        while (fa.launched < max_iter && fp1_seq - fa.next < 2) {
            KM_TRY(fp1_launch());
            ++fa.launched;
        }
        return KM_OK;
    }
    km_status fp1_async_poll(bool* finished) {
        *finished = false;
        while (fa.done_it < fa.max_iter && !fa.conv) {
            const km::IterMirror<A>& m = h_ring[fa.next % RING];
            if (*reinterpret_cast<const volatile int32_t*>(&m.seq) != (int32_t)fa.next) {
                // not written yet: every 256th miss, check that the stream is
                // still working on it (a fault or an idle stream is an error)
                if (++fa.misses % 256 == 0) {
                    const cudaError_t q = cudaStreamQuery(st);
                    if (q == cudaSuccess && *reinterpret_cast<const volatile int32_t*>(&m.seq) != (int32_t)fa.next)
                        return fail(KM_ECUDA, "iteration ring out of step (%d vs %lld)", m.seq, (long long)fa.next);
                    if (q != cudaSuccess && q != cudaErrorNotReady)
                        return fail(KM_ECUDA, "FastPAM1 iteration: %s", cudaGetErrorString(q));
                }
                return KM_OK;
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            *h_dec = m.d;
            *h_td = m.td;
            ++fa.next;
            ++fa.done_it;
            if (h_dec->apply) ++fa.sw; else fa.conv = true;
            while (!fa.conv && fa.launched < fa.max_iter && fp1_seq - fa.next < 2) {
                KM_TRY(fp1_launch());
                ++fa.launched;
            }
        }
        fp1_result(nullptr, nullptr);
        fp1_ring_polled = false;
        *finished = true;
        return KM_OK;
    }

    km_status step_prof_take(int gi) {
        // phases of the iteration (KM_STEP_PROF=1, measurement aid): launch ->
        // stream start, stream, combine, post
        float t[5];
        KM_CK(cudaEventElapsedTime(&t[0], sp_ev[0], g_ev[gi][0]));
        KM_CK(cudaEventElapsedTime(&t[1], g_ev[gi][0], g_ev[gi][1]));
        KM_CK(cudaEventElapsedTime(&t[2], g_ev[gi][1], sp_ev[2]));
        KM_CK(cudaEventElapsedTime(&t[3], sp_ev[2], sp_ev[3]));
        KM_CK(cudaEventElapsedTime(&t[4], sp_ev[3], sp_ev[4]));
        for (int i = 0; i < 5; ++i) sp_sum[i] += t[i];
        if (post_tph) {
            unsigned long long h[7];
            KM_CK(cudaMemcpy(h, post_tph, sizeof(h), cudaMemcpyDeviceToHost));
            const bool f = post_fuse;        // phase 0 (fused combine) stamped in h[6]
            post_ph_sum[5] += f ? 1e-3 * (double)(h[6] - h[0]) : 0.0;
            post_ph_sum[0] += 1e-3 * (double)(h[1] - (f ? h[6] : h[0]));
            for (int i = 1; i < 5; ++i) post_ph_sum[i] += 1e-3 * (double)(h[i + 1] - h[i]);
        }
        if (++sp_n % 50 == 0) {
            fprintf(stderr, "[kmedoids] step phases over %d iterations (us): launch %.1f stream %.1f combine %.1f "
                    "post %.1f copies %.1f\n", sp_n, 1e3 * sp_sum[0] / sp_n, 1e3 * sp_sum[1] / sp_n,
                    1e3 * sp_sum[2] / sp_n, 1e3 * sp_sum[3] / sp_n, 1e3 * sp_sum[4] / sp_n);
            if (post_tph)
                fprintf(stderr, "[kmedoids] post phases (us): combine0+sync %.1f select %.1f apply+rescan %.1f "
                        "count+sync %.1f scan+sync %.1f scatter/parts %.1f\n", post_ph_sum[5] / sp_n,
                        post_ph_sum[0] / sp_n, post_ph_sum[1] / sp_n,
                        post_ph_sum[2] / sp_n, post_ph_sum[3] / sp_n, post_ph_sum[4] / sp_n);
        }
        return KM_OK;
    }

    km_status fp2_alloc() {
        if (fp2_acc) return KM_OK;
        KM_TRY(alloc(&fp2_acc, (size_t)k * w));
        KM_TRY(alloc(&fp2_plus, w));
        KM_TRY(alloc(&fp2_best, k));
        KM_TRY(alloc(&fp2_part, (size_t)k * FP2_SPLIT));
        KM_TRY(alloc(&fp2_order, k));
        int dev = 0, per_sm = 0, nsm = 0;
        KM_CK(cudaGetDevice(&dev));
        KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        KM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, km::k_fp2_sequential<T, A>, 256, 0));
        // all co-resident blocks: a re-evaluation step is a strided gather of one
        // column (n sectors) and wants every SM's load units (measured: one
        // block per SM is ~1.6x slower despite cheaper grid syncs)
        fp2_blocks = (int)std::min<int64_t>((int64_t)nsm * std::max(per_sm, 1), std::max<int64_t>(1, cdiv(n, 256)));
        KM_TRY(alloc(&fp2_partials, (size_t)2 * fp2_blocks * km::FP2_B));
        KM_TRY(alloc(&fp2_cols, (size_t)km::FP2_B * n));
        KM_TRY(alloc(&fp2_m, 2));
        KM_TRY(alloc(&fp2_swaps_prev, 1));
        trace_cap = k;
        KM_TRY(alloc(&trace, trace_cap));
        h_best.resize(k);
        return KM_OK;
    }

    // FastPAM2 step 1-3 (reading R6), local part: per-slot best over this
    // handle's candidates into fp2_best (device).
    km_status fp2_eval_local(bool fused_plan = false) {
        KM_TRY(fp2_alloc());
        f2_mark(0);
        KM_TRY(prep());
        f2_mark(1);
        // FastPAM2 always uses the segment-aligned TMA stream (it stores acc_c[i]).
        if (profiling) KM_CK(record_ev(ev0));
        KM_TRY((launch_seg<SG_NC, SG_RB, SG_S, SG_MINB>(fp2_acc)));
        KM_CKL();
        if (profiling) { KM_CK(record_ev(ev1)); pending_prof = true; }
        f2_mark(2);
        KM_TRY(launch_combine(w, c0, P, o_plus, o_head, o_tail, o_imin, o_islot, head_slot, tail_slot, cand_v, cand_slot,
                              fp2_acc, fp2_plus));
        f2_mark(3);
        if (k >= FP2_SB_MIN_K)           // 4 slots per block: point_slot / plus loaded once per 4 rows of acc
            km::k_fp2_slot_best<A, 4><<<dim3((unsigned)cdiv(k, 4), FP2_SPLIT), 256, 0, st>>>(
                w, k, c0, fp2_acc, fp2_plus, R, seg_start, point_slot, fp2_part);
        else
            km::k_fp2_slot_best<A, 1><<<dim3(k, FP2_SPLIT), 256, 0, st>>>(w, k, c0, fp2_acc, fp2_plus, R, seg_start,
                                                                         point_slot, fp2_part);
        KM_CKL();
        if (!fused_plan) {                 // (single-GPU device plan: folded into k_fp2_plan_sort)
            km::k_fp2_slot_reduce<A><<<(unsigned)cdiv(k, 128), 128, 0, st>>>(k, FP2_SPLIT, fp2_part, fp2_best);
            KM_CKL();
        }
        return KM_OK;
    }

    // Steps 4-5 on the host (identical on every rank): improving slots of the
    // global per-slot bests h_best ordered by (v_i, i).
    std::vector<int> fp2_order_slots(A tdh) {
        std::vector<int> order;
        for (int i = 0; i < k; ++i) {
            const Rec& b = h_best[i];
            if (b.slot == INT_MAX) continue;
            const bool imp = km::Acc<T>::is_float ? ((double)b.v < -1e-12 * fabs((double)tdh)) : (b.v < 0);
            if (imp) order.push_back(i);
        }
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            return h_best[a].v < h_best[b].v || (h_best[a].v == h_best[b].v && a < b);
        });
        return order;
    }

    km_status fp2_finish_profiling() {
        if (profiling && pending_prof) {
            float ms = 0.f;
            KM_CK(cudaEventElapsedTime(&ms, ev0, ev1));
            prof_ms += ms; prof_launches += 1; pending_prof = false;
        }
        return KM_OK;
    }

    // Steps 6-7: the sequential phase (one cooperative kernel).  colsrc/colidx
    // give each order entry's candidate column (sharded: gathered columns);
    // nullptr = read the column from D.  Counts the iteration.
    km_status fp2_sequential(const std::vector<int>& order, const T* colsrc, const int* colidx_dev,
                             int32_t* swaps_out, void* td_out) {
        KM_CK(cudaMemcpyAsync(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        Dec hd = *h_dec;
        hd.iters += 1;
        hd.apply = 0;
        const int swaps0 = hd.swaps;
        last_swaps.clear();
        if (order.empty()) {
            KM_CK(cudaMemcpyAsync(dec, &hd, sizeof(Dec), cudaMemcpyHostToDevice, st));
            KM_CK(cudaStreamSynchronize(st));
            *h_dec = hd;
            if (swaps_out) *swaps_out = 0;
            copy_td(td_out);
            return KM_CONVERGED;
        }
        hd.swaps = 0;                       // the kernel counts this iteration's swaps from 0
        KM_CK(cudaMemcpyAsync(dec, &hd, sizeof(Dec), cudaMemcpyHostToDevice, st));
        KM_CK(cudaMemcpyAsync(fp2_order, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        int m = (int)order.size();
        KM_CK(cudaMemcpyAsync(fp2_m, &m, sizeof(int), cudaMemcpyHostToDevice, st));
        KM_TRY(launch_fp2_sequential(colsrc, colidx_dev));
        KM_CK(cudaMemcpyAsync(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        const int done = h_dec->swaps;
        last_swaps.resize(std::min(done, trace_cap));
        if (!last_swaps.empty())
            KM_CK(cudaMemcpy(last_swaps.data(), trace, last_swaps.size() * sizeof(Rec), cudaMemcpyDeviceToHost));
        hd = *h_dec;
        hd.swaps = swaps0 + done;
        KM_CK(cudaMemcpyAsync(dec, &hd, sizeof(Dec), cudaMemcpyHostToDevice, st));
        KM_CK(cudaStreamSynchronize(st));
        *h_dec = hd;
        if (swaps_out) *swaps_out = done;
        copy_td(td_out);
        return KM_OK;
    }

    // One single-GPU FastPAM2 iteration (reading R6).
    // One FastPAM2 iteration with the plan on the device (k_fp2_plan): the
    // host waits once, at the end (KM_FP2_HOSTPLAN=1: the host orders the
    // slots, as the sharded path does).
    int fp2_hostplan = -1;
    km_status swap_iter_fp2(int32_t* swaps_out, void* td_out) {
        fp1_prepped = false;
        inc_valid = false;
        if (fp2_hostplan < 0) {
            const char* e = getenv("KM_FP2_HOSTPLAN");
            fp2_hostplan = (e && e[0] == '1') ? 1 : 0;
        }
        const bool sort_plan = !fp2_hostplan && k <= km::FP2_SORT_MAX;
        KM_TRY(fp2_eval_local(sort_plan));
        if (fp2_hostplan) {
            A tdh;
            KM_CK(cudaMemcpyAsync(h_best.data(), fp2_best, k * sizeof(Rec), cudaMemcpyDeviceToHost, st));
            KM_CK(cudaMemcpyAsync(&tdh, td, sizeof(A), cudaMemcpyDeviceToHost, st));
            KM_CK(cudaStreamSynchronize(st));
            KM_TRY(fp2_finish_profiling());
            const std::vector<int> order = fp2_order_slots(tdh);
            return fp2_sequential(order, nullptr, nullptr, swaps_out, td_out);
        }
        KM_TRY(fp2_enqueue_tail(sort_plan, 0, false));
        f2_mark(6);
        f2_mark(7);
        KM_CK(cudaStreamSynchronize(st));
        f2_take();
        KM_TRY(fp2_finish_profiling());
        return fp2_read(0, swaps_out, td_out);
    }

    // Steps 4-7 on the device behind fp2_eval_local: the plan, then the
    // sequential kernel, which writes the outcome (decision, TD, this
    // iteration's swap count and trace) into pinned ring slot `slot`.
    // sticky: the plan kernels honour / set Decision::done (queued iterations).
    static constexpr int F2RING = 2;
    Rec* h_f2out = nullptr;          // pinned, F2RING slots of (trace_cap + 1) records: [0] swaps (int), [1..] trace
    Dec* h_f2dec = nullptr;          // pinned, F2RING decisions
    A* h_f2td = nullptr;             // pinned, F2RING TDs
    cudaEvent_t f2_done[F2RING] = {};
    km_status fp2_enqueue_tail(bool sort_plan, int slot, bool sticky) {
        f2_mark(4);
        if (sort_plan) {
            int np2 = 2;
            while (np2 < k) np2 <<= 1;
            km::k_fp2_plan_sort<A><<<1, 1024, (size_t)np2 * (sizeof(A) + sizeof(int)), st>>>(
                fp2_part, FP2_SPLIT, fp2_best, k, np2, td, dec, fp2_order, fp2_m, fp2_swaps_prev, sticky ? 1 : 0);
        } else {
            const size_t psm = (size_t)k * (sizeof(A) + 1);
            const bool pstaged = psm <= 40 * 1024;
            km::k_fp2_plan<A><<<1, 1024, pstaged ? psm : 0, st>>>(fp2_best, k, td, dec, fp2_order, fp2_m,
                                                                  fp2_swaps_prev, pstaged, sticky ? 1 : 0);
        }
        KM_CKL();
        ++launches;
        f2_mark(5);
        if (!h_f2out) {
            KM_CK(cudaMallocHost((void**)&h_f2out, sizeof(Rec) * (size_t)(trace_cap + 1) * F2RING));
            KM_CK(cudaMallocHost((void**)&h_f2dec, sizeof(Dec) * F2RING));
            KM_CK(cudaMallocHost((void**)&h_f2td, sizeof(A) * F2RING));
            for (auto& e : f2_done) KM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        Rec* out = h_f2out + (size_t)slot * (trace_cap + 1);
        km::F2HostOut<A> ho;
        ho.dec = h_f2dec + slot; ho.td = h_f2td + slot; ho.swaps = reinterpret_cast<int*>(out); ho.trace = out + 1;
        KM_TRY(launch_fp2_sequential(nullptr, nullptr, fp2_swaps_prev, ho));
        KM_CK(cudaEventRecord(f2_done[slot], st));
        return KM_OK;
    }
    // The outcome in ring slot `slot` (its iteration has completed).
    km_status fp2_read(int slot, int32_t* swaps_out, void* td_out) {
        const Rec* out = h_f2out + (size_t)slot * (trace_cap + 1);
        int done = 0;
        memcpy(&done, out, sizeof(int));
        last_swaps.assign(out + 1, out + 1 + std::min(done, trace_cap));
        *h_dec = h_f2dec[slot];
        *h_td = h_f2td[slot];
        if (swaps_out) *swaps_out = done;
        if (td_out) memcpy(td_out, h_td, sizeof(A));
        return done > 0 ? KM_OK : KM_CONVERGED;
    }

    // Up to max_iter FastPAM2 iterations, the next one queued on the device
    // while the host reads the current one (as fp1_run_pipelined): no host
    // round trip between iterations.  Each is exactly one swap_iter_fp2
    // (same plan, same swaps, same counts); stops after the first pass
    // without an improving slot (counted); passes queued behind
    // it are no-ops (sticky Decision::done).
    km_status fp2_run_pipelined(int32_t max_iter, int32_t* iters_out, int32_t* swaps_out, bool* converged) override {
        if (sharded) return fail(KM_EINVAL, "swap iterations on a sharded handle; use the kmedoids_fp2_shard_* phases");
        if (!ready) return fail(KM_EINVAL, "no medoids: call kmedoids_set_medoids or kmedoids_init_build first");
        if (fp2_hostplan < 0) {
            const char* e = getenv("KM_FP2_HOSTPLAN");
            fp2_hostplan = (e && e[0] == '1') ? 1 : 0;
        }
        int32_t it = 0, sw = 0;
        bool conv = false;
        if (fp2_hostplan) {                  // measurement override: the host plans, one iteration at a time
            while (it < max_iter && !conv) {
                int32_t s1 = 0;
                const km_status q = swap_iter(KM_FASTPAM2, &s1, nullptr);
                if (q != KM_OK && q != KM_CONVERGED) return q;
                ++it; sw += s1; conv = q == KM_CONVERGED;
            }
        } else {
            KM_TRY(clear_fp1_done());
            fp1_any_done = true;             // the plan may set Decision::done
            const bool sort_plan = k <= km::FP2_SORT_MAX;
            f2_skip = &dec->done;
            int64_t launched = 0, next = 0;
            km_status r = KM_OK;
            while (r == KM_OK && it < max_iter && !conv) {
                while (r == KM_OK && launched < max_iter && launched - next < F2RING) {
                    fp1_prepped = false;
                    inc_valid = false;
                    r = fp2_eval_local(sort_plan);
                    if (r == KM_OK) r = fp2_enqueue_tail(sort_plan, (int)(launched % F2RING), true);
                    ++launched;
                }
                if (r != KM_OK) break;
                if (cudaEventSynchronize(f2_done[next % F2RING]) != cudaSuccess) { r = fail(KM_ECUDA, "FastPAM2 iteration"); break; }
                int32_t s1 = 0;
                conv = fp2_read((int)(next % F2RING), &s1, nullptr) == KM_CONVERGED;
                ++next; ++it; sw += s1;
            }
            f2_skip = nullptr;
            if (r != KM_OK) return r;
            if (launched > next) KM_CK(cudaStreamSynchronize(st));   // the queued no-ops
            KM_TRY(fp2_finish_profiling());
        }
        if (iters_out) *iters_out = it;
        if (swaps_out) *swaps_out = sw;
        if (converged) *converged = conv;
        return KM_OK;
    }

    int* fp2_m = nullptr;            // [2]: improving slots m; swaps of the iteration
    int* fp2_swaps_prev = nullptr;
    km_status launch_fp2_sequential(const T* colsrc, const int* colidx_dev, const int* swaps_prev_dev = nullptr,
                                    km::F2HostOut<A> ho = km::F2HostOut<A>{nullptr, nullptr, nullptr, nullptr}) {
        const T* Dp = D; int64_t ldv = ld; int nn = (int)n; int kk = k;
        int* Mp = M; int* psp = point_slot; T* MCp = MC; int* nr = near; int* sc = sec; T* dnp = dn; T* dsp = ds;
        T* cb = fp2_cols; A* tdp = td; A* pp = fp2_partials; Dec* dp = dec; Rec* tr = trace; int tc = trace_cap;
        int* op = fp2_order; Rec* bp = fp2_best; const int* mp = fp2_m;
        const T* csp = colsrc; const int* cip = colidx_dev;
        int* rsp = rescan; int* rcp = rescan_count;
        int symv = symmetric ? 1 : 0;
        int* swi = fp2_m + 1;               // swaps of this iteration (written by the kernel)
        const int* swp = swaps_prev_dev;
        void* args[] = {&Dp, &ldv, &csp, &cip, &nn, &kk, &op, &mp, &bp, &Mp, &psp, &MCp, &nr, &sc, &dnp, &dsp, &cb,
                        &tdp, &pp, &dp, &tr, &tc, &rsp, &rcp, &symv, &swi, &swp, &ho};
        KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp2_sequential<T, A>, dim3(fp2_blocks), dim3(256), args, 0,
                                          st));
        ++launches;
        return KM_OK;
    }

    // ---- FasterPAM (Alg.4; readings F1-F5) -------------------------
    // Exact eager scan by speculative batches: evaluate the candidates of the
    // next scan positions [t, hi) on the current state in one stream pass,
    // accept the FIRST improving one (every candidate before it was evaluated
    // on exactly the state Alg.4's sequential loop sees), apply it, resume
    // at the position behind it.  Positions run t = 0, 1, 2, ... with
    // candidate c = t mod n (F1); the scan stops once n consecutive
    // positions passed without a swap (F2); a pass = n positions (F3).
    int64_t fp3_t = 0, fp3_tlast = 0;
    bool fp3_dirty = true;          // cache changed since the last prep()
    int fp3_wmax = 0, fp3_w0 = 0, fp3_pmax = 0;
    A *f3_plus = nullptr, *f3_head = nullptr, *f3_tail = nullptr, *f3_imin = nullptr, *f3_v = nullptr;
    int *f3_islot = nullptr, *f3_hs = nullptr, *f3_ts = nullptr, *f3_s = nullptr;
    int64_t fp3_batches = 0;

    void fp3_reset() { fp3_t = 0; fp3_tlast = 0; fp3_dirty = true; }

    // row parts for a window of ww columns: one wave of 3 CTAs per SM
    int fp3_parts(int ww) const {
        const int64_t ncb = cdiv(ww, SG_NC * 128);
        int64_t p = cdiv((int64_t)NUM_SMS * SG_MINB, ncb);
        p = std::min<int64_t>(p, std::max<int64_t>(1, n / 64));
        return (int)std::max<int64_t>(p, 1);
    }

    km_status fp3_alloc() {
        if (f3_plus) return KM_OK;
        const int tile = SG_NC * 128;
        const char* ew = getenv("KM_FASTER_WMAX");
        const char* e0 = getenv("KM_FASTER_W0");
        fp3_wmax = ew ? std::max(tile, atoi(ew) / tile * tile) : 16 * tile;
        fp3_w0 = e0 ? std::max(tile, atoi(e0) / tile * tile) : 2 * tile;
        fp3_w0 = std::min(fp3_w0, fp3_wmax);
        size_t cap = 0;
        for (int64_t nc = 1; nc <= cdiv(fp3_wmax + 3, tile); ++nc) {
            const int ww = (int)std::min<int64_t>(nc * tile, fp3_wmax + 3);
            cap = std::max(cap, (size_t)fp3_parts(ww) * ww);
        }
        fp3_pmax = fp3_parts(1);
        KM_TRY(alloc(&f3_plus, cap));
        KM_TRY(alloc(&f3_head, cap));
        KM_TRY(alloc(&f3_tail, cap));
        KM_TRY(alloc(&f3_imin, cap));
        KM_TRY(alloc(&f3_islot, cap));
        KM_TRY(alloc(&f3_hs, fp3_pmax));
        KM_TRY(alloc(&f3_ts, fp3_pmax));
        KM_TRY(alloc(&f3_v, fp3_wmax + 4));
        KM_TRY(alloc(&f3_s, fp3_wmax + 4));
        return KM_OK;
    }

    // One batch: scan positions [t, hi) of the pass starting at pass_base.
    km_status fp3_batch(int64_t pass_base, int64_t t, int64_t hi, bool new_pass) {
        const int clo = (int)(t - pass_base), chi = (int)(hi - pass_base);
        const int a = clo & ~3;                       // 16-byte aligned window start
        const int ww = chi - a, wpadw = (int)std::min<int64_t>(cdiv(ww, 4) * 4, ld - a);
        const int Pw = fp3_parts(ww);
        if (fp3_dirty) { KM_TRY(prep()); fp3_dirty = false; }
        km::k_part_meta<T><<<(unsigned)cdiv(Pw, 128), 128, 0, st>>>(ri, (int)n, Pw, f3_hs, f3_ts);
        KM_CKL();
        if (profiling) KM_CK(record_ev(ev0));
        KM_TRY((launch_seg_win<SG_NC, SG_RB, SG_S, SG_MINB>(D + a, ww, wpadw, Pw, f3_plus, f3_head, f3_tail, f3_imin,
                                                             f3_islot, nullptr)));
        KM_CKL();
        if (profiling) { KM_CK(record_ev(ev1)); pending_prof = true; }
        KM_TRY(launch_combine(ww, c0 + a, Pw, f3_plus, f3_head, f3_tail, f3_imin, f3_islot, f3_hs, f3_ts, f3_v, f3_s,
                              nullptr, nullptr));
        km::k_fp3_pick<A><<<1, 1024, 0, st>>>(f3_v, f3_s, clo - a, chi - a, c0 + a, td, M, point_slot, dec,
                                              rescan_count, new_pass ? 1 : 0);
        KM_CKL();
        KM_TRY(apply_local());                        // no-ops unless a swap was picked
        ++fp3_batches;
        return sync_dec();
    }

    // ---- FasterPAM, cooperative window scan (default; KM_FASTER=batch selects
    // the speculative batch path above).  A window is streamed once; one
    // cooperative kernel (km_fasterpam.cuh) scans it, swapping eagerly and
    // correcting the values ahead of each swap instead of re-streaming.
    int fp3_mode = -1;              // 1 = cooperative window scan, 0 = speculative batches
    int fp3c_ww = 0, fp3c_L = 0, fp3c_blocks = 0;
    A *f3_acc = nullptr, *f3_wplus = nullptr, *f3_pacc = nullptr, *f3_pplus = nullptr, *f3_pR = nullptr;
    int *f3_flag = nullptr, *f3_oldnear = nullptr, *f3_rescan = nullptr, *f3_blk = nullptr;
    T *f3_olddn = nullptr, *f3_oldds = nullptr, *f3_mct = nullptr;
    int *f3_tflag = nullptr, *f3_tmap = nullptr, *f3_tlist = nullptr;
    km::Fp3Chg<T>* f3_chg = nullptr;
    km::Fp3Ctl *f3_ctl = nullptr, *h_f3ctl = nullptr;
    Rec* f3_trace = nullptr;
    int64_t fp3_windows = 0, fp3_stale = 0;
    unsigned long long fp3_tphase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long fp3_stat[3] = {0, 0, 0};
    double fp3_host_ms = 0;

    km_status fp3c_alloc() {
        if (f3_acc) return KM_OK;
        const int tile = SG_NC * 128;
        const char* ew = getenv("KM_FASTER_COOP_W");
        const char* el = getenv("KM_FASTER_L");
        fp3c_ww = ew ? std::max(tile, atoi(ew) / tile * tile) : 8 * tile;
        fp3c_L = el ? std::max(32, atoi(el) / 32 * 32) : 4096;
        fp3c_ww = std::min(fp3c_ww, fp3_wmax);     // the stream's part buffers are sized for fp3_wmax
        fp3c_L = std::min(fp3c_L, fp3c_ww);
        const size_t wcap = (size_t)fp3c_ww + 4;
        KM_TRY(alloc(&f3_acc, (size_t)k * wcap));
        KM_TRY(alloc(&f3_wplus, wcap));
        KM_TRY(alloc(&f3_pacc, (size_t)km::FP3_G * km::FP3_TMAX * fp3c_L));
        KM_TRY(alloc(&f3_pplus, (size_t)km::FP3_G * fp3c_L));
        KM_TRY(alloc(&f3_pR, (size_t)km::FP3_G * km::FP3_TMAX));
        KM_TRY(alloc(&f3_flag, n));
        KM_TRY(alloc(&f3_oldnear, n));
        KM_TRY(alloc(&f3_olddn, n));
        KM_TRY(alloc(&f3_oldds, n));
        KM_TRY(alloc(&f3_rescan, n));
        KM_TRY(alloc(&f3_chg, n));
        KM_TRY(alloc(&f3_mct, (size_t)n * k));
        KM_TRY(alloc(&f3_tflag, k));
        KM_TRY(alloc(&f3_tmap, k));
        KM_TRY(alloc(&f3_tlist, k));
        KM_TRY(alloc(&f3_ctl, 1));
        KM_TRY(alloc(&f3_trace, wcap));
        KM_CK(cudaMemsetAsync(f3_tflag, 0, k * sizeof(int), st));
        KM_CK(cudaMallocHost((void**)&h_f3ctl, sizeof(km::Fp3Ctl)));
        auto kern = km::k_fp3_window<T, A, false>;
        KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, km::FP3_SMEM));
        KM_CK(cudaFuncSetAttribute(km::k_fp3_window<T, A, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   km::FP3_SMEM));
        int dev = 0, per_sm = 0, nsm = 0;
        KM_CK(cudaGetDevice(&dev));
        KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        KM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, km::FP3_THREADS, km::FP3_SMEM));
        if (per_sm < 1) return fail(KM_ECUDA, "k_fp3_window cannot be resident");
        fp3c_blocks = nsm * per_sm;
        KM_TRY(alloc(&f3_blk, fp3c_blocks));
        return KM_OK;
    }

    // One window of the scan: positions [t, hi) of the pass at pass_base.
    km_status fp3_window_coop(int64_t pass_base, int64_t t, int64_t hi, bool new_pass) {
        const int clo = (int)(t - pass_base), chi = (int)(hi - pass_base);
        const int a = clo & ~3;
        const int ww = chi - a, wpadw = (int)std::min<int64_t>(cdiv(ww, 4) * 4, ld - a);
        const int Pw = fp3_parts(ww);
        if (fp3_dirty) { KM_TRY(prep()); fp3_dirty = false; }
        KM_CK(cudaMemsetAsync(f3_acc, 0, (size_t)k * ww * sizeof(A), st));
        km::k_part_meta<T><<<(unsigned)cdiv(Pw, 128), 128, 0, st>>>(ri, (int)n, Pw, f3_hs, f3_ts);
        KM_CKL();
        if (profiling) KM_CK(record_ev(ev0));
        KM_TRY((launch_seg_win<SG_NC, SG_RB, SG_S, SG_MINB>(D + a, ww, wpadw, Pw, f3_plus, f3_head, f3_tail, f3_imin,
                                                             f3_islot, f3_acc)));
        KM_CKL();
        if (profiling) { KM_CK(record_ev(ev1)); pending_prof = true; }
        KM_TRY(launch_combine(ww, c0 + a, Pw, f3_plus, f3_head, f3_tail, f3_imin, f3_islot, f3_hs, f3_ts, f3_v, f3_s,
                              f3_acc, f3_wplus));
        km::Fp3Ctl hc;
        memset(&hc, 0, sizeof(hc));
        hc.first[0] = hc.first[1] = hc.first[2] = INT_MAX;
        *h_f3ctl = hc;
        KM_CK(cudaMemcpyAsync(f3_ctl, h_f3ctl, sizeof(hc), cudaMemcpyHostToDevice, st));
        km::Fp3Args<T, A> g;
        g.D = D; g.ld = ld; g.n = (int)n; g.k = k; g.c0 = c0; g.a = a; g.ww = ww;
        g.lo = clo - a; g.hi = chi - a; g.L = fp3c_L;
        g.acc = f3_acc; g.plus = f3_wplus; g.R = R; g.M = M; g.point_slot = point_slot; g.MC = MC; g.MCt = f3_mct;
        g.near = near; g.sec = sec; g.dn = dn; g.ds = ds; g.td = td; g.dec = dec;
        g.trace = f3_trace; g.trace_cap = fp3c_ww + 4;
        g.cand_v = f3_v; g.cand_s = f3_s; g.flag = f3_flag; g.old_near = f3_oldnear; g.old_dn = f3_olddn;
        g.old_ds = f3_oldds; g.rescan = f3_rescan; g.blk_cnt = f3_blk; g.chg = f3_chg; g.chg_cap = (int)n;
        g.touched_flag = f3_tflag; g.touched_map = f3_tmap; g.touched = f3_tlist;
        g.part_acc = f3_pacc; g.part_plus = f3_pplus; g.part_R = f3_pR; g.ctl = f3_ctl; g.new_pass = new_pass ? 1 : 0;
        g.max_iters = 0; g.gpart = nullptr;
        void* args[] = {&g};
        KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp3_window<T, A, false>, dim3(fp3c_blocks), dim3(km::FP3_THREADS),
                                          args, km::FP3_SMEM, st));
        ++launches;
        KM_CK(cudaMemcpyAsync(h_f3ctl, f3_ctl, sizeof(km::Fp3Ctl), cudaMemcpyDeviceToHost, st));
        KM_TRY(sync_dec());
        ++fp3_windows;
        const km::Fp3Ctl r = *h_f3ctl;
        if (r.status == km::FP3_STALE) ++fp3_stale;
        for (int q = 0; q < 8; ++q) fp3_tphase[q] += r.tphase[q];
        for (int q = 0; q < 3; ++q) fp3_stat[q] += r.pad[q];
        if (r.swaps > 0) {
            std::vector<Rec> tr((size_t)r.swaps);
            KM_CK(cudaMemcpy(tr.data(), f3_trace, tr.size() * sizeof(Rec), cudaMemcpyDeviceToHost));
            for (const Rec& x : tr) last_swaps.push_back(x);
            fp3_tlast = pass_base + (tr.back().c - c0);
            fp3_dirty = true;
        }
        fp3_t = pass_base + a + r.p_end;
        return KM_OK;
    }

    // One pass of Alg.4's scan (or its remainder up to the stop, F2).
    km_status swap_iter_fp3(int32_t* swaps_out, void* td_out) {
        fp1_prepped = false;
        inc_valid = false;
        if (fp3_mode < 0) {
            const char* e = getenv("KM_FASTER");
            fp3_mode = (e && strcmp(e, "batch") == 0) ? 0 : 1;
        }
        if (fp3_mode == 1) return swap_iter_fp3_coop(swaps_out, td_out);
        KM_TRY(fp3_alloc());
        fp3_dirty = true;           // another variant may have changed the cache
        last_swaps.clear();
        if (swaps_out) *swaps_out = 0;
        if (fp3_t - fp3_tlast >= n) { copy_td(td_out); return KM_CONVERGED; }
        const int64_t pass_base = fp3_t - fp3_t % n, pass_end = pass_base + n;
        int64_t wcur = fp3_w0;
        bool first = true;
        int done = 0;
        while (fp3_t < pass_end && fp3_t - fp3_tlast < n) {
            const int64_t hi = std::min(std::min(pass_end, fp3_tlast + n), fp3_t + wcur);
            KM_TRY(fp3_batch(pass_base, fp3_t, hi, first));
            first = false;
            if (h_dec->apply) {
                const int64_t pos = pass_base + h_dec->c;
                Rec r; r.v = h_dec->dtd; r.slot = h_dec->slot; r.c = h_dec->c;
                last_swaps.push_back(r);
                ++done;
                fp3_tlast = pos;
                fp3_t = pos + 1;
                fp3_dirty = true;
                wcur = fp3_w0;
            } else {
                fp3_t = hi;
                wcur = std::min<int64_t>(wcur * 2, fp3_wmax);
            }
        }
        if (swaps_out) *swaps_out = done;
        copy_td(td_out);
        return (fp3_t - fp3_tlast >= n) ? KM_CONVERGED : KM_OK;
    }

    km_status swap_iter_fp3_coop(int32_t* swaps_out, void* td_out) {
        KM_TRY(fp3_alloc());
        KM_TRY(fp3c_alloc());
        fp3_dirty = true;           // another variant may have changed the cache
        last_swaps.clear();
        if (swaps_out) *swaps_out = 0;
        if (fp3_t - fp3_tlast >= n) { copy_td(td_out); return KM_CONVERGED; }
        const int64_t pass_base = fp3_t - fp3_t % n, pass_end = pass_base + n;
        bool first = true;
        km::k_fp3_transpose_mc<T><<<dim3((unsigned)cdiv(n, 32), (unsigned)cdiv(k, 32)), dim3(32, 8), 0, st>>>(
            MC, (int)n, k, f3_mct);
        KM_CKL();
        while (fp3_t < pass_end && fp3_t - fp3_tlast < n) {
            const int64_t hi = std::min(std::min(pass_end, fp3_tlast + n), fp3_t + (int64_t)fp3c_ww - 3);
            const auto h0 = std::chrono::steady_clock::now();
            KM_TRY(fp3_window_coop(pass_base, fp3_t, hi, first));
            fp3_host_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
            first = false;
        }
        if (swaps_out) *swaps_out = (int32_t)last_swaps.size();
        copy_td(td_out);
        const char* ep = getenv("KM_FASTER_PROF");
        if (ep && ep[0] == '1')
            fprintf(stderr, "[fasterpam] pass: swaps %zu windows %lld stale %lld | ms pick %.2f apply %.2f rescan %.2f "
                    "compact %.2f correct %.2f fold %.2f | sum nres %lld m %lld T %lld | window host ms %.2f\n",
                    last_swaps.size(), (long long)fp3_windows, (long long)fp3_stale, fp3_tphase[0] * 1e-6,
                    fp3_tphase[1] * 1e-6, fp3_tphase[2] * 1e-6, fp3_tphase[4] * 1e-6, fp3_tphase[5] * 1e-6,
                    fp3_tphase[6] * 1e-6, fp3_stat[0], fp3_stat[1], fp3_stat[2], fp3_host_ms);
        return (fp3_t - fp3_tlast >= n) ? KM_CONVERGED : KM_OK;
    }

    // ---- incremental FastPAM1 (KM_FASTPAM1_INC; km_fasterpam.cuh GLOBAL mode) ---
    // The complete k-vectors of every candidate (acc[i][c], plus[c]) come from
    // one FastPAM2-mode stream; every iteration then takes Alg.3's best swap
    // over all candidates (key R1) from them and corrects them for the objects
    // whose (nearest, d_n, d_s) changed -- the same swaps as the streaming
    // FastPAM1 (bit-exact on u32), reading the changed rows instead of D.
    bool inc_valid = false;
    int64_t inc_restreams = 0;
    unsigned long long inc_tphase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long inc_stat[3] = {0, 0, 0};
    A *inc_pacc = nullptr, *inc_pplus = nullptr, *inc_pR = nullptr;
    Rec* inc_gpart = nullptr;
    Rec* inc_trace = nullptr;
    int inc_trace_cap = 0;

    km_status inc_alloc() {
        if (inc_pacc) return KM_OK;
        KM_TRY(fp2_alloc());
        KM_TRY(fp3_alloc());
        KM_TRY(fp3c_alloc());
        const int64_t nwarps = (int64_t)fp3c_blocks * km::FP3_WARPS;
        // partials of the GLOBAL correction: G groups x slots x w, for both item
        // shapes (128 columns x FP3_TV slots, 32 columns x FP3_TMAX slots)
        const int64_t Gw = std::min<int64_t>(km::FP3_G, std::max<int64_t>(1, nwarps / cdiv(w, 128)));
        const int64_t Gn = std::min<int64_t>(km::FP3_G, std::max<int64_t>(1, nwarps / cdiv(w, 32)));
        KM_TRY(alloc(&inc_pacc, (size_t)std::max(Gw * km::FP3_TV, Gn * km::FP3_TMAX) * w));
        KM_TRY(alloc(&inc_pplus, (size_t)std::max(Gw, Gn) * w));
        KM_TRY(alloc(&inc_pR, (size_t)km::FP3_G * km::FP3_TMAX));
        KM_TRY(alloc(&inc_gpart, fp3c_blocks));
        inc_trace_cap = 4096;
        KM_TRY(alloc(&inc_trace, inc_trace_cap));
        return KM_OK;
    }

    km_status inc_iters(int32_t max_iters, int32_t* swaps_out, void* td_out, int32_t* iters_out,
                        bool* conv_out) override {
        if (sharded) return fail(KM_EINVAL, "incremental FastPAM1 on a sharded handle");
        if (!ready) return fail(KM_EINVAL, "no medoids: call kmedoids_set_medoids or kmedoids_init_build first");
        KM_TRY(clear_fp1_done());
        KM_TRY(inc_alloc());
        fp1_prepped = false;
        last_swaps.clear();
        int done_iters = 0, done_swaps = 0;
        bool conv = false;
        while (done_iters < max_iters && !conv) {
            if (!inc_valid) {                         // exact k-vectors of the current state
                KM_CK(cudaMemsetAsync(fp2_acc, 0, (size_t)k * w * sizeof(A), st));
                KM_TRY(fp2_eval_local());
                KM_TRY(fp2_finish_profiling());
                km::k_fp3_transpose_mc<T><<<dim3((unsigned)cdiv(n, 32), (unsigned)cdiv(k, 32)), dim3(32, 8), 0, st>>>(
                    MC, (int)n, k, f3_mct);
                KM_CKL();
                inc_valid = true;
            }
            km::Fp3Ctl hc;
            memset(&hc, 0, sizeof(hc));
            hc.first[0] = hc.first[1] = hc.first[2] = INT_MAX;
            *h_f3ctl = hc;
            KM_CK(cudaMemcpyAsync(f3_ctl, h_f3ctl, sizeof(hc), cudaMemcpyHostToDevice, st));
            km::Fp3Args<T, A> g;
            g.D = D; g.ld = ld; g.n = (int)n; g.k = k; g.c0 = c0; g.a = 0; g.ww = w;
            g.lo = 0; g.hi = w; g.L = w;
            g.acc = fp2_acc; g.plus = fp2_plus; g.R = R; g.M = M; g.point_slot = point_slot; g.MC = MC; g.MCt = f3_mct;
            g.near = near; g.sec = sec; g.dn = dn; g.ds = ds; g.td = td; g.dec = dec;
            g.trace = inc_trace; g.trace_cap = inc_trace_cap;
            g.cand_v = f3_v; g.cand_s = f3_s; g.flag = f3_flag; g.old_near = f3_oldnear; g.old_dn = f3_olddn;
            g.old_ds = f3_oldds; g.rescan = f3_rescan; g.blk_cnt = f3_blk; g.chg = f3_chg; g.chg_cap = (int)n;
            g.touched_flag = f3_tflag; g.touched_map = f3_tmap; g.touched = f3_tlist;
            g.part_acc = inc_pacc; g.part_plus = inc_pplus; g.part_R = inc_pR; g.ctl = f3_ctl; g.new_pass = 0;
            g.max_iters = max_iters - done_iters; g.gpart = inc_gpart;
            void* args[] = {&g};
            KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp3_window<T, A, true>, dim3(fp3c_blocks),
                                              dim3(km::FP3_THREADS), args, km::FP3_SMEM, st));
            ++launches;
            KM_CK(cudaMemcpyAsync(h_f3ctl, f3_ctl, sizeof(km::Fp3Ctl), cudaMemcpyDeviceToHost, st));
            KM_TRY(sync_dec());
            const km::Fp3Ctl r = *h_f3ctl;
            if (r.swaps > 0) {
                std::vector<Rec> tr((size_t)std::min(r.swaps, inc_trace_cap));
                KM_CK(cudaMemcpy(tr.data(), inc_trace, tr.size() * sizeof(Rec), cudaMemcpyDeviceToHost));
                for (const Rec& x : tr) last_swaps.push_back(x);
            }
            done_swaps += r.swaps;
            done_iters += r.pad[4];
            conv = r.pad[3] != 0;
            if (r.status == km::FP3_STALE) { inc_valid = false; ++inc_restreams; }   // re-stream next
            for (int q = 0; q < 8; ++q) inc_tphase[q] += r.tphase[q];
            for (int q = 0; q < 3; ++q) inc_stat[q] += r.pad[q];
        }
        const char* ep = getenv("KM_FASTER_PROF");
        if (ep && ep[0] == '1')
            fprintf(stderr, "[fastpam1_inc] iters %d swaps %d restreams %lld | ms pick %.2f apply %.2f rescan %.2f "
                    "compact %.2f correct %.2f fold %.2f | sum nres %lld m %lld T %lld\n", done_iters, done_swaps,
                    (long long)inc_restreams, inc_tphase[0] * 1e-6, inc_tphase[1] * 1e-6, inc_tphase[2] * 1e-6,
                    inc_tphase[4] * 1e-6, inc_tphase[5] * 1e-6, inc_tphase[6] * 1e-6, inc_stat[0], inc_stat[1],
                    inc_stat[2]);
        if (swaps_out) *swaps_out = done_swaps;
        if (iters_out) *iters_out = done_iters;
        if (conv_out) *conv_out = conv;
        copy_td(td_out);
        return conv ? KM_CONVERGED : KM_OK;
    }

    // ---- sharded FastPAM2 ------------------------------------------------------
    // record_send: this rank's k per-slot bests; record_recv: R x k gathered.
    // col_send: the columns of the planned candidates this rank owns
    // (cap x n); col_recv: R x cap x n gathered (rank r's block at r*maxcnt).
    Rec* f2_rec_recv = nullptr;
    T* f2_col_send = nullptr;
    T* f2_col_recv = nullptr;
    int* f2_colidx = nullptr;
    int f2_ranks = 0, f2_maxcnt = 0, f2_cap = 0;
    int* f2_packcols = nullptr;        // [k] the owned candidates packed this iteration
    std::vector<int> f2_order;

    km_status fp2_shard_exchange(int32_t nr, km_fp2_exchange* out) override {
        if (nr < 1) return fail(KM_EINVAL, "nranks must be >= 1");
        KM_TRY(fp2_alloc());
        if (f2_ranks != nr) {
            if (f2_ranks != 0) return fail(KM_ECOMM, "fp2 exchange already sized for %d ranks", f2_ranks);
            f2_ranks = nr;
            KM_TRY(alloc(&f2_rec_recv, (size_t)nr * k));
            KM_TRY(alloc(&f2_colidx, k));
            KM_TRY(alloc(&f2_packcols, k));
            KM_TRY(f2_grow(std::min(k, 32)));
        }
        out->record_send = fp2_best;
        out->record_recv = f2_rec_recv;
        out->record_bytes = (size_t)k * sizeof(Rec);
        out->col_send = f2_col_send;
        out->col_recv = f2_col_recv;
        out->col_bytes_per_column = (size_t)n * sizeof(T);
        out->col_capacity = f2_cap;
        return KM_OK;
    }

    // column exchange buffers for `cap` columns per rank (grown on demand:
    // the plan needs max over ranks of the owned planned candidates, usually
    // far below k; round 1 sized them for k, i.e. R * k * n elements)
    km_status f2_grow(int cap) {
        if (cap <= f2_cap) return KM_OK;
        cap = std::min(k, std::max(cap, 2 * f2_cap));
        KM_CK(cudaStreamSynchronize(st));
        dealloc(f2_col_send);
        dealloc(f2_col_recv);
        f2_col_send = f2_col_recv = nullptr;
        KM_TRY(alloc(&f2_col_send, (size_t)cap * n));
        KM_TRY(alloc(&f2_col_recv, (size_t)f2_ranks * cap * n));
        f2_cap = cap;
        return KM_OK;
    }

    km_status fp2_shard_eval() override {
        if (!ready) return fail(KM_EINVAL, "no medoids set");
        if (!f2_ranks) return fail(KM_ECOMM, "call kmedoids_fp2_shard_exchange first");
        return fp2_eval_local();
    }

    km_status fp2_shard_plan(const int64_t* rcb, int32_t* m_out, int32_t* maxcnt_out) override {
        if (!f2_ranks) return fail(KM_ECOMM, "call kmedoids_fp2_shard_exchange first");
        const int nr = f2_ranks;
        int me = -1;
        for (int r = 0; r < nr; ++r)
            if (rcb[r] == c0 && rcb[r + 1] == c1) me = r;
        if (me < 0) return fail(KM_ECOMM, "rank_col_begin does not contain this handle's columns");
        std::vector<Rec> all((size_t)nr * k);
        A tdh;
        KM_CK(cudaMemcpyAsync(all.data(), f2_rec_recv, all.size() * sizeof(Rec), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaMemcpyAsync(&tdh, td, sizeof(A), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        KM_TRY(fp2_finish_profiling());
        for (int i = 0; i < k; ++i) {                // lexicographic min over ranks, rank order
            Rec b = km::rec_none<A>();
            for (int r = 0; r < nr; ++r)
                if (km::rec_less(all[(size_t)r * k + i], b)) b = all[(size_t)r * k + i];
            h_best[i] = b;
        }
        KM_CK(cudaMemcpyAsync(fp2_best, h_best.data(), k * sizeof(Rec), cudaMemcpyHostToDevice, st));
        f2_order = fp2_order_slots(tdh);
        // distinct candidates in order of first use, grouped by owner rank
        std::vector<std::vector<int>> owned(nr);
        std::vector<int> pos_of(f2_order.size()), own_of(f2_order.size());
        std::vector<std::pair<int, int>> seen;    // (candidate, index in owner list)
        for (size_t r = 0; r < f2_order.size(); ++r) {
            const int c = h_best[f2_order[r]].c;
            int ow = -1;
            for (int q = 0; q < nr; ++q)
                if (c >= rcb[q] && c < rcb[q + 1]) ow = q;
            if (ow < 0) return fail(KM_ECOMM, "candidate %d has no owner", c);
            int pos = -1;
            for (auto& sp : seen)
                if (sp.first == c) pos = sp.second;
            if (pos < 0) {
                pos = (int)owned[ow].size();
                owned[ow].push_back(c);
                seen.push_back({c, pos});
            }
            pos_of[r] = pos;
            own_of[r] = ow;
        }
        int maxcnt = 0;
        for (auto& v : owned) maxcnt = std::max(maxcnt, (int)v.size());
        f2_maxcnt = maxcnt;
        std::vector<int> colidx(f2_order.size());
        for (size_t r = 0; r < f2_order.size(); ++r) colidx[r] = own_of[r] * maxcnt + pos_of[r];
        if (!colidx.empty())
            KM_CK(cudaMemcpyAsync(f2_colidx, colidx.data(), colidx.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        KM_TRY(f2_grow(maxcnt));                     // (the caller re-queries the exchange when it grew)
        if (!owned[me].empty()) {
            KM_CK(cudaMemcpyAsync(f2_packcols, owned[me].data(), owned[me].size() * sizeof(int),
                                  cudaMemcpyHostToDevice, st));
            km::k_gather_cols<T><<<dim3((unsigned)cdiv(n, 256), (unsigned)owned[me].size()), 256, 0, st>>>(
                D, ld, (int)n, c0, f2_packcols, f2_col_send);
            KM_CKL();
        }
        KM_CK(cudaStreamSynchronize(st));
        f2_me = me;
        f2_round = 0;                                // owner-side rounds may follow (km_fp2_owner.cuh)
        if (m_out) *m_out = (int)f2_order.size();
        if (maxcnt_out) *maxcnt_out = maxcnt;
        return KM_OK;
    }

    km_status fp2_shard_apply(int32_t* swaps_out, void* td_out) override {
        f2_round = -1;
        return fp2_sequential(f2_order, f2_col_recv, f2_colidx, swaps_out, td_out);
    }

    // ---- sharded FastPAM2, owner-side rounds (km_fp2_owner.cuh) ---------------
    unsigned char* f2_rsend = nullptr;    // this rank's round buffer (header + column)
    unsigned char* f2_rrecv = nullptr;    // R round buffers, rank order
    size_t f2_rstride = 0;
    int* f2_state = nullptr;              // [2]: next plan position, another round needed
    int f2_round = -1;                    // rounds done in this iteration (-1: no plan)
    int f2_me = -1;
    Dec f2_hd{};                          // the iteration's decision bookkeeping (host)
    int f2_swaps0 = 0;

    km_status fp2_round_buffers(void** send, void** recv, size_t* stride) override {
        if (!f2_ranks) return fail(KM_ECOMM, "call kmedoids_fp2_shard_exchange first");
        if (!f2_rsend) {
            f2_rstride = km::fp2_round_stride<T>(n);
            KM_TRY(alloc(&f2_rsend, f2_rstride));
            KM_TRY(alloc(&f2_rrecv, f2_rstride * (size_t)f2_ranks));
            KM_TRY(alloc(&f2_state, 2));
        }
        if (send) *send = f2_rsend;
        if (recv) *recv = f2_rrecv;
        if (stride) *stride = f2_rstride;
        return KM_OK;
    }

    km_status fp2_round_eval() override {
        if (f2_round < 0) return fail(KM_EINVAL, "no FastPAM2 plan: call kmedoids_fp2_shard_plan first");
        if (f2_order.empty()) return fail(KM_EINVAL, "empty plan (converged): use kmedoids_fp2_shard_apply");
        KM_TRY(fp2_round_buffers(nullptr, nullptr, nullptr));
        if (f2_round == 0) {
            // the iteration's bookkeeping, as fp2_sequential: counted now, its
            // swaps counted from 0 by the apply kernels
            KM_CK(cudaMemcpyAsync(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost, st));
            KM_CK(cudaStreamSynchronize(st));
            f2_hd = *h_dec;
            f2_hd.iters += 1;
            f2_hd.apply = 0;
            f2_swaps0 = f2_hd.swaps;
            f2_hd.swaps = 0;
            KM_CK(cudaMemcpyAsync(dec, &f2_hd, sizeof(Dec), cudaMemcpyHostToDevice, st));
            KM_CK(cudaMemcpyAsync(fp2_order, f2_order.data(), f2_order.size() * sizeof(int), cudaMemcpyHostToDevice, st));
            const int m = (int)f2_order.size();
            const int init[2] = {0, 1};
            KM_CK(cudaMemcpyAsync(fp2_m, &m, sizeof(int), cudaMemcpyHostToDevice, st));
            KM_CK(cudaMemcpyAsync(f2_state, init, sizeof(init), cudaMemcpyHostToDevice, st));
            last_swaps.clear();
        }
        const T* csp = f2_col_send; const int* cip = f2_colidx; int me = f2_me; int mc = std::max(1, f2_maxcnt);
        int nn = (int)n; const int* op = fp2_order; const int* mp = fp2_m; const Rec* bp = fp2_best;
        const int* psp = point_slot; const int* nr = near; const T* dnp = dn; const T* dsp = ds; const A* tdp = td;
        A* pp = fp2_partials; const int* rp = f2_state; int* rcp = rescan_count; unsigned char* outp = f2_rsend;
        void* args[] = {&csp, &cip, &me, &mc, &nn, &op, &mp, &bp, &psp, &nr, &dnp, &dsp, &tdp, &pp, &rp, &rcp, &outp};
        KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp2_owned_eval<T, A>, dim3(fp2_blocks), dim3(256), args, 0, st));
        ++launches;
        return KM_OK;
    }

    km_status fp2_round_apply(int32_t* more_out, int32_t* swaps_out, void* td_out) override {
        if (f2_round < 0 || !f2_rsend) return fail(KM_EINVAL, "no FastPAM2 round: call kmedoids_fp2_round_eval first");
        const unsigned char* rv = f2_rrecv; int nrk = f2_ranks; size_t strd = f2_rstride; int nn = (int)n; int kk = k;
        const int* mp = fp2_m; int* Mp = M; int* psp = point_slot; T* MCp = MC; int* nr = near; int* sc = sec;
        T* dnp = dn; T* dsp = ds; A* tdp = td; Dec* dp = dec; Rec* tr = trace; int tc = trace_cap; int* rsp = rescan;
        int* rcp = rescan_count; int* stp = f2_state;
        void* args[] = {&rv, &nrk, &strd, &nn, &kk, &mp, &Mp, &psp, &MCp, &nr, &sc, &dnp, &dsp, &tdp, &dp, &tr, &tc,
                        &rsp, &rcp, &stp};
        KM_CK(cudaLaunchCooperativeKernel((void*)km::k_fp2_round_apply<T, A>, dim3(fp2_blocks), dim3(256), args, 0,
                                          st));
        ++launches;
        int hs[2];
        KM_CK(cudaMemcpyAsync(hs, f2_state, sizeof(hs), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        ++f2_round;
        if (more_out) *more_out = hs[1];
        if (hs[1]) return KM_OK;
        // the iteration is over: its swaps (the kernels counted them from 0)
        KM_CK(cudaMemcpyAsync(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        const int done = h_dec->swaps;
        last_swaps.resize(std::min(done, trace_cap));
        if (!last_swaps.empty())
            KM_CK(cudaMemcpy(last_swaps.data(), trace, last_swaps.size() * sizeof(Rec), cudaMemcpyDeviceToHost));
        Dec hd = *h_dec;
        hd.swaps = f2_swaps0 + done;
        KM_CK(cudaMemcpyAsync(dec, &hd, sizeof(Dec), cudaMemcpyHostToDevice, st));
        KM_CK(cudaStreamSynchronize(st));
        *h_dec = hd;
        f2_round = -1;
        if (swaps_out) *swaps_out = done;
        copy_td(td_out);
        return KM_OK;
    }

    // ---- NEXT-4 initialisations (km_init.cuh) ----------------------------------
    km_status init_common_alloc(T** w, int** flags) {
        if (!init_w) { KM_TRY(alloc(&init_w, n)); KM_TRY(alloc(&init_flags, n)); }
        KM_CK(cudaMemsetAsync(init_flags, 0, n * sizeof(int), st));
        *w = init_w; *flags = init_flags;
        return KM_OK;
    }
    T* init_w = nullptr;
    int* init_flags = nullptr;
    double* init_u = nullptr;
    int* init_seq = nullptr;
    size_t init_seq_cap = 0;
    T* init_sub = nullptr;
    size_t init_sub_cap = 0;
    int* initl_ctl = nullptr;
    Rec* initl_bmin = nullptr;
    int initl_blocks = 0;
    A* initw_bsum = nullptr;
    int* initw_picks = nullptr;
    int initw_blocks = 0, initw_picks_cap = 0;

    km_status finish_init(int32_t* M_out, void* td_out) {
        std::vector<int32_t> Mh((size_t)k);
        KM_CK(cudaMemcpyAsync(Mh.data(), M, k * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        KM_CK(cudaStreamSynchronize(st));
        KM_TRY(set_medoids(Mh.data()));
        if (M_out) memcpy(M_out, Mh.data(), k * sizeof(int32_t));
        copy_td(td_out);
        return KM_OK;
    }

    km_status init_weighted(const double* u, int32_t* M_out, void* td_out) override {
        KM_TRY(clear_fp1_done());
        if (sharded) return fail(KM_EINVAL, "init_weighted on a sharded handle");
        if (k < 2) return fail(KM_EINVAL, "SWAP needs k >= 2");
        for (int i = 0; i < k; ++i)
            if (!(u[i] >= 0.0 && u[i] < 1.0)) return fail(KM_EINVAL, "u[%d] = %g not in [0, 1)", i, u[i]);
        T* w; int* fl;
        KM_TRY(init_common_alloc(&w, &fl));
        if (!init_u) KM_TRY(alloc(&init_u, k));
        KM_CK(cudaMemcpyAsync(init_u, u, k * sizeof(double), cudaMemcpyHostToDevice, st));
        const char* ew = getenv("KM_INIT_WEIGHTED");       // "block": the single-block kernel
        if (ew && strcmp(ew, "block") == 0) {
            km::k_init_weighted<T, A><<<1, km::INIT_THREADS, 0, st>>>(D, ld, (int)n, k, init_u, M, w, fl);
            KM_CKL();
        } else {
            if (!initw_bsum) {
                int dev = 0, nsm = 0;
                KM_CK(cudaGetDevice(&dev));
                KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                initw_blocks = nsm;
                KM_TRY(alloc(&initw_bsum, initw_blocks));
            }
            if (k > initw_picks_cap) { KM_TRY(alloc(&initw_picks, k)); initw_picks_cap = k; }
            KM_CK(cudaMemsetAsync(initw_picks, 0x7f, (size_t)k * sizeof(int), st));   // > any index
            const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(initw_blocks, cdiv(n, km::INITW_THREADS)));
            const T* Dp = D; int64_t ldv = ld; int nn = (int)n; int kk = k; const double* up = init_u;
            int* Mp = M; T* wp = w; int* fp = fl; A* bp = initw_bsum; int* pp = initw_picks;
            void* args[] = {&Dp, &ldv, &nn, &kk, &up, &Mp, &wp, &fp, &bp, &pp};
            KM_CK(cudaLaunchCooperativeKernel((void*)km::k_init_weighted_coop<T, A>, dim3(nb),
                                              dim3(km::INITW_THREADS), args, 0, st));
        }
        ++launches;
        return finish_init(M_out, td_out);
    }

    km_status init_lab(int32_t s, const int32_t* seq, int32_t* M_out, void* td_out) override {
        KM_TRY(clear_fp1_done());
        if (sharded) return fail(KM_EINVAL, "init_lab on a sharded handle");
        if (k < 2) return fail(KM_EINVAL, "SWAP needs k >= 2");
        if (s < 1 || s > n) return fail(KM_EINVAL, "sample size s=%d must be in [1, n]", s);
        const size_t cnt = (size_t)k * (s + k);
        for (size_t j = 0; j < cnt; ++j)
            if (seq[j] < -1 || seq[j] >= n) return fail(KM_EINVAL, "seq[%zu] = %d out of range", j, seq[j]);
        T* w; int* fl;
        KM_TRY(init_common_alloc(&w, &fl));
        if (cnt + (size_t)s > init_seq_cap) {       // grows only (the handle owns its scratch)
            KM_TRY(alloc(&init_seq, cnt + (size_t)s));
            init_seq_cap = cnt + (size_t)s;
        }
        if ((size_t)s * s > init_sub_cap) {          // the sample's s x s sub-matrix (grows only)
            KM_TRY(alloc(&init_sub, (size_t)s * s));
            init_sub_cap = (size_t)s * s;
        }
        KM_CK(cudaMemcpyAsync(init_seq, seq, cnt * sizeof(int), cudaMemcpyHostToDevice, st));
        const char* el = getenv("KM_INIT_LAB");            // "block": the single-block kernel
        if (el && strcmp(el, "block") == 0) {
            km::k_init_lab<T, A><<<1, km::INIT_THREADS, 0, st>>>(D, ld, (int)n, k, s, init_seq, M, w, fl,
                                                                   init_seq + cnt, init_sub);
            KM_CKL();
        } else {
            if (!initl_ctl) {
                int dev = 0, nsm = 0;
                KM_CK(cudaGetDevice(&dev));
                KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
                initl_blocks = nsm;
                KM_TRY(alloc(&initl_ctl, 2));
                KM_TRY(alloc(&initl_bmin, initl_blocks));
            }
            const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(initl_blocks, cdiv(n, km::INIT_THREADS)));
            const T* Dp = D; int64_t ldv = ld; int nn = (int)n; int kk = k; int ss = s; const int* sq = init_seq;
            int* Mp = M; T* wp = w; int* fp = fl; int* Sp = init_seq + cnt; T* sp = init_sub; int* cp = initl_ctl;
            Rec* bp = initl_bmin;
            void* args[] = {&Dp, &ldv, &nn, &kk, &ss, &sq, &Mp, &wp, &fp, &Sp, &sp, &cp, &bp};
            KM_CK(cudaLaunchCooperativeKernel((void*)km::k_init_lab_coop<T, A>, dim3(nb), dim3(km::INIT_THREADS),
                                              args, 0, st));
        }
        ++launches;
        return finish_init(M_out, td_out);
    }

    // ---- NEXT-3 FastCLARA (reading C1) ------------------------------
    // Per sample: gather the s x s sub-matrix, PAM on it (BUILD + SWAP with
    // the requested variant, one nested handle reused for every sample), map
    // the medoids back and evaluate TD over ALL n objects with this handle's
    // cache kernels; keep the smallest (TD, sample).  Leaves this handle on
    // the winning medoids.
    // The samples are independent: up to CLARA_CONC of them run concurrently,
    // each on its own CUDA stream with its own nested handle and sub-matrix,
    // driven by its own host thread (the GPU overlaps the small, launch-bound
    // sub-problems).  The TD over all objects is then evaluated per sample on
    // this handle, in sample order.
    static constexpr int CLARA_CONC = 8;
    struct ClaraSlot {
        T* buf = nullptr;
        int* idx = nullptr;
        int* med = nullptr;                 // the sample's medoids as object indices
        A* part = nullptr;                  // TD block sums
        A* tdv = nullptr;
        int* h_med = nullptr;               // pinned: the sample's result
        A* h_td = nullptr;
        cudaEvent_t fin = nullptr;          // recorded behind the sample's TD pass
        cudaStream_t stream = nullptr;
        std::unique_ptr<Impl<T>> sub;
    };
    std::vector<ClaraSlot> clara_slots;
    int64_t clara_s = 0;

    km_status clara(int32_t ns, int32_t s, const int32_t* samples, km_variant v, int32_t* M_out, void* td_out,
                    int32_t* best_out) override {
        if (sharded) return fail(KM_EINVAL, "clara on a sharded handle");
        if (k < 2) return fail(KM_EINVAL, "CLARA needs k >= 2");
        if (ns < 1) return fail(KM_EINVAL, "nsamples must be >= 1");
        if (s <= k || s > n) return fail(KM_EINVAL, "sample size s=%d must satisfy k < s <= n", s);
        if (s > 65535) return fail(KM_EINVAL, "sample size s=%d exceeds 65535 (grid rows of the gather)", s);
        if (v != KM_FASTPAM1 && v != KM_FASTPAM2 && v != KM_FASTERPAM) return fail(KM_EINVAL, "unknown variant");
        std::vector<char> seen((size_t)n, 0);
        for (int j = 0; j < ns; ++j) {
            const int32_t* S = samples + (size_t)j * s;
            for (int a = 0; a < s; ++a) {
                if (S[a] < 0 || S[a] >= n) return fail(KM_EINVAL, "sample %d: index %d out of range", j, S[a]);
                if (seen[S[a]]) return fail(KM_EINVAL, "sample %d: duplicate index %d", j, S[a]);
                seen[S[a]] = 1;
            }
            for (int a = 0; a < s; ++a) seen[S[a]] = 0;
        }
        const int64_t lds = cdiv(s, 4) * 4;
        if (clara_s != 0 && clara_s != s) return fail(KM_EINVAL, "this handle already ran CLARA with s=%lld", (long long)clara_s);
        clara_s = s;
        const int conc = std::min(ns, CLARA_CONC);
        KM_CK(cudaStreamSynchronize(st));              // D and the cache are settled before other streams read D
        while ((int)clara_slots.size() < conc) {
            ClaraSlot sl;
            KM_TRY(alloc(&sl.buf, (size_t)s * lds));
            KM_TRY(alloc(&sl.idx, s));
            KM_TRY(alloc(&sl.med, k));
            KM_TRY(alloc(&sl.part, cdiv(n, 256)));
            KM_TRY(alloc(&sl.tdv, 1));
            KM_CK(cudaMallocHost(&sl.h_med, (size_t)k * sizeof(int)));
            KM_CK(cudaMallocHost(&sl.h_td, sizeof(A)));
            KM_CK(cudaEventCreateWithFlags(&sl.fin, cudaEventDisableTiming));
            KM_CK(cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking));
            KM_CK(cudaMemsetAsync(sl.buf, 0, (size_t)s * lds * sizeof(T), sl.stream));
            sl.sub.reset(new Impl<T>());
            KM_TRY(sl.sub->init(sl.buf, s, lds, 0, s, k, sl.stream));
            clara_slots.push_back(std::move(sl));
        }
        std::vector<std::vector<int32_t>> Mg((size_t)ns, std::vector<int32_t>((size_t)k));
        std::vector<km_status> res((size_t)ns, KM_OK);
        std::vector<std::string> errs((size_t)ns);
        auto worker = [&](int slot) {
            ClaraSlot& sl = clara_slots[slot];
            Impl<T>& sub = *sl.sub;
            for (int j = slot; j < ns; j += conc) {
                const int32_t* S = samples + (size_t)j * s;
                km_status r = KM_OK;
                if (cudaMemcpyAsync(sl.idx, S, s * sizeof(int32_t), cudaMemcpyHostToDevice, sl.stream) != cudaSuccess)
                    r = KM_ECUDA;
                if (r == KM_OK) {
                    km::k_gather_submatrix<T><<<dim3((unsigned)cdiv(s, 256), (unsigned)s), 256, 0, sl.stream>>>(
                        D, ld, sl.idx, s, sl.buf, lds);
                    if (cudaGetLastError() != cudaSuccess) r = KM_ECUDA;
                }
                if (r == KM_OK) r = sub.init_build(nullptr, nullptr);
                for (int it = 0; r == KM_OK && it < 2000; ++it) {
                    const km_status q = sub.swap_iter(v, nullptr, nullptr);
                    if (q == KM_CONVERGED) break;
                    if (q != KM_OK) r = q;
                }
                std::vector<int32_t> Mloc((size_t)k);
                if (r == KM_OK) r = sub.get_state(Mloc.data(), nullptr, nullptr, nullptr, nullptr);
                if (r == KM_OK)
                    for (int i = 0; i < k; ++i) Mg[j][i] = S[Mloc[i]];
                res[j] = r;
                if (r != KM_OK) errs[j] = g_err;
            }
        };
        std::vector<A> tds((size_t)ns);
        const int tdb = (int)cdiv(n, 256);
        if (v == KM_FASTPAM1) {
            // ONE host thread drives the samples, `conc` at a time, each on
            // its slot's stream (as kmedoids_clara_points): sub-matrix gather,
            // BUILD and the first two iterations enqueued at once, finished
            // iterations collected by event queries and the next queued,
            // then the medoids as object indices and their TD over all n
            // objects (Eq. eqn:td) into pinned memory behind the converging
            // pass.
            std::vector<int> cur((size_t)conc, -1), phase((size_t)conc, 0);
            int nextj = 0, left = ns, rj = -1;
            km_status r = KM_OK;
            while (left > 0 && r == KM_OK) {
                bool progress = false;
                for (int si = 0; si < conc && r == KM_OK; ++si) {
                    ClaraSlot& sl = clara_slots[si];
                    Impl<T>& sub = *sl.sub;
                    const int j = cur[si];
                    auto ck = [&](cudaError_t e, const char* what) {
                        if (r == KM_OK && e != cudaSuccess) r = fail(KM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
                    };
                    if (j < 0) {
                        if (nextj >= ns) continue;
                        const int jj = nextj++;
                        cur[si] = jj;
                        rj = jj;
                        ck(cudaMemcpyAsync(sl.idx, samples + (size_t)jj * s, s * sizeof(int32_t), cudaMemcpyHostToDevice,
                                           sl.stream), "sample indices");
                        if (r == KM_OK) {
                            km::k_gather_submatrix<T><<<dim3((unsigned)cdiv(s, 256), (unsigned)s), 256, 0, sl.stream>>>(
                                D, ld, sl.idx, s, sl.buf, lds);
                            ck(cudaGetLastError(), "sample gather");
                        }
                        sub.build_async = true;
                        if (r == KM_OK) r = sub.init_build(nullptr, nullptr);
                        sub.build_async = false;
                        if (r == KM_OK) r = sub.fp1_async_begin(2000);
                        phase[si] = 1;
                        progress = true;
                    } else if (phase[si] == 1) {
                        bool fin = false;
                        rj = j;
                        r = sub.fp1_async_poll(&fin);
                        if (r != KM_OK || !fin) continue;
                        km::k_map_sample_medoids<<<1, 256, 0, sl.stream>>>(sub.M, sl.idx, k, sl.med);
                        km::k_td_cols<T, A><<<tdb, 256, (size_t)k * sizeof(int), sl.stream>>>(D, ld, (int)n, sl.med, k,
                                                                                               sl.part);
                        km::k_sum_partials<A><<<1, 32, 0, sl.stream>>>(sl.part, tdb, sl.tdv);
                        ck(cudaGetLastError(), "sample TD");
                        ck(cudaMemcpyAsync(sl.h_med, sl.med, k * sizeof(int32_t), cudaMemcpyDeviceToHost, sl.stream), "medoids");
                        ck(cudaMemcpyAsync(sl.h_td, sl.tdv, sizeof(A), cudaMemcpyDeviceToHost, sl.stream), "TD");
                        ck(cudaEventRecord(sl.fin, sl.stream), "sample event");
                        phase[si] = 2;
                        progress = true;
                    } else {
                        rj = j;
                        const cudaError_t q = cudaEventQuery(sl.fin);
                        if (q == cudaErrorNotReady) continue;
                        ck(q, "sample");
                        if (r != KM_OK) continue;
                        memcpy(Mg[j].data(), sl.h_med, k * sizeof(int32_t));
                        tds[j] = *sl.h_td;
                        cur[si] = -1;
                        --left;
                        progress = true;
                    }
                }
                if (!progress) std::this_thread::yield();
            }
            if (r != KM_OK) {
                const std::string msg = g_err;
                for (int si = 0; si < conc; ++si) {
                    cudaStreamSynchronize(clara_slots[si].stream);
                    clara_slots[si].sub->fp1_ring_polled = false;
                }
                cudaGetLastError();
                return fail(r, "CLARA sample %d: %s", rj, msg.c_str());
            }
        } else {
            // FastPAM2 / FasterPAM iterations wait on the host inside
            // swap_iter: one worker thread per slot keeps the samples
            // concurrent; the TD of each sample's medoids by the same pass
            std::vector<std::thread> th;
            for (int t = 1; t < conc; ++t) th.emplace_back(worker, t);
            worker(0);
            for (auto& x : th) x.join();
            for (int j = 0; j < ns; ++j)
                if (res[j] != KM_OK) return fail(res[j], "CLARA sample %d: %s", j, errs[j].c_str());
            ClaraSlot& sl = clara_slots[0];
            for (int j = 0; j < ns; ++j) {
                KM_CK(cudaMemcpyAsync(sl.med, Mg[j].data(), k * sizeof(int32_t), cudaMemcpyHostToDevice, sl.stream));
                km::k_td_cols<T, A><<<tdb, 256, (size_t)k * sizeof(int), sl.stream>>>(D, ld, (int)n, sl.med, k, sl.part);
                km::k_sum_partials<A><<<1, 32, 0, sl.stream>>>(sl.part, tdb, sl.tdv);
                KM_CKL();
                KM_CK(cudaMemcpyAsync(sl.h_td, sl.tdv, sizeof(A), cudaMemcpyDeviceToHost, sl.stream));
                KM_CK(cudaStreamSynchronize(sl.stream));
                tds[j] = *sl.h_td;
            }
        }
        for (auto& sl : clara_slots) { launches += sl.sub->launches + 1; sl.sub->launches = 0; }
        int best_j = 0;
        for (int j = 1; j < ns; ++j)
            if (tds[j] < tds[best_j]) best_j = j;       // smallest (TD, sample index)
        KM_TRY(set_medoids(Mg[best_j].data()));
        if (M_out) memcpy(M_out, Mg[best_j].data(), k * sizeof(int32_t));
        if (best_out) *best_out = best_j;
        copy_td(td_out);
        return KM_OK;
    }

    // ---- BUILD ---------------------------------------------------------------
    template <int MODE>
    km_status launch_build_tma() {
        using C = km::SegCfg<T, SG_NC, SG_RB, SG_S>;
        auto kern = km::k_build_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB, MODE>;
        if (!build_attr_set) KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        dim3 g((unsigned)cdiv(w, C::COLS), Pbt);
        kern<<<g, C::THREADS, C::SMEM, st>>>(D, ld, w, wpad, (int)n, Pbt, dn, b_out);
        KM_CKL();
        km::k_build_combine<T, A, MODE><<<ncomb, 128, 0, st>>>(D, ld, w, c0, Pbt, b_out, point_slot, partials,
                                                                counters, rec_local);
        KM_CKL();
        return KM_OK;
    }

    km_status build_eval(int32_t step) override {
        if (step < 0 || step >= k) return fail(KM_EINVAL, "build step %d out of range", step);
        if (step == 0) {
            // a (re)started BUILD: no medoids yet, so the step-0 pass masks
            // nothing (a previous run's medoids must not be excluded)
            KM_CK(cudaMemsetAsync(point_slot, 0xff, n * sizeof(int), st));
            ready = false;
            build_step = 0;
        }
        {                                          // the phase-API BUILD is incremental too (own slab's gains)
            KM_TRY(bd_init());
            if (bd_mode == 1 && step >= 1) return bd_eval(step);
        }
        return step == 0 ? launch_build_tma<0>() : launch_build_tma<1>();
    }

    km_status build_finish() {
        if (k >= 2) KM_TRY(assign_full_and_td());
        KM_TRY(reset_counters());
        build_finish_host();
        return KM_OK;
    }
    void build_finish_host() {
        if (k >= 2) {
            ready = true;
            fp3_reset();
            fp1_prepped = false;
            inc_valid = false;
        }
    }

    // ---- incremental BUILD (km_build_delta.cuh; KM_BUILD=full recomputes every step)
    int bd_mode = -1;               // 1: incremental gains, 0: a full pass per step
    A* bd_gain = nullptr;
    T *bd_dnold = nullptr, *bd_lold = nullptr, *bd_lnew = nullptr;
    int *bd_flag = nullptr, *bd_cnt = nullptr, *bd_off = nullptr, *bd_lo = nullptr, *bd_m = nullptr;
    int bd_B = 1, bd_chunk = 1;

    km_status bd_alloc() {
        if (bd_gain) return KM_OK;
        bd_B = (int)std::min<int64_t>(1024, cdiv(n, km::BD_CHUNK_THREADS));
        bd_chunk = (int)cdiv(n, bd_B);
        KM_TRY(alloc(&bd_gain, w));
        KM_TRY(alloc(&bd_dnold, n));
        KM_TRY(alloc(&bd_lold, n));
        KM_TRY(alloc(&bd_lnew, n));
        KM_TRY(alloc(&bd_flag, n));
        KM_TRY(alloc(&bd_lo, n));
        KM_TRY(alloc(&bd_cnt, bd_B));
        KM_TRY(alloc(&bd_off, bd_B));
        KM_TRY(alloc(&bd_m, 1));
        return KM_OK;
    }

    // step >= 1 gains into bd_gain and the best record into rec_local:
    // a full pass (step 1) or the delta pass over the objects changed by the
    // previous step
    km_status bd_eval(int step, bool fuse_select = false) {
        using C = km::SegCfg<T, SG_NC, SG_RB, SG_S>;
        if (step == 1) {
            auto kern = km::k_build_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB, 1>;
            if (!build_attr_set) KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            dim3 g((unsigned)cdiv(w, C::COLS), Pbt);
            kern<<<g, C::THREADS, C::SMEM, st>>>(D, ld, w, wpad, (int)n, Pbt, dn, b_out);
        } else {
            auto kern = km::k_build_delta_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB>;
            if (!build_attr_set) KM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            dim3 g((unsigned)cdiv(w, C::COLS), Pbt);
            kern<<<g, C::THREADS, C::SMEM, st>>>(D, ld, w, wpad, Pbt, bd_m, bd_lo, bd_lold, bd_lnew, b_out);
        }
        KM_CKL();
        ++launches;
        // (the delta stream ran bd_parts(m, Pbt) parts; fused: the last block
        // also takes the step, as k_build_select)
        km::k_build_gain_combine<A><<<ncomb, 128, 0, st>>>(w, c0, Pbt, b_out, step == 1 ? 0 : 1, bd_gain, point_slot,
                                                            partials, counters, rec_local, step == 1 ? nullptr : bd_m,
                                                            fuse_select ? step : -1, td, M, dec);
        KM_CKL();
        ++launches;
        return KM_OK;
    }

    km_status bd_init() {
        if (bd_mode < 0) {
            const char* e = getenv("KM_BUILD");
            bd_mode = (e && (strcmp(e, "full") == 0 || strcmp(e, "ldg") == 0)) ? 0 : 1;
        }
        if (bd_mode == 1) KM_TRY(bd_alloc());
        return KM_OK;
    }

    // changed-object list of the step just applied (its column is in MC)
    int bd_coop = -1;               // 1: k_build_changed (cooperative) fits, 0: the three kernels
    km_status bd_changed_list(int from_mc) {
        if (bd_coop < 0) {
            int dev = 0, per_sm = 0, nsm = 0;
            KM_CK(cudaGetDevice(&dev));
            KM_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            KM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, km::k_build_changed<T, A>, km::BD_CHUNK_THREADS, 0));
            bd_coop = (int64_t)per_sm * nsm >= bd_B ? 1 : 0;
            if (const char* e = getenv("KM_BUILD_COOP")) bd_coop = bd_coop && e[0] != '0';   // measurement override
        }
        if (!from_mc && bd_coop) {
            const T* Dp = D; int64_t ldv = ld; int nn = (int)n; int64_t cbg = c0; const Dec* dp = dec; T* MCp = MC;
            const int* psp = point_slot; T* dnp = dn; T* dop = bd_dnold; int* fp = bd_flag; int ch = bd_chunk;
            int* cp = bd_cnt; int* lo = bd_lo; T* lold = bd_lold; T* lnew = bd_lnew; int* mp = bd_m;
            void* args[] = {&Dp, &ldv, &nn, &cbg, &dp, &MCp, &psp, &dnp, &dop, &fp, &ch, &cp, &lo, &lold, &lnew, &mp};
            KM_CK(cudaLaunchCooperativeKernel((void*)km::k_build_changed<T, A>, dim3(bd_B), dim3(km::BD_CHUNK_THREADS),
                                              args, 0, st));
            ++launches;
            return KM_OK;
        }
        km::k_build_dn_delta<T, A><<<bd_B, km::BD_CHUNK_THREADS, 0, st>>>(
            D, ld, (int)n, c0, dec, MC, point_slot, dn, bd_dnold, bd_flag, bd_chunk, bd_cnt, from_mc);
        KM_CKL();
        km::k_chunk_scan<<<1, 1024, 0, st>>>(bd_cnt, bd_B, bd_off, bd_m);
        KM_CKL();
        km::k_changed_scatter<T><<<bd_B, km::BD_CHUNK_THREADS, 0, st>>>(
            (int)n, bd_flag, bd_dnold, dn, bd_chunk, bd_off, bd_lo, bd_lold, bd_lnew);
        KM_CKL();
        launches += 3;
        return KM_OK;
    }

    // The k BUILD steps are ~6 small launches each with no host round trip;
    // they are captured once into a CUDA graph (pointers are fixed per handle,
    // so e.g. every CLARA sample of a nested handle replays the same graph).
    // KM_BUILD_GRAPH=0 launches them directly.
    cudaGraphExec_t build_exec = nullptr;
    int build_graph = -1;
    km_status init_build(int32_t* M_out, void* td_out) override {
        KM_TRY(clear_fp1_done());
        if (sharded) return fail(KM_EINVAL, "init_build on a sharded handle; use kmedoids_build_* phases");
        KM_TRY(bd_init());
        if (build_graph < 0) {
            const char* e = getenv("KM_BUILD_GRAPH");
            build_graph = (e && e[0] == '0') ? 0 : 1;
        }
        // a graph pays off only when replayed (capture + instantiate cost about
        // one direct BUILD): capture on the second BUILD of this handle
        const bool use_g = build_graph == 1 && (build_exec || build_calls >= 1);
        ++build_calls;
        if (use_g && !build_exec) {
            // kernel attributes are set outside the capture
            using C = km::SegCfg<T, SG_NC, SG_RB, SG_S>;
            KM_CK(cudaFuncSetAttribute(km::k_build_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB, 0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            KM_CK(cudaFuncSetAttribute(km::k_build_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            KM_CK(cudaFuncSetAttribute(km::k_build_delta_tma<T, A, SG_NC, SG_RB, SG_S, SG_MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
            build_attr_set = true;
            if (!cap_st) KM_CK(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
            cudaStream_t user_st = st;
            st = cap_st;
            const int64_t l0 = launches;
            cudaError_t be = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            km_status cs = KM_ECUDA;
            if (be == cudaSuccess) {
                capturing = true;
                cs = build_steps();
                capturing = false;
            }
            cudaGraph_t g = nullptr;
            cudaError_t ce = be == cudaSuccess ? cudaStreamEndCapture(st, &g) : be;
            st = user_st;
            bool ok = cs == KM_OK && ce == cudaSuccess;
            if (ok && cudaGraphInstantiate(&build_exec, g, 0) != cudaSuccess) { build_exec = nullptr; ok = false; }
            if (g) cudaGraphDestroy(g);
            build_graph_kernels = launches - l0;
            launches = l0;
            if (!ok) {
                cudaGetLastError();
                fprintf(stderr, "[kmedoids] BUILD graph unavailable (%s); launching directly\n", cudaGetErrorString(ce));
                build_graph = 0;
            }
        }
        if (use_g && build_graph == 1) {
            KM_CK(cudaGraphLaunch(build_exec, st));
            launches += build_graph_kernels;
        } else {
            KM_TRY(build_steps());
        }
        build_finish_host();                     // host-side state (not part of a graph replay)
        if (build_async && !M_out && !td_out) return KM_OK;   // stream-ordered (CLARA's single-thread driver)
        KM_CK(cudaStreamSynchronize(st));
        if (M_out) KM_CK(cudaMemcpy(M_out, M, k * sizeof(int32_t), cudaMemcpyDeviceToHost));
        copy_td(td_out);
        return KM_OK;
    }
    bool build_async = false;               // init_build without the closing host wait (no outputs requested)
    bool build_attr_set = false;
    int64_t build_graph_kernels = 0;
    int build_calls = 0;

    // the k steps of Alg.1 and the cache of the result, enqueued on st
    km_status build_steps() {
        KM_CK(cudaMemsetAsync(point_slot, 0xff, n * sizeof(int), st));
        ready = false;
        const int nb = (int)cdiv(n, 256);
        for (int step = 0; step < k; ++step) {
            if (bd_mode == 1 && step >= 1) {
                KM_TRY(bd_eval(step, true));             // the combine's last block takes the step
            } else {
                KM_TRY(build_eval(step));
                km::k_build_select<A><<<1, 1, 0, st>>>(rec_local, 1, step, td, M, point_slot, dec);
                KM_CKL();
            }
            if (bd_mode == 1 && step >= 1) {
                if (step + 1 < k) {
                    KM_TRY(bd_changed_list(0));
                } else {                                 // last step: only MC is needed
                    km::k_gather_decided_col<T, A><<<nb, 256, 0, st>>>(D, ld, (int)n, c0, c1, dec, MC, nullptr);
                    KM_CKL();
                }
            } else {
                km::k_gather_decided_col<T, A><<<nb, 256, 0, st>>>(D, ld, (int)n, c0, c1, dec, MC, nullptr);
                KM_CKL();
                km::k_build_dn<T, A><<<nb, 256, 0, st>>>(MC, (int)n, dec, point_slot, dn);
                KM_CKL();
            }
        }
        KM_TRY(build_finish());
        return KM_OK;
    }

    // FastPAM2 (reading R6 steps 2-5) of the last iteration: per-slot best
    // (v_i, c_i) (c_i = -1: no candidate) and the improving slots in the
    // order the sequential phase visited them.
    km_status fp2_last_plan(void* v, int32_t* c, int32_t* order, int32_t* m) override {
        if (!fp2_best) return fail(KM_EINVAL, "no FastPAM2 iteration has run on this handle");
        std::vector<Rec> b((size_t)k);
        int mm = 0;
        KM_CK(cudaStreamSynchronize(st));
        KM_CK(cudaMemcpy(b.data(), fp2_best, k * sizeof(Rec), cudaMemcpyDeviceToHost));
        KM_CK(cudaMemcpy(&mm, fp2_m, sizeof(int), cudaMemcpyDeviceToHost));
        if (order && mm > 0) KM_CK(cudaMemcpy(order, fp2_order, (size_t)mm * sizeof(int), cudaMemcpyDeviceToHost));
        for (int i = 0; i < k; ++i) {
            const bool none = b[i].slot == INT_MAX;
            if (v) static_cast<A*>(v)[i] = none ? (A)0 : b[i].v;
            if (c) c[i] = none ? -1 : b[i].c;
        }
        if (m) *m = mm;
        return KM_OK;
    }

    km_status last_swaps_out(int32_t* slots, int32_t* cands, void* dtds, int32_t cap, int32_t* count) override {
        const int m = (int)last_swaps.size();
        if (count) *count = m;
        for (int j = 0; j < m && j < cap; ++j) {
            if (slots) slots[j] = last_swaps[j].slot;
            if (cands) cands[j] = last_swaps[j].c;
            if (dtds) memcpy((char*)dtds + j * sizeof(A), &last_swaps[j].v, sizeof(A));
        }
        return KM_OK;
    }

    // ---- state ---------------------------------------------------------------
    km_status get_state(int32_t* Mo, int32_t* asg, void* td_out, int32_t* it, int32_t* sw) override {
        KM_CK(cudaStreamSynchronize(st));
        if (Mo) KM_CK(cudaMemcpy(Mo, M, k * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (asg) KM_CK(cudaMemcpy(asg, near, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        copy_td(td_out);
        KM_CK(cudaMemcpy(h_dec, dec, sizeof(Dec), cudaMemcpyDeviceToHost));
        if (it) *it = h_dec->iters;
        if (sw) *sw = h_dec->swaps;
        return KM_OK;
    }

    km_status get_cache(int32_t* nr, int32_t* sc, void* dno, void* dso) override {
        KM_CK(cudaStreamSynchronize(st));
        if (nr) KM_CK(cudaMemcpy(nr, near, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (sc) KM_CK(cudaMemcpy(sc, sec, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (dno) KM_CK(cudaMemcpy(dno, dn, n * sizeof(T), cudaMemcpyDeviceToHost));
        if (dso) KM_CK(cudaMemcpy(dso, ds, n * sizeof(T), cudaMemcpyDeviceToHost));
        return KM_OK;
    }

    km_status eval_candidates(void* vo, int32_t* so) override {
        if (!ready) return fail(KM_EINVAL, "no medoids set");
        KM_TRY(eval_local());
        KM_CK(cudaStreamSynchronize(st));
        if (vo) KM_CK(cudaMemcpy(vo, cand_v, (size_t)w * sizeof(A), cudaMemcpyDeviceToHost));
        if (so) KM_CK(cudaMemcpy(so, cand_slot, (size_t)w * sizeof(int32_t), cudaMemcpyDeviceToHost));
        pending_prof = false;
        return KM_OK;
    }

    // ---- sharded phases --------------------------------------------------------
    km_status shard_exchange(int32_t nr, km_exchange* out) override {
        if (nr < 1) return fail(KM_EINVAL, "nranks must be >= 1");
        if (!rec_recv || nr != nranks) {
            nranks = nr;
            KM_TRY(alloc(&rec_recv, nr));
        }
        out->record_send = rec_local;
        out->record_recv = rec_recv;
        out->record_bytes = sizeof(Rec);
        out->column = colbuf;
        out->column_bytes = (size_t)n * sizeof(T);
        return KM_OK;
    }

    km_status shard_set_medoids(const int32_t* Mh, const void* cols) override {
        if (k < 2) return fail(KM_EINVAL, "SWAP needs k >= 2");
        KM_TRY(set_point_slots(Mh));
        KM_CK(cudaMemcpyAsync(MC, cols, (size_t)k * n * sizeof(T), cudaMemcpyDeviceToDevice, st));
        KM_TRY(assign_full_and_td());
        KM_TRY(reset_counters());
        KM_TRY(sh_reset());
        ready = true;
        fp3_reset();
        fp1_prepped = false;
        inc_valid = false;
        return KM_OK;
    }

    km_status shard_eval() override {
        if (!ready) return fail(KM_EINVAL, "no medoids set");
        return eval_local();
    }

    static int owner_of(const int64_t* rcb, int nr, int64_t c) {
        for (int r = 0; r < nr; ++r)
            if (c >= rcb[r] && c < rcb[r + 1]) return r;
        return -1;
    }

    km_status shard_select(const int64_t* rcb, int32_t* found, int32_t* slot, int32_t* cand, int32_t* owner,
                           void* dtd) override {
        if (!rec_recv) return fail(KM_ECOMM, "call kmedoids_shard_exchange first");
        km::k_select<A><<<1, 1, 0, st>>>(rec_recv, nranks, td, M, point_slot, dec, rescan_count);
        KM_CKL();
        KM_TRY(sync_dec());
        if (found) *found = h_dec->apply;
        if (slot) *slot = h_dec->slot;
        if (cand) *cand = h_dec->c;
        if (owner) *owner = h_dec->apply ? owner_of(rcb, nranks, h_dec->c) : -1;
        if (dtd) memcpy(dtd, &h_dec->dtd, sizeof(A));
        return h_dec->apply ? KM_OK : KM_CONVERGED;
    }

    km_status shard_pack_column(int32_t cand) override {
        if (cand < c0 || cand >= c1) return fail(KM_ECOMM, "candidate %d is not in this rank's columns", cand);
        const int nb = (int)cdiv(n, 256);
        km::k_gather_col<T><<<nb, 256, 0, st>>>(D, ld, (int)n, c0, cand, colbuf);
        KM_CKL();
        KM_CK(cudaStreamSynchronize(st));
        return KM_OK;
    }

    km_status shard_apply() override {
        const int nb = (int)cdiv(n, 256);
        km::k_column_to_mc<T, A><<<nb, 256, 0, st>>>(colbuf, (int)n, dec, MC);
        KM_CKL();
        KM_TRY(assign_incremental());
        KM_CK(cudaStreamSynchronize(st));
        return KM_OK;
    }

    // ---- device-decided sharded iteration (no host round trip) ---------------
    using SStat = km::ShardStatus<A>;
    SStat* sh_status = nullptr;      // device
    SStat* sh_mirror = nullptr;      // pinned host
    Rec* sh_trace = nullptr;
    int sh_trace_cap = 0;
    int sh_calls = 0;                              // shard_decide calls enqueued since the reset
    cudaEvent_t sh_ev[2] = {nullptr, nullptr};   // recorded by alternate shard_apply_async calls
    int sh_ev_last = -1;                          // index of the most recent record (-1: none)
    int sh_ev_count = 0;
    km_status sh_alloc() {
        if (sh_status) return KM_OK;
        KM_TRY(alloc(&sh_status, 1));
        KM_CK(cudaMallocHost((void**)&sh_mirror, km::SHARD_MIRRORS * sizeof(SStat)));
        sh_trace_cap = 4096;
        KM_TRY(alloc(&sh_trace, sh_trace_cap));
        for (auto& e : sh_ev) KM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        return KM_OK;
    }
    // a new run starts at every set_medoids / BUILD: status zeroed (counted in
    // the stream order, before the first decide)
    km_status sh_reset() {
        KM_TRY(sh_alloc());
        SStat z{};
        KM_CK(cudaMemcpyAsync(sh_status, &z, sizeof(SStat), cudaMemcpyHostToDevice, st));
        KM_CK(cudaStreamSynchronize(st));
        for (int i = 0; i < km::SHARD_MIRRORS; ++i) sh_mirror[i] = z;
        sh_ev_last = -1;
        sh_ev_count = 0;
        sh_calls = 0;
        return KM_OK;
    }
    km_status shard_decide() override {
        if (!rec_recv) return fail(KM_ECOMM, "call kmedoids_shard_exchange first");
        prof_ring_mode = true;           // later evals of this handle time through the event ring
        if (!sh_status) KM_TRY(sh_reset());
        km::k_shard_decide<A><<<1, 1, 0, st>>>(rec_recv, nranks, td, M, point_slot, dec, rescan_count, sh_status,
                                              sh_mirror, sh_trace, sh_trace_cap);
        KM_CKL();
        ++sh_calls;
        km::k_shard_pack_decided<T, A><<<(unsigned)cdiv(n, 256), 256, 0, st>>>(D, ld, (int)n, c0, c1, dec, colbuf);
        KM_CKL();
        launches += 2;
        return KM_OK;
    }
    km_status shard_apply_async() override {
        const int nb = (int)cdiv(n, 256);
        km::k_column_to_mc<T, A><<<nb, 256, 0, st>>>(colbuf, (int)n, dec, MC);
        KM_CKL();
        KM_TRY(assign_incremental());
        sh_ev_last = sh_ev_last < 0 ? 0 : sh_ev_last ^ 1;
        KM_CK(cudaEventRecord(sh_ev[sh_ev_last], st));
        ++sh_ev_count;
        return KM_OK;
    }
    // After iterations the host did not enqueue itself (replays of a CUDA
    // graph that captured eval / decide / apply): wait for the stream, take
    // the decide count from the device status, forget the event ring.
    km_status shard_resync(int32_t* calls) override {
        if (!sh_status) KM_TRY(sh_reset());
        KM_CK(cudaStreamSynchronize(st));
        SStat m{};
        KM_CK(cudaMemcpy(&m, sh_status, sizeof(SStat), cudaMemcpyDeviceToHost));
        sh_calls = m.calls;
        sh_ev_last = -1;
        sh_ev_count = 0;
        if (calls) *calls = m.calls;
        return KM_OK;
    }
    // wait: 0 = read the mirror as it is, 1 = after all enqueued work, 2 =
    // after the iteration BEFORE the most recently enqueued one (so the host
    // can keep one iteration queued ahead of the one it inspects)
    km_status shard_status(int32_t wait, int32_t* conv, int32_t* iters, int32_t* swaps, void* tdo) override {
        if (!sh_status) KM_TRY(sh_reset());
        // the status after decide call `which` (1-based; 0 = the reset state)
        int which = sh_calls;
        if (wait == 1) KM_CK(cudaStreamSynchronize(st));
        else if (wait == 2) {
            which = sh_calls - 1;
            if (sh_ev_count >= 2) KM_CK(cudaEventSynchronize(sh_ev[sh_ev_last ^ 1]));
            else KM_CK(cudaStreamSynchronize(st));
        }
        SStat m{};
        if (which > 0) m = sh_mirror[(which - 1) % km::SHARD_MIRRORS];
        if (conv) *conv = m.conv;
        if (iters) *iters = m.iters;
        if (swaps) *swaps = m.swaps;
        if (tdo) memcpy(tdo, &m.td, sizeof(A));
        return KM_OK;
    }
    km_status shard_trace(int32_t* slots, int32_t* cands, void* dtds, int32_t cap, int32_t* count) override {
        if (!sh_status) KM_TRY(sh_reset());
        KM_CK(cudaStreamSynchronize(st));
        const int cnt = sh_calls > 0 ? std::min(sh_mirror[(sh_calls - 1) % km::SHARD_MIRRORS].swaps, sh_trace_cap) : 0;
        std::vector<Rec> h(cnt);
        if (cnt) KM_CK(cudaMemcpy(h.data(), sh_trace, cnt * sizeof(Rec), cudaMemcpyDeviceToHost));
        const int m = std::min(cnt, cap);
        for (int i = 0; i < m; ++i) {
            if (slots) slots[i] = h[i].slot;
            if (cands) cands[i] = h[i].c;
            if (dtds) memcpy((char*)dtds + (size_t)i * sizeof(A), &h[i].v, sizeof(A));
        }
        if (count) *count = cnt;
        return KM_OK;
    }

    int build_step = 0;
    km_status build_select(const int64_t* rcb, int32_t* cand, int32_t* owner, void* gain) override {
        if (!rec_recv) return fail(KM_ECOMM, "call kmedoids_shard_exchange first");
        if (build_step == 0) {
            KM_CK(cudaMemsetAsync(point_slot, 0xff, n * sizeof(int), st));
            ready = false;
        }
        km::k_build_select<A><<<1, 1, 0, st>>>(rec_recv, nranks, build_step, td, M, point_slot, dec);
        KM_CKL();
        KM_TRY(sync_dec());
        if (cand) *cand = h_dec->c;
        if (owner) *owner = owner_of(rcb, nranks, h_dec->c);
        if (gain) memcpy(gain, &h_dec->dtd, sizeof(A));
        return KM_OK;
    }

    // Device-decided BUILD step (kmedoids.h): the decision stays on the device,
    // the owner packs column c* and the other ranks zeros (SUM all-reduce).
    km_status build_decide(int32_t step) override {
        if (!rec_recv) return fail(KM_ECOMM, "call kmedoids_shard_exchange first");
        if (step != build_step) return fail(KM_EINVAL, "build step %d out of order (expected %d)", step, build_step);
        if (step == 0) {
            KM_CK(cudaMemsetAsync(point_slot, 0xff, n * sizeof(int), st));
            ready = false;
        }
        km::k_build_select<A><<<1, 1, 0, st>>>(rec_recv, nranks, build_step, td, M, point_slot, dec);
        KM_CKL();
        km::k_shard_pack_decided<T, A><<<(unsigned)cdiv(n, 256), 256, 0, st>>>(D, ld, (int)n, c0, c1, dec, colbuf);
        KM_CKL();
        launches += 2;
        return KM_OK;
    }
    km_status build_apply_async(int32_t step) override { return build_apply_impl(step, false); }
    km_status build_apply(int32_t step) override { return build_apply_impl(step, true); }

    km_status build_apply_impl(int32_t step, bool sync) {
        const int nb = (int)cdiv(n, 256);
        km::k_column_to_mc<T, A><<<nb, 256, 0, st>>>(colbuf, (int)n, dec, MC);
        KM_CKL();
        if (bd_mode == 1 && step >= 1) {
            if (step + 1 < k) KM_TRY(bd_changed_list(1));   // column from MC (broadcast)
        } else {
            km::k_build_dn<T, A><<<nb, 256, 0, st>>>(MC, (int)n, dec, point_slot, dn);
            KM_CKL();
        }
        build_step = step + 1;
        if (step == k - 1) {
            KM_TRY(build_finish());
            build_step = 0;
            KM_TRY(sh_reset());
        }
        if (sync) KM_CK(cudaStreamSynchronize(st));
        return KM_OK;
    }
};

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* kmedoids_last_error(void) { return g_err.c_str(); }

km_status kmedoids_create(km_handle** out, const void* D, km_dtype dtype, int64_t n, int64_t ld, int64_t col_begin,
                          int64_t col_end, int32_t k, void* cuda_stream) {
    g_err.clear();
    if (!out) return fail(KM_EINVAL, "out is NULL");
    *out = nullptr;
    if (!D) return fail(KM_EINVAL, "D is NULL");
    if (dtype != KM_U32 && dtype != KM_F32) return fail(KM_EINVAL, "unknown dtype %d", (int)dtype);
    if (n < 3 || n >= (int64_t)INT32_MAX) return fail(KM_EINVAL, "n=%lld out of range [3, 2^31)", (long long)n);
    if (k < 1 || k >= n) return fail(KM_EINVAL, "k=%d must satisfy 1 <= k < n", k);
    if (k > MAX_K) return fail(KM_EINVAL, "k=%d exceeds the supported maximum %d", k, MAX_K);
    if (col_begin < 0 || col_end > n || col_begin >= col_end)
        return fail(KM_EINVAL, "column range [%lld,%lld) invalid for n=%lld", (long long)col_begin,
                    (long long)col_end, (long long)n);
    if (ld < col_end - col_begin || ld % 4 != 0)
        return fail(KM_EINVAL, "ld=%lld must be >= the slab width and a multiple of 4", (long long)ld);
    if (((uintptr_t)D) % 16 != 0) return fail(KM_EINVAL, "D must be 16-byte aligned");
    std::unique_ptr<km_handle> h(new km_handle());
    km_status s;
    if (dtype == KM_U32) {
        auto* im = new Impl<uint32_t>();
        h->impl.reset(im);
        s = im->init(D, n, ld, col_begin, col_end, k, (cudaStream_t)cuda_stream);
    } else {
        auto* im = new Impl<float>();
        h->impl.reset(im);
        s = im->init(D, n, ld, col_begin, col_end, k, (cudaStream_t)cuda_stream);
    }
    if (s != KM_OK) return s;
    *out = h.release();
    return KM_OK;
}

km_status kmedoids_destroy(km_handle* h) {
    delete h;
    return KM_OK;
}

#define KM_H()                                                  \
    do {                                                        \
        g_err.clear();                                          \
        if (!h || !h->impl) return fail(KM_EINVAL, "null handle"); \
    } while (0)

km_status kmedoids_set_medoids(km_handle* h, const int32_t* medoids) {
    KM_H();
    if (!medoids) return fail(KM_EINVAL, "medoids is NULL");
    return h->impl->set_medoids(medoids);
}

km_status kmedoids_init_build(km_handle* h, int32_t* medoids_out, void* td_out) {
    KM_H();
    return h->impl->init_build(medoids_out, td_out);
}

km_status kmedoids_init_weighted(km_handle* h, const double* u, int32_t* medoids_out, void* td_out) {
    KM_H();
    if (!u) return fail(KM_EINVAL, "u is NULL");
    return h->impl->init_weighted(u, medoids_out, td_out);
}

km_status kmedoids_init_lab(km_handle* h, int32_t s, const int32_t* seq, int32_t* medoids_out, void* td_out) {
    KM_H();
    if (!seq) return fail(KM_EINVAL, "seq is NULL");
    return h->impl->init_lab(s, seq, medoids_out, td_out);
}

km_status kmedoids_clara(km_handle* h, int32_t nsamples, int32_t s, const int32_t* samples, km_variant variant,
                         int32_t* medoids_out, void* td_out, int32_t* best_sample_out) {
    KM_H();
    if (!samples) return fail(KM_EINVAL, "samples is NULL");
    return h->impl->clara(nsamples, s, samples, variant, medoids_out, td_out, best_sample_out);
}

// ---- FastCLARA from points (NEXT-3 without the n x n matrix) ----------------
}  // extern "C"
namespace {

template <typename T>
struct ClaraPointsCache {
    using A = typename km::Acc<T>::type;
    struct Slot {
        T* buf = nullptr; int* idx = nullptr; int* med = nullptr; A* part = nullptr; A* tdv = nullptr;
        int* h_med = nullptr; A* h_td = nullptr;       // pinned: the sample's result
        cudaEvent_t fin = nullptr;                     // recorded behind the sample's TD pass
        cudaStream_t st = nullptr; std::unique_ptr<Impl<T>> sub;
    };
    std::mutex mu;
    int dev = -1, s = 0, k = 0;
    int64_t n = 0;
    std::vector<Slot> slots;
    void clear() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (dev >= 0 && dev != cur) cudaSetDevice(dev);
        for (auto& sl : slots) {
            sl.sub.reset();
            if (sl.st) cudaStreamDestroy(sl.st);
            if (sl.fin) cudaEventDestroy(sl.fin);
            cudaFree(sl.buf); cudaFree(sl.idx); cudaFree(sl.med); cudaFree(sl.part); cudaFree(sl.tdv);
            cudaFreeHost(sl.h_med); cudaFreeHost(sl.h_td);
        }
        if (dev >= 0 && dev != cur) cudaSetDevice(cur);
        slots.clear();
        dev = -1; s = 0; k = 0; n = 0;
    }
    static ClaraPointsCache& get() {
        static ClaraPointsCache* c = new ClaraPointsCache;   // never destroyed: no CUDA calls at exit
        return *c;
    }
};

template <typename T>
km_status clara_points_run(const void* Xv, int64_t n, int32_t d, int32_t k, int32_t ns, int32_t s,
                           const int32_t* samples, km_variant variant, cudaStream_t ust, int32_t* M_out,
                           void* td_out, int32_t* best_out, int32_t* asg_out) {
    using A = typename km::Acc<T>::type;
    using P = typename km::PointOf<T>::type;
    const P* X = static_cast<const P*>(Xv);
    // sample validation: distinct indices in range
    {
        std::vector<char> seen((size_t)n, 0);
        for (int j = 0; j < ns; ++j) {
            const int32_t* S = samples + (size_t)j * s;
            for (int a = 0; a < s; ++a) {
                if (S[a] < 0 || S[a] >= n) return fail(KM_EINVAL, "sample %d: index %d out of range", j, S[a]);
                if (seen[S[a]]) return fail(KM_EINVAL, "sample %d: duplicate index %d", j, S[a]);
                seen[S[a]] = 1;
            }
            for (int a = 0; a < s; ++a) seen[S[a]] = 0;
        }
    }
    const int64_t lds = cdiv(s, 4) * 4;
    const int conc = std::min(ns, 8);
    const int tdb = (int)cdiv(n, km::TDP_THREADS);          // k_td_points blocks
    // medoid rows per chunk (widened): the staged objects plus kc rows in 96 KB
    const int kc = std::max(1, std::min<int>(k, (int)((96 * 1024 - km::td_points_xs_bytes<T>(d)) /
                                                      ((size_t)d * sizeof(typename km::PointWide<T>::type)))));
    const size_t td_smem = km::td_points_smem<T>(d, kc);
    const size_t sd_smem = 64 * (size_t)km::clara_row_stride(d) * sizeof(P);   // k_subdist_exact
    KM_CK(cudaFuncSetAttribute(km::k_td_points<T, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)td_smem));
    // the per-sample slots (stream, s x s buffer, nested handle) are kept
    // between calls with the same (device, s, k, n) so a handle's BUILD is
    // replayed from its CUDA graph on later samples and calls
    auto& cache = ClaraPointsCache<T>::get();
    std::unique_lock<std::mutex> lk(cache.mu);
    int dev = 0;
    KM_CK(cudaGetDevice(&dev));
    using Slot = typename ClaraPointsCache<T>::Slot;
    std::vector<Slot>& slots = cache.slots;
    if (cache.dev != dev || cache.s != s || cache.k != k || cache.n != n) {
        cache.clear();
        cache.dev = dev; cache.s = s; cache.k = k; cache.n = n;
    }
    auto cleanup = [&]() { cache.clear(); };
    KM_CK(cudaStreamSynchronize(ust));                      // X is ready before other streams read it
    while ((int)slots.size() < conc) {
        slots.emplace_back();
        Slot& sl = slots.back();
        cudaError_t e = cudaMalloc(&sl.buf, (size_t)s * lds * sizeof(T));
        if (e == cudaSuccess) e = cudaMalloc(&sl.idx, (size_t)s * sizeof(int));
        if (e == cudaSuccess) e = cudaMalloc(&sl.med, (size_t)k * sizeof(int));
        if (e == cudaSuccess) e = cudaMalloc(&sl.part, (size_t)tdb * sizeof(A));
        if (e == cudaSuccess) e = cudaMalloc(&sl.tdv, sizeof(A));
        if (e == cudaSuccess) e = cudaMallocHost(&sl.h_med, (size_t)k * sizeof(int));
        if (e == cudaSuccess) e = cudaMallocHost(&sl.h_td, sizeof(A));
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.fin, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaMemsetAsync(sl.buf, 0, (size_t)s * lds * sizeof(T), sl.st);
        if (e != cudaSuccess) { cleanup(); cudaGetLastError(); return fail(KM_ENOMEM, "CLARA scratch: %s", cudaGetErrorString(e)); }
        sl.sub.reset(new Impl<T>());
        const km_status r = sl.sub->init(sl.buf, s, lds, 0, s, k, sl.st);
        if (r != KM_OK) { cleanup(); return r; }
    }
    std::vector<std::vector<int32_t>> Mg((size_t)ns, std::vector<int32_t>((size_t)k));
    std::vector<A> tds((size_t)ns);
    std::vector<km_status> res((size_t)ns, KM_OK);
    std::vector<std::string> errs((size_t)ns);
    auto worker = [&](int si) {
        Slot& sl = slots[si];
        Impl<T>& sub = *sl.sub;
        for (int j = si; j < ns; j += conc) {
            const int32_t* S = samples + (size_t)j * s;
            km_status r = KM_OK;
            auto ck = [&](cudaError_t e, const char* what) {
                if (r == KM_OK && e != cudaSuccess) r = fail(KM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
            };
            ck(cudaMemcpyAsync(sl.idx, S, s * sizeof(int32_t), cudaMemcpyHostToDevice, sl.st), "sample indices");
            if (r == KM_OK) {
                const dim3 g((unsigned)cdiv(s, 32), (unsigned)cdiv(s, 32));
                km::k_subdist_exact<T><<<g, 256, sd_smem, sl.st>>>(X, d, sl.idx, s, sl.buf, lds);
                ck(cudaGetLastError(), "sample dissimilarities");
            }
            if (r == KM_OK) r = sub.init_build(nullptr, nullptr);
            if (r == KM_OK) {
                if (variant == KM_FASTPAM1) {
                    bool conv = false;
                    r = sub.fp1_run_pipelined(2000, nullptr, nullptr, &conv);
                } else {
                    for (int it = 0; r == KM_OK && it < 2000; ++it) {
                        const km_status q = sub.swap_iter(variant, nullptr, nullptr);
                        if (q == KM_CONVERGED) break;
                        if (q != KM_OK) r = q;
                    }
                }
            }
            std::vector<int32_t> Mloc((size_t)k);
            if (r == KM_OK) r = sub.get_state(Mloc.data(), nullptr, nullptr, nullptr, nullptr);
            if (r == KM_OK) {
                for (int i = 0; i < k; ++i) Mg[j][i] = S[Mloc[i]];
                // TD over all n objects from the points (Eq. eqn:td, reading C2)
                ck(cudaMemcpyAsync(sl.med, Mg[j].data(), k * sizeof(int32_t), cudaMemcpyHostToDevice, sl.st), "medoids");
                if (r == KM_OK) {
                    km::k_td_points<T, A><<<tdb, km::TDP_THREADS, td_smem, sl.st>>>(X, (int)n, d, sl.med, k, kc, sl.part, nullptr);
                    km::k_sum_partials<A><<<1, 32, 0, sl.st>>>(sl.part, tdb, sl.tdv);
                    ck(cudaGetLastError(), "TD from points");
                }
                A v = 0;
                ck(cudaMemcpyAsync(&v, sl.tdv, sizeof(A), cudaMemcpyDeviceToHost, sl.st), "TD");
                ck(cudaStreamSynchronize(sl.st), "sample");
                tds[j] = v;
            }
            res[j] = r;
            if (r != KM_OK) errs[j] = g_err;
        }
    };
    if (variant == KM_FASTPAM1) {
        // ONE host thread drives the samples, `conc` at a time, each on its
        // slot's stream: sample indices, s x s dissimilarities, BUILD and the
        // first two FastPAM1 iterations are enqueued at once; finished
        // iterations are collected by event queries (never a blocking wait)
        // and the next queued; behind the converging pass the medoids are
        // mapped to object indices and the TD over all n objects computed,
        // then copied into pinned memory (the slot's `fin` event).
        std::vector<int> cur((size_t)conc, -1), phase((size_t)conc, 0);
        int nextj = 0, left = ns;
        km_status r = KM_OK;
        int rj = -1;
        while (left > 0 && r == KM_OK) {
            bool progress = false;
            for (int si = 0; si < conc && r == KM_OK; ++si) {
                Slot& sl = slots[si];
                Impl<T>& sub = *sl.sub;
                const int j = cur[si];
                auto ck = [&](cudaError_t e, const char* what) {
                    if (r == KM_OK && e != cudaSuccess) { r = fail(KM_ECUDA, "%s: %s", what, cudaGetErrorString(e)); rj = j; }
                };
                if (j < 0) {
                    if (nextj >= ns) continue;
                    const int jj = nextj++;
                    cur[si] = jj;
                    rj = jj;
                    const int32_t* S = samples + (size_t)jj * s;
                    ck(cudaMemcpyAsync(sl.idx, S, s * sizeof(int32_t), cudaMemcpyHostToDevice, sl.st), "sample indices");
                    if (r == KM_OK) {
                        const dim3 g((unsigned)cdiv(s, 32), (unsigned)cdiv(s, 32));
                        km::k_subdist_exact<T><<<g, 256, sd_smem, sl.st>>>(X, d, sl.idx, s, sl.buf, lds);
                        ck(cudaGetLastError(), "sample dissimilarities");
                    }
                    sub.build_async = true;
                    if (r == KM_OK) r = sub.init_build(nullptr, nullptr);
                    sub.build_async = false;
                    if (r == KM_OK) r = sub.fp1_async_begin(2000);
                    phase[si] = 1;
                    progress = true;
                } else if (phase[si] == 1) {
                    bool fin = false;
                    rj = j;
                    r = sub.fp1_async_poll(&fin);
                    if (r != KM_OK || !fin) continue;
                    // the medoids as object indices, the TD over all n objects
                    // (Eq. eqn:td, reading C2), both into pinned memory
                    km::k_map_sample_medoids<<<1, 256, 0, sl.st>>>(sub.M, sl.idx, k, sl.med);
                    km::k_td_points<T, A><<<tdb, km::TDP_THREADS, td_smem, sl.st>>>(X, (int)n, d, sl.med, k, kc, sl.part, nullptr);
                    km::k_sum_partials<A><<<1, 32, 0, sl.st>>>(sl.part, tdb, sl.tdv);
                    ck(cudaGetLastError(), "TD from points");
                    ck(cudaMemcpyAsync(sl.h_med, sl.med, k * sizeof(int32_t), cudaMemcpyDeviceToHost, sl.st), "medoids");
                    ck(cudaMemcpyAsync(sl.h_td, sl.tdv, sizeof(A), cudaMemcpyDeviceToHost, sl.st), "TD");
                    ck(cudaEventRecord(sl.fin, sl.st), "sample event");
                    phase[si] = 2;
                    progress = true;
                } else {
                    const cudaError_t q = cudaEventQuery(sl.fin);
                    if (q == cudaErrorNotReady) continue;
                    ck(q, "sample");
                    if (r != KM_OK) continue;
                    memcpy(Mg[j].data(), sl.h_med, k * sizeof(int32_t));
                    tds[j] = *sl.h_td;
                    cur[si] = -1;
                    --left;
                    progress = true;
                }
            }
            if (!progress) std::this_thread::yield();
        }
        if (r != KM_OK) {
            const std::string msg = g_err;
            for (int si = 0; si < conc; ++si) cudaStreamSynchronize(slots[si].st);
            cleanup();
            cudaGetLastError();
            return fail(r, "CLARA sample %d: %s", rj, msg.c_str());
        }
    } else {
        // FastPAM2 / FasterPAM iterations wait on the host inside swap_iter:
        // one worker thread per slot keeps the samples concurrent
        std::vector<std::thread> th;
        for (int t = 1; t < conc; ++t) th.emplace_back(worker, t);
        worker(0);
        for (auto& x : th) x.join();
    }
    for (int j = 0; j < ns; ++j)
        if (res[j] != KM_OK) { cleanup(); return fail(res[j], "CLARA sample %d: %s", j, errs[j].c_str()); }
    int bj = 0;
    for (int j = 1; j < ns; ++j)
        if (tds[j] < tds[bj]) bj = j;                       // smallest (TD, sample index)
    if (asg_out) {
        // the assignment of every object to the winning medoids
        Slot& sl = slots[0];
        int* asg = nullptr;
        cudaError_t e = cudaMalloc(&asg, (size_t)n * sizeof(int));
        if (e == cudaSuccess) e = cudaMemcpyAsync(sl.med, Mg[bj].data(), k * sizeof(int32_t), cudaMemcpyHostToDevice, sl.st);
        if (e == cudaSuccess) {
            km::k_td_points<T, A><<<tdb, km::TDP_THREADS, td_smem, sl.st>>>(X, (int)n, d, sl.med, k, kc, sl.part, asg);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(asg_out, asg, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost, sl.st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(sl.st);
        cudaFree(asg);
        if (e != cudaSuccess) { cleanup(); return fail(KM_ECUDA, "CLARA assignment: %s", cudaGetErrorString(e)); }
    }
    if (M_out) memcpy(M_out, Mg[bj].data(), k * sizeof(int32_t));
    if (td_out) memcpy(td_out, &tds[bj], sizeof(A));
    if (best_out) *best_out = bj;
    return KM_OK;
}

}  // namespace

void clara_points_release() {
    {
        auto& c = ClaraPointsCache<float>::get();
        std::lock_guard<std::mutex> lk(c.mu);
        c.clear();
    }
    auto& c = ClaraPointsCache<uint32_t>::get();
    std::lock_guard<std::mutex> lk(c.mu);
    c.clear();
}

extern "C" {

km_status kmedoids_clara_points(const void* X, km_metric metric, int64_t n, int32_t d, int32_t k, int32_t nsamples,
                                int32_t s, const int32_t* samples, km_variant variant, void* cuda_stream,
                                int32_t* medoids_out, void* td_out, int32_t* best_sample_out,
                                int32_t* assignment_out) {
    g_err.clear();
    if (!X || !samples) return fail(KM_EINVAL, "X and samples must not be NULL");
    if (n < 3 || n >= (int64_t)INT32_MAX) return fail(KM_EINVAL, "n=%lld out of range [3, 2^31)", (long long)n);
    if (d < 1 || d > km::CLARA_MAXD) return fail(KM_EINVAL, "d=%d must be in [1, %d]", d, km::CLARA_MAXD);
    if (k < 2 || k > MAX_K) return fail(KM_EINVAL, "k=%d out of range [2, %d]", k, MAX_K);
    if (nsamples < 1) return fail(KM_EINVAL, "nsamples must be >= 1");
    if (s <= k || s > n) return fail(KM_EINVAL, "sample size s=%d must satisfy k < s <= n", s);
    if (variant != KM_FASTPAM1 && variant != KM_FASTPAM2 && variant != KM_FASTERPAM)
        return fail(KM_EINVAL, "unknown variant %d", (int)variant);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (metric == KM_METRIC_L2_F32)
        return clara_points_run<float>(X, n, d, k, nsamples, s, samples, variant, st, medoids_out, td_out,
                                       best_sample_out, assignment_out);
    if (metric == KM_METRIC_L1_U32)
        return clara_points_run<uint32_t>(X, n, d, k, nsamples, s, samples, variant, st, medoids_out, td_out,
                                          best_sample_out, assignment_out);
    return fail(KM_EINVAL, "unknown metric %d", (int)metric);
}

km_status kmedoids_swap_iter(km_handle* h, km_variant variant, int32_t* swaps_done_out, void* td_out) {
    KM_H();
    return h->impl->swap_iter(variant, swaps_done_out, td_out);
}

km_status kmedoids_run(km_handle* h, int32_t use_build, km_variant variant, int32_t max_iter, int32_t* medoids_out,
                       int32_t* assignment_out, void* td_out, int32_t* n_iter_out, int32_t* n_swaps_out) {
    KM_H();
    if (h->impl->sharded) return fail(KM_EINVAL, "kmedoids_run on a sharded handle; drive the shard phases");
    if (max_iter <= 0) max_iter = 2000;
    if (use_build) KM_TRY(h->impl->init_build(nullptr, nullptr));
    km_status st = KM_NOT_CONVERGED;
    if (variant == KM_FASTPAM1_INC) {              // all iterations in cooperative launches
        bool conv = false;
        const km_status s = h->impl->inc_iters(max_iter, nullptr, nullptr, nullptr, &conv);
        if (s != KM_OK && s != KM_CONVERGED) return s;
        KM_TRY(h->impl->get_state(medoids_out, assignment_out, td_out, n_iter_out, n_swaps_out));
        return conv ? KM_OK : KM_NOT_CONVERGED;
    }
    if (variant == KM_FASTPAM1 || variant == KM_FASTPAM2) {   // iterations queued one ahead (no host round trip)
        bool conv = false;
        if (variant == KM_FASTPAM1) KM_TRY(h->impl->fp1_run_pipelined(max_iter, nullptr, nullptr, &conv));
        else KM_TRY(h->impl->fp2_run_pipelined(max_iter, nullptr, nullptr, &conv));
        if (conv) st = KM_OK;
    } else {
        for (int it = 0; it < max_iter; ++it) {
            km_status s = h->impl->swap_iter(variant, nullptr, nullptr);
            if (s == KM_CONVERGED) { st = KM_OK; break; }
            if (s != KM_OK) return s;
        }
    }
    KM_TRY(h->impl->get_state(medoids_out, assignment_out, td_out, n_iter_out, n_swaps_out));
    return st;
}

km_status kmedoids_swap_iters_variant(km_handle* h, km_variant variant, int32_t count, int32_t* iters_out,
                                      int32_t* swaps_out, void* td_out) {
    KM_H();
    if (count < 1) return fail(KM_EINVAL, "count=%d must be >= 1", count);
    if (variant != KM_FASTPAM1 && variant != KM_FASTPAM2)
        return fail(KM_EINVAL, "queued iterations: variant must be KM_FASTPAM1 or KM_FASTPAM2");
    bool conv = false;
    int32_t it = 0, sw = 0;
    if (variant == KM_FASTPAM1) KM_TRY(h->impl->fp1_run_pipelined(count, &it, &sw, &conv));
    else KM_TRY(h->impl->fp2_run_pipelined(count, &it, &sw, &conv));
    if (iters_out) *iters_out = it;
    if (swaps_out) *swaps_out = sw;
    if (td_out) KM_TRY(h->impl->get_state(nullptr, nullptr, td_out, nullptr, nullptr));
    return conv ? KM_CONVERGED : KM_OK;
}

km_status kmedoids_swap_iters(km_handle* h, int32_t count, int32_t* iters_out, int32_t* swaps_out, void* td_out) {
    KM_H();
    if (count < 1) return fail(KM_EINVAL, "count=%d must be >= 1", count);
    bool conv = false;
    int32_t it = 0, sw = 0;
    KM_TRY(h->impl->fp1_run_pipelined(count, &it, &sw, &conv));
    if (iters_out) *iters_out = it;
    if (swaps_out) *swaps_out = sw;
    if (td_out) KM_TRY(h->impl->get_state(nullptr, nullptr, td_out, nullptr, nullptr));
    return conv ? KM_CONVERGED : KM_OK;
}

// The device copy of D of kmedoids_run_host is kept between calls (one
// buffer per process, reused when large enough) so a repeated job pays no
// 10 GB cudaMalloc / cudaFree (round 1: occasional 0.3-0.6 s stalls around
// them); kmedoids_release_host_cache frees it.  A call that finds the buffer
// busy (concurrent jobs) allocates its own.
namespace {
struct HostJobCache {
    std::mutex mu;
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    // the handle of the last job, reused by a job of the same shape on the
    // same buffer and stream (its scratch, graphs and events stay allocated:
    // destroying a handle measured 4-380 ms per job in round 2)
    km_handle* h = nullptr;
    int64_t hn = 0, hld = 0;
    int32_t hk = 0;
    km_dtype hdt = KM_U32;
    void* hst = nullptr;
};
HostJobCache g_job;
}  // namespace

km_status kmedoids_release_host_cache(void) {
    g_err.clear();
    clara_points_release();
    std::lock_guard<std::mutex> lk(g_job.mu);
    if (g_job.h) { kmedoids_destroy(g_job.h); g_job.h = nullptr; }
    if (g_job.p) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (g_job.dev != cur) cudaSetDevice(g_job.dev);
        cudaError_t e = cudaFree(g_job.p);
        if (g_job.dev != cur) cudaSetDevice(cur);
        g_job.p = nullptr;
        g_job.bytes = 0;
        if (e != cudaSuccess) return fail(KM_ECUDA, "cudaFree: %s", cudaGetErrorString(e));
    }
    return KM_OK;
}

km_status kmedoids_run_host(const void* D_host, km_dtype dtype, int64_t n, int64_t ld, int32_t k, int32_t use_build,
                            const int32_t* initial_medoids, km_variant variant, int32_t max_iter, void* cuda_stream,
                            int32_t* medoids_out, int32_t* assignment_out, void* td_out, int32_t* n_iter_out,
                            int32_t* n_swaps_out) {
    g_err.clear();
    if (!D_host) return fail(KM_EINVAL, "D_host is NULL");
    if (!use_build && !initial_medoids) return fail(KM_EINVAL, "initial_medoids required without BUILD");
    if (n < 3 || ld < n) return fail(KM_EINVAL, "bad n/ld");
    const size_t bytes = (size_t)n * (size_t)ld * 4;
    const char* ep = getenv("KM_E2E_PROF");              // measurement aid: phase times to stderr
    const bool prof = ep && ep[0] == '1';
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t0 = now();
    void* Dd = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    std::unique_lock<std::mutex> lk(g_job.mu, std::try_to_lock);
    const bool cached = lk.owns_lock();
    cudaError_t e = cudaSuccess;
    if (cached && g_job.p && (g_job.bytes < bytes || g_job.dev != dev)) {
        if (g_job.h) { kmedoids_destroy(g_job.h); g_job.h = nullptr; }
        if (g_job.dev == dev) cudaFree(g_job.p);
        else { cudaSetDevice(g_job.dev); cudaFree(g_job.p); cudaSetDevice(dev); }
        g_job.p = nullptr; g_job.bytes = 0;
    }
    if (cached && g_job.p) {
        Dd = g_job.p;
    } else {
        e = cudaMalloc(&Dd, bytes);
        if (e != cudaSuccess) return fail(KM_ENOMEM, "cudaMalloc(%zu) for D failed: %s", bytes, cudaGetErrorString(e));
        if (cached) { g_job.p = Dd; g_job.bytes = bytes; g_job.dev = dev; }
    }
    const auto t1 = now();
    cudaStream_t st = (cudaStream_t)cuda_stream;
    km_status s = KM_OK;
    km_handle* h = nullptr;
    // (the H2D is one copy: 2 or 4 concurrent chunked copies on their own
    // streams measured no faster, ~55.5 GB/s from pinned memory either way)
    e = cudaMemcpyAsync(Dd, D_host, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) s = fail(KM_ECUDA, "H2D copy of D failed: %s", cudaGetErrorString(e));
    if (prof) cudaStreamSynchronize(st);
    const auto t2 = now();
    if (s == KM_OK && cached && g_job.h && g_job.hn == n && g_job.hld == ld && g_job.hk == k && g_job.hdt == dtype &&
        g_job.hst == cuda_stream && g_job.dev == dev) {
        h = g_job.h;                                     // same shape, buffer and stream: reuse
        s = h->impl->check_diagonal();                   // the new D is validated like a new handle's
    } else if (s == KM_OK) {
        if (cached && g_job.h) { kmedoids_destroy(g_job.h); g_job.h = nullptr; }
        s = kmedoids_create(&h, Dd, dtype, n, ld, 0, n, k, cuda_stream);
        if (s == KM_OK && cached) {
            g_job.h = h; g_job.hn = n; g_job.hld = ld; g_job.hk = k; g_job.hdt = dtype; g_job.hst = cuda_stream;
        }
    }
    if (s == KM_OK && !use_build) s = kmedoids_set_medoids(h, initial_medoids);
    const auto t3 = now();
    if (s == KM_OK) {
        km_status r = kmedoids_run(h, use_build, variant, max_iter, medoids_out, assignment_out, td_out, n_iter_out,
                                   n_swaps_out);
        s = r;
    }
    const auto t4 = now();
    if (!(cached && g_job.h == h)) kmedoids_destroy(h);
    cudaStreamSynchronize(st);
    const auto t5 = now();
    if (!cached) cudaFree(Dd);
    const auto t6 = now();
    if (prof)
        fprintf(stderr, "[kmedoids_run_host] ms: malloc %.1f h2d %.1f create %.1f run %.1f destroy %.1f free %.1f\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, t6));
    return s;
}

km_status kmedoids_get_state(km_handle* h, int32_t* medoids_out, int32_t* assignment_out, void* td_out,
                             int32_t* n_iter_out, int32_t* n_swaps_out) {
    KM_H();
    return h->impl->get_state(medoids_out, assignment_out, td_out, n_iter_out, n_swaps_out);
}

km_status kmedoids_get_cache(km_handle* h, int32_t* nearest_out, int32_t* second_out, void* dn_out, void* ds_out) {
    KM_H();
    return h->impl->get_cache(nearest_out, second_out, dn_out, ds_out);
}

km_status kmedoids_eval_candidates(km_handle* h, void* dtd_out, int32_t* slot_out) {
    KM_H();
    return h->impl->eval_candidates(dtd_out, slot_out);
}

km_status kmedoids_last_swaps(km_handle* h, int32_t* slots_out, int32_t* cands_out, void* dtds_out, int32_t cap,
                              int32_t* count_out) {
    KM_H();
    return h->impl->last_swaps_out(slots_out, cands_out, dtds_out, cap, count_out);
}

km_status kmedoids_fp2_last_plan(km_handle* h, void* v_out, int32_t* c_out, int32_t* order_out, int32_t* m_out) {
    KM_H();
    return h->impl->fp2_last_plan(v_out, c_out, order_out, m_out);
}

km_status kmedoids_set_symmetric(km_handle* h, int32_t symmetric) {
    KM_H();
    return h->impl->set_symmetric(symmetric);
}

km_status kmedoids_set_profiling(km_handle* h, int32_t enable) {
    KM_H();
    h->impl->profiling = enable != 0;
    return KM_OK;
}

km_status kmedoids_stream_time(km_handle* h, double* ms_out, int64_t* launches_out, int32_t reset) {
    KM_H();
    KM_TRY(h->impl->prof_harvest());
    if (ms_out) *ms_out = h->impl->prof_ms;
    if (launches_out) *launches_out = h->impl->prof_launches;
    if (reset) { h->impl->prof_ms = 0.0; h->impl->prof_launches = 0; }
    return KM_OK;
}

namespace {
std::mutex g_dist_mu;
struct DistScratch { void* p = nullptr; size_t bytes = 0; cudaEvent_t done = nullptr; };
DistScratch g_dist_scr[64];
// Grow-only scratch of device dev; a larger request waits for the stream
// (earlier launches may still read the old buffer) before replacing it.
cudaError_t dist_scratch(int dev, size_t bytes, cudaStream_t st, float** out) {
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    DistScratch& s = g_dist_scr[dev];
    if (s.bytes < bytes) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        if (s.p) cudaFree(s.p);
        s.p = nullptr; s.bytes = 0;
        e = cudaMalloc(&s.p, bytes);
        if (e != cudaSuccess) { cudaGetLastError(); return e; }
        s.bytes = bytes;
    }
    if (!s.done) {
        cudaError_t e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    } else {
        // a call on another stream may still use the scratch
        cudaError_t e = cudaStreamWaitEvent(st, s.done, 0);
        if (e != cudaSuccess) return e;
    }
    *out = (float*)s.p;
    return cudaSuccess;
}
}  // namespace

km_status kmedoids_dissimilarity(const void* X, km_metric metric, int64_t n, int32_t d, void* D, int64_t ld,
                                 int64_t col_begin, int64_t col_end, void* cuda_stream) {
    g_err.clear();
    if (!X || !D) return fail(KM_EINVAL, "X and D must be device pointers");
    if (n < 1 || n >= (int64_t)INT32_MAX) return fail(KM_EINVAL, "n=%lld out of range", (long long)n);
    if (d < 1) return fail(KM_EINVAL, "d=%d must be >= 1", d);
    if (col_begin < 0 || col_end > n || col_begin >= col_end)
        return fail(KM_EINVAL, "column range [%lld,%lld) invalid for n=%lld", (long long)col_begin, (long long)col_end,
                    (long long)n);
    if (ld < col_end - col_begin) return fail(KM_EINVAL, "ld=%lld smaller than the slab width", (long long)ld);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if (metric == KM_METRIC_L2_F32 || metric == KM_METRIC_L2_F32_EXACT) {
        if (d > 64) return fail(KM_EINVAL, "L2 on tensor cores supports d <= 64 (d=%d)", d);
        if (ld % 4 != 0 || ((uintptr_t)D) % 16 != 0) return fail(KM_EINVAL, "D must be 16-byte aligned, ld % 4 == 0");
        const int dpad = (d + 7) / 8 * 8;
        const int64_t nm = cdiv(n, km::DT_M), ntc = cdiv(col_end - col_begin, km::DT_N);
        int dev = 0, nsm = 0, smax = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        std::lock_guard<std::mutex> lock(g_dist_mu);   // one scratch per device
        const char* ek = getenv("KM_DIST_KERNEL");     // "simple": the single-role kernel
        const bool ws = !(ek && strcmp(ek, "simple") == 0) && km::dw_smem_bytes(dpad, 1) <= (size_t)smax;
        int wstage = 1;                                 // measured: a second staging buffer is slower (L1 carve-out)
        if (const char* es = getenv("KM_DIST_STAGES"))
            if (atoi(es) == 2 && km::dw_smem_bytes(dpad, 2) <= (size_t)smax) wstage = 2;
        // pairs with d^2 < tau (|x - mu|^2 + |y - mu|^2) are recomputed exactly
        // from the raw points in the epilogue (KM_DIST_TAU: measurement
        // override), KM_METRIC_L2_F32_EXACT only
        float tau = metric == KM_METRIC_L2_F32_EXACT ? 1.0f / 16.0f : 0.f;
        if (const char* et = getenv("KM_DIST_TAU")) tau = (float)atof(et);
        const bool fixup = ws && tau > 0.f;
        const int64_t RFl = km::dw_raw_floats(dpad);
        const bool same = (col_begin == 0);
        const int64_t TF = ws ? km::dw_tile_floats(dpad) : km::dt_tile_floats(dpad);
        const size_t nrm_floats = (size_t)cdiv(n, 64) * 64;          // keeps the packed tiles 256-byte aligned
        const size_t mu_floats = 64 + 2 * (size_t)km::DM_BLOCKS * 64;  // mu (d <= 64) + the fp64 block partials
        const size_t raw_floats = fixup ? (size_t)nm * RFl + (same ? 0 : (size_t)ntc * RFl) : 0;
        const size_t scratch = nrm_floats + (size_t)nm * TF + (same ? 0 : (size_t)ntc * TF) + mu_floats + raw_floats;
        // persistent per-device scratch (norms + packed operands), grown on
        // demand: a stream-ordered allocation per call pays the pool's page
        // mapping again whenever the pool was trimmed at a synchronisation
        float* nrm = nullptr;
        cudaError_t e = dist_scratch(dev, scratch * sizeof(float), st, &nrm);
        if (e != cudaSuccess) return fail(KM_ENOMEM, "dissimilarity scratch: %s", cudaGetErrorString(e));
        float* PA = nrm + nrm_floats;
        float* PB = same ? PA : PA + nm * TF;
        float* mu = PA + nm * TF + (same ? 0 : ntc * TF);
        float* RA = mu + mu_floats;                                   // raw point tiles (exact fix-up)
        float* RB = same ? RA : RA + nm * RFl;
        const char* ec = getenv("KM_DIST_CENTER");       // measurement override: 0 = no centring
        const bool center = !(ec && ec[0] == '0');
        if (center) {
            double* mpart = reinterpret_cast<double*>(mu + 64);
            km::k_dist_mean_part<<<km::DM_BLOCKS, 256, 0, st>>>((const float*)X, (int)n, d, mpart);
            km::k_dist_mean_fin<<<1, 64, 0, st>>>(mpart, km::DM_BLOCKS, (int)n, d, mu);
        }
        const float* mup = center ? mu : nullptr;
        km::k_dist_norms<<<(unsigned)cdiv(n, 256), 256, 0, st>>>((const float*)X, mup, (int)n, d, nrm);
        // work items (row tile x column range): at least 8 per SM for balance
        const int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(ntc, cdiv((int64_t)nsm * 8, nm)));
        const int grid = (int)std::min<int64_t>(nsm, nm * nsplit);
        if (ws) {
            km::k_dist_pack2<<<(unsigned)nm, 256, 0, st>>>((const float*)X, mup, d, dpad, 0, n, PA);
            if (!same)
                km::k_dist_pack2<<<(unsigned)ntc, 256, 0, st>>>((const float*)X, mup, d, dpad, col_begin, col_end, PB);
            if (fixup) {
                km::k_dist_pack_raw<<<(unsigned)nm, 256, 0, st>>>((const float*)X, d, dpad, 0, n, RA);
                if (!same)
                    km::k_dist_pack_raw<<<(unsigned)ntc, 256, 0, st>>>((const float*)X, d, dpad, col_begin, col_end, RB);
            }
            static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
            if (!encode) {
                void* fn = nullptr;
                cudaDriverEntryPointQueryResult qr;
                e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
                if (e != cudaSuccess || !fn) { return fail(KM_ECUDA, "cuTensorMapEncodeTiled unavailable"); }
                encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
            }
            CUtensorMap tm;
            cuuint64_t gdim[2] = {(cuuint64_t)(col_end - col_begin), (cuuint64_t)n};
            cuuint64_t gstride[1] = {(cuuint64_t)ld * sizeof(float)};
            cuuint32_t box[2] = {32, 32};                 // one warp's 32 x 32 staging box
            cuuint32_t estr[2] = {1, 1};
            CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, gdim, gstride, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) { return fail(KM_ECUDA, "tensor map encode failed (%d)", (int)cr); }
            const size_t smem = km::dw_smem_bytes(dpad, wstage);
            e = cudaFuncSetAttribute(km::k_dist_l2_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) { return fail(KM_ECUDA, "smem attribute: %s", cudaGetErrorString(e)); }
            km::k_dist_l2_ws<<<grid, km::DW_THREADS, smem, st>>>(tm, PA, PB, nrm, (int)n, dpad, nsplit, wstage,
                                                                  col_begin, col_end, RA, RB, fixup ? tau : 0.f);
        } else {
            km::k_dist_pack<<<(unsigned)nm, 256, 0, st>>>((const float*)X, mup, nrm, d, dpad, 0, n, PA);
            if (!same)
                km::k_dist_pack<<<(unsigned)ntc, 256, 0, st>>>((const float*)X, mup, nrm, d, dpad, col_begin, col_end,
                                                               PB);
            const int nstage = km::dt_smem_bytes(dpad, 2) + 1024 <= (size_t)smax ? 2 : 1;
            const size_t smem = km::dt_smem_bytes(dpad, nstage);
            e = cudaFuncSetAttribute(km::k_dist_l2_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) { return fail(KM_ECUDA, "smem attribute: %s", cudaGetErrorString(e)); }
            km::k_dist_l2_tc<<<grid, km::DT_THREADS, smem, st>>>(PA, PB, (int)n, dpad, nstage, nsplit, (float*)D, ld,
                                                                  col_begin, col_end);
        }
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaEventRecord(g_dist_scr[dev].done, st);
        if (e != cudaSuccess) return fail(KM_ECUDA, "k_dist_l2_tc: %s", cudaGetErrorString(e));
        return KM_OK;
    }
    if (metric == KM_METRIC_L1_U32) {
        // Exactness of the fp32 kernel is decided on the device (coordinate
        // ranges), and both kernels are launched: the one not chosen exits at
        // its first instruction, so the call never waits for the GPU.
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lock(g_dist_mu);
        float* scr = nullptr;
        // scratch: ranges + flag [2d + 1], row sums [n], packed 16-bit operand
        // tiles of the rows (A) and of the slab's columns (B; shared when c0 == 0)
        const int dp = (d + 1) / 2;
        const int64_t ntr = cdiv(n, km::L1F_TB), ntc = cdiv(col_end - col_begin, km::L1F_TB);
        const size_t off_pa = (size_t)cdiv(2 * d + 1 + n, 32) * 32;            // 128-byte aligned
        const size_t pa_words = (size_t)ntr * dp * km::L1F_TB;
        const size_t pb_words = col_begin == 0 ? 0 : (size_t)ntc * dp * km::L1F_TB;
        cudaError_t e = dist_scratch(dev, (off_pa + pa_words + pb_words) * sizeof(int), st, &scr);
        if (e != cudaSuccess) return fail(KM_ENOMEM, "dissimilarity scratch: %s", cudaGetErrorString(e));
        int* rng = (int*)scr;
        // measurement / test override: "int" = the integer kernel only, "f32" =
        // no packed 16-bit kernel
        const char* ek = getenv("KM_DIST_L1");
        const bool try_f32 = !(ek && strcmp(ek, "int") == 0);
        const int allow_packed = (ek && (strcmp(ek, "int") == 0 || strcmp(ek, "f32") == 0)) ? 0 : 1;
        if (try_f32) {
            km::k_dist_l1_range_init<<<1, 256, 0, st>>>(d, rng);
            km::k_dist_l1_range<<<dim3((unsigned)std::min<int64_t>(cdiv(n, 256), 64), (unsigned)d), 256, 0, st>>>(
                (const int32_t*)X, (int)n, d, rng);
            km::k_dist_l1_decide<<<1, 256, 0, st>>>(d, rng, allow_packed);
            km::k_dist_l1_rowsum<<<(unsigned)cdiv(n, 256), 256, 0, st>>>((const int32_t*)X, (int)n, d, rng,
                                                                        rng + 2 * d + 1);
            const bool vec = (ld % 4 == 0) && (((uintptr_t)D) % 16 == 0);
            dim3 gf((unsigned)cdiv(col_end - col_begin, km::L1F_TB), (unsigned)cdiv(n, km::L1F_TB));
            uint32_t* PA = (uint32_t*)scr + off_pa;
            uint32_t* PB = col_begin == 0 ? PA : PA + pa_words;
            km::k_dist_l1_pack16<<<(unsigned)ntr, 256, 0, st>>>((const int32_t*)X, d, 0, n, rng, PA);
            if (col_begin != 0)
                km::k_dist_l1_pack16<<<(unsigned)ntc, 256, 0, st>>>((const int32_t*)X, d, col_begin, col_end, rng, PB);
            km::k_dist_l1_u16x2<<<gf, 256, 0, st>>>(PA, PB, (int)n, d, (uint32_t*)D, ld, col_begin, col_end, vec, rng,
                                                     rng + 2 * d + 1);
            km::k_dist_l1_f32x<<<gf, 256, 0, st>>>((const int32_t*)X, (int)n, d, (uint32_t*)D, ld, col_begin, col_end,
                                                    vec, rng, rng + 2 * d + 1);
        }
        dim3 g((unsigned)cdiv(col_end - col_begin, 64), (unsigned)cdiv(n, 64));
        km::k_dist_l1_u32<<<g, 256, 0, st>>>((const int32_t*)X, (int)n, d, (uint32_t*)D, ld, col_begin, col_end,
                                             try_f32 ? rng + 2 * d : nullptr);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaEventRecord(g_dist_scr[dev].done, st);
        if (e != cudaSuccess) return fail(KM_ECUDA, "k_dist_l1: %s", cudaGetErrorString(e));
        return KM_OK;
    }
    return fail(KM_EINVAL, "unknown metric %d", (int)metric);
}

km_status kmedoids_stream_kernel(km_handle* h, const char** name_out) {
    KM_H();
    if (!name_out) return fail(KM_EINVAL, "name_out is NULL");
    *name_out = h->impl->stream_kernel_name();
    return KM_OK;
}

km_status kmedoids_launch_count(km_handle* h, int64_t* count_out) {
    KM_H();
    if (count_out) *count_out = h->impl->launches;
    return KM_OK;
}

km_status kmedoids_shard_exchange(km_handle* h, int32_t nranks, km_exchange* out) {
    KM_H();
    if (!out) return fail(KM_EINVAL, "out is NULL");
    return h->impl->shard_exchange(nranks, out);
}

km_status kmedoids_shard_set_medoids(km_handle* h, const int32_t* medoids, const void* columns_dev) {
    KM_H();
    if (!medoids || !columns_dev) return fail(KM_EINVAL, "NULL argument");
    return h->impl->shard_set_medoids(medoids, columns_dev);
}

km_status kmedoids_shard_eval(km_handle* h) {
    KM_H();
    return h->impl->shard_eval();
}

km_status kmedoids_build_decide(km_handle* h, int32_t step) {
    KM_H();
    return h->impl->build_decide(step);
}

km_status kmedoids_build_apply_async(km_handle* h, int32_t step) {
    KM_H();
    if (step < 0 || step >= h->impl->k) return fail(KM_EINVAL, "build step %d out of range", step);
    return h->impl->build_apply_async(step);
}

km_status kmedoids_shard_decide(km_handle* h) {
    KM_H();
    return h->impl->shard_decide();
}

km_status kmedoids_shard_apply_async(km_handle* h) {
    KM_H();
    return h->impl->shard_apply_async();
}

km_status kmedoids_shard_status(km_handle* h, int32_t wait, int32_t* converged, int32_t* n_iter, int32_t* n_swaps,
                                void* td_out) {
    KM_H();
    if (wait < 0 || wait > 2) return fail(KM_EINVAL, "wait must be 0, 1 or 2");
    return h->impl->shard_status(wait, converged, n_iter, n_swaps, td_out);
}

km_status kmedoids_shard_resync(km_handle* h, int32_t* calls_out) {
    KM_H();
    return h->impl->shard_resync(calls_out);
}

km_status kmedoids_shard_trace(km_handle* h, int32_t* slots_out, int32_t* cands_out, void* dtds_out, int32_t cap,
                               int32_t* count_out) {
    KM_H();
    return h->impl->shard_trace(slots_out, cands_out, dtds_out, cap, count_out);
}

km_status kmedoids_shard_select(km_handle* h, const int64_t* rank_col_begin, int32_t* found, int32_t* slot,
                                int32_t* cand, int32_t* owner, void* dtd) {
    KM_H();
    if (!rank_col_begin) return fail(KM_EINVAL, "rank_col_begin is NULL");
    return h->impl->shard_select(rank_col_begin, found, slot, cand, owner, dtd);
}

km_status kmedoids_shard_pack_column(km_handle* h, int32_t cand) {
    KM_H();
    return h->impl->shard_pack_column(cand);
}

km_status kmedoids_shard_apply(km_handle* h) {
    KM_H();
    return h->impl->shard_apply();
}

km_status kmedoids_fp2_shard_exchange(km_handle* h, int32_t nranks, km_fp2_exchange* out) {
    KM_H();
    if (!out) return fail(KM_EINVAL, "out is NULL");
    return h->impl->fp2_shard_exchange(nranks, out);
}

km_status kmedoids_fp2_shard_eval(km_handle* h) {
    KM_H();
    return h->impl->fp2_shard_eval();
}

km_status kmedoids_fp2_shard_plan(km_handle* h, const int64_t* rank_col_begin, int32_t* m_out, int32_t* maxcnt_out) {
    KM_H();
    if (!rank_col_begin) return fail(KM_EINVAL, "rank_col_begin is NULL");
    return h->impl->fp2_shard_plan(rank_col_begin, m_out, maxcnt_out);
}

km_status kmedoids_fp2_shard_apply(km_handle* h, int32_t* swaps_done_out, void* td_out) {
    KM_H();
    return h->impl->fp2_shard_apply(swaps_done_out, td_out);
}

km_status kmedoids_fp2_round_buffers(km_handle* h, void** send_out, void** recv_out, size_t* stride_out) {
    KM_H();
    return h->impl->fp2_round_buffers(send_out, recv_out, stride_out);
}

km_status kmedoids_fp2_round_eval(km_handle* h) {
    KM_H();
    return h->impl->fp2_round_eval();
}

km_status kmedoids_fp2_round_apply(km_handle* h, int32_t* more_out, int32_t* swaps_done_out, void* td_out) {
    KM_H();
    return h->impl->fp2_round_apply(more_out, swaps_done_out, td_out);
}

km_status kmedoids_build_eval(km_handle* h, int32_t step) {
    KM_H();
    return h->impl->build_eval(step);
}

km_status kmedoids_build_select(km_handle* h, const int64_t* rank_col_begin, int32_t* cand, int32_t* owner,
                                void* gain) {
    KM_H();
    if (!rank_col_begin) return fail(KM_EINVAL, "rank_col_begin is NULL");
    return h->impl->build_select(rank_col_begin, cand, owner, gain);
}

km_status kmedoids_build_apply(km_handle* h, int32_t step) {
    KM_H();
    return h->impl->build_apply(step);
}

}  // extern "C"
