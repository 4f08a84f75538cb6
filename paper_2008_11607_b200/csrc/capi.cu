// capi.cu — the C ABI of librexi.so (include/rexi.h): plan lifetime, the stream-ordered
// step S1..S5, pole-range partial steps for pole-parallel multi-GPU runs, host-buffer
// entry, multi-step driver and pole-kernel timing. No exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <complex>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include "../../include/rexi.h"
#include "launch.h"
#include "planner.h"

using rexi::cd;

namespace {

thread_local std::string g_last_error;

rexi_status_t fail(rexi_status_t s, const std::string &msg) {
    g_last_error = msg;
    return s;
}

rexi_status_t cuda_fail(cudaError_t e, const char *where) {
    return fail(REXI_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                       \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);            \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

// shared with scalar.cu (launch.h): its entry points report through the same thread-local text
void rexi::set_last_error(const char *msg) { g_last_error = msg ? msg : ""; }

struct rexi_plan_s {
    rexi::Plan host;
    int device = 0;
    int variant = REXI_VARIANT_PFHX;
    int method = REXI_METHOD_REXII;
    // pole-kernel tuning per kernel kind (0 REXII-DZ, 1 REXII-UV, 2 REXI): modes per thread,
    // poles per loop trip, min blocks/SM
    int mpt[8] = {4, 4, 4, 4, 4, 4, 8, 8}, pu[8] = {1, 1, 1, 1, 1, 2, 8, 8}, minb[8] = {4, 3, 4, 4, 3, 2, 2, 2};
    int occ_cache[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // resident blocks per SM of the current tuning
    int sk_occ = 0;                            // same, stream-K R2C kernel
    int schedule = REXI_SCHEDULE_AUTO;
    int fused_clusters = 0;   // rexi_plan_set_fused_clusters (0: from the pole count)
    int last_schedule = REXI_SCHEDULE_AUTO;
    // pole-kernel kind: 0 REXII DZ, 1 REXII UV, 2 REXI, 3 REXII DZ3, 4 REXII PF, 5 REXII PFH,
    // 6 REXII PFH on R2C pairs, collapsed (real input only; spectral calls use kind 5),
    // 7 REXII PFHX: explicit solves on R2C pairs (real input only; spectral calls use kind 5)
    int kind() const {
        if (method == REXI_METHOD_REXI) {
            // REXI: w2 = 0, so the partial-fraction weights are W1 = w1, W2 = 0 and the PF / PFH /
            // R2C rearrangements hold unchanged (one solve per term and mode: a {K, -K} pair
            // takes the solves at K and, through the Hermitian symmetry, at -K)
            switch (variant) {
                case REXI_VARIANT_PF: return 4;
                case REXI_VARIANT_PFH: return 5;
                case REXI_VARIANT_PFHR: return 6;
                case REXI_VARIANT_PFHX: return 7;
                default: return 2;
            }
        }
        // tau = 0: every symbol vanishes, (delta, zeta) carry no velocity anywhere -> UV route
        if (host.tau == 0.0) return 1;
        switch (variant) {
            case REXI_VARIANT_UV: return 1;
            case REXI_VARIANT_DZ3: return 3;
            case REXI_VARIANT_PF: return 4;
            case REXI_VARIANT_PFH: return 5;
            case REXI_VARIANT_PFHR: return 6;
            case REXI_VARIANT_PFHX: return 7;
            default: return 0;
        }
    }
    long n_modes = 0;
    int num_sms = 0;
    int max_chunks = 1;
    // device buffers
    rexi::PoleConst *d_poles = nullptr;
    rexi::R2CPole *d_rpoles = nullptr;
    rexi::R2XPole *d_xpoles = nullptr;
    double *d_ksym = nullptr;
    cd *d_tw = nullptr;
    cd *d_fhat = nullptr;   // [3][n_modes]
    cd *d_acc = nullptr;    // [3][n_modes]
    cd *d_tmp = nullptr;    // [3][n_modes]
    cd *d_partial = nullptr;  // [max_chunks][3][n_modes]
    unsigned *d_counter = nullptr;  // fused DSMEM step: clusters arrived (0 between launches)
    long long *d_trace = nullptr;   // REXI_SMALL_TRACE measurement buffer (allocated on first use)
    double *d_stage = nullptr;  // [6][n_modes] (rexi_apply_host)
    double *d_stage2 = nullptr;  // [6][n_modes] second set (rexi_apply_host_batch)
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_step[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev;  // pairs
    size_t ev_used = 0;
    long launches = 0;
    long pole_launches = 0;
    // CUDA-graph cache of whole steps (S1..S5 for a pole range and fixed buffers)
    struct GraphEntry {
        const void *key[6];
        int mode;               // 0: physical step S1..S5, 1: spectral step (S2, S3, Re projection)
        long b, e;
        int kind, method, mpt, pu, minb;
        bool timing;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t ev_node[2] = {nullptr, nullptr};
        long n_launches = 0, n_pole = 0;
        unsigned long long last_use = 0;
    };
    bool use_graphs = true;
    bool capturing = false;
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t ev_cap[2] = {nullptr, nullptr};
    // side stream for the K = 0 fix-up, which runs concurrently with the pole kernel (R2C kind)
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<GraphEntry> graphs;
    unsigned long long graph_clock = 0;

    void clear_graphs() {
        for (GraphEntry &g : graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        graphs.clear();
    }

    ~rexi_plan_s() {
        DeviceGuard g(device);
        clear_graphs();
        if (cap_stream) cudaStreamDestroy(cap_stream);
        if (aux_stream) cudaStreamDestroy(aux_stream);
        if (h2d_stream) cudaStreamDestroy(h2d_stream);
        if (d2h_stream) cudaStreamDestroy(d2h_stream);
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t e : {ev_in[i], ev_step[i], ev_out[i]})
                if (e) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        for (cudaEvent_t e : ev_cap)
            if (e) cudaEventDestroy(e);
        for (void *p : {(void *)d_poles, (void *)d_rpoles, (void *)d_xpoles, (void *)d_ksym, (void *)d_tw, (void *)d_fhat, (void *)d_acc,
                        (void *)d_tmp, (void *)d_partial, (void *)d_counter, (void *)d_trace, (void *)d_stage,
                        (void *)d_stage2})
            if (p) cudaFree(p);
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
};

namespace {

rexi_status_t check_plan(rexi_plan_t p) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    return REXI_OK;
}

// Number of pole chunks (grid.y) for a pole range: minimise the tail of the last wave of
// blocks (grid sized in multiples of SMs x resident blocks), at most max_chunks, at least
// 4 poles per chunk.
int choose_chunks(const rexi_plan_s *p, long n_range, int v) {
    if (n_range <= 0) return 0;
    const long tiles = v == 7   ? rexi::pole_r2x_blocks(p->host.D, p->minb[v])
                       : v == 6 ? rexi::pole_r2c_blocks(p->host.D, p->mpt[v])
                              : (p->n_modes + rexi::pole_modes_per_block(p->mpt[v]) - 1) /
                                    rexi::pole_modes_per_block(p->mpt[v]);
    int &occ = const_cast<rexi_plan_s *>(p)->occ_cache[v];
    if (occ <= 0) {
        cudaError_t e = v == 7   ? rexi::pole_r2x_occupancy(p->pu[v], p->minb[v], &occ)
                        : v == 6 ? rexi::pole_r2c_occupancy(p->mpt[v], p->pu[v], p->minb[v], &occ)
                                 : rexi::pole_occupancy(v, p->mpt[v], p->pu[v], p->minb[v], &occ);
        if (e != cudaSuccess) occ = 1;
    }
    const long conc = (long)p->num_sms * std::max(1, occ);
    const long max_c = std::max(1L, std::min<long>(p->max_chunks, n_range / 4));
    int best = 1;
    double best_eff = 0.0;
    for (long c = 1; c <= max_c; ++c) {
        const long blocks = tiles * c;
        const long waves = (blocks + conc - 1) / conc;
        const double eff = (double)blocks / (double)(waves * conc);
        if (eff > best_eff + 0.02) {
            best_eff = eff;
            best = (int)c;
        }
        if (best_eff > 0.97) break;
    }
    return best;
}

rexi_status_t next_event(rexi_plan_s *p, cudaEvent_t *out) {
    if (p->ev_used >= p->ev.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        p->ev.push_back(e);
    }
    *out = p->ev[p->ev_used++];
    return REXI_OK;
}

// Bracket the pole kernel with timing events (start = true before, false after). While a step
// is being captured into a graph, two placeholder events become event-record nodes that each
// replay re-targets to fresh events from the pool.
rexi_status_t record(rexi_plan_s *p, cudaStream_t st, bool start) {
    if (!p->timing) return REXI_OK;
    if (p->capturing) {
        CK(cudaEventRecordWithFlags(p->ev_cap[start ? 0 : 1], st, cudaEventRecordExternal));
        return REXI_OK;
    }
    cudaEvent_t e;
    rexi_status_t s = next_event(p, &e);
    if (s != REXI_OK) return s;
    CK(cudaEventRecord(e, st));
    return REXI_OK;
}

// half_out: write only the spectrum's rows l <= D/2, which hold the representative of every
// {K, -K} pair — enough for the R2C pole kernels and their finish / fix-up (internal steps only;
// rexi_forward writes the full spectrum)
rexi_status_t do_forward(rexi_plan_s *p, const double *eta, const double *u, const double *v,
                         cd *fhat, cudaStream_t st, bool half_out = false) {
    const long n = p->n_modes;
    const int D = p->host.D;
    const double *in[3] = {eta, u, v};
    cd *half[3] = {p->d_tmp, p->d_tmp + n, p->d_tmp + 2 * n};
    cd *out[3] = {fhat, fhat + n, fhat + 2 * n};
    CK(rexi::launch_fft_forward(in, half, out, p->d_tw, D, 1.0 / ((double)D * (double)D), st, half_out));
    p->launches += 2;
    return REXI_OK;
}

// hermitian: acc is known to be a Hermitian spectrum (the R2C accumulator, or a spectrum after
// the Re projection), so the inverse skips the symmetrisation loads.
rexi_status_t do_inverse(rexi_plan_s *p, const cd *acc, double *eta, double *u, double *v,
                         cudaStream_t st, bool hermitian = false) {
    const long n = p->n_modes;
    const int D = p->host.D;
    const cd *in[3] = {acc, acc + n, acc + 2 * n};
    cd *half[3] = {p->d_tmp, p->d_tmp + n, p->d_tmp + 2 * n};
    double *out[3] = {eta, u, v};
    CK(rexi::launch_fft_inverse(in, half, out, hermitian, p->d_tw, D, st));
    p->launches += 2;
    return REXI_OK;
}

// real_input: fhat is the spectrum of real fields (Hermitian), so the R2C pair kernel may be
// used; rexi_poles (arbitrary complex spectra) passes false.
// half_acc (R2C kinds): the finish writes only the modes with k <= D/2, all that the inverse
// transform of the Hermitian accumulator reads (internal physical steps only)
rexi_status_t do_poles(rexi_plan_s *p, long b, long e, const cd *fhat, cd *acc, cudaStream_t st,
                       bool real_input, bool half_acc = false) {
    const long n = p->n_modes;
    if (e <= b) {
        CK(cudaMemsetAsync(acc, 0, sizeof(cd) * 3 * (size_t)n, st));
        return REXI_OK;
    }
    int kd = p->kind();
    if ((kd == 6 || kd == 7) && !real_input) kd = 5;
    // R2C with octet items, REXI_SCHEDULE_STREAMK: a persistent grid when the segment partials
    // fit the partial buffer (AUTO = chunked: measured 2-4 % faster, rexi.h)
    long sk_tiles = 0;
    int sk_slots = 0, sk_ctas = 0;
    if (kd == 6 && p->mpt[6] == 8 && p->schedule == REXI_SCHEDULE_STREAMK) {
        if (p->sk_occ <= 0 && rexi::pole_r2c_sk_occupancy(p->pu[6], &p->sk_occ) != cudaSuccess)
            p->sk_occ = -1;
        if (p->sk_occ > 0) {
            const long T = rexi::pole_r2c_sk_tiles(p->host.D);
            const long P = (long)p->num_sms * p->sk_occ;
            const long slots = rexi::sk_slots_bound(T, e - b, P);
            const size_t need = (size_t)T * (size_t)std::max(0L, slots) * 8 * 256 * sizeof(cd);
            if (p->schedule == REXI_SCHEDULE_STREAMK && T * (e - b) / P >= 1 && slots > 0 &&
                need <= sizeof(cd) * 3 * (size_t)n * p->max_chunks) {
                sk_tiles = T;
                sk_slots = (int)slots;
                sk_ctas = (int)P;
            }
        }
    }
    const int chunks = sk_tiles ? 1 : choose_chunks(p, e - b, kd);
    rexi::PoleArgs a;
    a.fhat = fhat;
    a.partial = p->d_partial;
    a.poles = p->d_poles;
    a.rpoles = p->d_rpoles;
    a.xpoles = p->d_xpoles;
    a.ksym = p->d_ksym;
    a.pole_begin = b;
    a.pole_end = e;
    a.n_modes = n;
    a.n_chunks = chunks;
    a.D = p->host.D;
    a.log2D = 0;
    while ((1 << a.log2D) < a.D) ++a.log2D;
    a.tau = p->host.tau;
    a.hmu = p->host.poles[0].ar;
    a.sk_tiles = sk_tiles;
    a.sk_slots = sk_slots;
    a.partial_cap = 3 * n * (long)p->max_chunks;
    a.n_poles = p->host.n_poles;
    rexi_status_t s;
    const bool fork = (kd == 6 || kd == 7);
    if (fork) {
        // K = 0 corners on a side stream, concurrently with the pole kernel (disjoint outputs)
        if (!p->aux_stream) {
            CK(cudaStreamCreateWithFlags(&p->aux_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
        }
        rexi::FixupArgs x;
        x.method = p->method;
        x.write_eta = 1;
        {
            const long double sr = p->host.spre_re[(size_t)e] - p->host.spre_re[(size_t)b];
            const long double si = p->host.spre_im[(size_t)e] - p->host.spre_im[(size_t)b];
            x.S = cd{(double)sr, (double)si};
        }
        x.fhat = fhat;
        x.acc = acc;
        x.poles = p->d_poles;
        x.pole_begin = b;
        x.pole_end = e;
        x.n_modes = n;
        x.D = p->host.D;
        CK(cudaEventRecord(p->ev_fork, st));
        CK(cudaStreamWaitEvent(p->aux_stream, p->ev_fork, 0));
        CK(rexi::launch_fixup_k0(x, p->aux_stream, true));
        CK(cudaEventRecord(p->ev_join, p->aux_stream));
        p->launches += 1;
    }
    if ((s = record(p, st, true)) != REXI_OK) return s;
    p->last_schedule = sk_tiles ? REXI_SCHEDULE_STREAMK : REXI_SCHEDULE_CHUNKED;
    if (sk_tiles) CK(rexi::launch_poles_r2c_sk(a, p->pu[kd], sk_ctas, st));
    else if (kd == 7) CK(rexi::launch_poles_r2x(a, p->pu[kd], p->minb[kd], st));
    else if (kd == 6) CK(rexi::launch_poles_r2c(a, p->mpt[kd], p->pu[kd], p->minb[kd], st));
    else CK(rexi::launch_poles(a, kd, p->mpt[kd], p->pu[kd], p->minb[kd], st));
    if ((s = record(p, st, false)) != REXI_OK) return s;
    p->pole_launches += 1;
    rexi::FinishArgs f;
    f.partial = p->d_partial;
    f.acc = acc;
    f.ksym = p->d_ksym;
    f.n_modes = n;
    f.n_chunks = chunks;
    f.D = a.D;
    f.log2D = a.log2D;
    f.kind = kd;
    f.fhat = fhat;
    f.tau = p->host.tau;
    {
        const long double sr = p->host.spre_re[(size_t)e] - p->host.spre_re[(size_t)b];
        const long double si = p->host.spre_im[(size_t)e] - p->host.spre_im[(size_t)b];
        f.S = cd{(double)sr, (double)si};
        const long double wr = p->host.wpre_re[(size_t)e] - p->host.wpre_re[(size_t)b];
        const long double wi = p->host.wpre_im[(size_t)e] - p->host.wpre_im[(size_t)b];
        f.Sd = cd{(double)wr, (double)wi};
    }
    f.sk_tiles = sk_tiles;
    f.sk_slots = sk_slots;
    f.sk_ctas = sk_ctas;
    f.sk_poles = e - b;
    f.partial_cap = 3 * n * (long)p->max_chunks;
    f.half_out = (half_acc && kd >= 6) ? 1 : 0;
    if (sk_tiles) CK(rexi::launch_finish_r2c_sk(f, st));
    else CK(rexi::launch_finish(f, st));
    p->launches += 2;
    if (fork) {
        CK(cudaStreamWaitEvent(st, p->ev_join, 0));
    } else if (kd != 1) {   // DZ accumulators carry no velocity at K = 0
        rexi::FixupArgs x;
        x.method = p->method;
        x.write_eta = kd >= 6;
        x.S = f.S;
        x.fhat = fhat;
        x.acc = acc;
        x.poles = p->d_poles;
        x.pole_begin = b;
        x.pole_end = e;
        x.n_modes = n;
        x.D = a.D;
        CK(rexi::launch_fixup_k0(x, st, false));
        p->launches += 1;
    }
    return REXI_OK;
}

rexi_status_t check_range(const rexi_plan_s *p, long b, long e) {
    if (b < 0 || e < b || e > p->host.n_poles)
        return fail(REXI_ERANGE, "pole range must satisfy 0 <= begin <= end <= n_poles");
    return REXI_OK;
}

template <class F>
rexi_status_t guarded(rexi_plan_t p, F &&f) {
    rexi_status_t s = check_plan(p);
    if (s != REXI_OK) return s;
    try {
        DeviceGuard g(p->device);
        if (!g.ok) return fail(REXI_ECUDA, "cudaSetDevice failed");
        return f();
    } catch (const std::bad_alloc &) {
        return fail(REXI_ENOMEM, "host allocation failed");
    } catch (...) {
        return fail(REXI_EINVAL, "unexpected exception");
    }
}

// Pole-range sums used by the finish / fix-up kernels: S = sum (w1/alpha + w2/|alpha|^2) and
// Sd = sum w1 over [b, e), from the planner's extended-precision prefix sums.
void range_sums(const rexi_plan_s *p, long b, long e, cd *S, cd *Sd) {
    const long double sr = p->host.spre_re[(size_t)e] - p->host.spre_re[(size_t)b];
    const long double si = p->host.spre_im[(size_t)e] - p->host.spre_im[(size_t)b];
    *S = cd{(double)sr, (double)si};
    const long double wr = p->host.wpre_re[(size_t)e] - p->host.wpre_re[(size_t)b];
    const long double wi = p->host.wpre_im[(size_t)e] - p->host.wpre_im[(size_t)b];
    *Sd = cd{(double)wr, (double)wi};
}

// The fused small-grid step (REXI_SCHEDULE_FUSED / AUTO, include/rexi.h): PFHX kind, D <= 128,
// a non-empty pole range, cluster launch available; under AUTO for pole work up to 2^19 octet
// item-poles (measured, tools/sweep_fused.py, profiles/r02y_sweep_fused.jsonl: at 64^2 the fused
// step takes half the chunked path's time up to 604 poles, at 128^2 it is 3-8 % faster up to 149
// poles and slower from 377 on).
constexpr long kSmallWorkMax = 1L << 19;   // octet items x poles
bool small_eligible(const rexi_plan_s *p, long b, long e) {
    if (p->kind() != 7 || e <= b || p->host.D > 128) return false;
    if (p->schedule != REXI_SCHEDULE_FUSED && p->schedule != REXI_SCHEDULE_AUTO) return false;
    if (p->schedule == REXI_SCHEDULE_AUTO && rexi::small_step_items(p->host.D) * (e - b) > kSmallWorkMax)
        return false;
    // AUTO falls back to the multi-launch path without a cluster launch; an explicit FUSED
    // request then fails in do_step_small (no silent change of schedule)
    return p->schedule == REXI_SCHEDULE_FUSED || rexi::small2_cluster(nullptr) > 0;
}

// Clusters of the fused step when the plan leaves the choice open, from the pole work w = octet
// items x poles of the range (measured on B200, tools/sweep_fused.py): one
// cluster up to w = 30 000 (C1: 558 x 47), then 4..8 clusters, one per ~40 000 item-poles.
int fused_clusters_auto(long items, long n) {
    const long w = items * n;
    if (w <= 30000) return 1;
    return (int)std::min(8L, std::max(4L, (w + 39999) / 40000));
}

// steps > 1: a spectral-resident run of `steps` steps in the one launch (one cluster; rexi_run)
rexi_status_t do_step_small(rexi_plan_s *p, long b, long e, const double *eta, const double *u,
                            const double *v, double *eo, double *uo, double *vo, cudaStream_t st,
                            int steps = 1) {
    int resident = 0;
    const int cs = rexi::small2_cluster(&resident);
    if (cs <= 0) return fail(REXI_ECUDA, "fused small-grid step: thread-block cluster launch unavailable");
    if (e - b > (1L << 27)) return fail(REXI_EINVAL, "fused small-grid step: pole range above 2^27");
    const long n = p->n_modes;
    const int D = p->host.D;
    const long items = rexi::small_step_items(D);
    rexi::SmallArgs a;
    a.in[0] = eta; a.in[1] = u; a.in[2] = v;
    a.out[0] = eo; a.out[1] = uo; a.out[2] = vo;
    a.tw = p->d_tw;
    a.scale = 1.0 / ((double)D * (double)D);
    a.n_items = items;
    {
        // measurement knob: REXI_SMALL_STOP=k ends the kernel after stage k (results invalid)
        static const int stop = [] { const char *v = getenv("REXI_SMALL_STOP"); return v ? atoi(v) : 99; }();
        a.stop_after = stop;
    }
    a.steps = steps;
    rexi::PoleArgs &q = a.pole;
    q = rexi::PoleArgs{};
    q.xpoles = p->d_xpoles;
    q.ksym = p->d_ksym;
    q.pole_begin = b;
    q.pole_end = e;
    q.n_modes = n;
    q.D = D;
    q.log2D = 0;
    while ((1 << q.log2D) < D) ++q.log2D;
    q.tau = p->host.tau;
    q.hmu = p->host.poles[0].ar;
    q.n_poles = p->host.n_poles;
    a.poles = p->d_poles;
    a.method = p->method;
    // the pole range split over nc clusters, each with its own range sums
    int nc = steps > 1 ? 1 : p->fused_clusters > 0 ? p->fused_clusters : fused_clusters_auto(items, e - b);
    nc = (int)std::max(1L, std::min<long>({(long)nc, (long)rexi::kSmallMaxClusters, e - b}));
    if (resident > 0) nc = std::min(nc, resident);
    if ((long)nc * 3 * D * (D / 2 + 1) > 3 * n * (long)p->max_chunks) nc = 1;
    a.n_clusters = nc;
    for (int g = 0; g < nc; ++g) {
        const long gb = b + (e - b) * g / nc, ge = b + (e - b) * (g + 1) / nc;
        range_sums(p, gb, ge, &a.Sg[g], &a.Sdg[g]);
    }
    a.cl_acc = p->d_partial;
    a.counter = p->d_counter;
    rexi_status_t s;
    if ((s = record(p, st, true)) != REXI_OK) return s;
    // REXI_SMALL_TRACE=1 (measurement knob, graphs off): clock64 marks per CTA, printed to stderr
    static const bool trace = [] { const char *v = getenv("REXI_SMALL_TRACE"); return v && atoi(v) != 0; }();
    const size_t trace_n = (size_t)cs * nc * 2 * 16;
    a.trace = nullptr;
    if (trace && !p->capturing) {
        if (!p->d_trace)
            CK(cudaMalloc((void **)&p->d_trace, (size_t)rexi::kSmallMaxClusters * 16 * 2 * 16 * sizeof(long long)));
        CK(cudaMemsetAsync(p->d_trace, 0, trace_n * sizeof(long long), st));
        a.trace = p->d_trace;
    }
    CK(rexi::launch_step_small2(a, cs, st));
    if (a.trace) {
        std::vector<long long> h(trace_n);
        CK(cudaMemcpyAsync(h.data(), p->d_trace, trace_n * sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (size_t c = 0; c < (size_t)cs * nc; ++c)
            for (int w = 0; w < 2; ++w) {
                const long long *t = h.data() + (c * 2 + w) * 16;
                fprintf(stderr, "REXI_SMALL_TRACE cta %zu t%d:", c, w ? 255 : 0);
                for (int k = 1; k < 16; ++k) fprintf(stderr, " %lld", t[k] ? t[k] - t[0] : -1LL);
                fprintf(stderr, "\n");
            }
    }
    if ((s = record(p, st, false)) != REXI_OK) return s;
    p->pole_launches += 1;
    p->launches += 1;
    p->last_schedule = REXI_SCHEDULE_FUSED;
    return REXI_OK;
}

// REXI_CHECKED builds: every workspace array a step writes before reading is filled with NaN
// first, so a read of a slot the step did not write shows up in the result (checked tests).
rexi_status_t poison_workspace(rexi_plan_s *p, cudaStream_t st, bool fhat) {
#ifdef REXI_CHECKED
    const size_t field = sizeof(cd) * 3 * (size_t)p->n_modes;
    CK(cudaMemsetAsync(p->d_tmp, 0xFF, field, st));
    CK(cudaMemsetAsync(p->d_acc, 0xFF, field, st));
    CK(cudaMemsetAsync(p->d_partial, 0xFF, field * (size_t)p->max_chunks, st));
    if (fhat) CK(cudaMemsetAsync(p->d_fhat, 0xFF, field, st));
#else
    (void)p;
    (void)st;
    (void)fhat;
#endif
    return REXI_OK;
}

rexi_status_t do_step_direct(rexi_plan_s *p, long b, long e, const double *eta, const double *u,
                             const double *v, double *eo, double *uo, double *vo, cudaStream_t st) {
    {
        rexi_status_t s0 = poison_workspace(p, st, true);
        if (s0 != REXI_OK) return s0;
    }
    if (small_eligible(p, b, e)) return do_step_small(p, b, e, eta, u, v, eo, uo, vo, st);
    rexi_status_t s;
    const bool r2c = p->kind() >= 6;
    if ((s = do_forward(p, eta, u, v, p->d_fhat, st, r2c)) != REXI_OK) return s;
    if ((s = do_poles(p, b, e, p->d_fhat, p->d_acc, st, true, r2c)) != REXI_OK) return s;
    return do_inverse(p, p->d_acc, eo, uo, vo, st, r2c);
}

// One spectral-resident step: acc = poles(fhat), fhat = H(acc) (the Re projection, spectral).
rexi_status_t do_spectral_step_direct(rexi_plan_s *p, long b, long e, cudaStream_t st) {
    rexi_status_t s;
    if ((s = poison_workspace(p, st, false)) != REXI_OK) return s;
    if ((s = do_poles(p, b, e, p->d_fhat, p->d_acc, st, true)) != REXI_OK) return s;
    CK(rexi::launch_hermitian(p->d_acc, p->d_fhat, p->n_modes, p->host.D, st));
    p->launches += 1;
    return REXI_OK;
}

// One step through a cached CUDA graph (captured on the plan's private stream the first time
// these buffers / pole range / tuning are seen; replayed on the caller's stream afterwards).
// mode 0: physical step (S1..S5) on the given fields; mode 1: spectral step on plan buffers.
rexi_status_t do_step_graph(rexi_plan_s *p, int mode, long b, long e, const double *eta,
                            const double *u, const double *v, double *eo, double *uo, double *vo,
                            cudaStream_t st) {
    const void *key[6] = {eta, u, v, eo, uo, vo};
    const int kd = p->kind();
    rexi_plan_s::GraphEntry *hit = nullptr;
    for (auto &g : p->graphs)
        if (g.mode == mode && std::equal(key, key + 6, g.key) && g.b == b && g.e == e && g.kind == kd &&
            g.method == p->method &&
            g.mpt == p->mpt[kd] && g.pu == p->pu[kd] && g.minb == p->minb[kd] && g.timing == p->timing)
            hit = &g;
    if (!hit) {
        if (!p->cap_stream) {
            CK(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&p->ev_cap[0], cudaEventDefault));
            CK(cudaEventCreateWithFlags(&p->ev_cap[1], cudaEventDefault));
        }
        if (p->graphs.size() >= 8) {  // evict the least recently used entry
            auto it = std::min_element(p->graphs.begin(), p->graphs.end(),
                                       [](const auto &x, const auto &y) { return x.last_use < y.last_use; });
            if (it->exec) cudaGraphExecDestroy(it->exec);
            if (it->graph) cudaGraphDestroy(it->graph);
            p->graphs.erase(it);
        }
        rexi_plan_s::GraphEntry g;
        std::copy(key, key + 6, g.key);
        g.mode = mode;
        g.b = b;
        g.e = e;
        g.kind = kd;
        g.method = p->method;
        g.mpt = p->mpt[kd];
        g.pu = p->pu[kd];
        g.minb = p->minb[kd];
        g.timing = p->timing;
        const long l0 = p->launches, pl0 = p->pole_launches;
        CK(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
        p->capturing = true;
        rexi_status_t s = mode == 0 ? do_step_direct(p, b, e, eta, u, v, eo, uo, vo, p->cap_stream)
                                    : do_spectral_step_direct(p, b, e, p->cap_stream);
        p->capturing = false;
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &graph);
        if (s != REXI_OK) {
            if (graph) cudaGraphDestroy(graph);
            return s;
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
        g.n_launches = p->launches - l0;
        g.n_pole = p->pole_launches - pl0;
        p->launches = l0;
        p->pole_launches = pl0;
        g.graph = graph;
        ce = cudaGraphInstantiate(&g.exec, graph, 0);
        if (ce != cudaSuccess) {
            cudaGraphDestroy(graph);
            return cuda_fail(ce, "cudaGraphInstantiate");
        }
        if (g.timing) {
            size_t nn = 0;
            CK(cudaGraphGetNodes(graph, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                CK(cudaGraphNodeGetType(nd, &t));
                if (t != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t ev;
                CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
                for (int i = 0; i < 2; ++i)
                    if (ev == p->ev_cap[i]) g.ev_node[i] = nd;
            }
        }
        p->graphs.push_back(g);
        hit = &p->graphs.back();
    }
    hit->last_use = ++p->graph_clock;
    if (hit->timing && hit->ev_node[0] && hit->ev_node[1]) {
        cudaEvent_t e0, e1;
        rexi_status_t s;
        if ((s = next_event(p, &e0)) != REXI_OK) return s;
        if ((s = next_event(p, &e1)) != REXI_OK) return s;
        CK(cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[0], e0));
        CK(cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[1], e1));
    }
    CK(cudaGraphLaunch(hit->exec, st));
    p->launches += hit->n_launches;
    p->pole_launches += hit->n_pole;
    return REXI_OK;
}

rexi_status_t do_step(rexi_plan_s *p, long b, long e, const double *eta, const double *u,
                      const double *v, double *eo, double *uo, double *vo, cudaStream_t st) {
    if (p->use_graphs) return do_step_graph(p, 0, b, e, eta, u, v, eo, uo, vo, st);
    return do_step_direct(p, b, e, eta, u, v, eo, uo, vo, st);
}

rexi_status_t do_spectral_step(rexi_plan_s *p, long b, long e, cudaStream_t st) {
    if (p->use_graphs) return do_step_graph(p, 1, b, e, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st);
    return do_spectral_step_direct(p, b, e, st);
}

}  // namespace

extern "C" {

int rexi_abi_version(void) { return REXI_ABI_VERSION; }

const char *rexi_status_string(rexi_status_t s) {
    switch (s) {
        case REXI_OK: return "REXI_OK";
        case REXI_EINVAL: return "REXI_EINVAL: invalid argument";
        case REXI_ENOMEM: return "REXI_ENOMEM: out of memory";
        case REXI_ECUDA: return "REXI_ECUDA: CUDA error";
        case REXI_ERANGE: return "REXI_ERANGE: bad pole range";
    }
    return "unknown rexi status";
}

const char *rexi_last_error(void) { return g_last_error.c_str(); }

rexi_status_t rexi_plan_create(rexi_plan_t *out, int D, double tau, double tol, double h, long M,
                               int device) {
    if (!out) return fail(REXI_EINVAL, "out is NULL");
    *out = nullptr;
    rexi_plan_s *p = nullptr;
    try {
        p = new rexi_plan_s();
    } catch (...) {
        return fail(REXI_ENOMEM, "host allocation failed");
    }
    std::vector<char> err;
    int st;
    try {
        st = rexi::make_plan(p->host, D, tau, tol, h, M, err);
    } catch (...) {
        delete p;
        return fail(REXI_ENOMEM, "planner allocation failed");
    }
    if (st != REXI_OK) {
        delete p;
        return fail((rexi_status_t)st, err.empty() ? "invalid argument" : std::string(err.data()));
    }
    p->device = device;
    p->n_modes = (long)D * D;
    {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || device < 0 || device >= ndev) {
            delete p;
            return e != cudaSuccess ? cuda_fail(e, "cudaGetDeviceCount")
                                    : fail(REXI_EINVAL, "device ordinal out of range");
        }
    }
    DeviceGuard g(device);
    if (!g.ok) {
        delete p;
        return fail(REXI_ECUDA, "cudaSetDevice failed");
    }
    auto cleanup_fail = [&](rexi_status_t s) {
        delete p;
        return s;
    };
    cudaError_t e;
    if ((e = cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device)))
        return cleanup_fail(cuda_fail(e, "cudaDeviceGetAttribute"));
    if ((e = rexi::fft_setup_attributes())) return cleanup_fail(cuda_fail(e, "cudaFuncSetAttribute"));
    const size_t field = sizeof(cd) * 3 * (size_t)p->n_modes;
    // Partial-sum buffer: at most 64 chunks and at most ~2 GiB.
    const size_t budget = (size_t)2 << 30;
    p->max_chunks = (int)std::max<size_t>(1, std::min<size_t>(64, budget / field));
    auto alloc = [&](void **ptr, size_t bytes) -> cudaError_t { return cudaMalloc(ptr, bytes); };
    if ((e = alloc((void **)&p->d_poles, sizeof(rexi::PoleConst) * (size_t)p->host.n_poles)) ||
        (e = alloc((void **)&p->d_rpoles, sizeof(rexi::R2CPole) * (size_t)p->host.n_poles)) ||
        (e = alloc((void **)&p->d_xpoles, sizeof(rexi::R2XPole) * (size_t)p->host.n_poles)) ||
        (e = alloc((void **)&p->d_ksym, sizeof(double) * (size_t)D)) ||
        (e = alloc((void **)&p->d_tw, 2 * sizeof(double) * (size_t)D)) ||
        (e = alloc((void **)&p->d_fhat, field)) || (e = alloc((void **)&p->d_acc, field)) ||
        (e = alloc((void **)&p->d_tmp, field)) ||
        (e = alloc((void **)&p->d_partial, field * (size_t)p->max_chunks)) ||
        (e = alloc((void **)&p->d_counter, sizeof(unsigned))) || (e = cudaMemset(p->d_counter, 0, sizeof(unsigned)))) {
        cudaGetLastError();
        return cleanup_fail(e == cudaErrorMemoryAllocation ? fail(REXI_ENOMEM, "cudaMalloc failed")
                                                           : cuda_fail(e, "cudaMalloc"));
    }
    if ((e = cudaMemcpy(p->d_poles, p->host.poles.data(), sizeof(rexi::PoleConst) * (size_t)p->host.n_poles,
                        cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(p->d_rpoles, p->host.r2c.data(), sizeof(rexi::R2CPole) * (size_t)p->host.n_poles,
                        cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(p->d_xpoles, p->host.r2x.data(), sizeof(rexi::R2XPole) * (size_t)p->host.n_poles,
                        cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(p->d_ksym, p->host.ksym.data(), sizeof(double) * (size_t)D, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(p->d_tw, p->host.twiddle.data(), 2 * sizeof(double) * (size_t)D, cudaMemcpyHostToDevice)))
        return cleanup_fail(cuda_fail(e, "cudaMemcpy"));
    *out = p;
    return REXI_OK;
}

rexi_status_t rexi_plan_destroy(rexi_plan_t p) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    delete p;
    return REXI_OK;
}

rexi_status_t rexi_plan_info(rexi_plan_t p, rexi_plan_info_t *info) {
    if (!p || !info) return fail(REXI_EINVAL, "null argument");
    const rexi::Plan &h = p->host;
    info->D = h.D;
    info->variant = p->variant;
    info->method = p->method;
    info->tau = h.tau;
    info->tol = h.tol;
    info->h = h.h;
    info->mu = h.mu;
    info->M = h.M;
    info->L = h.L;
    info->N = h.N;
    info->n_poles = h.n_poles;
    info->m0 = h.m0;
    info->rho = h.rho;
    info->predicted_floor = h.predicted_floor;
    info->flops_per_pole_mode = rexi::pole_flops(p->kind(), p->mpt[p->kind()], p->host.D);
    info->fp64_ops_per_pole_mode = rexi::pole_ops(p->kind(), p->mpt[p->kind()], p->host.D);
    info->schedule = p->schedule;
    info->last_schedule = p->last_schedule;
    return REXI_OK;
}

rexi_status_t rexi_plan_set_variant(rexi_plan_t p, int variant) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    if (variant < REXI_VARIANT_DZ || variant > REXI_VARIANT_PFHX) return fail(REXI_EINVAL, "unknown variant");
    p->variant = variant;
    return REXI_OK;
}

rexi_status_t rexi_plan_set_method(rexi_plan_t p, int method) {
    return guarded(p, [&]() -> rexi_status_t {
        if (method != REXI_METHOD_REXII && method != REXI_METHOD_REXI)
            return fail(REXI_EINVAL, "unknown method");
        if (method == REXI_METHOD_REXI && p->host.tau == 0.0)
            return fail(REXI_EINVAL, "REXI method needs tau != 0 (its kernel back-substitutes in delta, zeta)");
        if (method == p->method) return REXI_OK;
        rexi::Plan np;
        std::vector<char> err;
        const rexi::Plan &h = p->host;
        int st = rexi::make_plan(np, h.D, h.tau, h.tol, h.h, h.M, err, method, &h.table);
        if (st != REXI_OK) return fail((rexi_status_t)st, err.empty() ? "planner" : std::string(err.data()));
        CK(cudaDeviceSynchronize());
        // cached graphs hold the old method's finish / fix-up arguments (pole sums S, Sd)
        p->clear_graphs();
        CK(cudaMemcpy(p->d_poles, np.poles.data(), sizeof(rexi::PoleConst) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_rpoles, np.r2c.data(), sizeof(rexi::R2CPole) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_xpoles, np.r2x.data(), sizeof(rexi::R2XPole) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        p->host = std::move(np);
        p->method = method;
        return REXI_OK;
    });
}

rexi_status_t rexi_plan_set_table(rexi_plan_t p, int L, double mu, const double *a) {
    return guarded(p, [&]() -> rexi_status_t {
        if (L < 1 || L > 64 || !a || !std::isfinite(mu)) return fail(REXI_EINVAL, "bad coefficient table");
        rexi::GaussTable t;
        t.L = L;
        t.mu = mu;
        t.a.resize((size_t)L + 1);
        for (int l = 0; l <= L; ++l) t.a[(size_t)l] = std::complex<long double>(a[2 * l], a[2 * l + 1]);
        rexi::Plan np;
        std::vector<char> err;
        const rexi::Plan &h = p->host;
        // M is kept (the term count of the plan); N = M + L follows the new L
        int st = rexi::make_plan(np, h.D, h.tau, h.tol, h.h, h.M, err, p->method, &t);
        if (st != REXI_OK) return fail((rexi_status_t)st, err.empty() ? "planner" : std::string(err.data()));
        CK(cudaDeviceSynchronize());
        p->clear_graphs();
        if (np.n_poles != h.n_poles) {
            rexi::PoleConst *d = nullptr;
            rexi::R2CPole *dr = nullptr;
            rexi::R2XPole *dx = nullptr;
            cudaError_t e = cudaMalloc((void **)&d, sizeof(rexi::PoleConst) * (size_t)np.n_poles);
            if (e == cudaSuccess) e = cudaMalloc((void **)&dr, sizeof(rexi::R2CPole) * (size_t)np.n_poles);
            if (e == cudaSuccess) e = cudaMalloc((void **)&dx, sizeof(rexi::R2XPole) * (size_t)np.n_poles);
            if (e != cudaSuccess) {
                cudaGetLastError();
                if (d) cudaFree(d);
                if (dr) cudaFree(dr);
                return fail(REXI_ENOMEM, "cudaMalloc (pole table) failed");
            }
            cudaFree(p->d_poles);
            cudaFree(p->d_rpoles);
            cudaFree(p->d_xpoles);
            p->d_poles = d;
            p->d_rpoles = dr;
            p->d_xpoles = dx;
        }
        CK(cudaMemcpy(p->d_poles, np.poles.data(), sizeof(rexi::PoleConst) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_rpoles, np.r2c.data(), sizeof(rexi::R2CPole) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_xpoles, np.r2x.data(), sizeof(rexi::R2XPole) * (size_t)np.n_poles,
                      cudaMemcpyHostToDevice));
        p->host = std::move(np);
        return REXI_OK;
    });
}

rexi_status_t rexi_plan_set_tuning(rexi_plan_t p, int modes_per_thread, int poles_per_iter,
                                   int min_blocks_per_sm) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    const int v = p->kind();
    const bool ok = v == 7   ? rexi::pole_r2x_supported(modes_per_thread, poles_per_iter, min_blocks_per_sm)
                    : v == 6 ? rexi::pole_r2c_supported(modes_per_thread, poles_per_iter, min_blocks_per_sm)
                             : rexi::pole_config_supported(v, modes_per_thread, poles_per_iter, min_blocks_per_sm);
    if (!ok) return fail(REXI_EINVAL, "unsupported pole-kernel tuning for this variant");
    p->mpt[v] = modes_per_thread;
    p->pu[v] = poles_per_iter;
    p->minb[v] = min_blocks_per_sm;
    p->occ_cache[v] = 0;
    p->sk_occ = 0;
    return REXI_OK;
}

rexi_status_t rexi_plan_set_schedule(rexi_plan_t p, int schedule) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    if (schedule != REXI_SCHEDULE_AUTO && schedule != REXI_SCHEDULE_CHUNKED && schedule != REXI_SCHEDULE_STREAMK &&
        schedule != REXI_SCHEDULE_FUSED)
        return fail(REXI_EINVAL, "unknown schedule");
    DeviceGuard g(p->device);
    p->schedule = schedule;
    p->clear_graphs();
    return REXI_OK;
}

rexi_status_t rexi_plan_set_fused_clusters(rexi_plan_t p, int clusters) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    if (clusters < 0 || clusters > rexi::kSmallMaxClusters) return fail(REXI_EINVAL, "clusters outside 0..9");
    DeviceGuard g(p->device);
    p->fused_clusters = clusters;
    p->clear_graphs();
    return REXI_OK;
}

rexi_status_t rexi_plan_coeffs(rexi_plan_t p, double *alpha, double *C1, double *C2, double *gamma) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    const rexi::Plan &h = p->host;
    const size_t n = (size_t)h.n_poles;
    if (alpha) std::memcpy(alpha, h.alpha.data(), 2 * n * sizeof(double));
    if (C1) std::memcpy(C1, h.C1.data(), 2 * n * sizeof(double));
    if (C2) std::memcpy(C2, h.C2.data(), 2 * n * sizeof(double));
    if (gamma) std::memcpy(gamma, h.gamma.data(), n * sizeof(double));
    return REXI_OK;
}

rexi_status_t rexi_forward(rexi_plan_t p, const double *eta, const double *u, const double *v,
                           double *fhat, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!eta || !u || !v || !fhat) return fail(REXI_EINVAL, "null pointer");
        return do_forward(p, eta, u, v, reinterpret_cast<cd *>(fhat), (cudaStream_t)stream);
    });
}

rexi_status_t rexi_poles(rexi_plan_t p, long b, long e, const double *fhat, double *acc, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!fhat || !acc) return fail(REXI_EINVAL, "null pointer");
        if (fhat == acc) return fail(REXI_EINVAL, "fhat and acc must not alias");
        rexi_status_t s = check_range(p, b, e);
        if (s != REXI_OK) return s;
        return do_poles(p, b, e, reinterpret_cast<const cd *>(fhat), reinterpret_cast<cd *>(acc),
                        (cudaStream_t)stream, false);
    });
}

rexi_status_t rexi_poles_real(rexi_plan_t p, long b, long e, const double *fhat, double *acc, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!fhat || !acc) return fail(REXI_EINVAL, "null pointer");
        if (fhat == acc) return fail(REXI_EINVAL, "fhat and acc must not alias");
        rexi_status_t s = check_range(p, b, e);
        if (s != REXI_OK) return s;
        const cudaStream_t st = (cudaStream_t)stream;
        const cd *in = reinterpret_cast<const cd *>(fhat);
        cd *out = reinterpret_cast<cd *>(acc);
        if (p->kind() >= 6) return do_poles(p, b, e, in, out, st, true);   // R2C: Hermitian already
        // generic kernels: the complex pole sum, then its Hermitian part (the spectral Re)
        if ((s = do_poles(p, b, e, in, p->d_tmp, st, true)) != REXI_OK) return s;
        CK(rexi::launch_hermitian(p->d_tmp, out, p->n_modes, p->host.D, st));
        p->launches += 1;
        return REXI_OK;
    });
}

rexi_status_t rexi_hermitian_mirror(rexi_plan_t p, double *acc, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!acc) return fail(REXI_EINVAL, "null pointer");
        CK(rexi::launch_mirror_rows(reinterpret_cast<cd *>(acc), p->n_modes, p->host.D, (cudaStream_t)stream));
        p->launches += 1;
        return REXI_OK;
    });
}

rexi_status_t rexi_inverse(rexi_plan_t p, const double *acc, double *eta, double *u, double *v,
                           void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!acc || !eta || !u || !v) return fail(REXI_EINVAL, "null pointer");
        return do_inverse(p, reinterpret_cast<const cd *>(acc), eta, u, v, (cudaStream_t)stream);
    });
}

rexi_status_t rexi_apply_partial(rexi_plan_t p, long b, long e, const double *eta, const double *u,
                                 const double *v, double *eo, double *uo, double *vo, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!eta || !u || !v || !eo || !uo || !vo) return fail(REXI_EINVAL, "null pointer");
        rexi_status_t s = check_range(p, b, e);
        if (s != REXI_OK) return s;
        return do_step(p, b, e, eta, u, v, eo, uo, vo, (cudaStream_t)stream);
    });
}

rexi_status_t rexi_plan_set_graphs(rexi_plan_t p, int enable) {
    return guarded(p, [&]() -> rexi_status_t {
        p->use_graphs = enable != 0;
        if (!p->use_graphs) p->clear_graphs();
        return REXI_OK;
    });
}

rexi_status_t rexi_apply(rexi_plan_t p, const double *eta, const double *u, const double *v,
                         double *eo, double *uo, double *vo, void *stream) {
    if (!p) return fail(REXI_EINVAL, "null plan");
    return rexi_apply_partial(p, 0, p->host.n_poles, eta, u, v, eo, uo, vo, stream);
}

rexi_status_t rexi_apply_host(rexi_plan_t p, const double *eta, const double *u, const double *v,
                              double *eo, double *uo, double *vo, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!eta || !u || !v || !eo || !uo || !vo) return fail(REXI_EINVAL, "null pointer");
        const size_t n = (size_t)p->n_modes;
        if (!p->d_stage) {
            cudaError_t e = cudaMalloc((void **)&p->d_stage, 6 * n * sizeof(double));
            if (e != cudaSuccess) {
                p->d_stage = nullptr;
                cudaGetLastError();
                return fail(REXI_ENOMEM, "cudaMalloc (staging) failed");
            }
        }
        cudaStream_t st = (cudaStream_t)stream;
        double *d[6];
        for (int i = 0; i < 6; ++i) d[i] = p->d_stage + i * n;
        const double *hin[3] = {eta, u, v};
        double *hout[3] = {eo, uo, vo};
        // every failure path below still drains the stream: no queued copy may touch the
        // caller's host buffers once this call has returned
        rexi_status_t s = REXI_OK;
        for (int i = 0; i < 3 && s == REXI_OK; ++i) {
            const cudaError_t e = cudaMemcpyAsync(d[i], hin[i], n * sizeof(double), cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync (H2D)");
        }
        if (s == REXI_OK) s = do_step(p, 0, p->host.n_poles, d[0], d[1], d[2], d[3], d[4], d[5], st);
        for (int i = 0; i < 3 && s == REXI_OK; ++i) {
            const cudaError_t e = cudaMemcpyAsync(hout[i], d[3 + i], n * sizeof(double), cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync (D2H)");
        }
        const cudaError_t es = cudaStreamSynchronize(st);
        if (s != REXI_OK) return s;
        if (es != cudaSuccess) return cuda_fail(es, "cudaStreamSynchronize");
        return REXI_OK;
    });
}

rexi_status_t rexi_apply_host_batch(rexi_plan_t p, long batch, const double *eta, const double *u,
                                    const double *v, double *eo, double *uo, double *vo, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (batch < 0) return fail(REXI_EINVAL, "batch must be >= 0");
        if (batch == 0) return REXI_OK;
        if (!eta || !u || !v || !eo || !uo || !vo) return fail(REXI_EINVAL, "null pointer");
        const size_t n = (size_t)p->n_modes;
        for (double **buf : {&p->d_stage, &p->d_stage2}) {
            if (*buf) continue;
            cudaError_t e = cudaMalloc((void **)buf, 6 * n * sizeof(double));
            if (e != cudaSuccess) {
                *buf = nullptr;
                cudaGetLastError();
                return fail(REXI_ENOMEM, "cudaMalloc (staging) failed");
            }
        }
        if (!p->h2d_stream) CK(cudaStreamCreateWithFlags(&p->h2d_stream, cudaStreamNonBlocking));
        if (!p->d2h_stream) CK(cudaStreamCreateWithFlags(&p->d2h_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t *e : {&p->ev_in[i], &p->ev_step[i], &p->ev_out[i]})
                if (!*e) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        cudaStream_t st = (cudaStream_t)stream;
        const size_t bytes = n * sizeof(double);
        const double *hin[3] = {eta, u, v};
        double *hout[3] = {eo, uo, vo};
        auto pipeline = [&]() -> rexi_status_t {
        // order the copy streams after whatever the caller queued on `stream` before this call
        CK(cudaEventRecord(p->ev_step[0], st));
        CK(cudaStreamWaitEvent(p->h2d_stream, p->ev_step[0], 0));
        for (long i = 0; i < batch; ++i) {
            const int b = (int)(i & 1);
            double *d = b ? p->d_stage2 : p->d_stage;
            // H2D of step i into set b, once step i-2 (the last user of set b's inputs) is done
            if (i >= 2) CK(cudaStreamWaitEvent(p->h2d_stream, p->ev_step[b], 0));
            for (int f = 0; f < 3; ++f)
                CK(cudaMemcpyAsync(d + f * n, hin[f] + (size_t)i * n, bytes, cudaMemcpyHostToDevice,
                                   p->h2d_stream));
            CK(cudaEventRecord(p->ev_in[b], p->h2d_stream));
            // step i on `stream`, once its inputs landed and step i-2's outputs left set b
            CK(cudaStreamWaitEvent(st, p->ev_in[b], 0));
            if (i >= 2) CK(cudaStreamWaitEvent(st, p->ev_out[b], 0));
            rexi_status_t s = do_step(p, 0, p->host.n_poles, d, d + n, d + 2 * n, d + 3 * n, d + 4 * n,
                                      d + 5 * n, st);
            if (s != REXI_OK) return s;
            CK(cudaEventRecord(p->ev_step[b], st));
            // D2H of step i
            CK(cudaStreamWaitEvent(p->d2h_stream, p->ev_step[b], 0));
            for (int f = 0; f < 3; ++f)
                CK(cudaMemcpyAsync(hout[f] + (size_t)i * n, d + (3 + f) * n, bytes, cudaMemcpyDeviceToHost,
                                   p->d2h_stream));
            CK(cudaEventRecord(p->ev_out[b], p->d2h_stream));
        }
        return REXI_OK;
        };
        const rexi_status_t s = pipeline();
        // drain all three streams, also after an error: no copy may touch the caller's host
        // buffers once this call has returned
        const cudaError_t e1 = cudaStreamSynchronize(p->h2d_stream);
        const cudaError_t e2 = cudaStreamSynchronize(p->d2h_stream);
        const cudaError_t e3 = cudaStreamSynchronize(st);
        if (s != REXI_OK) return s;
        if (e1 != cudaSuccess) return cuda_fail(e1, "cudaStreamSynchronize (h2d)");
        if (e2 != cudaSuccess) return cuda_fail(e2, "cudaStreamSynchronize (d2h)");
        if (e3 != cudaSuccess) return cuda_fail(e3, "cudaStreamSynchronize");
        return REXI_OK;
    });
}

rexi_status_t rexi_run(rexi_plan_t p, int steps, double *eta, double *u, double *v, void *stream) {
    return guarded(p, [&]() -> rexi_status_t {
        if (!eta || !u || !v) return fail(REXI_EINVAL, "null pointer");
        if (steps < 0) return fail(REXI_EINVAL, "steps must be >= 0");
        if (steps == 0) return REXI_OK;
        cudaStream_t st = (cudaStream_t)stream;
        const long N1 = p->host.n_poles;
        if (steps == 1) return do_step(p, 0, N1, eta, u, v, eta, u, v, st);
        rexi_status_t s;
        // small steps whose fused step runs on one cluster: the whole run as ONE launch, the
        // state kept in the cluster's shared memory between steps (kernels.cu step_small2_kernel)
        if (small_eligible(p, 0, N1) &&
            (p->fused_clusters > 0 ? p->fused_clusters : fused_clusters_auto(rexi::small_step_items(p->host.D), N1)) == 1) {
            if ((s = poison_workspace(p, st, true)) != REXI_OK) return s;
            return do_step_small(p, 0, N1, eta, u, v, eta, u, v, st, steps);
        }
        // spectral-resident: forward once, (poles + Re projection) per step, inverse once
        if ((s = do_forward(p, eta, u, v, p->d_fhat, st, p->kind() >= 6)) != REXI_OK) return s;
        for (int k = 0; k < steps; ++k)
            if ((s = do_spectral_step(p, 0, N1, st)) != REXI_OK) return s;
        return do_inverse(p, p->d_fhat, eta, u, v, st, true);
    });
}

rexi_status_t rexi_timing_enable(rexi_plan_t p, int enable) {
    return guarded(p, [&]() -> rexi_status_t {
        p->timing = enable != 0;
        // pre-create events so that no cudaEventCreate happens inside a timed region
        while (p->timing && p->ev.size() < 2048) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            p->ev.push_back(e);
        }
        return REXI_OK;
    });
}

rexi_status_t rexi_timing_read(rexi_plan_t p, double *ms, long *pole_launches, long *total_launches) {
    return guarded(p, [&]() -> rexi_status_t {
        double sum = 0.0;
        for (size_t i = 0; i + 1 < p->ev_used; i += 2) {
            CK(cudaEventSynchronize(p->ev[i + 1]));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, p->ev[i], p->ev[i + 1]));
            sum += t;
        }
        if (ms) *ms = sum;
        if (pole_launches) *pole_launches = p->pole_launches;
        if (total_launches) *total_launches = p->launches;
        p->ev_used = 0;
        p->pole_launches = 0;
        p->launches = 0;
        return REXI_OK;
    });
}

}  // extern "C"
