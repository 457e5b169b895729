// C-ABI layer of the B200 DOT library: problem state, workspace, field caches
// and the paper-level calls set_params / misfit / jacobian / optimize_directions
// (include/dot_b200.h documents every entry point).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "arena.h"
#include "kernels.h"
#include "optimize.h"

using namespace dot;

struct FieldCache {
    bool valid = false;
    bool identity = false;
    int ncols = 0;
    std::vector<double> coeff;        // [n_side][ncols] host copy (empty for identity)
    std::vector<int> sel;             // cached columns are the point sources sel[j] (selection / identity)
    std::shared_ptr<DBuf<double2>> blk;   // the solve's output block (shared by the sides solved together)
    double2* X = nullptr;             // [n_freq][ncols][nP] inside blk
};

struct dot_problem {
    // ---- configuration
    int nx = 0, ny = 0, nz = 0, n_freq = 0, n_src = 0, n_det = 0, n_rbf = 0, n_p = 0, max_iter = 0;
    size_t N = 0;
    double Lx = 0, Ly = 0, Lz = 0, D = 0, mua_in = 0, mua_out = 0, nu = 0, gamma = 0, eps = 0,
           cutoff = 0, tol = 0;
    double hx = 0, hy = 0, hz = 0;
    std::vector<double> omega;
    std::vector<int32_t> src, det;
    std::vector<double> src_scale, det_scale;
    OpConst op{};
    CgTiling tl{};
    PalsConst pc{};
    cudaStream_t stream = nullptr;
    std::string err;

    // ---- device state
    Arena arena;
    DBuf<int32_t> d_src, d_det;
    DBuf<double> d_src_scale, d_det_scale, d_omega_nu, d_mu, d_params;
    DBuf<int32_t> d_flagS, d_flagP, d_posS, d_posP, d_scan_tmp, d_tot;
    DBuf<int> d_count;
    bool have_params = false, have_data = false;
    std::vector<double> params;
    // support S and sample set P = S u detectors
    int K = 0, nP = 0;
    DBuf<int32_t> d_S, d_P, d_S_slot, d_det_slot, d_src_slot, d_off;
    DBuf<double> d_G;
    DBuf<int32_t> d_seg, d_segoff;    // block sparsity of G by basis (GSparse)
    DBuf<int32_t> d_segslot;          // [T] sample slot of the basis-ordered support points
    DBuf<double> d_Gseg;              // [T][5] basis-ordered weights
    DBuf<int32_t> d_ktile, d_kto, d_jorder;   // segment GEMM k-tiles / work order (GSparse)
    GSparse gsp;
    DBuf<double2> d_Dt;               // data, [n_freq][n_src][n_det]
    FieldCache cache[2];              // 0: sources, 1: detectors

    // ---- stats / timing
    dot_stats stats{};
    bool timing = false;
    std::vector<cudaEvent_t> events;
    int* h_count = nullptr;          // [2] pinned, pipelined convergence polls
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    int num_sms = 148;
    // second stream of the pass groups (half of a multi-wave batch runs there, so one half's
    // wave tail is filled by the other half's CTAs) and its fork / join events
    cudaStream_t side = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // stream of the folds (they run beside the next passes; history ring of two fold periods)
    cudaStream_t fold_stream = nullptr;
    cudaEvent_t fold_in = nullptr, fold_done = nullptr;

    ~dot_problem() {
        if (fold_in) cudaEventDestroy(fold_in);
        if (fold_done) cudaEventDestroy(fold_done);
        if (fold_stream) cudaStreamDestroy(fold_stream);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (join_ev) cudaEventDestroy(join_ev);
        if (side) cudaStreamDestroy(side);
        for (auto e : events) cudaEventDestroy(e);
        for (auto e : poll_ev)
            if (e) cudaEventDestroy(e);
        if (h_count) cudaFreeHost(h_count);
    }
};

namespace {

std::string g_create_error;

void sync(dot_problem* P) { DOT_CUDA_TRY(cudaStreamSynchronize(P->stream)); }

cudaEvent_t event_at(dot_problem* P, size_t i) {
    while (P->events.size() <= i) {
        cudaEvent_t e;
        DOT_CUDA_TRY(cudaEventCreate(&e));
        P->events.push_back(e);
    }
    return P->events[i];
}

void require_bound(dot_problem* P) {
    if (!P->arena.bound()) throw Error(DOT_ERR_STATE, "no workspace bound (dot_bind_workspace)");
}
void require_params(dot_problem* P) {
    require_bound(P);
    if (!P->have_params) throw Error(DOT_ERR_STATE, "no parameters (dot_set_params)");
}

// copy `count` elements of T from (host|device) src to a device buffer
template <class T>
DBuf<T> to_device(dot_problem* P, const T* src, size_t count, int where) {
    DBuf<T> b(P->arena, std::max<size_t>(count, 1));
    if (count) {
        DOT_CUDA_TRY(cudaMemcpyAsync(b.get(), src, count * sizeof(T),
                                     where == DOT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                     P->stream));
    }
    return b;
}

template <class T>
void from_device(dot_problem* P, T* dst, const T* src, size_t count, int where) {
    if (!count) return;
    DOT_CUDA_TRY(cudaMemcpyAsync(dst, src, count * sizeof(T),
                                 where == DOT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                 P->stream));
    if (where == DOT_HOST) sync(P);
}

// host copy of a (host|device) real matrix
std::vector<double> host_copy(dot_problem* P, const double* src, size_t count, int where) {
    std::vector<double> h(count);
    if (!count) return h;
    if (where == DOT_HOST) {
        std::memcpy(h.data(), src, count * sizeof(double));
    } else {
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), src, count * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
        sync(P);
    }
    return h;
}

// device bytes per pair of seeds iterated together (r, p ping-pong; history, shifted state
// on the samples; partial slots; states)
// hist: passes between folds (history ring depth); nsl: shifts kept per seed
size_t per_pair_bytes(const dot_problem* P, int nP, int hist, int nsl) {
    const size_t vec = P->N * sizeof(double2);
    const size_t zmax = (size_t)std::max(1, P->nz / 4);
    const size_t samp = (size_t)std::max(nP, 1) * sizeof(double2) * ((size_t)hist + 4 * (size_t)nsl);
    return 4 * vec + samp + 2 * P->tl.ntiles * zmax * kNumPartials * sizeof(double) +
           4 * sizeof(SeedState) + 4 * kMaxShift * sizeof(ShiftState) + 2 * hist * kMaxShift * sizeof(ShiftCoef) +
           8 * sizeof(int32_t) + 10 * Arena::kAlign;
}

// ---------------------------------------------------------------- batched solve
// One segment of point-combination right-hand sides: RHS (f, c) = side's point
// combination with coefficient column c at frequency f, f-major (nf * ncols outputs).
struct Seg {
    int side;
    const double* d_coeff;   // device [n_side][ncols] or null (identity)
    int ncols;
};

// Seeds of a batch: point mode -- one real seed per column c of each
// segment, delivering all n_freq shifts, output (f, c) of the segment; dense mode -- the
// complex RHS r is the seed pair (Re, Im) at its own frequency only.
struct SeedPlan {
    int nseeds = 0;                  // even (a dummy seed pads an odd count)
    std::vector<uint32_t> mask;      // needed shifts
    std::vector<int32_t> omap;       // 3 per seed: output base, stride per shift, imaginary part
    std::vector<int32_t> seg, col;   // point mode: segment and column (-1: dummy)
};

SeedPlan plan_point(const dot_problem* P, const std::vector<Seg>& segs) {
    SeedPlan sp;
    const uint32_t all = P->n_freq >= 32 ? 0xffffffffu : ((1u << P->n_freq) - 1u);
    int base = 0;
    for (int g = 0; g < (int)segs.size(); ++g) {
        for (int c = 0; c < segs[g].ncols; ++c) {
            sp.mask.push_back(all);
            sp.omap.insert(sp.omap.end(), {base + c, segs[g].ncols, 0});
            sp.seg.push_back(g);
            sp.col.push_back(c);
        }
        base += P->n_freq * segs[g].ncols;
    }
    if (sp.mask.size() % 2) {
        sp.mask.push_back(0);
        sp.omap.insert(sp.omap.end(), {-1, 0, 0});
        sp.seg.push_back(-1);
        sp.col.push_back(-1);
    }
    sp.nseeds = (int)sp.mask.size();
    return sp;
}

SeedPlan plan_dense(const dot_problem* P, const std::vector<int32_t>& freq_of) {
    SeedPlan sp;
    for (int r = 0; r < (int)freq_of.size(); ++r) {
        if (freq_of[r] < 0 || freq_of[r] >= P->n_freq) throw Error(DOT_ERR_ARG, "frequency index out of range");
        for (int e = 0; e < 2; ++e) {
            sp.mask.push_back(1u << freq_of[r]);
            sp.omap.insert(sp.omap.end(), {r, 0, e});
            sp.seg.push_back(-1);
            sp.col.push_back(-1);
        }
    }
    sp.nseeds = (int)sp.mask.size();
    return sp;
}

// Batched multi-shift solve.  Outputs XP [n_out][nP_out] on the sample list (samp_nodes,
// samp_off; the problem's P, or every node for dense solutions).  Point mode: segs;
// dense mode: dense [n_rhs][N] complex with host frequency list freq_of.  Returns per-output
// seed iterations (dense mode).
std::vector<int32_t> solve_batch(dot_problem* P, const std::vector<Seg>& segs, const double2* dense,
                                 const std::vector<int32_t>& freq_of, double2* XP, int n_out, int nP_out,
                                 const int32_t* samp_nodes, const int32_t* samp_off) {
    const SeedPlan sp = dense ? plan_dense(P, freq_of) : plan_point(P, segs);
    std::vector<int32_t> iters(n_out, 0);
    if (sp.nseeds == 0) return iters;
    if (P->n_freq > kMaxShift) throw Error(DOT_ERR_ARG, "more frequencies than the solver's shift capacity (8)");
    const size_t N = P->N;
    const int nf = P->n_freq, nP = nP_out;
    const int npairs = sp.nseeds / 2;
    // Sampled solves of less than two waves of CTAs (latency-bound passes: the sketched regimes) fold
    // every kHist passes on a side stream while the next passes run; their history rings hold two fold
    // periods (the passes of one period write one half while the fold reads the other).  Larger
    // batches fold in the pass stream (beside multi-wave passes the fold only competes for HBM:
    // measured equal step time).  Dense solutions sample every node: they fold every poll
    // group in the pass stream.  DOT_CG_FOLD_SIDE=0 / 1 forces either (sampled solves).
    const char* eFS = std::getenv("DOT_CG_FOLD_SIDE");
    const bool fold_side = !dense && (eFS ? std::atoi(eFS) != 0 : (long long)P->tl.ntiles * npairs < 2LL * P->num_sms);
    const int fold_n = dense ? 8 : kHist;    // passes per fold
    const int hist = fold_side ? 2 * fold_n : fold_n;
    const int nsl = dense ? 1 : nf;
    const size_t ppb = per_pair_bytes(P, nP, hist, nsl);
    size_t fit = P->arena.largest_free() / ppb;
    fit = fit > 2 ? fit - 1 : fit;      // several allocations fragment the arena: keep a margin
    if (fit < 1)
        throw Error(DOT_ERR_WORKSPACE, "workspace too small for one pair of right-hand sides (pair needs " +
                                           std::to_string(ppb) + " B, largest free block " +
                                           std::to_string(P->arena.largest_free()) + " B of " +
                                           std::to_string(P->arena.capacity()) + " B, " +
                                           std::to_string(P->arena.used_bytes()) + " B in use; nP " +
                                           std::to_string(nP) + ", N " + std::to_string(N) + ")");
    const int chunk = (int)std::min<size_t>(fit, (size_t)npairs);
    const int CHK = 8;
    // z chunks: enough CTAs to fill the GPU when few pairs iterate together on a deep grid
    // (DESIGN.md "z chunks"); at least 4 planes per chunk.  DOT_CG_ZCHUNKS overrides.
    auto zchunks = [&](int nb) {
        int n = 1;
        const char* e = std::getenv("DOT_CG_ZCHUNKS");
        if (e) {
            n = std::min(std::max(1, std::atoi(e)), std::max(1, P->nz / 4));
        } else {
            // wave model: a pass costs ~ ceil(CTAs / SMs) waves x (planes per chunk + 4 halo planes +
            // ~2 planes of start-up); pick the chunk count that minimises it.  sketch32 at 8 pairs:
            // 4 / 8 chunks 0.13 / 0.17 of the HBM peak (latency-bound: one wave of 16-64 CTAs).
            // Measured (tools/pass_bench.py): opt96 at 12 pairs 0.41 / 0.51 / 0.47 of the HBM peak with
            // 1 / 2 / 4 chunks -- the model's choice is 2.
            const long long have = (long long)P->tl.ntiles * nb;
            const int nmax = std::max(1, P->nz / 4);           // chunks of >= 4 planes
            double best = 0;
            for (int c = 1; c <= nmax; ++c) {
                const long long waves = (have * c + P->num_sms - 1) / P->num_sms;
                const double t = (double)waves * ((P->nz + c - 1) / c + 6);
                if (c == 1 || t < best - 1e-9) {
                    best = t;
                    n = c;
                }
            }
        }
        const int zlen = (P->nz + n - 1) / n;
        return (P->nz + zlen - 1) / zlen;
    };
    DOT_CUDA_TRY(cudaMemsetAsync(XP, 0, (size_t)n_out * nP * sizeof(double2), P->stream));
    int mx = 0, mn = 1 << 30;
    for (int p0 = 0; p0 < npairs; p0 += chunk) {
        const int nb = std::min(chunk, npairs - p0);
        const int s0 = 2 * p0, ns = 2 * nb;               // seeds of this chunk
        DBuf<double2> R0(P->arena, nb * N), R1(P->arena, nb * N), P0(P->arena, nb * N), P1(P->arena, nb * N);
        const int nzch = zchunks(nb);
        const size_t nslot = (size_t)P->tl.ntiles * nzch;
        DBuf<double> part(P->arena, 2 * (size_t)nb * nslot * kNumPartials);
        DBuf<SeedState> st(P->arena, 2 * (size_t)ns);
        DBuf<ShiftState> shs(P->arena, 2 * (size_t)ns * kMaxShift);
        DBuf<ShiftCoef> coef(P->arena, (size_t)hist * ns * kMaxShift);
        DBuf<double2> H(P->arena, (size_t)hist * nb * std::max(nP, 1));
        DBuf<double2> Ps(P->arena, (size_t)ns * nsl * std::max(nP, 1)), Xs(P->arena, (size_t)ns * nsl * std::max(nP, 1));
        DBuf<int32_t> act(P->arena, nb);
        DBuf<uint32_t> dmask = to_device(P, sp.mask.data() + s0, ns, DOT_HOST);
        DBuf<int32_t> domap = to_device(P, sp.omap.data() + 3 * s0, 3 * ns, DOT_HOST);
        int nb_launch = nb;
        DOT_CUDA_TRY(cudaMemsetAsync(coef.get(), 0, (size_t)hist * ns * kMaxShift * sizeof(ShiftCoef), P->stream));
        DOT_CUDA_TRY(cudaMemsetAsync(P0.get(), 0, (size_t)nb * N * sizeof(double2), P->stream));   // p_{-1} = 0
        DOT_CUDA_TRY(cudaMemsetAsync(Ps.get(), 0, (size_t)ns * nsl * std::max(nP, 1) * sizeof(double2), P->stream));
        DOT_CUDA_TRY(cudaMemsetAsync(Xs.get(), 0, (size_t)ns * nsl * std::max(nP, 1) * sizeof(double2), P->stream));

        // ---- right-hand sides of the seeds (scaled by theta^-1/2)
        if (dense) {
            launch_split_dense(R0.get(), dense + (size_t)p0 * N, N, nb, P->op, P->stream);
            P->stats.kernel_launches++;
        } else {
            DOT_CUDA_TRY(cudaMemsetAsync(R0.get(), 0, (size_t)nb * N * sizeof(double2), P->stream));
            for (int q = s0; q < s0 + ns;) {           // runs of consecutive columns of one segment
                const int g = sp.seg[q];
                int e = q + 1;
                while (e < s0 + ns && sp.seg[e] == g && sp.col[e] == sp.col[e - 1] + 1) ++e;
                if (g >= 0) {
                    const Seg& sg = segs[g];
                    launch_scatter_seeds(R0.get(), N, sg.side == 0 ? P->d_src.get() : P->d_det.get(),
                                         sg.side == 0 ? P->n_src : P->n_det, sg.d_coeff, sg.ncols,
                                         sg.side == 0 ? P->d_src_scale.get() : P->d_det_scale.get(), sp.col[q],
                                         q - s0, e - q, P->op, P->stream);
                    P->stats.kernel_launches++;
                }
                q = e;
            }
        }

        PassArgs a;
        a.op = P->op;
        set_edge_coefs(a);
        a.tl = P->tl;
        a.max_iter = P->max_iter;
        a.tol2 = P->tol * P->tol;
        a.nshift = nf;
        for (int f = 0; f < nf; ++f) a.sigma[f] = P->omega[f] / P->nu;
        a.mu = P->d_mu.get();
        a.R[0] = R0.get();
        a.R[1] = R1.get();
        a.Pv[0] = P0.get();
        a.Pv[1] = P1.get();
        a.part[0] = part.get();
        a.part[1] = part.get() + (size_t)nb * nslot * kNumPartials;
        a.nzch = nzch;
        a.nzch_tot = nzch;
        a.zc0 = 0;
        a.zlen = (P->nz + nzch - 1) / nzch;
        a.st[0] = st.get();
        a.st[1] = st.get() + ns;
        a.sh[0] = shs.get();
        a.sh[1] = shs.get() + (size_t)ns * kMaxShift;
        a.mask = dmask.get();
        a.coef = coef.get();
        a.hist = hist;
        a.npairs = nb;
        a.samp_nodes = samp_nodes;
        a.samp_off = samp_off;
        a.nP = nP;
        a.H = H.get();
        set_pass_tmaps(a);
        FoldArgs fa;
        fa.s0 = 0;
        fa.s1 = nP;
        fa.npairs = nb;
        fa.nshift = nf;
        fa.hist = hist;
        fa.nsl = nsl;
        fa.nP = std::max(nP, 1);
        fa.mask = dmask.get();
        fa.coef = coef.get();
        fa.H = H.get();
        fa.Ps = Ps.get();
        fa.Xs = Xs.get();

        launch_cg_init(a, nb, P->stream);
        P->stats.kernel_launches++;
        // Groups of CHK passes; each ends with a convergence count into pinned memory.  The
        // poll is pipelined: group g+1 is enqueued before the host reads group g-1's count,
        // so the GPU never idles on the host round trip (a group launched after the last
        // pair finished runs as no-ops).  Every kHist passes the fold kernel applies the
        // shifted recurrences of those passes on the samples.
        int k = 0, g = 0, kf = 0, nfold = 0;
        size_t ev = 0;
        for (;;) {
            if (P->timing) DOT_CUDA_TRY(cudaEventRecord(event_at(P, ev++), P->stream));
            // a batch of two or more waves runs as two half batches on two streams: pass k of
            // one half fills the SMs the other half's wave tail leaves idle (the halves are
            // independent seeds; they join before the fold / convergence count of the group)
            const long long ctas = (long long)P->tl.ntiles * nzch * nb_launch;
            const bool split = nb_launch >= 2 && ctas >= 2LL * P->num_sms && !std::getenv("DOT_CG_NOSPLIT");
            const int h = nb_launch / 2;
            if (split) {
                if (!P->side) {
                    DOT_CUDA_TRY(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking));
                    DOT_CUDA_TRY(cudaEventCreateWithFlags(&P->fork_ev, cudaEventDisableTiming));
                    DOT_CUDA_TRY(cudaEventCreateWithFlags(&P->join_ev, cudaEventDisableTiming));
                }
                DOT_CUDA_TRY(cudaEventRecord(P->fork_ev, P->stream));
                DOT_CUDA_TRY(cudaStreamWaitEvent(P->side, P->fork_ev, 0));
            }
            for (int i = 0; i < CHK; ++i) {
                a.k = k++;
                if (split) {
                    a.pair0 = 0;
                    launch_cg_pass(a, h, P->stream);
                    a.pair0 = h;
                    launch_cg_pass(a, nb_launch - h, P->side);
                    a.pair0 = 0;
                    P->stats.kernel_launches++;
                } else {
                    launch_cg_pass(a, nb_launch, P->stream);
                }
                P->stats.kernel_launches++;
                P->stats.pass_launches++;
            }
            if (split) {
                DOT_CUDA_TRY(cudaEventRecord(P->join_ev, P->side));
                DOT_CUDA_TRY(cudaStreamWaitEvent(P->stream, P->join_ev, 0));
            }
            if (P->timing) DOT_CUDA_TRY(cudaEventRecord(event_at(P, ev++), P->stream));
            if (k - kf >= fold_n) {
                fa.k0 = kf;
                fa.k1 = k;
                if (fold_side) {
                    if (!P->fold_stream) {
                        DOT_CUDA_TRY(cudaStreamCreateWithFlags(&P->fold_stream, cudaStreamNonBlocking));
                        DOT_CUDA_TRY(cudaEventCreateWithFlags(&P->fold_in, cudaEventDisableTiming));
                        DOT_CUDA_TRY(cudaEventCreateWithFlags(&P->fold_done, cudaEventDisableTiming));
                    }
                    // the passes from here on overwrite the ring half the previous fold read
                    if (nfold > 0) DOT_CUDA_TRY(cudaStreamWaitEvent(P->stream, P->fold_done, 0));
                    DOT_CUDA_TRY(cudaEventRecord(P->fold_in, P->stream));          // passes [kf, k) done
                    DOT_CUDA_TRY(cudaStreamWaitEvent(P->fold_stream, P->fold_in, 0));
                    launch_cg_fold(fa, P->fold_stream);
                    DOT_CUDA_TRY(cudaEventRecord(P->fold_done, P->fold_stream));
                    ++nfold;
                } else {
                    launch_cg_fold(fa, P->stream);
                }
                P->stats.kernel_launches++;
                kf = k;
            }
            launch_count_active(a.st[(k - 1) & 1], nb, P->d_count.get() + (g & 1), P->stream, act.get());
            P->stats.kernel_launches++;
            DOT_CUDA_TRY(cudaMemcpyAsync(P->h_count + (g & 1), P->d_count.get() + (g & 1), sizeof(int),
                                         cudaMemcpyDeviceToHost, P->stream));
            DOT_CUDA_TRY(cudaEventRecord(P->poll_ev[g & 1], P->stream));
            if (g > 0) {
                DOT_CUDA_TRY(cudaEventSynchronize(P->poll_ev[(g - 1) & 1]));
                const int c = P->h_count[(g - 1) & 1];
                if (c == 0) break;
                a.act = act.get();      // later passes launch only the pairs still iterating
                nb_launch = c;
            }
            ++g;
        }
        fa.k0 = kf;
        fa.k1 = k;
        if (nfold > 0) DOT_CUDA_TRY(cudaStreamWaitEvent(P->stream, P->fold_done, 0));   // folds are ordered
        launch_cg_fold(fa, P->stream);
        launch_cg_finalize(fa, P->op, XP, nP, domap.get(), samp_nodes, P->stream);
        P->stats.kernel_launches += 2;
        sync(P);
        if (P->timing) {
            for (size_t e = 0; e + 1 < ev; e += 2) {
                float ms = 0;
                DOT_CUDA_TRY(cudaEventElapsedTime(&ms, P->events[e], P->events[e + 1]));
                P->stats.pass_ms += ms;
            }
        }
        std::vector<SeedState> hs(ns);
        DOT_CUDA_TRY(cudaMemcpyAsync(hs.data(), a.st[(k - 1) & 1], ns * sizeof(SeedState), cudaMemcpyDeviceToHost,
                                     P->stream));
        sync(P);
        for (int q = 0; q < ns; ++q) {
            const int seed = s0 + q;
            if (!sp.mask[seed]) continue;
            if (hs[q].flag == DOT_ERR_NOCONV)
                throw Error(DOT_ERR_NOCONV, "CG did not converge within max_iter for seed " + std::to_string(seed));
            if (hs[q].flag == DOT_ERR_BREAKDOWN)
                throw Error(DOT_ERR_BREAKDOWN, "CG breakdown for seed " + std::to_string(seed) + " at iteration " +
                                                   std::to_string(hs[q].iters));
            const int it = hs[q].iters;
            const int systems = dense ? (sp.omap[3 * seed + 2] ? 0 : 1) : __builtin_popcount(sp.mask[seed]);
            if (dense) {
                int& o = iters[sp.omap[3 * seed]];
                o = std::max(o, it);
            }
            P->stats.seeds_solved++;
            P->stats.seed_iterations += it;
            P->stats.rhs_solved += systems;
            P->stats.rhs_iterations += (int64_t)systems * it;
            P->stats.pass_bytes += 32.0 * (double)N * it;
            mx = std::max(mx, it);
            mn = std::min(mn, it);
        }
    }
    P->stats.last_max_iters = mx;
    P->stats.last_min_iters = mn;
    return iters;
}

// ---------------------------------------------------------------- field caches
// cache[side] holds sampled solutions [n_freq][ncols][nP] of one coefficient matrix
// (identity, a selection, or a general combination).
struct Req {
    int side;
    std::vector<double> hc;   // host [n_side][ncols]; empty for identity
    bool identity;
    int ncols;
};

// Can the fields of this request be served from the cache (directly or, for a
// combination of cached point sources, by linear combination without solves)?
bool cache_hit(dot_problem* P, const Req& q) {
    const int n_side = q.side == 0 ? P->n_src : P->n_det;
    const FieldCache& c = P->cache[q.side];
    if (!c.valid) return false;
    if (q.identity && c.identity) return true;
    if (!q.identity && !c.identity && c.ncols == q.ncols && c.coeff == q.hc) return true;
    if (!q.identity && !c.sel.empty()) {
        std::vector<char> in_sel(n_side, 0);
        for (int j : c.sel) in_sel[j] = 1;
        for (int a = 0; a < n_side; ++a)
            if (!in_sel[a])
                for (int k = 0; k < q.ncols; ++k)
                    if (q.hc[(size_t)a * q.ncols + k] != 0.0) return false;
        return true;
    }
    return false;
}

// Solve every request in ONE batch (all their RHS iterate together) and cache them.
void solve_and_cache(dot_problem* P, const std::vector<Req>& reqs) {
    std::vector<Seg> segs;
    std::vector<DBuf<double>> dcs;
    int total = 0;
    for (const Req& q : reqs) {
        dcs.emplace_back();
        if (!q.identity) dcs.back() = to_device(P, q.hc.data(), q.hc.size(), DOT_HOST);
        segs.push_back(Seg{q.side, q.identity ? nullptr : dcs.back().get(), q.ncols});
        total += P->n_freq * q.ncols;
    }
    const size_t nPp = (size_t)std::max(P->nP, 1);
    for (const Req& q : reqs) {              // the caches being replaced free their memory first
        FieldCache& c = P->cache[q.side];
        c.valid = false;
        c.blk.reset();
        c.X = nullptr;
    }
    auto blk = std::make_shared<DBuf<double2>>(P->arena, (size_t)total * nPp);
    solve_batch(P, segs, nullptr, {}, blk->get(), total, P->nP, P->d_P.get(), P->d_off.get());
    size_t off = 0;
    for (const Req& q : reqs) {
        const int n_side = q.side == 0 ? P->n_src : P->n_det;
        FieldCache& c = P->cache[q.side];
        const size_t n = (size_t)P->n_freq * q.ncols * nPp;
        c.blk = blk;
        c.X = blk->get() + off;
        off += n;
        c.valid = true;
        c.identity = q.identity;
        c.ncols = q.ncols;
        c.coeff = q.identity ? std::vector<double>() : q.hc;
        c.sel.clear();
        if (q.identity) {
            for (int a = 0; a < n_side; ++a) c.sel.push_back(a);
        } else {
            // selection matrix? every column a unit vector e_a
            bool is_sel = true;
            std::vector<int> sel(q.ncols, -1);
            for (int k = 0; k < q.ncols && is_sel; ++k)
                for (int a = 0; a < n_side; ++a) {
                    const double v = q.hc[(size_t)a * q.ncols + k];
                    if (v == 0.0) continue;
                    if (v != 1.0 || sel[k] >= 0) { is_sel = false; break; }
                    sel[k] = a;
                }
            for (int k = 0; k < q.ncols && is_sel; ++k) is_sel = sel[k] >= 0;
            if (is_sel) c.sel = sel;
        }
    }
    sync(P);
}

// Before a call that needs the fields of several requests: solve all uncached ones
// together (e.g. the forward W and adjoint V solves of dot_jacobian, L966).
void prefetch_fields(dot_problem* P, const std::vector<Req>& reqs) {
    std::vector<Req> miss;
    for (const Req& q : reqs)
        if (!cache_hit(P, q)) miss.push_back(q);
    if (!miss.empty()) solve_and_cache(P, miss);
}

// Sampled fields for `side` and coefficients (host copy hc; empty = identity):
// returns a pointer to [n_freq][ncols][nP]; `tmp` receives storage when the
// fields are formed by combination rather than taken from the cache.
const double2* get_fields(dot_problem* P, int side, const std::vector<double>& hc, bool identity, int ncols,
                          DBuf<double2>& tmp) {
    const Req q{side, hc, identity, ncols};
    if (!cache_hit(P, q)) solve_and_cache(P, {q});
    FieldCache& c = P->cache[side];
    if (identity && c.identity) return c.X;
    if (!identity && !c.identity && c.ncols == ncols && c.coeff == hc) return c.X;
    // combination of the cached point sources sel[0..m):
    // X'[f][c][q] = sum_j coeff[sel_j][c] X[f][j][q]
    const int m = (int)c.sel.size();
    std::vector<double> X((size_t)m * ncols);
    for (int j = 0; j < m; ++j)
        for (int k = 0; k < ncols; ++k) X[(size_t)j * ncols + k] = hc[(size_t)c.sel[j] * ncols + k];
    DBuf<double> dc = to_device(P, X.data(), X.size(), DOT_HOST);
    tmp = DBuf<double2>(P->arena, (size_t)P->n_freq * ncols * std::max(P->nP, 1));
    launch_rc_gemm(P->n_freq, ncols, P->nP, m, dc.get(), ncols, c.X, (size_t)m * P->nP, P->nP, 1, tmp.get(),
                   (size_t)ncols * P->nP, P->nP, 1, P->stream);
    P->stats.kernel_launches++;
    sync(P);
    return tmp.get();
}

void invalidate_caches(dot_problem* P) {
    for (auto& c : P->cache) {
        c.valid = false;
        c.blk.reset();
        c.X = nullptr;
        c.coeff.clear();
        c.sel.clear();
    }
}

int fail(dot_problem* P, const Error& e) {
    if (P) P->err = e.msg;
    else g_create_error = e.msg;
    return e.code;
}

#define DOT_API_BEGIN try {
#define DOT_API_END(P)                                 \
    }                                                  \
    catch (const Error& e) { return fail(P, e); }      \
    catch (const std::exception& e) { return fail(P, Error(DOT_ERR_ARG, e.what())); } \
    return DOT_OK;

void check_side_matrix(const double* M, int n_side, int ncols, const char* name) {
    if (ncols <= 0) throw Error(DOT_ERR_ARG, std::string(name) + ": number of columns must be positive");
    if (!M && ncols != n_side) throw Error(DOT_ERR_ARG, std::string(name) + " = NULL (identity) needs ncols = n");
}


// ======================================================== z-slab domain decomposition
// (BASELINE north_star: "by z-slab domain decomposition with NCCL halo exchange and an
// allreduce of Krylov inner products in the few-simultaneous-source regime";
// DESIGN.md "Domain decomposition").  Rank r owns the z chunks [cb[r], cb[r+1]) of a
// global chunking (zlen planes per chunk) and runs the z pass on them; after every
// pass the two boundary planes of r_{k+1} and p_k are exchanged with the neighbours
// and the per-chunk partial sums (disjoint slots) are all-reduced, so every rank
// derives the same Krylov scalars.  Sampled solutions are all-reduced at the end.
// Ranks live either in one process (several dot_problem, exchanged with device
// copies: the single-GPU emulation the tests use) or one per process with NCCL.

struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
};

// NCCL is loaded on first use (libnccl.so.2: the one torch already loaded, else the system one)
static NcclApi load_nccl_api() {
    NcclApi api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
        return api;
    }
    bool ok = true;
    auto sym = [&](const char* n) {
        void* f = dlsym(h, n);
        if (!f) ok = false;
        return f;
    };
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(sym("ncclAllReduce"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
    api.errStr = reinterpret_cast<decltype(api.errStr)>(sym("ncclGetErrorString"));
    api.ok = ok;
    if (!ok) api.why = "libnccl.so.2 lacks a required symbol";
    return api;
}

NcclApi& nccl_api() {
    static NcclApi api = load_nccl_api();     // thread-safe one-time load
    return api;
}

#define DOT_NCCL_TRY(expr)                                                                        \
    do {                                                                                          \
        ncclResult_t _r = (expr);                                                                 \
        if (_r != ncclSuccess)                                                                    \
            throw Error(DOT_ERR_CUDA, std::string(#expr) + ": " + nccl_api().errStr(_r));         \
    } while (0)

struct DDPlan {
    int C = 1, zlen = 0;
    std::vector<int> cb;            // chunk boundaries of the global ranks, size world + 1
    int zs(int r, int nz) const { return std::min(cb[r] * zlen, nz); }
    int ze(int r, int nz) const { return std::min(cb[r + 1] * zlen, nz); }
};

}  // namespace

struct dot_dd {
    std::vector<dot_problem*> loc;  // local ranks rank0 .. rank0 + loc.size() - 1
    int rank0 = 0, world = 1;
    ncclComm_t comm = nullptr;      // one local rank per process, NCCL transport
    bool host = false;              // one local rank per process, host-staged caller transport
    dot_transport tr{};
    std::string err;
};

namespace {

DDPlan dd_plan(const dot_dd* G, int nb) {
    const dot_problem* P = G->loc[0];
    DDPlan pl;
    const int W = G->world, nz = P->nz;
    // chunks per rank from the fill target of one GPU (4 CTAs per SM), at least 2 planes each
    const long long target = 4LL * P->num_sms, have = (long long)P->tl.ntiles * nb;
    int m = have < target ? (int)((target + have - 1) / have) : 1;
    int zlen = std::max(2, (nz + W * m - 1) / (W * m));
    int C = (nz + zlen - 1) / zlen;
    if (C < W) {
        zlen = std::max(2, nz / W);
        C = (nz + zlen - 1) / zlen;
    }
    if (C < W) throw Error(DOT_ERR_ARG, "z-slab decomposition: nz too small for this many ranks (need 2 planes per rank)");
    pl.C = C;
    pl.zlen = zlen;
    pl.cb.resize(W + 1);
    for (int r = 0; r <= W; ++r) pl.cb[r] = (int)((long long)r * C / W);
    return pl;
}

// Exchange step of the decomposition for one rank per process: halo planes with the two
// neighbours and the in-place sum of the Krylov partials / sampled solutions over all ranks.
// Buffers are device buffers on `s`.
struct Transport {
    virtual ~Transport() = default;
    // send s_lo (n_lo_s) to rank - 1 and s_hi (n_hi_s) to rank + 1; receive r_lo (n_lo_r) from
    // rank - 1 and r_hi (n_hi_r) from rank + 1 (counts in double2; 0 = no such neighbour)
    virtual void halo(const double2* s_lo, size_t n_lo_s, double2* r_lo, size_t n_lo_r, const double2* s_hi,
                      size_t n_hi_s, double2* r_hi, size_t n_hi_r, cudaStream_t s) = 0;
    virtual void allreduce(double* buf, size_t n, cudaStream_t s) = 0;
    virtual bool synchronous() const = 0;
};

struct NcclTransport : Transport {
    ncclComm_t comm;
    int rank;
    explicit NcclTransport(ncclComm_t c, int r) : comm(c), rank(r) {}
    void halo(const double2* s_lo, size_t n_lo_s, double2* r_lo, size_t n_lo_r, const double2* s_hi, size_t n_hi_s,
              double2* r_hi, size_t n_hi_r, cudaStream_t s) override {
        NcclApi& nc = nccl_api();
        DOT_NCCL_TRY(nc.groupStart());
        if (n_hi_s) DOT_NCCL_TRY(nc.send(s_hi, 2 * n_hi_s, ncclDouble, rank + 1, comm, s));
        if (n_hi_r) DOT_NCCL_TRY(nc.recv(r_hi, 2 * n_hi_r, ncclDouble, rank + 1, comm, s));
        if (n_lo_s) DOT_NCCL_TRY(nc.send(s_lo, 2 * n_lo_s, ncclDouble, rank - 1, comm, s));
        if (n_lo_r) DOT_NCCL_TRY(nc.recv(r_lo, 2 * n_lo_r, ncclDouble, rank - 1, comm, s));
        DOT_NCCL_TRY(nc.groupEnd());
    }
    void allreduce(double* buf, size_t n, cudaStream_t s) override {
        DOT_NCCL_TRY(nccl_api().allReduce(buf, buf, n, ncclDouble, ncclSum, comm, s));
    }
    bool synchronous() const override { return false; }
};

// host-staged exchange through the caller's callbacks (e.g. torch.distributed on gloo)
struct HostTransport : Transport {
    dot_transport t;
    int rank;
    std::vector<char> a, b;        // staging (pageable; the copies are synchronous here)
    HostTransport(const dot_transport& tr, int r) : t(tr), rank(r) {}
    void stage(std::vector<char>& v, size_t bytes) {
        if (v.size() < bytes) v.resize(bytes);
    }
    void one(int peer, const double2* sd, size_t ns, double2* rd, size_t nr, cudaStream_t s) {
        if (!ns && !nr) return;
        stage(a, ns * sizeof(double2));
        stage(b, nr * sizeof(double2));
        if (ns) DOT_CUDA_TRY(cudaMemcpyAsync(a.data(), sd, ns * sizeof(double2), cudaMemcpyDeviceToHost, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
        if (t.sendrecv(t.ctx, peer, a.data(), ns * sizeof(double2), b.data(), nr * sizeof(double2)) != 0)
            throw Error(DOT_ERR_CUDA, "transport sendrecv failed");
        if (nr) DOT_CUDA_TRY(cudaMemcpyAsync(rd, b.data(), nr * sizeof(double2), cudaMemcpyHostToDevice, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
    }
    void halo(const double2* s_lo, size_t n_lo_s, double2* r_lo, size_t n_lo_r, const double2* s_hi, size_t n_hi_s,
              double2* r_hi, size_t n_hi_r, cudaStream_t s) override {
        one(rank - 1, s_lo, n_lo_s, r_lo, n_lo_r, s);     // lower neighbour first: the chain resolves from rank 0
        one(rank + 1, s_hi, n_hi_s, r_hi, n_hi_r, s);
    }
    void allreduce(double* buf, size_t n, cudaStream_t s) override {
        stage(a, n * sizeof(double));
        DOT_CUDA_TRY(cudaMemcpyAsync(a.data(), buf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
        if (t.allreduce_sum(t.ctx, reinterpret_cast<double*>(a.data()), n) != 0)
            throw Error(DOT_ERR_CUDA, "transport allreduce failed");
        DOT_CUDA_TRY(cudaMemcpyAsync(buf, a.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
    }
    bool synchronous() const override { return true; }
};

// DD solve of the point-combination requests: fills the field caches of every local rank.
// Every rank runs the same multi-shift passes on its own z chunks; after each pass the two
// boundary planes of r_{k+1} and p_k of ALL pairs are packed into one buffer per direction
// and exchanged, and the partial sums (each rank writes only its own slots) are summed.
void dd_solve(dot_dd* G, const std::vector<Req>& reqs) {
    const int L = (int)G->loc.size();
    dot_problem* P0 = G->loc[0];
    const size_t N = P0->N;
    const int PS = P0->nx * P0->ny;
    const int nz = P0->nz, nP = P0->nP, nf = P0->n_freq;
    std::vector<Seg> segs0;
    int n_out = 0;
    for (const Req& q : reqs) {
        segs0.push_back(Seg{q.side, nullptr, q.ncols});
        n_out += nf * q.ncols;
    }
    if (n_out == 0) return;
    if (nf > kMaxShift) throw Error(DOT_ERR_ARG, "more frequencies than the solver's shift capacity (8)");
    const SeedPlan sp = plan_point(P0, segs0);
    const int nb = sp.nseeds / 2, ns = sp.nseeds;
    const DDPlan pl = dd_plan(G, nb);
    const int ntiles = P0->tl.ntiles, nslots = ntiles * pl.C;
    const bool local = (L == G->world) && !G->comm && !G->host;
    std::unique_ptr<Transport> tr;
    if (!local) {
        if (G->comm) tr.reset(new NcclTransport(G->comm, G->rank0));
        else tr.reset(new HostTransport(G->tr, G->rank0));
    }
    // sample ranges of the slabs (samples ascend by node id, slabs are contiguous node ranges)
    std::vector<int32_t> hsamp(nP);
    DOT_CUDA_TRY(cudaMemcpyAsync(hsamp.data(), P0->d_P.get(), nP * sizeof(int32_t), cudaMemcpyDeviceToHost, P0->stream));
    sync(P0);

    struct RankBufs {
        std::vector<DBuf<double>> dcs;
        DBuf<double2> R[2], Pv[2], XP, H, Ps, Xs, sbuf[2], rbuf[2];
        DBuf<double> part;
        DBuf<SeedState> st;
        DBuf<ShiftState> sh;
        DBuf<ShiftCoef> coef;
        DBuf<uint32_t> mask;
        DBuf<int32_t> omap;
        PassArgs a;
        FoldArgs fa;
        int zs = 0, ze = 0, n_lo_s = 0, n_lo_r = 0, n_hi_s = 0, n_hi_r = 0;
    };
    std::vector<RankBufs> B(L);
    const size_t nPp = (size_t)std::max(nP, 1);
    for (int q = 0; q < L; ++q) {
        dot_problem* P = G->loc[q];
        RankBufs& b = B[q];
        const int r = G->rank0 + q;
        std::vector<Seg> segs;
        for (const Req& rq : reqs) {
            b.dcs.emplace_back();
            if (!rq.identity) b.dcs.back() = to_device(P, rq.hc.data(), rq.hc.size(), DOT_HOST);
            segs.push_back(Seg{rq.side, rq.identity ? nullptr : b.dcs.back().get(), rq.ncols});
        }
        for (int i = 0; i < 2; ++i) {
            b.R[i] = DBuf<double2>(P->arena, (size_t)nb * N);
            b.Pv[i] = DBuf<double2>(P->arena, (size_t)nb * N);
        }
        b.XP = DBuf<double2>(P->arena, (size_t)n_out * nPp);
        b.H = DBuf<double2>(P->arena, (size_t)kHist * nb * nPp);
        b.Ps = DBuf<double2>(P->arena, (size_t)ns * nf * nPp);
        b.Xs = DBuf<double2>(P->arena, (size_t)ns * nf * nPp);
        b.part = DBuf<double>(P->arena, 2 * (size_t)nb * nslots * kNumPartials);
        b.st = DBuf<SeedState>(P->arena, 2 * (size_t)ns);
        b.sh = DBuf<ShiftState>(P->arena, 2 * (size_t)ns * kMaxShift);
        b.coef = DBuf<ShiftCoef>(P->arena, (size_t)kHist * ns * kMaxShift);
        b.mask = to_device(P, sp.mask.data(), ns, DOT_HOST);
        b.omap = to_device(P, sp.omap.data(), 3 * ns, DOT_HOST);
        b.zs = pl.zs(r, nz);
        b.ze = pl.ze(r, nz);
        b.n_hi_s = r + 1 < G->world ? std::min(2, b.ze - b.zs) : 0;
        b.n_hi_r = r + 1 < G->world ? std::min(b.ze + 2, pl.ze(r + 1, nz)) - b.ze : 0;
        b.n_lo_s = r > 0 ? std::min(2, b.ze - b.zs) : 0;
        b.n_lo_r = r > 0 ? std::min(2, b.zs - pl.zs(r - 1, nz)) : 0;
        for (int d = 0; d < 2; ++d) {
            b.sbuf[d] = DBuf<double2>(P->arena, (size_t)2 * nb * 2 * PS);
            b.rbuf[d] = DBuf<double2>(P->arena, (size_t)2 * nb * 2 * PS);
        }
        cudaStream_t s = P->stream;
        DOT_CUDA_TRY(cudaMemsetAsync(b.R[0].get(), 0, (size_t)nb * N * sizeof(double2), s));
        DOT_CUDA_TRY(cudaMemsetAsync(b.Pv[0].get(), 0, (size_t)nb * N * sizeof(double2), s));   // p_{-1} = 0
        DOT_CUDA_TRY(cudaMemsetAsync(b.part.get(), 0, 2 * (size_t)nb * nslots * kNumPartials * sizeof(double), s));
        DOT_CUDA_TRY(cudaMemsetAsync(b.coef.get(), 0, (size_t)kHist * ns * kMaxShift * sizeof(ShiftCoef), s));
        DOT_CUDA_TRY(cudaMemsetAsync(b.Ps.get(), 0, (size_t)ns * nf * nPp * sizeof(double2), s));
        DOT_CUDA_TRY(cudaMemsetAsync(b.Xs.get(), 0, (size_t)ns * nf * nPp * sizeof(double2), s));
        DOT_CUDA_TRY(cudaMemsetAsync(b.XP.get(), 0, (size_t)n_out * nPp * sizeof(double2), s));
        for (int e = 0; e < ns;) {
            const int g = sp.seg[e];
            int e2 = e + 1;
            while (e2 < ns && sp.seg[e2] == g && sp.col[e2] == sp.col[e2 - 1] + 1) ++e2;
            if (g >= 0) {
                const Seg& sg = segs[g];
                launch_scatter_seeds(b.R[0].get(), N, sg.side == 0 ? P->d_src.get() : P->d_det.get(),
                                     sg.side == 0 ? P->n_src : P->n_det, sg.d_coeff, sg.ncols,
                                     sg.side == 0 ? P->d_src_scale.get() : P->d_det_scale.get(), sp.col[e], e, e2 - e,
                                     P->op, s);
                P->stats.kernel_launches++;
            }
            e = e2;
        }
        PassArgs& a = b.a;
        a.op = P->op;
        set_edge_coefs(a);
        a.tl = P->tl;
        a.max_iter = P->max_iter;
        a.tol2 = P->tol * P->tol;
        a.nshift = nf;
        for (int f = 0; f < nf; ++f) a.sigma[f] = P->omega[f] / P->nu;
        a.mu = P->d_mu.get();
        for (int i = 0; i < 2; ++i) {
            a.R[i] = b.R[i].get();
            a.Pv[i] = b.Pv[i].get();
            a.part[i] = b.part.get() + (size_t)i * nb * nslots * kNumPartials;
            a.st[i] = b.st.get() + (size_t)i * ns;
            a.sh[i] = b.sh.get() + (size_t)i * ns * kMaxShift;
        }
        a.mask = b.mask.get();
        a.coef = b.coef.get();
        a.npairs = nb;
        a.samp_nodes = P->d_P.get();
        a.samp_off = P->d_off.get();
        a.nP = nP;
        a.H = b.H.get();
        a.zlen = pl.zlen;
        a.nzch_tot = pl.C;
        a.zc0 = pl.cb[r];
        a.nzch = pl.cb[r + 1] - pl.cb[r];
        set_pass_tmaps(a);
        FoldArgs& fa = b.fa;
        fa.s0 = (int)(std::lower_bound(hsamp.begin(), hsamp.end(), (int32_t)((size_t)b.zs * PS)) - hsamp.begin());
        fa.s1 = (int)(std::lower_bound(hsamp.begin(), hsamp.end(), (int32_t)((size_t)b.ze * PS)) - hsamp.begin());
        fa.npairs = nb;
        fa.nshift = nf;
        fa.hist = kHist;
        fa.nsl = nf;
        fa.nP = (int)nPp;
        fa.mask = b.mask.get();
        fa.coef = b.coef.get();
        fa.H = b.H.get();
        fa.Ps = b.Ps.get();
        fa.Xs = b.Xs.get();
        launch_cg_init(a, nb, s);      // full-domain sums of b: identical on every rank
        P->stats.kernel_launches++;
    }
    const size_t halo_per_plane = (size_t)2 * nb * PS;     // double2 per plane: both vectors, all pairs
    const int CHK = 8;
    int k = 0, g = 0, kf = 0;
    for (;;) {
        const int kout = (k + 1) & 1;
        for (int q = 0; q < L; ++q) {
            dot_problem* P = G->loc[q];
            PassArgs& a = B[q].a;
            a.k = k;
            if (!local)   // this rank's slots only; the others arrive through the sum
                DOT_CUDA_TRY(cudaMemsetAsync(a.part[kout], 0, (size_t)nb * nslots * kNumPartials * sizeof(double),
                                             P->stream));
            launch_cg_pass(a, nb, P->stream);
            P->stats.kernel_launches++;
            P->stats.pass_launches++;
            RankBufs& b = B[q];
            // pack the boundary planes of r_{k+1}, p_k (kout arrays) for the neighbours
            launch_pack_planes(a.R[kout], a.Pv[kout], nb, N, PS, b.zs, b.n_lo_s, b.sbuf[0].get(), P->stream);
            launch_pack_planes(a.R[kout], a.Pv[kout], nb, N, PS, b.ze - b.n_hi_s, b.n_hi_s, b.sbuf[1].get(), P->stream);
            P->stats.kernel_launches += 2;
        }
        if (local) {
            for (int q = 0; q < L; ++q) DOT_CUDA_TRY(cudaStreamSynchronize(G->loc[q]->stream));
            cudaStream_t s = G->loc[0]->stream;
            for (int q = 0; q + 1 < L; ++q) {
                DOT_CUDA_TRY(cudaMemcpyAsync(B[q + 1].rbuf[0].get(), B[q].sbuf[1].get(),
                                             B[q + 1].n_lo_r * halo_per_plane * sizeof(double2), cudaMemcpyDeviceToDevice, s));
                DOT_CUDA_TRY(cudaMemcpyAsync(B[q].rbuf[1].get(), B[q + 1].sbuf[0].get(),
                                             B[q].n_hi_r * halo_per_plane * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            }
            for (int q = 0; q < L; ++q)            // owned slot ranges to every other local rank
                for (int q2 = 0; q2 < L; ++q2) {
                    if (q2 == q) continue;
                    const int r = G->rank0 + q;
                    const size_t off = (size_t)pl.cb[r] * ntiles * kNumPartials;
                    const size_t w = (size_t)(pl.cb[r + 1] - pl.cb[r]) * ntiles * kNumPartials * sizeof(double);
                    DOT_CUDA_TRY(cudaMemcpy2DAsync(B[q2].a.part[kout] + off, nslots * kNumPartials * sizeof(double),
                                                   B[q].a.part[kout] + off, nslots * kNumPartials * sizeof(double), w,
                                                   nb, cudaMemcpyDeviceToDevice, s));
                }
            DOT_CUDA_TRY(cudaStreamSynchronize(s));
        } else {
            RankBufs& b = B[0];
            cudaStream_t s = G->loc[0]->stream;
            tr->halo(b.sbuf[0].get(), b.n_lo_s * halo_per_plane, b.rbuf[0].get(), b.n_lo_r * halo_per_plane,
                     b.sbuf[1].get(), b.n_hi_s * halo_per_plane, b.rbuf[1].get(), b.n_hi_r * halo_per_plane, s);
            tr->allreduce(b.a.part[kout], (size_t)nb * nslots * kNumPartials, s);
        }
        for (int q = 0; q < L; ++q) {
            dot_problem* P = G->loc[q];
            RankBufs& b = B[q];
            PassArgs& a = b.a;
            launch_unpack_planes(a.R[kout], a.Pv[kout], nb, N, PS, b.zs - b.n_lo_r, b.n_lo_r, b.rbuf[0].get(), P->stream);
            launch_unpack_planes(a.R[kout], a.Pv[kout], nb, N, PS, b.ze, b.n_hi_r, b.rbuf[1].get(), P->stream);
            P->stats.kernel_launches += 2;
        }
        ++k;
        if (k - kf >= kHist) {
            for (int q = 0; q < L; ++q) {
                B[q].fa.k0 = kf;
                B[q].fa.k1 = k;
                launch_cg_fold(B[q].fa, G->loc[q]->stream);
                G->loc[q]->stats.kernel_launches++;
            }
            kf = k;
        }
        if (k % CHK == 0) {   // pipelined poll (every rank holds the same scalars; rank 0's count)
            dot_problem* P = G->loc[0];
            launch_count_active(B[0].a.st[(k - 1) & 1], nb, P->d_count.get() + (g & 1), P->stream);
            DOT_CUDA_TRY(cudaMemcpyAsync(P->h_count + (g & 1), P->d_count.get() + (g & 1), sizeof(int),
                                         cudaMemcpyDeviceToHost, P->stream));
            DOT_CUDA_TRY(cudaEventRecord(P->poll_ev[g & 1], P->stream));
            bool stop = false;
            if (local || (tr && tr->synchronous())) {
                DOT_CUDA_TRY(cudaEventSynchronize(P->poll_ev[g & 1]));
                stop = P->h_count[g & 1] == 0;
            } else if (g > 0) {
                DOT_CUDA_TRY(cudaEventSynchronize(P->poll_ev[(g - 1) & 1]));
                stop = P->h_count[(g - 1) & 1] == 0;
            }
            ++g;
            if (stop) break;
        }
    }
    // ---- shifted solutions on each rank's own samples, then the sum over ranks
    const size_t nx = (size_t)n_out * nPp;
    for (int q = 0; q < L; ++q) {
        dot_problem* P = G->loc[q];
        B[q].fa.k0 = kf;
        B[q].fa.k1 = k;
        launch_cg_fold(B[q].fa, P->stream);
        launch_cg_finalize(B[q].fa, P->op, B[q].XP.get(), nP, B[q].omap.get(), P->d_P.get(), P->stream);
        P->stats.kernel_launches += 2;
    }
    if (local) {
        for (int q = 0; q < L; ++q) DOT_CUDA_TRY(cudaStreamSynchronize(G->loc[q]->stream));
        cudaStream_t s = G->loc[0]->stream;
        for (int q = 1; q < L; ++q) launch_cadd_inplace(B[0].XP.get(), B[q].XP.get(), nx, s);
        for (int q = 1; q < L; ++q)
            DOT_CUDA_TRY(cudaMemcpyAsync(B[q].XP.get(), B[0].XP.get(), nx * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
    } else {
        tr->allreduce(reinterpret_cast<double*>(B[0].XP.get()), 2 * nx, G->loc[0]->stream);
    }
    // ---- convergence flags, statistics and the field caches of every local rank
    for (int q = 0; q < L; ++q) {
        dot_problem* P = G->loc[q];
        std::vector<SeedState> hs(ns);
        DOT_CUDA_TRY(cudaMemcpyAsync(hs.data(), B[q].a.st[(k - 1) & 1], ns * sizeof(SeedState), cudaMemcpyDeviceToHost,
                                     P->stream));
        sync(P);
        int mx = 0, mn = 1 << 30;
        for (int i = 0; i < ns; ++i) {
            if (!sp.mask[i]) continue;
            if (hs[i].flag == DOT_ERR_NOCONV) throw Error(DOT_ERR_NOCONV, "CG (domain decomposition) did not converge");
            if (hs[i].flag == DOT_ERR_BREAKDOWN) throw Error(DOT_ERR_BREAKDOWN, "CG (domain decomposition) breakdown");
            const int it = hs[i].iters, systems = __builtin_popcount(sp.mask[i]);
            mx = std::max(mx, it);
            mn = std::min(mn, it);
            P->stats.seeds_solved++;
            P->stats.seed_iterations += it;
            P->stats.rhs_solved += systems;
            P->stats.rhs_iterations += (int64_t)systems * it;
            P->stats.pass_bytes += 32.0 * (double)N * it / G->world;
        }
        P->stats.last_max_iters = mx;
        P->stats.last_min_iters = mn;
        size_t off = 0;
        auto blk = std::make_shared<DBuf<double2>>(std::move(B[q].XP));
        for (const Req& rq : reqs) {
            const int n_side = rq.side == 0 ? P->n_src : P->n_det;
            FieldCache& c = P->cache[rq.side];
            const size_t n = (size_t)nf * rq.ncols * nPp;
            c.blk = blk;
            c.X = blk->get() + off;
            off += n;
            c.valid = true;
            c.identity = rq.identity;
            c.ncols = rq.ncols;
            c.coeff = rq.identity ? std::vector<double>() : rq.hc;
            c.sel.clear();
            if (rq.identity)
                for (int a2 = 0; a2 < n_side; ++a2) c.sel.push_back(a2);
        }
        sync(P);
    }
}
}  // namespace

// ===================================================================== C ABI
extern "C" {

const char* dot_version(void) { return "dot_b200 0.1 (sm_100a)"; }

const char* dot_last_error(const dot_problem* P) { return P ? P->err.c_str() : g_create_error.c_str(); }

int dot_create(const dot_config* cfg, dot_problem** out) {
    dot_problem* P = nullptr;
    try {
        if (!cfg || !out) throw Error(DOT_ERR_ARG, "null argument");
        if (cfg->nx < 1 || cfg->ny < 1 || cfg->nz < 2) throw Error(DOT_ERR_ARG, "need nx, ny >= 1, nz >= 2");
        if (cfg->nx > 256) throw Error(DOT_ERR_ARG, "nx > 256 not supported");
        if (!(cfg->Lx > 0 && cfg->Ly > 0 && cfg->Lz > 0 && cfg->D > 0 && cfg->nu > 0))
            throw Error(DOT_ERR_ARG, "extents, D and nu must be positive");
        if (cfg->n_freq < 1 || !cfg->omega) throw Error(DOT_ERR_ARG, "need at least one frequency");
        if (cfg->n_src < 1 || cfg->n_det < 1 || !cfg->src_nodes || !cfg->det_nodes)
            throw Error(DOT_ERR_ARG, "need sources and detectors");
        if (cfg->n_rbf < 0) throw Error(DOT_ERR_ARG, "n_rbf < 0");
        if (!(cfg->gamma > 0 && cfg->eps > 0)) throw Error(DOT_ERR_ARG, "gamma and eps must be positive");
        std::unique_ptr<dot_problem> p(new dot_problem());
        P = p.get();
        P->nx = cfg->nx; P->ny = cfg->ny; P->nz = cfg->nz;
        P->N = (size_t)cfg->nx * cfg->ny * cfg->nz;
        if (P->N >= (1ull << 31)) throw Error(DOT_ERR_ARG, "grid too large (N >= 2^31)");
        P->Lx = cfg->Lx; P->Ly = cfg->Ly; P->Lz = cfg->Lz;
        P->D = cfg->D; P->mua_in = cfg->mua_in; P->mua_out = cfg->mua_out; P->nu = cfg->nu;
        P->gamma = cfg->gamma; P->eps = cfg->eps; P->cutoff = cfg->cutoff;
        P->tol = cfg->tol > 0 ? cfg->tol : 1e-17;
        P->max_iter = cfg->max_iter > 0 ? cfg->max_iter : 4000;
        P->n_freq = cfg->n_freq; P->n_src = cfg->n_src; P->n_det = cfg->n_det;
        P->n_rbf = cfg->n_rbf; P->n_p = 5 * cfg->n_rbf;
        P->omega.assign(cfg->omega, cfg->omega + cfg->n_freq);
        P->hx = P->Lx / (P->nx + 1);
        P->hy = P->Ly / (P->ny + 1);
        P->hz = P->Lz / (P->nz - 1);
        const double V = P->hx * P->hy * P->hz;
        auto take_nodes = [&](const int64_t* nodes, int n, std::vector<int32_t>& dst, std::vector<double>& scale,
                              bool source) {
            std::vector<int64_t> sorted(nodes, nodes + n);
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                throw Error(DOT_ERR_ARG, "duplicate node on one side");
            for (int a = 0; a < n; ++a) {
                if (nodes[a] < 0 || (size_t)nodes[a] >= P->N) throw Error(DOT_ERR_ARG, "node index out of range");
                dst.push_back((int32_t)nodes[a]);
                const int k = (int)(nodes[a] / ((int64_t)P->nx * P->ny));
                const double th = (k == 0 || k == P->nz - 1) ? 0.5 : 1.0;
                scale.push_back(source ? th / V : 1.0);      // b_s = theta e/(hx hy hz), c_d = e (R6)
            }
        };
        take_nodes(cfg->src_nodes, cfg->n_src, P->src, P->src_scale, true);
        take_nodes(cfg->det_nodes, cfg->n_det, P->det, P->det_scale, false);
        P->op.nx = P->nx; P->op.ny = P->ny; P->op.nz = P->nz;
        P->op.cx = P->D / (P->hx * P->hx);
        P->op.cy = P->D / (P->hy * P->hy);
        P->op.cz = P->D / (P->hz * P->hz);
        P->op.robin = 1.0 / (2.0 * P->hz);
        P->op.dint = 2.0 * P->op.cx + 2.0 * P->op.cy + 2.0 * P->op.cz;
        {
            // test knobs: TMA planes in flight, forced tile height
            const char* ePD = std::getenv("DOT_CG_PREFETCH");
            const char* eTY = std::getenv("DOT_CG_TY");
            const char* eRW = std::getenv("DOT_CG_ROWS");
            const char* eNM = std::getenv("DOT_CG_NOMU");
            const char* eXS = std::getenv("DOT_CG_XS");
            P->tl = cg_tiling(P->nx, P->ny, P->nz, ePD ? std::max(1, std::atoi(ePD)) : 2, eTY ? std::atoi(eTY) : 0,
                              eRW ? std::atoi(eRW) : 0, eNM && std::atoi(eNM) != 0, eXS ? std::atoi(eXS) : 0);
            const char* ePL = std::getenv("DOT_CG_PDL");
            P->tl.pdl = !(ePL && std::atoi(ePL) == 0);
        }
        P->pc = PalsConst{P->nx, P->ny, P->nz, P->n_rbf, P->hx, P->hy, P->hz, P->gamma, P->eps, P->cutoff,
                          P->mua_in, P->mua_out};
        DOT_CUDA_TRY(cudaMallocHost(&P->h_count, 2 * sizeof(int)));
        for (auto& e : P->poll_ev) DOT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        {
            int dev = 0;
            DOT_CUDA_TRY(cudaGetDevice(&dev));
            DOT_CUDA_TRY(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, dev));
        }
        *out = p.release();
        return DOT_OK;
    } catch (const Error& e) {
        g_create_error = e.msg;
        return e.code;
    }
}

int dot_destroy(dot_problem* P) {
    if (!P) return DOT_OK;
    cudaStreamSynchronize(P->stream);   // outstanding work may still use the bound workspace
    delete P;
    return DOT_OK;
}

int dot_set_stream(dot_problem* P, void* s) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    P->stream = static_cast<cudaStream_t>(s);
    DOT_API_END(P)
}

size_t dot_workspace_bytes(const dot_problem* P, int32_t max_rhs) {
    if (!P) return 0;
    const size_t N = P->N;
    size_t fixed = N * (sizeof(double) + 4 * sizeof(int32_t)) + scan_temp_bytes(N) + 64 * 1024;
    // support / samples: budget 5% of the nodes on large grids, every node on small ones
    const size_t Kb = std::min(N, std::max(N / 20 + P->n_det + P->n_src, (size_t)65536));
    fixed += Kb * (3 * sizeof(int32_t) + P->n_p * sizeof(double)) + (size_t)P->nz * P->tl.ntiles * 4;
    fixed += (size_t)P->n_freq * P->n_src * P->n_det * sizeof(double2);
    // field caches (sources + detectors, all frequencies) on the samples, plus as much again for
    // the Jacobian's support panels / combined fields, and the host-staged full Jacobian
    fixed += 2 * (size_t)P->n_freq * (P->n_src + P->n_det) * Kb * sizeof(double2);
    fixed += (size_t)P->n_freq * P->n_src * P->n_det * std::max(P->n_p, 1) * sizeof(double2);
    // two frequencies' operand tiles of the segment GEMM (support budget Kb points over all bases)
    fixed += 2 * contract_seg_tma_bytes(P->n_det, P->n_src, (long long)Kb, P->n_rbf);   // double-buffered
    // max_rhs systems = max_rhs / n_freq real seeds (all shifts of one seed together), in pairs
    const size_t pairs = ((size_t)std::max(max_rhs, 1) + 2 * P->n_freq - 1) / (2 * P->n_freq) + 1;
    // dense solutions (dot_solve: every node sampled) of up to 3 complex right-hand sides
    const size_t dense = 3 * per_pair_bytes(P, (int)N, 8, 1) + 6 * N * sizeof(double2);
    // (batches of less than two waves keep a history ring of two fold periods)
    const size_t small_pairs = std::min(pairs, (size_t)(2 * P->num_sms / std::max(P->tl.ntiles, 1) + 1));
    const size_t ring2 = small_pairs * (per_pair_bytes(P, (int)Kb, 2 * kHist, P->n_freq) -
                                        per_pair_bytes(P, (int)Kb, kHist, P->n_freq));
    return fixed + std::max(pairs * per_pair_bytes(P, (int)Kb, kHist, P->n_freq) + ring2, dense) + 64 * Arena::kAlign;
}

int dot_bind_workspace(dot_problem* P, void* ptr, size_t bytes) {
    DOT_API_BEGIN
    if (!P || !ptr) throw Error(DOT_ERR_ARG, "null argument");
    if ((reinterpret_cast<uintptr_t>(ptr) & 255) != 0) throw Error(DOT_ERR_ARG, "workspace must be 256-byte aligned");
    // drop everything allocated from the old workspace
    invalidate_caches(P);
    P->d_S.reset(); P->d_P.reset(); P->d_S_slot.reset(); P->d_det_slot.reset(); P->d_src_slot.reset(); P->d_off.reset(); P->d_G.reset();
    P->d_Dt.reset(); P->d_src.reset(); P->d_det.reset(); P->d_src_scale.reset(); P->d_det_scale.reset();
    P->d_omega_nu.reset(); P->d_mu.reset(); P->d_params.reset(); P->d_flagS.reset(); P->d_flagP.reset();
    P->d_posS.reset(); P->d_posP.reset(); P->d_scan_tmp.reset(); P->d_tot.reset(); P->d_count.reset();
    P->have_params = P->have_data = false;
    P->arena.reset(ptr, bytes);
    const size_t N = P->N;
    P->d_src = to_device(P, P->src.data(), P->src.size(), DOT_HOST);
    P->d_det = to_device(P, P->det.data(), P->det.size(), DOT_HOST);
    P->d_src_scale = to_device(P, P->src_scale.data(), P->src_scale.size(), DOT_HOST);
    P->d_det_scale = to_device(P, P->det_scale.data(), P->det_scale.size(), DOT_HOST);
    std::vector<double> wn(P->n_freq);
    for (int f = 0; f < P->n_freq; ++f) wn[f] = P->omega[f] / P->nu;
    P->d_omega_nu = to_device(P, wn.data(), wn.size(), DOT_HOST);
    P->d_mu = DBuf<double>(P->arena, N);
    P->d_params = DBuf<double>(P->arena, std::max(P->n_p, 1));
    P->d_flagS = DBuf<int32_t>(P->arena, N);
    P->d_flagP = DBuf<int32_t>(P->arena, N);
    P->d_posS = DBuf<int32_t>(P->arena, N);
    P->d_posP = DBuf<int32_t>(P->arena, N);
    P->d_scan_tmp = DBuf<int32_t>(P->arena, scan_temp_bytes(N) / 4 + 1);
    P->d_tot = DBuf<int32_t>(P->arena, 4);
    P->d_count = DBuf<int>(P->arena, 4);
    sync(P);
    DOT_API_END(P)
}

int dot_enable_timing(dot_problem* P, int on) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    P->timing = on != 0;
    DOT_API_END(P)
}

int dot_get_stats(const dot_problem* P, dot_stats* out) {
    if (!P || !out) return DOT_ERR_ARG;
    *out = P->stats;
    out->support_K = P->K;
    out->n_samples = P->nP;
    return DOT_OK;
}

int dot_reset_stats(dot_problem* P) {
    if (!P) return DOT_ERR_ARG;
    P->stats = dot_stats{};
    return DOT_OK;
}

int dot_set_data(dot_problem* P, const double* data, int where) {
    DOT_API_BEGIN
    if (!P || !data) throw Error(DOT_ERR_ARG, "null argument");
    require_bound(P);
    const size_t n = (size_t)P->n_freq * P->n_det * P->n_src;
    DBuf<double2> tmp = to_device(P, reinterpret_cast<const double2*>(data), n, where);
    P->d_Dt.reset();
    P->d_Dt = DBuf<double2>(P->arena, n);
    launch_transpose_data(tmp.get(), P->n_freq, P->n_det, P->n_src, P->d_Dt.get(), P->stream);
    P->stats.kernel_launches++;
    sync(P);
    P->have_data = true;
    DOT_API_END(P)
}

int dot_set_params(dot_problem* P, const double* p, int where) {
    DOT_API_BEGIN
    if (!P || (!p && P->n_p > 0)) throw Error(DOT_ERR_ARG, "null argument");
    require_bound(P);
    const size_t N = P->N;
    invalidate_caches(P);
    P->params = host_copy(P, p, P->n_p, where);
    for (double v : P->params)
        if (!std::isfinite(v)) throw Error(DOT_ERR_ARG, "non-finite parameter");
    DOT_CUDA_TRY(cudaMemcpyAsync(P->d_params.get(), P->params.data(), P->n_p * sizeof(double), cudaMemcpyHostToDevice,
                                 P->stream));
    cudaStream_t s = P->stream;
    launch_pals_eval(P->pc, P->d_params.get(), P->d_mu.get(), P->d_flagS.get(), P->d_flagP.get(), s);
    launch_mark_nodes(P->d_flagP.get(), P->d_det.get(), P->n_det, s);
    launch_mark_nodes(P->d_flagP.get(), P->d_src.get(), P->n_src, s);   // reciprocity / adjoint samples
    launch_exclusive_scan(P->d_flagS.get(), P->d_posS.get(), N, P->d_tot.get(), P->d_scan_tmp.get(), s);
    launch_exclusive_scan(P->d_flagP.get(), P->d_posP.get(), N, P->d_tot.get() + 1, P->d_scan_tmp.get(), s);
    P->stats.kernel_launches += 8;
    int32_t tot[2];
    DOT_CUDA_TRY(cudaMemcpyAsync(tot, P->d_tot.get(), 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    sync(P);
    P->K = tot[0];
    P->nP = tot[1];
    P->d_S.reset(); P->d_P.reset(); P->d_S_slot.reset(); P->d_det_slot.reset(); P->d_src_slot.reset(); P->d_off.reset(); P->d_G.reset();
    P->d_S = DBuf<int32_t>(P->arena, std::max(P->K, 1));
    P->d_P = DBuf<int32_t>(P->arena, std::max(P->nP, 1));
    P->d_S_slot = DBuf<int32_t>(P->arena, std::max(P->K, 1));
    P->d_det_slot = DBuf<int32_t>(P->arena, P->n_det);
    P->d_src_slot = DBuf<int32_t>(P->arena, P->n_src);
    P->d_off = DBuf<int32_t>(P->arena, (size_t)P->nz * P->tl.ntiles + 1);
    P->d_G = DBuf<double>(P->arena, std::max<size_t>((size_t)P->K * P->n_p, 1));
    P->d_seg.reset();
    P->d_segoff.reset();
    P->d_segslot.reset();
    P->d_Gseg.reset();
    P->d_ktile.reset();
    P->d_kto.reset();
    P->d_jorder.reset();
    P->gsp = GSparse{};
    launch_compact(P->d_flagS.get(), P->d_posS.get(), N, P->d_S.get(), s);
    launch_compact(P->d_flagP.get(), P->d_posP.get(), N, P->d_P.get(), s);
    launch_gather_rank(P->d_posP.get(), P->d_S.get(), P->K, P->d_S_slot.get(), s);
    launch_gather_rank(P->d_posP.get(), P->d_det.get(), P->n_det, P->d_det_slot.get(), s);
    launch_gather_rank(P->d_posP.get(), P->d_src.get(), P->n_src, P->d_src_slot.get(), s);
    launch_pals_grad(P->pc, P->d_params.get(), P->d_S.get(), P->K, P->d_G.get(), s);
    {   // block sparsity of G by basis for the Jacobian contraction (L972); DOT_CONTRACT=dense skips it
        const char* eC = std::getenv("DOT_CONTRACT");
        const size_t nfl = (size_t)P->n_rbf * P->K;
        if (nfl > 0 && !(eC && std::string(eC) == "dense")) {
            DBuf<int32_t> F(P->arena, nfl), Fpos(P->arena, nfl), tmp(P->arena, scan_temp_bytes(nfl) / 4 + 1);
            launch_rbf_flags(P->d_G.get(), P->K, P->n_rbf, F.get(), s);
            launch_exclusive_scan(F.get(), Fpos.get(), nfl, P->d_tot.get() + 2, tmp.get(), s);
            int32_t T = 0;
            DOT_CUDA_TRY(cudaMemcpyAsync(&T, P->d_tot.get() + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            sync(P);
            P->d_seg = DBuf<int32_t>(P->arena, std::max(T, 1));
            P->d_segoff = DBuf<int32_t>(P->arena, P->n_rbf + 1);
            launch_rbf_segments(F.get(), Fpos.get(), P->K, P->n_rbf, P->d_tot.get() + 2, P->d_seg.get(),
                                P->d_segoff.get(), s);
            std::vector<int32_t> hoff(P->n_rbf + 1);
            DOT_CUDA_TRY(cudaMemcpyAsync(hoff.data(), P->d_segoff.get(), hoff.size() * sizeof(int32_t),
                                         cudaMemcpyDeviceToHost, s));
            P->stats.kernel_launches += 5;
            sync(P);
            // k-tiles of 16 points per basis (the segment GEMM's blocks never straddle bases)
            std::vector<int32_t> kto(P->n_rbf + 1, 0), ktile;
            for (int j = 0; j < P->n_rbf; ++j) {
                kto[j + 1] = kto[j] + (hoff[j + 1] - hoff[j] + 15) / 16;
                for (int t = hoff[j]; t < hoff[j + 1]; t += 16) {
                    ktile.push_back(t);
                    ktile.push_back(hoff[j + 1]);
                    ktile.push_back(j);
                    ktile.push_back(0);
                }
            }
            if (ktile.empty()) ktile.assign(4, 0);
            std::vector<int32_t> jorder(P->n_rbf);
            for (int j = 0; j < P->n_rbf; ++j) jorder[j] = j;
            std::stable_sort(jorder.begin(), jorder.end(),
                             [&](int a, int b) { return kto[a + 1] - kto[a] > kto[b + 1] - kto[b]; });
            P->d_kto = to_device(P, kto.data(), kto.size(), DOT_HOST);
            P->d_ktile = to_device(P, ktile.data(), ktile.size(), DOT_HOST);
            P->d_jorder = to_device(P, jorder.data(), std::max<size_t>(jorder.size(), 1), DOT_HOST);
            int maxkt = 0;
            for (int j = 0; j < P->n_rbf; ++j) maxkt = std::max(maxkt, kto[j + 1] - kto[j]);
            P->gsp = GSparse{P->d_seg.get(), P->d_segoff.get(), P->n_rbf, T,
                             reinterpret_cast<const int4*>(P->d_ktile.get()), P->d_kto.get(), kto[P->n_rbf],
                             P->d_jorder.get(), maxkt};
            P->d_segslot = DBuf<int32_t>(P->arena, std::max(T, 1));
            P->d_Gseg = DBuf<double>(P->arena, 5 * (size_t)std::max(T, 1));
            launch_compose_index(P->d_seg.get(), T, P->d_S_slot.get(), P->d_segslot.get(), s);
            launch_seg_weights(P->d_G.get(), P->n_p, P->gsp, P->d_Gseg.get(), s);
            P->stats.kernel_launches += 2;
        }
    }
    launch_sample_offsets(P->d_P.get(), P->nP, P->nx, P->ny, P->nz, P->tl.TY, P->tl.nty, P->d_off.get(), s);
    P->stats.kernel_launches += 6;
    sync(P);
    P->have_params = true;
    DOT_API_END(P)
}

int dot_misfit(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld, int where,
               double* misfit_out, double* resid_out) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    require_params(P);
    if (!P->have_data) throw Error(DOT_ERR_STATE, "no data (dot_set_data)");
    check_side_matrix(W, P->n_src, ls, "W");
    check_side_matrix(V, P->n_det, ld, "V");
    cudaStream_t s = P->stream;
    const int nf = P->n_freq, ns = P->n_src, nd = P->n_det;
    std::vector<double> hW = W ? host_copy(P, W, (size_t)ns * ls, where) : std::vector<double>();
    DBuf<double2> tmpX;
    const double2* X = get_fields(P, 0, hW, W == nullptr, ls, tmpX);
    // Mt[f][i][d] = X[f][i][det_slot[d]]
    DBuf<double2> Rt(P->arena, (size_t)nf * ls * nd);
    launch_gather_cols(nf, ls, nd, X, (size_t)ls * P->nP, P->nP, P->d_det_slot.get(), Rt.get(), (size_t)ls * nd, nd, s);
    // DWt[f][i][d] = sum_s W[s][i] Dt[f][s][d]
    DBuf<double2> DWt(P->arena, (size_t)nf * ls * nd);
    DBuf<double> dW;
    if (W) dW = to_device(P, hW.data(), hW.size(), DOT_HOST);
    launch_rc_gemm(nf, ls, nd, ns, W ? dW.get() : nullptr, ls, P->d_Dt.get(), (size_t)ns * nd, nd, 1, DWt.get(),
                   (size_t)ls * nd, nd, 1, s);
    launch_csub_inplace(Rt.get(), DWt.get(), (size_t)nf * ls * nd, s);
    // S[f][j][i] = sum_d V[d][j] Rt[f][i][d]
    DBuf<double2> S(P->arena, (size_t)nf * ld * ls);
    DBuf<double> dV;
    std::vector<double> hV;
    if (V) {
        hV = host_copy(P, V, (size_t)nd * ld, where);
        dV = to_device(P, hV.data(), hV.size(), DOT_HOST);
    }
    launch_rc_gemm(nf, ld, ls, nd, V ? dV.get() : nullptr, ld, Rt.get(), (size_t)ls * nd, 1, nd, S.get(),
                   (size_t)ld * ls, ls, 1, s);
    DBuf<double> d_m(P->arena, 1);
    launch_sumsq(S.get(), (size_t)nf * ld * ls, d_m.get(), s);
    P->stats.kernel_launches += 5;
    double m = 0;
    DOT_CUDA_TRY(cudaMemcpyAsync(&m, d_m.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    if (resid_out)
        DOT_CUDA_TRY(cudaMemcpyAsync(resid_out, S.get(), (size_t)nf * ld * ls * sizeof(double2),
                                     where == DOT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    sync(P);
    if (misfit_out) *misfit_out = m;
    DOT_API_END(P)
}

// block-sparse segment GEMM of basis-ordered panels
static void contract_seg(dot_problem* P, int nf, int T, int ld, int ls, const double2* L, size_t lbs, const double2* U,
                         size_t ubs, double2* J) {
    contract_seg_tma(nf, T, ld, ls, P->n_p, L, lbs, U, ubs, P->d_Gseg.get(), P->gsp, J, P->arena, P->stream,
                     &P->stats.kernel_launches, &P->stats.contract_dmma_flops);
}

int dot_jacobian(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld, int where,
                 double* J_out) {
    DOT_API_BEGIN
    if (!P || !J_out) throw Error(DOT_ERR_ARG, "null argument");
    require_params(P);
    check_side_matrix(W, P->n_src, ls, "W");
    check_side_matrix(V, P->n_det, ld, "V");
    cudaStream_t s = P->stream;
    const int nf = P->n_freq, K = P->K;
    std::vector<double> hW = W ? host_copy(P, W, (size_t)P->n_src * ls, where) : std::vector<double>();
    std::vector<double> hV = V ? host_copy(P, V, (size_t)P->n_det * ld, where) : std::vector<double>();
    prefetch_fields(P, {Req{0, hW, W == nullptr, ls}, Req{1, hV, V == nullptr, ld}});   // one joint batch
    DBuf<double2> tmpU, tmpL;
    const double2* XU = get_fields(P, 0, hW, W == nullptr, ls, tmpU);
    const double2* XL = get_fields(P, 1, hV, V == nullptr, ld, tmpL);
    const size_t nJ = (size_t)nf * ld * ls * P->n_p;
    DBuf<double2> Jtmp;
    double2* J = reinterpret_cast<double2*>(J_out);
    if (where == DOT_HOST) {
        Jtmp = DBuf<double2>(P->arena, std::max<size_t>(nJ, 1));
        J = Jtmp.get();
    }
    // large panels: support fields gathered in basis order (contiguous k per basis); else S order
    const bool seg = contract_seg_applies(ld, ls, &P->gsp, P->n_p);
    const int Kp = seg ? (int)P->gsp.total : K;
    const int32_t* gidx = seg ? P->d_segslot.get() : P->d_S_slot.get();
    DBuf<double2> US(P->arena, std::max<size_t>((size_t)nf * ls * Kp, 1)), LS(P->arena, std::max<size_t>((size_t)nf * ld * Kp, 1));
    launch_gather_cols(nf, ls, Kp, XU, (size_t)ls * P->nP, P->nP, gidx, US.get(), (size_t)ls * Kp, Kp, s);
    launch_gather_cols(nf, ld, Kp, XL, (size_t)ld * P->nP, P->nP, gidx, LS.get(), (size_t)ld * Kp, Kp, s);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (P->timing) {
        e0 = event_at(P, 0);
        e1 = event_at(P, 1);
        DOT_CUDA_TRY(cudaEventRecord(e0, s));
    }
    if (seg)
        contract_seg(P, nf, Kp, ld, ls, LS.get(), (size_t)ld * Kp, US.get(), (size_t)ls * Kp, J);
    else
        launch_contract(nf, K, ld, ls, P->n_p, LS.get(), (size_t)ld * K, US.get(), (size_t)ls * K, P->d_G.get(), J, s,
                        &P->gsp, &P->arena, &P->stats.kernel_launches);
    P->stats.kernel_launches += 3;
    if (P->timing) {
        DOT_CUDA_TRY(cudaEventRecord(e1, s));
        DOT_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        DOT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        P->stats.contract_ms += ms;
        if (seg) P->stats.gemm_ms += ms;
    }
    // useful flops: 4 per (pair, point, parameter) with a nonzero weight block (5 per basis
    // over its points when the block-sparse kernel runs; the dense K x n_p otherwise)
    P->stats.contract_flops += 4.0 * nf * ld * ls * (P->gsp.seg ? 5.0 * (double)P->gsp.total : (double)K * P->n_p);
    if (seg) P->stats.gemm_flops += 4.0 * nf * ld * ls * 5.0 * (double)P->gsp.total;
    P->stats.contract_flops_dense += 4.0 * nf * ld * ls * (double)K * P->n_p;
    if (where == DOT_HOST) {
        DOT_CUDA_TRY(cudaMemcpyAsync(J_out, J, nJ * sizeof(double2), cudaMemcpyDeviceToHost, s));
    }
    sync(P);
    DOT_API_END(P)
}

int dot_optimize_directions(dot_problem* P, int32_t k, const double* W, int32_t ls, const double* V, int32_t ld,
                            int where, double* W_out, double* V_out, double* objective_out) {
    DOT_API_BEGIN
    if (!P || !W || !V || !W_out || !V_out) throw Error(DOT_ERR_ARG, "null argument");
    require_params(P);
    if (k < 0 || k >= ls || k >= ld) throw Error(DOT_ERR_ARG, "need 0 <= k < min(ls, ld)");
    std::vector<double> hW = host_copy(P, W, (size_t)P->n_src * ls, where);
    std::vector<double> hV = host_copy(P, V, (size_t)P->n_det * ld, where);
    prefetch_fields(P, {Req{0, {}, true, P->n_src}, Req{1, {}, true, P->n_det}});
    DBuf<double2> t0, t1;
    const double2* XU = get_fields(P, 0, {}, true, P->n_src, t0);
    const double2* XL = get_fields(P, 1, {}, true, P->n_det, t1);
    OptContext oc{P->arena, P->stream, P->n_freq, P->n_src, P->n_det, P->n_p, P->K, P->nP,
                  XU, XL, P->d_S_slot.get(), P->d_G.get(), &P->stats.kernel_launches, &P->gsp};
    double obj = optimize_two_phase(oc, k, hW, ls, hV, ld);
    if (objective_out) *objective_out = obj;
    if (where == DOT_HOST) {
        std::memcpy(W_out, hW.data(), hW.size() * sizeof(double));
        std::memcpy(V_out, hV.data(), hV.size() * sizeof(double));
    } else {
        DOT_CUDA_TRY(cudaMemcpyAsync(W_out, hW.data(), hW.size() * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        DOT_CUDA_TRY(cudaMemcpyAsync(V_out, hV.data(), hV.size() * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        sync(P);
    }
    DOT_API_END(P)
}

int dot_optimize_directions_subspace(dot_problem* P, int32_t k, int32_t iters, int32_t block, const double* W,
                                     int32_t ls, const double* V, int32_t ld, const double* X0_src,
                                     const double* X0_det, int where, double* W_out, double* V_out,
                                     double* objective_out) {
    DOT_API_BEGIN
    if (!P || !W || !V || !X0_src || !X0_det || !W_out || !V_out) throw Error(DOT_ERR_ARG, "null argument");
    require_params(P);
    if (k < 0 || k >= ls || k >= ld) throw Error(DOT_ERR_ARG, "need 0 <= k < min(ls, ld)");
    if (iters < 1 || block < 1) throw Error(DOT_ERR_ARG, "need iters >= 1 and block >= 1");
    if (block > P->n_src - ls + k || block > P->n_det - ld + k)
        throw Error(DOT_ERR_ARG, "block larger than the complement of the kept directions");
    std::vector<double> hW = host_copy(P, W, (size_t)P->n_src * ls, where);
    std::vector<double> hV = host_copy(P, V, (size_t)P->n_det * ld, where);
    std::vector<double> hXs = host_copy(P, X0_src, (size_t)P->n_src * block * std::max(k, 1), where);
    std::vector<double> hXd = host_copy(P, X0_det, (size_t)P->n_det * block * std::max(k, 1), where);
    const int nf = P->n_freq, K = P->K, nP = P->nP;
    cudaStream_t s = P->stream;
    SubspaceOps ops;
    ops.fields = [&](int side, const double* d_coeff, int ncols, double2* out, double2* outP) {
        DBuf<double2> XPt;
        double2* XP = outP;
        if (!XP) {
            XPt = DBuf<double2>(P->arena, std::max<size_t>((size_t)nf * ncols * nP, 1));
            XP = XPt.get();
        }
        solve_batch(P, {Seg{side, d_coeff, ncols}}, nullptr, {}, XP, nf * ncols, nP, P->d_P.get(), P->d_off.get());
        launch_gather_cols(nf, ncols, K, XP, (size_t)ncols * nP, nP, P->d_S_slot.get(), out, (size_t)ncols * K, K, s);
        P->stats.kernel_launches++;
    };
    ops.solve_support = [&](const double2* w, int nvec, int side, double2* out) {
        const int nr = nf * nvec;
        DBuf<double2> R(P->arena, (size_t)nr * P->N);
        DOT_CUDA_TRY(cudaMemsetAsync(R.get(), 0, (size_t)nr * P->N * sizeof(double2), s));
        launch_scatter_support(R.get(), P->N, nr, P->d_S.get(), K, w, s);
        std::vector<int32_t> fo(nr);
        for (int r = 0; r < nr; ++r) fo[r] = r / nvec;
        DBuf<double2> XP(P->arena, std::max<size_t>((size_t)nr * nP, 1));
        solve_batch(P, {}, R.get(), fo, XP.get(), nr, nP, P->d_P.get(), P->d_off.get());
        const int n_side = side == 0 ? P->n_src : P->n_det;
        launch_gather_cols(nf, nvec, n_side, XP.get(), (size_t)nvec * nP, nP,
                           side == 0 ? P->d_src_slot.get() : P->d_det_slot.get(), out, (size_t)nvec * n_side, n_side, s);
        // b_s^T x = theta_s / (hx hy hz) x[src_s]  (reading R6), on the device
        if (side == 0) launch_scale_cols(out, (size_t)nr, n_side, P->d_src_scale.get(), s);
        P->stats.kernel_launches += side == 0 ? 3 : 2;
    };
    ops.start_fields = [&](const std::vector<double>& W0, int l0, const std::vector<double>& V0, int d0, double2* zw,
                           double2* yv, double2* zwP, double2* yvP) {
        prefetch_fields(P, {Req{0, W0, false, l0}, Req{1, V0, false, d0}});   // no solves after jacobian(W, V)
        DBuf<double2> t0, t1;
        const double2* XZ = get_fields(P, 0, W0, false, l0, t0);
        const double2* XY = get_fields(P, 1, V0, false, d0, t1);
        launch_gather_cols(nf, l0, K, XZ, (size_t)l0 * nP, nP, P->d_S_slot.get(), zw, (size_t)l0 * K, K, s);
        launch_gather_cols(nf, d0, K, XY, (size_t)d0 * nP, nP, P->d_S_slot.get(), yv, (size_t)d0 * K, K, s);
        DOT_CUDA_TRY(cudaMemcpyAsync(zwP, XZ, (size_t)nf * l0 * nP * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        DOT_CUDA_TRY(cudaMemcpyAsync(yvP, XY, (size_t)nf * d0 * nP * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        P->stats.kernel_launches += 2;
        sync(P);                                       // t0 / t1 are released on return
    };
    ops.finish = [&](const std::vector<double>& W1, int a1, DBuf<double2>& zwP, const std::vector<double>& V1, int b1,
                     DBuf<double2>& yvP) {
        const std::vector<double>* cf[2] = {&W1, &V1};
        const int nc[2] = {a1, b1};
        DBuf<double2>* fb[2] = {&zwP, &yvP};
        for (int side = 0; side < 2; ++side) {
            FieldCache& c = P->cache[side];
            c.blk = std::make_shared<DBuf<double2>>(std::move(*fb[side]));
            c.X = c.blk->get();
            c.valid = true;
            c.identity = false;
            c.ncols = nc[side];
            c.coeff = *cf[side];
            c.sel.clear();
        }
    };
    OptContext oc{P->arena, P->stream, P->n_freq, P->n_src, P->n_det, P->n_p, P->K, P->nP,
                  nullptr, nullptr, P->d_S_slot.get(), P->d_G.get(), &P->stats.kernel_launches, &P->gsp};
    double obj = optimize_two_phase_subspace(oc, ops, k, iters, block, hW, ls, hV, ld, hXs, hXd);
    if (objective_out) *objective_out = obj;
    if (where == DOT_HOST) {
        std::memcpy(W_out, hW.data(), hW.size() * sizeof(double));
        std::memcpy(V_out, hV.data(), hV.size() * sizeof(double));
    } else {
        DOT_CUDA_TRY(cudaMemcpyAsync(W_out, hW.data(), hW.size() * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        DOT_CUDA_TRY(cudaMemcpyAsync(V_out, hV.data(), hV.size() * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        sync(P);
    }
    DOT_API_END(P)
}

int dot_prefetch_fields(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld, int where) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    require_params(P);
    std::vector<Req> reqs;
    if (ls > 0) {
        check_side_matrix(W, P->n_src, ls, "W");
        reqs.push_back(Req{0, W ? host_copy(P, W, (size_t)P->n_src * ls, where) : std::vector<double>(), W == nullptr, ls});
    }
    if (ld > 0) {
        check_side_matrix(V, P->n_det, ld, "V");
        reqs.push_back(Req{1, V ? host_copy(P, V, (size_t)P->n_det * ld, where) : std::vector<double>(), V == nullptr, ld});
    }
    prefetch_fields(P, reqs);
    DOT_API_END(P)
}

int dot_absorption(dot_problem* P, double* mu_out, int where) {
    DOT_API_BEGIN
    if (!P || !mu_out) throw Error(DOT_ERR_ARG, "null argument");
    require_params(P);
    from_device(P, mu_out, P->d_mu.get(), P->N, where);
    sync(P);
    DOT_API_END(P)
}

int dot_support(dot_problem* P, int32_t* K_out, int64_t* nodes_out, double* G_out, int where) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    require_params(P);
    if (K_out) *K_out = P->K;
    if (nodes_out && P->K) {
        std::vector<int32_t> h(P->K);
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), P->d_S.get(), P->K * sizeof(int32_t), cudaMemcpyDeviceToHost, P->stream));
        sync(P);
        std::vector<int64_t> h64(h.begin(), h.end());
        if (where == DOT_HOST) std::memcpy(nodes_out, h64.data(), h64.size() * 8);
        else DOT_CUDA_TRY(cudaMemcpyAsync(nodes_out, h64.data(), h64.size() * 8, cudaMemcpyHostToDevice, P->stream));
    }
    if (G_out && P->K) from_device(P, G_out, P->d_G.get(), (size_t)P->K * P->n_p, where);
    sync(P);
    DOT_API_END(P)
}

int dot_samples(dot_problem* P, int32_t* n_out, int64_t* nodes_out, int where) {
    DOT_API_BEGIN
    if (!P) throw Error(DOT_ERR_ARG, "null problem");
    require_params(P);
    if (n_out) *n_out = P->nP;
    if (nodes_out && P->nP) {
        std::vector<int32_t> h(P->nP);
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), P->d_P.get(), P->nP * sizeof(int32_t), cudaMemcpyDeviceToHost, P->stream));
        sync(P);
        std::vector<int64_t> h64(h.begin(), h.end());
        if (where == DOT_HOST) std::memcpy(nodes_out, h64.data(), h64.size() * 8);
        else DOT_CUDA_TRY(cudaMemcpyAsync(nodes_out, h64.data(), h64.size() * 8, cudaMemcpyHostToDevice, P->stream));
        sync(P);
    }
    DOT_API_END(P)
}

int dot_apply(dot_problem* P, int32_t freq, int32_t nrhs, const double* u, double* Au, int where) {
    DOT_API_BEGIN
    if (!P || !u || !Au) throw Error(DOT_ERR_ARG, "null argument");
    require_params(P);
    if (freq < 0 || freq >= P->n_freq || nrhs < 1) throw Error(DOT_ERR_ARG, "bad freq / nrhs");
    const size_t n = (size_t)nrhs * P->N;
    DBuf<double2> du = to_device(P, reinterpret_cast<const double2*>(u), n, where);
    DBuf<double2> dA(P->arena, n);
    std::vector<double> sh(nrhs, P->omega[freq] / P->nu);
    DBuf<double> dsh = to_device(P, sh.data(), sh.size(), DOT_HOST);
    launch_apply(P->op, P->d_mu.get(), dsh.get(), du.get(), dA.get(), nrhs, P->stream);
    P->stats.kernel_launches++;
    from_device(P, reinterpret_cast<double2*>(Au), dA.get(), n, where);
    sync(P);
    DOT_API_END(P)
}

int dot_solve(dot_problem* P, int32_t nrhs, const int32_t* freq, const double* b, double* x, int where,
              int32_t* iters_out) {
    DOT_API_BEGIN
    if (!P || !freq || !b || !x || nrhs < 1) throw Error(DOT_ERR_ARG, "bad argument");
    require_params(P);
    const size_t n = (size_t)nrhs * P->N;
    DBuf<double2> db = to_device(P, reinterpret_cast<const double2*>(b), n, where);
    std::vector<int32_t> fh(nrhs);
    if (where == DOT_HOST) {
        std::copy(freq, freq + nrhs, fh.begin());
    } else {
        DOT_CUDA_TRY(cudaMemcpyAsync(fh.data(), freq, nrhs * sizeof(int32_t), cudaMemcpyDeviceToHost, P->stream));
        sync(P);
    }
    // dense solutions: the sample list is every node (identity), with its (plane, tile) ranges
    std::vector<int32_t> all(P->N);
    for (size_t i = 0; i < P->N; ++i) all[i] = (int32_t)i;
    DBuf<int32_t> dall = to_device(P, all.data(), all.size(), DOT_HOST);
    DBuf<int32_t> doff(P->arena, (size_t)P->nz * P->tl.ntiles + 1);
    launch_sample_offsets(dall.get(), (int)P->N, P->nx, P->ny, P->nz, P->tl.TY, P->tl.nty, doff.get(), P->stream);
    DBuf<double2> dx(P->arena, n);
    auto it = solve_batch(P, {}, db.get(), fh, dx.get(), nrhs, (int)P->N, dall.get(), doff.get());
    from_device(P, reinterpret_cast<double2*>(x), dx.get(), n, where);
    sync(P);
    if (iters_out) std::copy(it.begin(), it.end(), iters_out);
    DOT_API_END(P)
}

int dot_solve_sampled(dot_problem* P, int32_t side, const double* coeff, int32_t ncols, int where, double* X_out) {
    DOT_API_BEGIN
    if (!P || (side != 0 && side != 1)) throw Error(DOT_ERR_ARG, "bad argument");
    require_params(P);
    const int n_side = side == 0 ? P->n_src : P->n_det;
    check_side_matrix(coeff, n_side, ncols, "coeff");
    std::vector<double> hc = coeff ? host_copy(P, coeff, (size_t)n_side * ncols, where) : std::vector<double>();
    DBuf<double2> tmp;
    const double2* X = get_fields(P, side, hc, coeff == nullptr, ncols, tmp);
    if (X_out) from_device(P, reinterpret_cast<double2*>(X_out), X, (size_t)P->n_freq * ncols * P->nP, where);
    sync(P);
    DOT_API_END(P)
}

int dot_fields_on_support(dot_problem* P, int32_t side, const double* coeff, int32_t ncols, int where,
                          double* out) {
    DOT_API_BEGIN
    if (!P || (side != 0 && side != 1) || !out) throw Error(DOT_ERR_ARG, "bad argument");
    require_params(P);
    const int n_side = side == 0 ? P->n_src : P->n_det;
    check_side_matrix(coeff, n_side, ncols, "coeff");
    std::vector<double> hc = coeff ? host_copy(P, coeff, (size_t)n_side * ncols, where) : std::vector<double>();
    DBuf<double2> tmp;
    const double2* X = get_fields(P, side, hc, coeff == nullptr, ncols, tmp);
    const size_t n = (size_t)P->n_freq * ncols * P->K;
    if (n) {
        DBuf<double2> g;
        double2* dst = reinterpret_cast<double2*>(out);
        if (where == DOT_HOST) {
            g = DBuf<double2>(P->arena, n);
            dst = g.get();
        }
        launch_gather_cols(P->n_freq, ncols, P->K, X, (size_t)ncols * P->nP, P->nP, P->d_S_slot.get(), dst,
                           (size_t)ncols * P->K, P->K, P->stream);
        P->stats.kernel_launches++;
        if (where == DOT_HOST) from_device(P, reinterpret_cast<double2*>(out), g.get(), n, where);
    }
    sync(P);
    DOT_API_END(P)
}

int dot_nccl_unique_id(unsigned char* out) {
    try {
        if (!out) throw Error(DOT_ERR_ARG, "null argument");
        NcclApi& nc = nccl_api();
        if (!nc.ok) throw Error(DOT_ERR_CUDA, nc.why);
        ncclUniqueId id;
        DOT_NCCL_TRY(nc.getUniqueId(&id));
        std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
        return DOT_OK;
    } catch (const Error& e) {
        g_create_error = e.msg;
        return e.code;
    }
}

int dot_dd_create(dot_problem* const* local, int32_t nlocal, int32_t rank0, int32_t world,
                  const unsigned char* nccl_id, dot_dd** out) {
    std::unique_ptr<dot_dd> G;
    try {
        if (!local || !out || nlocal < 1 || world < 1 || rank0 < 0 || rank0 + nlocal > world)
            throw Error(DOT_ERR_ARG, "bad rank layout");
        if (nlocal < world && nlocal != 1)
            throw Error(DOT_ERR_ARG, "either all ranks in this process or one rank per process");
        G.reset(new dot_dd());
        for (int q = 0; q < nlocal; ++q) {
            if (!local[q]) throw Error(DOT_ERR_ARG, "null problem");
            const dot_problem* A = local[0];
            const dot_problem* Bq = local[q];
            if (Bq->nx != A->nx || Bq->ny != A->ny || Bq->nz != A->nz || Bq->n_src != A->n_src ||
                Bq->n_det != A->n_det || Bq->n_freq != A->n_freq || Bq->tl.TY != A->tl.TY)
                throw Error(DOT_ERR_ARG, "ranks must hold the same problem");
            G->loc.push_back(local[q]);
        }
        G->rank0 = rank0;
        G->world = world;
        if (nlocal < world || (nccl_id && world == 1)) {   // one rank per process (world 1: NCCL smoke)
            if (!nccl_id) throw Error(DOT_ERR_ARG, "multi-process decomposition needs an NCCL unique id");
            NcclApi& nc = nccl_api();
            if (!nc.ok) throw Error(DOT_ERR_CUDA, nc.why);
            ncclUniqueId id;
            std::memcpy(id.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
            DOT_NCCL_TRY(nc.commInitRank(&G->comm, world, id, rank0));
        }
        *out = G.release();
        return DOT_OK;
    } catch (const Error& e) {
        g_create_error = e.msg;
        return e.code;
    }
}

int dot_dd_create_transport(dot_problem* local, int32_t rank, int32_t world, const dot_transport* t, dot_dd** out) {
    try {
        if (!local || !out || !t || !t->sendrecv || !t->allreduce_sum || world < 2 || rank < 0 || rank >= world)
            throw Error(DOT_ERR_ARG, "bad transport decomposition arguments");
        std::unique_ptr<dot_dd> G(new dot_dd());
        G->loc.push_back(local);
        G->rank0 = rank;
        G->world = world;
        G->host = true;
        G->tr = *t;
        *out = G.release();
        return DOT_OK;
    } catch (const Error& e) {
        g_create_error = e.msg;
        return e.code;
    }
}

int dot_dd_destroy(dot_dd* G) {
    if (!G) return DOT_OK;
    if (G->comm) nccl_api().commDestroy(G->comm);
    delete G;
    return DOT_OK;
}

const char* dot_dd_last_error(const dot_dd* G) { return G ? G->err.c_str() : g_create_error.c_str(); }

int dot_dd_fields(dot_dd* G, const double* W, int32_t ls, const double* V, int32_t ld, int where) {
    if (!G) return DOT_ERR_ARG;
    try {
        dot_problem* P = G->loc[0];
        for (dot_problem* Q : G->loc) require_params(Q);
        std::vector<Req> reqs;
        if (ls > 0) {
            check_side_matrix(W, P->n_src, ls, "W");
            reqs.push_back(Req{0, W ? host_copy(P, W, (size_t)P->n_src * ls, where) : std::vector<double>(),
                               W == nullptr, ls});
        }
        if (ld > 0) {
            check_side_matrix(V, P->n_det, ld, "V");
            reqs.push_back(Req{1, V ? host_copy(P, V, (size_t)P->n_det * ld, where) : std::vector<double>(),
                               V == nullptr, ld});
        }
        for (dot_problem* Q : G->loc)
            for (auto& c : Q->cache) {
                c.valid = false;
                c.blk.reset();
                c.X = nullptr;
            }
        dd_solve(G, reqs);
        return DOT_OK;
    } catch (const Error& e) {
        G->err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        G->err = e.what();
        return DOT_ERR_ARG;
    }
}

int dot_contract_fields(dot_problem* P, int32_t ld, int32_t ls, const double* Lam, const double* U, double* J) {
    DOT_API_BEGIN
    if (!P || !Lam || !U || !J || ld < 1 || ls < 1) throw Error(DOT_ERR_ARG, "bad argument");
    require_params(P);
    const int nf = P->n_freq, K = P->K;
    cudaStream_t s = P->stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto start_timer = [&]() {                 // brackets the contraction kernel only
        if (P->timing) {
            e0 = event_at(P, 0);
            e1 = event_at(P, 1);
            DOT_CUDA_TRY(cudaEventRecord(e0, s));
        }
    };
    const bool segp = contract_seg_applies(ld, ls, &P->gsp, P->n_p);
    if (segp) {
        // reorder the S-ordered panels into basis order (one gather), then the segment GEMM
        const int T = (int)P->gsp.total;
        DBuf<double2> Lg(P->arena, std::max<size_t>((size_t)nf * ld * T, 1)), Ug(P->arena, std::max<size_t>((size_t)nf * ls * T, 1));
        launch_gather_cols(nf, ld, T, reinterpret_cast<const double2*>(Lam), (size_t)ld * K, K, P->gsp.seg, Lg.get(),
                           (size_t)ld * T, T, s);
        launch_gather_cols(nf, ls, T, reinterpret_cast<const double2*>(U), (size_t)ls * K, K, P->gsp.seg, Ug.get(),
                           (size_t)ls * T, T, s);
        start_timer();
        contract_seg(P, nf, T, ld, ls, Lg.get(), (size_t)ld * T, Ug.get(), (size_t)ls * T, reinterpret_cast<double2*>(J));
        P->stats.kernel_launches += 3;
    } else {
        start_timer();
        launch_contract(nf, K, ld, ls, P->n_p, reinterpret_cast<const double2*>(Lam), (size_t)ld * K,
                        reinterpret_cast<const double2*>(U), (size_t)ls * K, P->d_G.get(), reinterpret_cast<double2*>(J),
                        s, &P->gsp, &P->arena, &P->stats.kernel_launches);
    }
    if (P->timing) {
        DOT_CUDA_TRY(cudaEventRecord(e1, s));
        DOT_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        DOT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        P->stats.contract_ms += ms;
        if (segp) P->stats.gemm_ms += ms;
    }
    P->stats.contract_flops += 4.0 * nf * ld * ls * (P->gsp.seg ? 5.0 * (double)P->gsp.total : (double)K * P->n_p);
    if (segp) P->stats.gemm_flops += 4.0 * nf * ld * ls * 5.0 * (double)P->gsp.total;
    P->stats.contract_flops_dense += 4.0 * nf * ld * ls * (double)K * P->n_p;
    DOT_API_END(P)
}

int dot_contract(void* stream, int32_t nb, int32_t K, int32_t ld, int32_t ls, int32_t n_p, const double* Lam,
                 const double* U, const double* G, double* J) {
    try {
        if (nb < 1 || K < 0 || ld < 1 || ls < 1 || n_p < 1 || n_p > 256 || !Lam || !U || !G || !J)
            throw Error(DOT_ERR_ARG, "bad argument");
        launch_contract(nb, K, ld, ls, n_p, reinterpret_cast<const double2*>(Lam), (size_t)ld * K,
                        reinterpret_cast<const double2*>(U), (size_t)ls * K, G, reinterpret_cast<double2*>(J),
                        static_cast<cudaStream_t>(stream));
        return DOT_OK;
    } catch (const Error& e) {
        g_create_error = e.msg;
        return e.code;
    }
}

}  // extern "C"
