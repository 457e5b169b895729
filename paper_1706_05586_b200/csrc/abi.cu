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
    DBuf<double2> X;                  // [n_freq][ncols][nP]
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
    CocgTiling tl{};
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

    ~dot_problem() {
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

size_t per_rhs_bytes(const dot_problem* P) {
    const size_t vec = P->N * sizeof(double2);
    const size_t zmax = (size_t)std::max(1, P->nz / 4);
    return 4 * vec + 2 * P->tl.ntiles * zmax * kNumPartials * sizeof(double) + 2 * sizeof(RhsState) +
           sizeof(double) + 4 * Arena::kAlign;
}

// ---------------------------------------------------------------- batched solve
// Solve the global RHS list r = f*ncols + c, f < n_freq, c < ncols, where RHS
// (f, c) is either the point-combination `side` (0: B coeff[:,c], 1: C coeff[:,c])
// or, if dense != null, the dense vector dense[r].  Outputs: XP [n_rhs][nP]
// (sampled) or, if Xfull != null, Xfull [n_rhs][N].  freq_of: optional per-RHS
// frequency (dense mode).  Returns per-RHS iterations.
// One segment of point-combination right-hand sides: RHS (f, c) = side's point
// combination with coefficient column c at frequency f, f-major (nf * ncols RHS).
struct Seg {
    int side;
    const double* d_coeff;   // device [n_side][ncols] or null (identity)
    int ncols;
};

std::vector<int32_t> solve_batch(dot_problem* P, const std::vector<Seg>& segs, int n_rhs, const double2* dense,
                                 const int32_t* d_freq_of, double2* XP, double2* Xfull);

std::vector<int32_t> solve_rhs(dot_problem* P, int side, const double* d_coeff, int ncols, int n_rhs,
                               const double2* dense, const int32_t* d_freq_of, double2* XP,
                               double2* Xfull) {
    std::vector<Seg> segs;
    if (!dense) segs.push_back(Seg{side, d_coeff, ncols});
    return solve_batch(P, segs, n_rhs, dense, d_freq_of, XP, Xfull);
}

// R0 [nb][N] and shift [nb] of global RHS r0 .. r0+nb-1 of the concatenated segments.
void build_point_rhs(dot_problem* P, const std::vector<Seg>& segs, long long r0, int nb, double2* R0, double* shift) {
    const size_t N = P->N;
    DOT_CUDA_TRY(cudaMemsetAsync(R0, 0, (size_t)nb * N * sizeof(double2), P->stream));
    long long gs = 0;
    for (const Seg& sg : segs) {                 // the part of each segment inside [r0, r0 + nb)
        const long long ge = gs + (long long)P->n_freq * sg.ncols;
        const long long rs = std::max<long long>(r0, gs), re = std::min<long long>(r0 + nb, ge);
        if (rs < re) {
            const int nn = sg.side == 0 ? P->n_src : P->n_det;
            launch_scatter_rhs(R0 + (size_t)(rs - r0) * N, N, (int)(re - rs), rs - gs, sg.ncols,
                               sg.side == 0 ? P->d_src.get() : P->d_det.get(), nn, sg.d_coeff,
                               sg.side == 0 ? P->d_src_scale.get() : P->d_det_scale.get(), P->stream);
            launch_fill_shift(shift + (rs - r0), (int)(re - rs), rs - gs, sg.ncols, P->d_omega_nu.get(), P->stream);
            P->stats.kernel_launches += 2;
        }
        gs = ge;
    }
}

// Batched solve of the concatenated RHS lists of `segs` (point mode) or of the dense
// vectors `dense` (with per-RHS frequency d_freq_of).  All RHS iterate together in
// chunks of what fits the workspace.
std::vector<int32_t> solve_batch(dot_problem* P, const std::vector<Seg>& segs, int n_rhs, const double2* dense,
                                 const int32_t* d_freq_of, double2* XP, double2* Xfull) {
    std::vector<int32_t> iters(n_rhs, 0);
    if (n_rhs == 0) return iters;
    const size_t N = P->N;
    const size_t prb = per_rhs_bytes(P);
    size_t fit = P->arena.largest_free() / prb;
    // multiple allocations fragment the arena: keep a safety margin
    fit = fit > 2 ? fit - 1 : fit;
    if (fit < 1) throw Error(DOT_ERR_WORKSPACE, "workspace too small for one right-hand side");
    const int chunk = (int)std::min<size_t>(fit, (size_t)n_rhs);
    const int CHK = 8;
    // z chunks (z pass): enough CTAs to fill the GPU when few RHS iterate together on a
    // deep grid; at least 8 planes per chunk.  DOT_COCG_ZCHUNKS overrides.
    auto zchunks = [&](int nb) {
        if (P->tl.kind != 1) return 1;
        int n = 1;
        const char* e = std::getenv("DOT_COCG_ZCHUNKS");
        if (e) {
            n = std::min(std::max(1, std::atoi(e)), std::max(1, P->nz / 4));
        } else {
            // measured (tools/rowsweep.sh): chunks pay off on deep grids (opt96, 96^3: 94 -> 110
            // RHS solves/s) but not on shallow ones, where a chunk's halo planes and CTA start-up
            // dominate (sketch32, 32^3: 4 chunks 3720 vs none 4180)
            const long long target = 4LL * P->num_sms;
            const long long have = (long long)P->tl.ntiles * nb;
            if (have < target && P->nz >= 64) n = (int)((target + have - 1) / have);
            n = std::min(n, std::max(1, P->nz / 8));
        }
        const int zlen = (P->nz + n - 1) / n;
        return (P->nz + zlen - 1) / zlen;
    };

    for (int r0 = 0; r0 < n_rhs; r0 += chunk) {
        const int nb = std::min(chunk, n_rhs - r0);
        DBuf<double2> R0(P->arena, nb * N), R1(P->arena, nb * N), P0(P->arena, nb * N), P1(P->arena, nb * N);
        const int nzch = zchunks(nb);
        DBuf<double> part(P->arena, 2 * (size_t)nb * P->tl.ntiles * nzch * kNumPartials);
        DBuf<RhsState> st(P->arena, 2 * (size_t)nb);
        DBuf<double> shift(P->arena, nb);
        DBuf<int32_t> act(P->arena, nb);                 // active-RHS list of the tail passes
        int nb_launch = nb;

        // ---- right-hand sides
        if (dense) {
            DOT_CUDA_TRY(cudaMemcpyAsync(R0.get(), dense + (size_t)r0 * N, (size_t)nb * N * sizeof(double2),
                                         cudaMemcpyDeviceToDevice, P->stream));
        } else {
            build_point_rhs(P, segs, r0, nb, R0.get(), shift.get());
        }
        if (d_freq_of) {
            // shift[r] = omega_nu[freq_of[r0 + r]] : reuse fill_shift with ncols = 1 on a gathered table
            std::vector<int32_t> fh(nb);
            DOT_CUDA_TRY(cudaMemcpyAsync(fh.data(), d_freq_of + r0, nb * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                         P->stream));
            sync(P);
            std::vector<double> sh(nb);
            for (int r = 0; r < nb; ++r) {
                if (fh[r] < 0 || fh[r] >= P->n_freq) throw Error(DOT_ERR_ARG, "frequency index out of range");
                sh[r] = P->omega[fh[r]] / P->nu;
            }
            DOT_CUDA_TRY(cudaMemcpyAsync(shift.get(), sh.data(), nb * sizeof(double), cudaMemcpyHostToDevice,
                                         P->stream));
            sync(P);
        }
        if (XP) DOT_CUDA_TRY(cudaMemsetAsync(XP + (size_t)r0 * P->nP, 0, (size_t)nb * P->nP * sizeof(double2), P->stream));
        if (Xfull) DOT_CUDA_TRY(cudaMemsetAsync(Xfull + (size_t)r0 * N, 0, (size_t)nb * N * sizeof(double2), P->stream));

        PassArgs a;
        a.op = P->op;
        a.tl = P->tl;
        a.max_iter = P->max_iter;
        a.tol2 = P->tol * P->tol;
        a.mu = P->d_mu.get();
        a.shift = shift.get();
        a.R[0] = R0.get();
        a.R[1] = R1.get();
        a.Pv[0] = P0.get();
        a.Pv[1] = P1.get();
        a.part[0] = part.get();
        a.part[1] = part.get() + (size_t)nb * P->tl.ntiles * nzch * kNumPartials;
        a.nzch = nzch;
        a.nzch_tot = nzch;
        a.zc0 = 0;
        a.zlen = (P->nz + nzch - 1) / nzch;
        a.st[0] = st.get();
        a.st[1] = st.get() + nb;
        a.samp_nodes = P->d_P.get();
        a.samp_off = P->d_off.get();
        a.XP = XP ? XP + (size_t)r0 * P->nP : nullptr;
        a.nP = XP ? P->nP : 0;
        a.X = Xfull ? Xfull + (size_t)r0 * N : nullptr;

        launch_cocg_init(a, nb, P->stream);
        P->stats.kernel_launches++;
        // Groups of CHK passes; each ends with a convergence count into pinned memory.  The
        // poll is pipelined: group g+1 is enqueued before the host reads group g-1's count,
        // so the GPU never idles on the host round trip (a group launched after the last
        // RHS finished runs as no-ops).
        int k = 0, g = 0;
        size_t ev = 0;
        for (;;) {
            if (P->timing) DOT_CUDA_TRY(cudaEventRecord(event_at(P, ev++), P->stream));
            for (int i = 0; i < CHK; ++i) {
                a.k = k++;
                launch_cocg_pass(a, nb_launch, P->stream);
                P->stats.kernel_launches++;
                P->stats.pass_launches++;
            }
            if (P->timing) DOT_CUDA_TRY(cudaEventRecord(event_at(P, ev++), P->stream));
            launch_count_active(a.st[(k - 1) & 1], nb, P->d_count.get() + (g & 1), P->stream,
                                P->tl.kind == 1 ? act.get() : nullptr);
            P->stats.kernel_launches++;
            DOT_CUDA_TRY(cudaMemcpyAsync(P->h_count + (g & 1), P->d_count.get() + (g & 1), sizeof(int),
                                         cudaMemcpyDeviceToHost, P->stream));
            DOT_CUDA_TRY(cudaEventRecord(P->poll_ev[g & 1], P->stream));
            if (g > 0) {
                DOT_CUDA_TRY(cudaEventSynchronize(P->poll_ev[(g - 1) & 1]));
                const int c = P->h_count[(g - 1) & 1];
                if (c == 0) break;
                if (P->tl.kind == 1) {     // later passes launch only the RHS still iterating
                    a.act = act.get();
                    nb_launch = c;
                }
            }
            ++g;
        }
        sync(P);
        if (P->timing) {
            for (size_t e = 0; e + 1 < ev; e += 2) {
                float ms = 0;
                DOT_CUDA_TRY(cudaEventElapsedTime(&ms, P->events[e], P->events[e + 1]));
                P->stats.pass_ms += ms;
            }
        }
        std::vector<RhsState> hs(nb);
        DOT_CUDA_TRY(cudaMemcpyAsync(hs.data(), a.st[(k - 1) & 1], nb * sizeof(RhsState), cudaMemcpyDeviceToHost,
                                     P->stream));
        sync(P);
        int mx = 0, mn = 1 << 30;
        for (int r = 0; r < nb; ++r) {
            if (hs[r].flag == DOT_ERR_NOCONV)
                throw Error(DOT_ERR_NOCONV, "COCG did not converge within max_iter for rhs " + std::to_string(r0 + r));
            if (hs[r].flag == DOT_ERR_BREAKDOWN)
                throw Error(DOT_ERR_BREAKDOWN, "COCG breakdown for rhs " + std::to_string(r0 + r) + " at iteration " +
                                                   std::to_string(hs[r].iters) + " (batch of " + std::to_string(nb) +
                                                   ", chunk start " + std::to_string(r0) + ")");
            iters[r0 + r] = hs[r].iters;
            mx = std::max(mx, hs[r].iters);
            mn = std::min(mn, hs[r].iters);
            P->stats.rhs_iterations += hs[r].iters;
            P->stats.pass_bytes += 64.0 * (double)N * hs[r].iters;
        }
        P->stats.rhs_solved += nb;
        P->stats.last_max_iters = mx;
        P->stats.last_min_iters = mn;
    }
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
    DBuf<double2> XPj(P->arena, (size_t)total * nPp);
    solve_batch(P, segs, total, nullptr, nullptr, XPj.get(), nullptr);
    size_t off = 0;
    for (const Req& q : reqs) {
        const int n_side = q.side == 0 ? P->n_src : P->n_det;
        FieldCache& c = P->cache[q.side];
        c.valid = false;
        c.X.reset();
        const size_t n = (size_t)P->n_freq * q.ncols * nPp;
        c.X = DBuf<double2>(P->arena, n);
        DOT_CUDA_TRY(cudaMemcpyAsync(c.X.get(), XPj.get() + off, n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                     P->stream));
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
    if (identity && c.identity) return c.X.get();
    if (!identity && !c.identity && c.ncols == ncols && c.coeff == hc) return c.X.get();
    // combination of the cached point sources sel[0..m):
    // X'[f][c][q] = sum_j coeff[sel_j][c] X[f][j][q]
    const int m = (int)c.sel.size();
    std::vector<double> X((size_t)m * ncols);
    for (int j = 0; j < m; ++j)
        for (int k = 0; k < ncols; ++k) X[(size_t)j * ncols + k] = hc[(size_t)c.sel[j] * ncols + k];
    DBuf<double> dc = to_device(P, X.data(), X.size(), DOT_HOST);
    tmp = DBuf<double2>(P->arena, (size_t)P->n_freq * ncols * std::max(P->nP, 1));
    launch_rc_gemm(P->n_freq, ncols, P->nP, m, dc.get(), ncols, c.X.get(), (size_t)m * P->nP, P->nP, 1, tmp.get(),
                   (size_t)ncols * P->nP, P->nP, 1, P->stream);
    P->stats.kernel_launches++;
    sync(P);
    return tmp.get();
}

void invalidate_caches(dot_problem* P) {
    for (auto& c : P->cache) {
        c.valid = false;
        c.X.reset();
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
    ncclComm_t comm = nullptr;      // one local rank per process when set
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

// DD solve of the point-combination requests: fills the field caches of every local rank.
void dd_solve(dot_dd* G, const std::vector<Req>& reqs) {
    const int L = (int)G->loc.size();
    dot_problem* P0 = G->loc[0];
    const size_t N = P0->N, PS = (size_t)P0->nx * P0->ny;
    const int nz = P0->nz, nP = P0->nP, nf = P0->n_freq;
    int nb = 0;
    for (const Req& q : reqs) nb += nf * q.ncols;
    if (nb == 0) return;
    const DDPlan pl = dd_plan(G, nb);
    const int ntiles = P0->tl.ntiles, nslots = ntiles * pl.C;
    const bool use_nccl = G->comm != nullptr;
    if (P0->tl.kind != 1) throw Error(DOT_ERR_ARG, "domain decomposition needs the z pass (DOT_COCG_KERNEL != ring)");

    struct RankBufs {
        std::vector<DBuf<double>> dcs;
        DBuf<double2> R[2], Pv[2], XP;
        DBuf<double> part, shift;
        DBuf<RhsState> st;
        PassArgs a;
    };
    std::vector<RankBufs> B(L);
    for (int q = 0; q < L; ++q) {
        dot_problem* P = G->loc[q];
        RankBufs& b = B[q];
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
        b.XP = DBuf<double2>(P->arena, (size_t)nb * std::max(nP, 1));
        b.part = DBuf<double>(P->arena, 2 * (size_t)nb * nslots * kNumPartials);
        b.shift = DBuf<double>(P->arena, nb);
        b.st = DBuf<RhsState>(P->arena, 2 * (size_t)nb);
        build_point_rhs(P, segs, 0, nb, b.R[0].get(), b.shift.get());
        DOT_CUDA_TRY(cudaMemsetAsync(b.XP.get(), 0, (size_t)nb * std::max(nP, 1) * sizeof(double2), P->stream));
        DOT_CUDA_TRY(cudaMemsetAsync(b.part.get(), 0, 2 * (size_t)nb * nslots * kNumPartials * sizeof(double), P->stream));
        PassArgs& a = b.a;
        a.op = P->op;
        a.tl = P->tl;
        a.max_iter = P->max_iter;
        a.tol2 = P->tol * P->tol;
        a.mu = P->d_mu.get();
        a.shift = b.shift.get();
        for (int i = 0; i < 2; ++i) {
            a.R[i] = b.R[i].get();
            a.Pv[i] = b.Pv[i].get();
            a.part[i] = b.part.get() + (size_t)i * nb * nslots * kNumPartials;
            a.st[i] = b.st.get() + (size_t)i * nb;
        }
        a.samp_nodes = P->d_P.get();
        a.samp_off = P->d_off.get();
        a.XP = b.XP.get();
        a.nP = nP;
        a.X = nullptr;
        const int r = G->rank0 + q;
        a.zlen = pl.zlen;
        a.nzch_tot = pl.C;
        a.zc0 = pl.cb[r];
        a.nzch = pl.cb[r + 1] - pl.cb[r];
        launch_cocg_init(a, nb, P->stream);      // full-domain sums of b: identical on every rank
        P->stats.kernel_launches += 1;
    }
    // boundary planes [z, z + n) of vector arrays V (nb vectors of N) : (dst rank q', src rank q)
    auto copy_planes = [&](double2* dst, const double2* src, int z, int n, cudaStream_t s) {
        if (n <= 0) return;
        DOT_CUDA_TRY(cudaMemcpy2DAsync(dst + (size_t)z * PS, N * sizeof(double2), src + (size_t)z * PS,
                                       N * sizeof(double2), (size_t)n * PS * sizeof(double2), nb,
                                       cudaMemcpyDeviceToDevice, s));
    };
    const int CHK = 8;
    int k = 0;
    for (;;) {
        const int kout = (k + 1) & 1;
        for (int q = 0; q < L; ++q) {
            dot_problem* P = G->loc[q];
            PassArgs& a = B[q].a;
            a.k = k;
            if (use_nccl)   // this rank's slots only; the others arrive through the all-reduce
                DOT_CUDA_TRY(cudaMemsetAsync(a.part[kout], 0, (size_t)nb * nslots * kNumPartials * sizeof(double),
                                             P->stream));
            launch_cocg_pass(a, nb, P->stream);
            P->stats.kernel_launches++;
            P->stats.pass_launches++;
        }
        // ---- halo exchange of r_{k+1}, p_k (kout arrays) and all-reduce of the partials
        if (!use_nccl) {
            for (int q = 0; q < L; ++q) DOT_CUDA_TRY(cudaStreamSynchronize(G->loc[q]->stream));
            cudaStream_t s = G->loc[0]->stream;
            for (int q = 0; q + 1 < L; ++q) {
                const int r = G->rank0 + q;
                const int zt = pl.ze(r, nz);                         // boundary between r and r + 1
                for (int v = 0; v < 2; ++v) {
                    double2* lo = v == 0 ? B[q].a.R[kout] : B[q].a.Pv[kout];
                    double2* hi = v == 0 ? B[q + 1].a.R[kout] : B[q + 1].a.Pv[kout];
                    copy_planes(hi, lo, std::max(zt - 2, pl.zs(r, nz)), std::min(2, zt - pl.zs(r, nz)), s);
                    copy_planes(lo, hi, zt, std::min(zt + 2, pl.ze(r + 1, nz)) - zt, s);
                }
            }
            for (int q = 0; q < L; ++q)            // owned slot ranges to every other local rank
                for (int q2 = 0; q2 < L; ++q2) {
                    if (q2 == q) continue;
                    const int r = G->rank0 + q;
                    const size_t off = (size_t)pl.cb[r] * ntiles * kNumPartials;
                    const size_t w = (size_t)(pl.cb[r + 1] - pl.cb[r]) * ntiles * kNumPartials * sizeof(double);
                    DOT_CUDA_TRY(cudaMemcpy2DAsync(B[q2].a.part[kout] + off, nslots * kNumPartials * sizeof(double),
                                                   B[q].a.part[kout] + off, nslots * kNumPartials * sizeof(double),
                                                   w, nb, cudaMemcpyDeviceToDevice, s));
                }
            DOT_CUDA_TRY(cudaStreamSynchronize(s));
        } else {
            NcclApi& nc = nccl_api();
            dot_problem* P = G->loc[0];
            const int r = G->rank0;
            const int zs = pl.zs(r, nz), ze = pl.ze(r, nz);
            DOT_NCCL_TRY(nc.groupStart());
            for (int v = 0; v < 2; ++v) {
                double2* X = v == 0 ? B[0].a.R[kout] : B[0].a.Pv[kout];
                for (int i = 0; i < nb; ++i) {
                    double2* Xi = X + (size_t)i * N;
                    if (r + 1 < G->world) {                 // top planes up, halo from above
                        const int n_up = std::min(2, ze - zs), n_dn = std::min(ze + 2, pl.ze(r + 1, nz)) - ze;
                        DOT_NCCL_TRY(nc.send(Xi + (size_t)(ze - n_up) * PS, 2 * n_up * PS, ncclDouble, r + 1, G->comm,
                                             P->stream));
                        DOT_NCCL_TRY(nc.recv(Xi + (size_t)ze * PS, 2 * n_dn * PS, ncclDouble, r + 1, G->comm, P->stream));
                    }
                    if (r > 0) {                            // bottom planes down, halo from below
                        const int n_dn = std::min(2, ze - zs), n_up = std::min(2, zs - pl.zs(r - 1, nz));
                        DOT_NCCL_TRY(nc.send(Xi + (size_t)zs * PS, 2 * n_dn * PS, ncclDouble, r - 1, G->comm, P->stream));
                        DOT_NCCL_TRY(nc.recv(Xi + (size_t)(zs - n_up) * PS, 2 * n_up * PS, ncclDouble, r - 1, G->comm,
                                             P->stream));
                    }
                }
            }
            DOT_NCCL_TRY(nc.groupEnd());
            DOT_NCCL_TRY(nc.allReduce(B[0].a.part[kout], B[0].a.part[kout], (size_t)nb * nslots * kNumPartials,
                                      ncclDouble, ncclSum, G->comm, P->stream));
        }
        ++k;
        if (k % CHK == 0 || k > P0->max_iter) {
            dot_problem* P = G->loc[0];
            launch_count_active(B[0].a.st[(k - 1) & 1], nb, P->d_count.get(), P->stream);
            DOT_CUDA_TRY(cudaMemcpyAsync(P->h_count, P->d_count.get(), sizeof(int), cudaMemcpyDeviceToHost, P->stream));
            sync(P);
            if (*P->h_count == 0) break;
        }
    }
    // ---- sampled solutions: each sample node belongs to one slab -> sum over ranks
    const size_t nx = (size_t)nb * std::max(nP, 1);
    if (!use_nccl) {
        for (int q = 1; q < L; ++q) launch_cadd_inplace(B[0].XP.get(), B[q].XP.get(), nx, G->loc[0]->stream);
        for (int q = 1; q < L; ++q)
            DOT_CUDA_TRY(cudaMemcpyAsync(B[q].XP.get(), B[0].XP.get(), nx * sizeof(double2), cudaMemcpyDeviceToDevice,
                                         G->loc[0]->stream));
        DOT_CUDA_TRY(cudaStreamSynchronize(G->loc[0]->stream));
    } else {
        DOT_NCCL_TRY(nccl_api().allReduce(B[0].XP.get(), B[0].XP.get(), 2 * nx, ncclDouble, ncclSum, G->comm,
                                          G->loc[0]->stream));
    }
    // ---- convergence flags, statistics and the field caches of every local rank
    for (int q = 0; q < L; ++q) {
        dot_problem* P = G->loc[q];
        std::vector<RhsState> hs(nb);
        DOT_CUDA_TRY(cudaMemcpyAsync(hs.data(), B[q].a.st[(k - 1) & 1], nb * sizeof(RhsState), cudaMemcpyDeviceToHost,
                                     P->stream));
        sync(P);
        int mx = 0, mn = 1 << 30;
        for (int i = 0; i < nb; ++i) {
            if (hs[i].flag == DOT_ERR_NOCONV) throw Error(DOT_ERR_NOCONV, "COCG (domain decomposition) did not converge");
            if (hs[i].flag == DOT_ERR_BREAKDOWN) throw Error(DOT_ERR_BREAKDOWN, "COCG (domain decomposition) breakdown");
            mx = std::max(mx, hs[i].iters);
            mn = std::min(mn, hs[i].iters);
            P->stats.rhs_iterations += hs[i].iters;
            P->stats.pass_bytes += 64.0 * (double)N * hs[i].iters / G->world;
        }
        P->stats.rhs_solved += nb;
        P->stats.last_max_iters = mx;
        P->stats.last_min_iters = mn;
        size_t off = 0;
        const size_t nPp = (size_t)std::max(nP, 1);
        for (const Req& rq : reqs) {
            const int n_side = rq.side == 0 ? P->n_src : P->n_det;
            FieldCache& c = P->cache[rq.side];
            c.valid = false;
            c.X.reset();
            const size_t n = (size_t)nf * rq.ncols * nPp;
            c.X = DBuf<double2>(P->arena, n);
            DOT_CUDA_TRY(cudaMemcpyAsync(c.X.get(), B[q].XP.get() + off, n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                         P->stream));
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
            // tuning knobs: planes prefetched, smem budget per CTA
            const char* ePD = std::getenv("DOT_COCG_PREFETCH");
            const char* eSM = std::getenv("DOT_COCG_SMEM_KB");
            const char* eTH = std::getenv("DOT_COCG_THREADS");
            const char* eK = std::getenv("DOT_COCG_KERNEL");      // "ring" selects the padded-ring pass
            const char* eTY = std::getenv("DOT_COCG_TY");         // z-pass tile height
            const int kind = (eK && std::string(eK) == "ring") ? 0 : 1;
            const int pd = ePD ? std::max(1, std::atoi(ePD)) : (kind == 1 ? 2 : 1);
            const size_t sm = eSM ? (size_t)std::atoi(eSM) * 1024 : 0;
            P->tl = cocg_tiling(P->nx, P->ny, P->nz, pd, sm, eTH ? std::atoi(eTH) : 0, kind,
                                eTY ? std::atoi(eTY) : 0);
            // cluster of consecutive tiles of one RHS: the largest size <= request dividing ntiles
            const char* eCL = std::getenv("DOT_COCG_CLUSTER");
            int cs = eCL ? std::max(1, std::min(8, std::atoi(eCL))) : 1;
            while (cs > 1 && P->tl.ntiles % cs != 0) --cs;
            P->tl.cluster = cs;
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
    // support / samples: budget 5% of the nodes
    const size_t Kb = N / 20 + P->n_det;
    fixed += Kb * (3 * sizeof(int32_t) + P->n_p * sizeof(double)) + (size_t)P->nz * P->tl.ntiles * 4;
    fixed += (size_t)P->n_freq * P->n_src * P->n_det * sizeof(double2);
    // field caches (sources + detectors, all frequencies) on the samples
    fixed += (size_t)P->n_freq * (P->n_src + P->n_det) * Kb * sizeof(double2);
    return fixed + (size_t)std::max(max_rhs, 1) * per_rhs_bytes(P) + 64 * Arena::kAlign;
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
            P->stats.kernel_launches += 5;
            sync(P);
            P->gsp = GSparse{P->d_seg.get(), P->d_segoff.get(), P->n_rbf, T};
        }
    }
    launch_sample_offsets(P->d_P.get(), P->nP, P->nx, P->ny, P->nz, P->tl.TY, P->tl.ntiles, P->d_off.get(), s);
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
    DBuf<double2> US(P->arena, std::max<size_t>((size_t)nf * ls * K, 1)), LS(P->arena, std::max<size_t>((size_t)nf * ld * K, 1));
    launch_gather_cols(nf, ls, K, XU, (size_t)ls * P->nP, P->nP, P->d_S_slot.get(), US.get(), (size_t)ls * K, K, s);
    launch_gather_cols(nf, ld, K, XL, (size_t)ld * P->nP, P->nP, P->d_S_slot.get(), LS.get(), (size_t)ld * K, K, s);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (P->timing) {
        e0 = event_at(P, 0);
        e1 = event_at(P, 1);
        DOT_CUDA_TRY(cudaEventRecord(e0, s));
    }
    launch_contract(nf, K, ld, ls, P->n_p, LS.get(), (size_t)ld * K, US.get(), (size_t)ls * K, P->d_G.get(), J, s,
                    &P->gsp);
    P->stats.kernel_launches += 3;
    if (P->timing) {
        DOT_CUDA_TRY(cudaEventRecord(e1, s));
        DOT_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        DOT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        P->stats.contract_ms += ms;
    }
    // useful flops: 4 per (pair, point, parameter) with a nonzero weight block (5 per basis
    // over its points when the block-sparse kernel runs; the dense K x n_p otherwise)
    P->stats.contract_flops += 4.0 * nf * ld * ls * (P->gsp.seg ? 5.0 * (double)P->gsp.total : (double)K * P->n_p);
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
    ops.fields = [&](int side, const std::vector<double>& coeff, int ncols, double2* out) {
        DBuf<double> dc = to_device(P, coeff.data(), coeff.size(), DOT_HOST);
        DBuf<double2> XP(P->arena, std::max<size_t>((size_t)nf * ncols * nP, 1));
        solve_rhs(P, side, dc.get(), ncols, nf * ncols, nullptr, nullptr, XP.get(), nullptr);
        launch_gather_cols(nf, ncols, K, XP.get(), (size_t)ncols * nP, nP, P->d_S_slot.get(), out, (size_t)ncols * K,
                           K, s);
        P->stats.kernel_launches++;
        sync(P);
    };
    ops.solve_support = [&](const double2* w, int nvec, int side, double2* out) {
        const int nr = nf * nvec;
        DBuf<double2> R(P->arena, (size_t)nr * P->N);
        DOT_CUDA_TRY(cudaMemsetAsync(R.get(), 0, (size_t)nr * P->N * sizeof(double2), s));
        launch_scatter_support(R.get(), P->N, nr, P->d_S.get(), K, w, s);
        std::vector<int32_t> fo(nr);
        for (int r = 0; r < nr; ++r) fo[r] = r / nvec;
        DBuf<int32_t> dfo = to_device(P, fo.data(), fo.size(), DOT_HOST);
        DBuf<double2> XP(P->arena, std::max<size_t>((size_t)nr * nP, 1));
        solve_rhs(P, -1, nullptr, 1, nr, R.get(), dfo.get(), XP.get(), nullptr);
        const int n_side = side == 0 ? P->n_src : P->n_det;
        launch_gather_cols(nf, nvec, n_side, XP.get(), (size_t)nvec * nP, nP,
                           side == 0 ? P->d_src_slot.get() : P->d_det_slot.get(), out, (size_t)nvec * n_side, n_side, s);
        P->stats.kernel_launches += 2;
        if (side == 0) {     // b_s^T x = theta_s / (hx hy hz) x[src_s]  (reading R6)
            std::vector<double2> h((size_t)nr * n_side);
            DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), out, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, s));
            sync(P);
            for (int r = 0; r < nr; ++r)
                for (int a = 0; a < n_side; ++a) {
                    double2& v = h[(size_t)r * n_side + a];
                    v.x *= P->src_scale[a];
                    v.y *= P->src_scale[a];
                }
            DOT_CUDA_TRY(cudaMemcpyAsync(out, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
        }
        sync(P);
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
    DBuf<int32_t> df = to_device(P, freq, nrhs, where);
    DBuf<double2> dx(P->arena, n);
    auto it = solve_rhs(P, -1, nullptr, 1, nrhs, db.get(), df.get(), nullptr, dx.get());
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
        if (nlocal < world) {
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
                c.X.reset();
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
    if (P->timing) {
        e0 = event_at(P, 0);
        e1 = event_at(P, 1);
        DOT_CUDA_TRY(cudaEventRecord(e0, s));
    }
    launch_contract(nf, K, ld, ls, P->n_p, reinterpret_cast<const double2*>(Lam), (size_t)ld * K,
                    reinterpret_cast<const double2*>(U), (size_t)ls * K, P->d_G.get(), reinterpret_cast<double2*>(J), s,
                    &P->gsp);
    P->stats.kernel_launches++;
    if (P->timing) {
        DOT_CUDA_TRY(cudaEventRecord(e1, s));
        DOT_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        DOT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        P->stats.contract_ms += ms;
    }
    P->stats.contract_flops += 4.0 * nf * ld * ls * (P->gsp.seg ? 5.0 * (double)P->gsp.total : (double)K * P->n_p);
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
