// Simultaneous optimized sources and detectors (Sec. 3.2 Theorems
// 3.4-3.7, Sec. 3.3.2 "two-phase alternating approach").  All contractions
// (sketched Jacobians J(W, V), J(I, V), J(W, I)) and Gram matrices run on the
// GPU; only the small symmetric eigenproblems (Table 1 sizes, Lemma 3.2) are
// solved on the host.
#include <cmath>

#include "optimize.h"

namespace dot {

namespace {

// Gram tile kernel: Gr[r][c] = Re sum_l X[l-th (o,i)][r] conj(X[..][c]); 32x32 tiles, 16x16 threads.
__global__ void __launch_bounds__(256) gram_kernel(const double2* __restrict__ X, int outer, int R, int inner,
                                                   double* Gr) {
    __shared__ double2 As[32][17], Bs[32][17];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const long long L = (long long)outer * inner;
    double acc[2][2] = {{0, 0}, {0, 0}};
    for (long long l0 = 0; l0 < L; l0 += 16) {
        for (int e = threadIdx.x; e < 32 * 16; e += 256) {
            const int rr = e / 16, ll = e % 16;
            const long long l = l0 + ll;
            double2 va = make_double2(0, 0), vb = make_double2(0, 0);
            if (l < L) {
                const long long o = l / inner, i = l % inner;
                if (r0 + rr < R) va = X[(o * R + r0 + rr) * inner + i];
                if (c0 + rr < R) vb = X[(o * R + c0 + rr) * inner + i];
            }
            As[rr][ll] = va;
            Bs[rr][ll] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int ll = 0; ll < 16; ++ll) {
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const double2 x = As[ty * 2 + a][ll];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const double2 y = Bs[tx * 2 + b][ll];
                    acc[a][b] = fma(x.x, y.x, fma(x.y, y.y, acc[a][b]));
                }
            }
        }
        __syncthreads();
    }
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            const int r = r0 + ty * 2 + a, c = c0 + tx * 2 + b;
            if (r < R && c < R) Gr[(size_t)r * R + c] = acc[a][b];
        }
}

// host helpers ----------------------------------------------------------------
std::vector<double> matmul(const std::vector<double>& A, int m, int k, const std::vector<double>& B, int n) {
    std::vector<double> C((size_t)m * n, 0.0);
    for (int i = 0; i < m; ++i)
        for (int p = 0; p < k; ++p) {
            const double a = A[(size_t)i * k + p];
            if (a == 0.0) continue;
            for (int j = 0; j < n; ++j) C[(size_t)i * n + j] += a * B[(size_t)p * n + j];
        }
    return C;
}

// orthonormal basis (n x l) of the column span of M (n x l), modified Gram-Schmidt twice
std::vector<double> orth_basis(const std::vector<double>& M, int n, int l) {
    std::vector<double> Q = M;
    for (int j = 0; j < l; ++j) {
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i < j; ++i) {
                double d = 0;
                for (int r = 0; r < n; ++r) d += Q[(size_t)r * l + i] * Q[(size_t)r * l + j];
                for (int r = 0; r < n; ++r) Q[(size_t)r * l + j] -= d * Q[(size_t)r * l + i];
            }
        double nr = 0;
        for (int r = 0; r < n; ++r) nr += Q[(size_t)r * l + j] * Q[(size_t)r * l + j];
        nr = std::sqrt(nr);
        if (nr == 0) throw Error(DOT_ERR_ARG, "simultaneous source/detector matrix is rank deficient");
        for (int r = 0; r < n; ++r) Q[(size_t)r * l + j] /= nr;
    }
    return Q;
}

}  // namespace

void launch_gram(const double2* X, int outer, int R, int inner, double* Gr, cudaStream_t s) {
    dim3 grid((R + 31) / 32, (R + 31) / 32);
    gram_kernel<<<grid, 256, 0, s>>>(X, outer, R, inner, Gr);
    DOT_CUDA_TRY(cudaGetLastError());
}

double optimize_two_phase(OptContext& c, int k, std::vector<double>& W, int ls, std::vector<double>& V, int ld) {
    const int nf = c.nf, ns = c.ns, nd = c.nd, n_p = c.n_p, K = c.K;
    cudaStream_t s = c.stream;
    // sampled full-data fields restricted to the support S: [nf][n][K]
    DBuf<double2> US(c.arena, std::max<size_t>((size_t)nf * ns * K, 1)), LS(c.arena, std::max<size_t>((size_t)nf * nd * K, 1));
    launch_gather_cols(nf, ns, K, c.XU, (size_t)ns * c.nP, c.nP, c.S_slot, US.get(), (size_t)ns * K, K, s);
    launch_gather_cols(nf, nd, K, c.XL, (size_t)nd * c.nP, c.nP, c.S_slot, LS.get(), (size_t)nd * K, K, s);
    *c.launches += 2;

    // sketched Jacobian J[f][b][a][n_p] for W (ns x a) / V (nd x b); null = identity
    auto jac = [&](const std::vector<double>* Wm, int a, const std::vector<double>* Vm, int b) {
        DBuf<double2> J(c.arena, std::max<size_t>((size_t)nf * b * a * n_p, 1));
        DBuf<double2> UW, LV;
        DBuf<double> dW, dV;
        const double2* u = US.get();
        const double2* lam = LS.get();
        if (Wm) {
            dW = DBuf<double>(c.arena, Wm->size());
            DOT_CUDA_TRY(cudaMemcpyAsync(dW.get(), Wm->data(), Wm->size() * 8, cudaMemcpyHostToDevice, s));
            UW = DBuf<double2>(c.arena, std::max<size_t>((size_t)nf * a * K, 1));
            launch_rc_gemm(nf, a, K, ns, dW.get(), a, US.get(), (size_t)ns * K, K, 1, UW.get(), (size_t)a * K, K, 1, s);
            u = UW.get();
        }
        if (Vm) {
            dV = DBuf<double>(c.arena, Vm->size());
            DOT_CUDA_TRY(cudaMemcpyAsync(dV.get(), Vm->data(), Vm->size() * 8, cudaMemcpyHostToDevice, s));
            LV = DBuf<double2>(c.arena, std::max<size_t>((size_t)nf * b * K, 1));
            launch_rc_gemm(nf, b, K, nd, dV.get(), b, LS.get(), (size_t)nd * K, K, 1, LV.get(), (size_t)b * K, K, 1, s);
            lam = LV.get();
        }
        launch_contract(nf, K, b, a, n_p, lam, (size_t)b * K, u, (size_t)a * K, c.G, J.get(), s, c.gsp);
        *c.launches += 3;
        DOT_CUDA_TRY(cudaStreamSynchronize(s));   // host copies above must outlive their async use
        return J;
    };
    auto gram = [&](const DBuf<double2>& J, int outer, int R, int inner) {
        DBuf<double> dG(c.arena, (size_t)R * R);
        launch_gram(J.get(), outer, R, inner, dG.get(), s);
        *c.launches += 1;
        std::vector<double> h((size_t)R * R);
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), dG.get(), h.size() * 8, cudaMemcpyDeviceToHost, s));
        DOT_CUDA_TRY(cudaStreamSynchronize(s));
        for (int i = 0; i < R; ++i)          // symmetrise (rounding)
            for (int j = i + 1; j < R; ++j) {
                const double m = 0.5 * (h[(size_t)i * R + j] + h[(size_t)j * R + i]);
                h[(size_t)i * R + j] = h[(size_t)j * R + i] = m;
            }
        return h;
    };
    // top-q eigenvectors of an R x R Gram -> R x q
    auto top = [&](const std::vector<double>& Gr, int R, int q) {
        std::vector<double> w, Z;
        sym_eig(R, Gr, w, Z);
        std::vector<double> T((size_t)R * q);
        for (int r = 0; r < R; ++r)
            for (int j = 0; j < q; ++j) T[(size_t)r * q + j] = Z[(size_t)r * R + j];
        return T;
    };
    // best unit direction in the orthogonal complement of span(M): eigvec of Pc Gr Pc
    auto add_dir = [&](const std::vector<double>& Gr, int R, const std::vector<double>& M, int l) {
        std::vector<double> Q = orth_basis(M, R, l);
        std::vector<double> T = matmul(Gr, R, R, Q, l);                 // Gr Q (R x l)
        std::vector<double> Qt((size_t)l * R);
        for (int r = 0; r < R; ++r)
            for (int j = 0; j < l; ++j) Qt[(size_t)j * R + r] = Q[(size_t)r * l + j];
        std::vector<double> U = matmul(Qt, l, R, T, l);                 // Q^T Gr Q (l x l)
        std::vector<double> QU = matmul(Q, R, l, U, l);                 // Q U (R x l)
        std::vector<double> Gc = Gr;
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < R; ++j) {
                double v = 0;
                for (int p = 0; p < l; ++p)
                    v += -Q[(size_t)i * l + p] * T[(size_t)j * l + p] - T[(size_t)i * l + p] * Q[(size_t)j * l + p] +
                         QU[(size_t)i * l + p] * Q[(size_t)j * l + p];
                Gc[(size_t)i * R + j] += v;
            }
        std::vector<double> q = top(Gc, R, 1);
        // project once more onto the complement (rounding) and normalise
        for (int p = 0; p < l; ++p) {
            double d = 0;
            for (int r = 0; r < R; ++r) d += Q[(size_t)r * l + p] * q[r];
            for (int r = 0; r < R; ++r) q[r] -= d * Q[(size_t)r * l + p];
        }
        double nr = 0;
        for (double v : q) nr += v * v;
        nr = std::sqrt(nr);
        for (double& v : q) v /= nr;
        return q;
    };
    auto append_col = [](std::vector<double>& M, int n, int l, const std::vector<double>& q, double scale) {
        std::vector<double> out((size_t)n * (l + 1));
        for (int r = 0; r < n; ++r) {
            for (int j = 0; j < l; ++j) out[(size_t)r * (l + 1) + j] = M[(size_t)r * l + j];
            out[(size_t)r * (l + 1) + l] = scale * q[r];
        }
        M.swap(out);
    };

    int a = ls, b = ld;
    for (int step = 0; step < k; ++step) {       // phase one: remove a source, then a detector
        {
            DBuf<double2> J = jac(&W, a, &V, b);
            std::vector<double> Gam = top(gram(J, nf * b, a, n_p), a, a - 1);     // Theorem 3.5
            W = matmul(W, ns, a, Gam, a - 1);
            --a;
        }
        {
            DBuf<double2> J = jac(&W, a, &V, b);
            std::vector<double> Gam = top(gram(J, nf, b, a * n_p), b, b - 1);     // Theorem 3.4
            V = matmul(V, nd, b, Gam, b - 1);
            --b;
        }
    }
    for (int step = 0; step < k; ++step) {       // phase two: add a source, then a detector
        {
            DBuf<double2> J = jac(nullptr, ns, &V, b);                           // J(I, V)
            std::vector<double> q = add_dir(gram(J, nf * b, ns, n_p), ns, W, a);  // Theorem 3.7
            append_col(W, ns, a, q, std::sqrt((double)ns));
            ++a;
        }
        {
            DBuf<double2> J = jac(&W, a, nullptr, nd);                           // J(W, I)
            std::vector<double> q = add_dir(gram(J, nf, nd, a * n_p), nd, V, b);  // Theorem 3.6
            append_col(V, nd, b, q, std::sqrt((double)nd));
            ++b;
        }
    }
    DBuf<double2> J = jac(&W, a, &V, b);
    DBuf<double> d_obj(c.arena, 1);
    launch_sumsq(J.get(), (size_t)nf * b * a * n_p, d_obj.get(), s);
    *c.launches += 1;
    double obj = 0;
    DOT_CUDA_TRY(cudaMemcpyAsync(&obj, d_obj.get(), 8, cudaMemcpyDeviceToHost, s));
    DOT_CUDA_TRY(cudaStreamSynchronize(s));
    return obj;
}


// ------------------------------------------------------------------------------
// Matrix-free variant (reading R16).  Notation of PAPER.md Sec. 3.2: for adding a
// detector, X_f[d, (i,k)] = (W^T (x) I) J = - y_d^T diag(G_k) z_i with y_d = A^-T c_d,
// z_i = A^-1 B w_i; Xr = [Re X_f, Im X_f]_f.  K = P Xr Xr^T P with P the projector onto
// the complement of span(V):
//   Xr^T q  = contraction of the adjoint field of C q with the z_i       (1 solve / f)
//   Xr t    = - Re( c_d^T A^-1 w_f ),  w_f = sum_ik conj(T_f,ik) G_k z_i  (1 solve / f)
// with T = Xr^T q in complex form (t = [Re T, Im T] -> coefficient conj(T)).  Adding a
// source is the same with the roles of (W, z, B) and (V, y, C) exchanged.
double optimize_two_phase_subspace(OptContext& c, SubspaceOps& ops, int k, int iters, int blk,
                                   std::vector<double>& W, int ls, std::vector<double>& V, int ld,
                                   const std::vector<double>& X0s, const std::vector<double>& X0d) {
    const int nf = c.nf, ns = c.ns, nd = c.nd, n_p = c.n_p, K = c.K;
    cudaStream_t s = c.stream;
    auto sync = [&]() { DOT_CUDA_TRY(cudaStreamSynchronize(s)); };
    auto fields = [&](int side, const std::vector<double>& coeff, int ncols) {
        DBuf<double2> out(c.arena, std::max<size_t>((size_t)nf * ncols * K, 1));
        ops.fields(side, coeff, ncols, out.get());
        return out;
    };
    // z fields of W and y fields of V on S: [nf][cols][K]
    DBuf<double2> ZW = fields(0, W, ls), YV = fields(1, V, ld);
    int a = ls, b = ld;

    auto contract = [&](const double2* lam, int nl, const double2* u, int nu) {
        DBuf<double2> J(c.arena, std::max<size_t>((size_t)nf * nl * nu * n_p, 1));
        launch_contract(nf, K, nl, nu, n_p, lam, (size_t)nl * K, u, (size_t)nu * K, c.G, J.get(), s, c.gsp);
        *c.launches += 1;
        return J;
    };
    auto to_host = [&](const double2* d, size_t n) {
        std::vector<double2> h(n);
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), d, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
        sync();
        return h;
    };
    // new fields F' [nf][m][K] = sum_j Gam[j][m] F[f][j][K]  (Gam host [ncols][m])
    auto combine = [&](const DBuf<double2>& F, int ncols, const std::vector<double>& Gam, int m) {
        DBuf<double> dG(c.arena, Gam.size());
        DOT_CUDA_TRY(cudaMemcpyAsync(dG.get(), Gam.data(), Gam.size() * 8, cudaMemcpyHostToDevice, s));
        DBuf<double2> out(c.arena, std::max<size_t>((size_t)nf * m * K, 1));
        launch_rc_gemm(nf, m, K, ncols, dG.get(), m, F.get(), (size_t)ncols * K, K, 1, out.get(), (size_t)m * K, K, 1, s);
        *c.launches += 1;
        sync();
        return out;
    };
    auto gram_of = [&](const DBuf<double2>& J, int outer, int R, int inner) {
        DBuf<double> dG(c.arena, (size_t)R * R);
        launch_gram(J.get(), outer, R, inner, dG.get(), s);
        *c.launches += 1;
        std::vector<double> h((size_t)R * R);
        DOT_CUDA_TRY(cudaMemcpyAsync(h.data(), dG.get(), h.size() * 8, cudaMemcpyDeviceToHost, s));
        sync();
        for (int i = 0; i < R; ++i)
            for (int j = i + 1; j < R; ++j) {
                const double m = 0.5 * (h[(size_t)i * R + j] + h[(size_t)j * R + i]);
                h[(size_t)i * R + j] = h[(size_t)j * R + i] = m;
            }
        return h;
    };
    auto top = [&](const std::vector<double>& Gr, int R, int q) {
        std::vector<double> w, Z;
        sym_eig(R, Gr, w, Z);
        std::vector<double> T((size_t)R * q);
        for (int r = 0; r < R; ++r)
            for (int j = 0; j < q; ++j) T[(size_t)r * q + j] = Z[(size_t)r * R + j];
        return T;
    };

    // ---- phase one: remove a source (Theorem 3.5), then a detector (Theorem 3.4)
    for (int step = 0; step < k; ++step) {
        {
            DBuf<double2> J = contract(YV.get(), b, ZW.get(), a);
            std::vector<double> Gam = top(gram_of(J, nf * b, a, n_p), a, a - 1);
            W = matmul(W, ns, a, Gam, a - 1);
            ZW = combine(ZW, a, Gam, a - 1);
            --a;
        }
        {
            DBuf<double2> J = contract(YV.get(), b, ZW.get(), a);
            std::vector<double> Gam = top(gram_of(J, nf, b, a * n_p), b, b - 1);
            V = matmul(V, nd, b, Gam, b - 1);
            YV = combine(YV, b, Gam, b - 1);
            --b;
        }
    }

    // ---- one matrix-free add step.  side 0: new source (kept fields F = YV, b cols);
    // side 1: new detector (kept fields F = ZW, a cols).  M = current directions.
    auto add_step = [&](int side, std::vector<double>& M, int l, const DBuf<double2>& F, int nF,
                        const std::vector<double>& X0all, int step, DBuf<double2>& newfield) {
        const int n = side == 0 ? ns : nd;
        const std::vector<double> QM = orth_basis(M, n, l);
        auto project = [&](std::vector<double>& X, int cols) {      // X <- (I - QM QM^T) X
            for (int j = 0; j < cols; ++j)
                for (int p = 0; p < l; ++p) {
                    double d = 0;
                    for (int r = 0; r < n; ++r) d += QM[(size_t)r * l + p] * X[(size_t)r * cols + j];
                    for (int r = 0; r < n; ++r) X[(size_t)r * cols + j] -= d * QM[(size_t)r * l + p];
                }
        };
        // K Q (Q: n x blk, already in range(P)); also returns the fields of Q on S
        auto applyK = [&](const std::vector<double>& Q, DBuf<double2>& FQ) {
            FQ = fields(side, Q, blk);                                  // [nf][blk][K]
            // T[f][..] = Xr^T q in complex form
            DBuf<double2> J = side == 0 ? contract(F.get(), nF, FQ.get(), blk)    // [nf][nF][blk][n_p]
                                        : contract(FQ.get(), blk, F.get(), nF);   // [nf][blk][nF][n_p]
            std::vector<double2> T = to_host(J.get(), (size_t)nf * nF * blk * n_p);
            // coefficients C[f][q][i][k] = conj(T)
            std::vector<double2> Cc((size_t)nf * blk * nF * n_p);
            for (int f = 0; f < nf; ++f)
                for (int q = 0; q < blk; ++q)
                    for (int i = 0; i < nF; ++i)
                        for (int kk = 0; kk < n_p; ++kk) {
                            const size_t src = side == 0 ? (((size_t)f * nF + i) * blk + q) * n_p + kk
                                                         : (((size_t)f * blk + q) * nF + i) * n_p + kk;
                            const double2 t = T[src];
                            Cc[(((size_t)f * blk + q) * nF + i) * n_p + kk] = make_double2(t.x, -t.y);
                        }
            DBuf<double2> dC(c.arena, Cc.size()), w(c.arena, std::max<size_t>((size_t)nf * blk * K, 1));
            DOT_CUDA_TRY(cudaMemcpyAsync(dC.get(), Cc.data(), Cc.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
            launch_form_support_rhs(nf, blk, K, nF, n_p, dC.get(), F.get(), c.G, w.get(), s);
            *c.launches += 1;
            DBuf<double2> out(c.arena, (size_t)nf * blk * n);
            ops.solve_support(w.get(), blk, side, out.get());
            std::vector<double2> hs = to_host(out.get(), (size_t)nf * blk * n);
            std::vector<double> Y((size_t)n * blk, 0.0);
            for (int f = 0; f < nf; ++f)
                for (int q = 0; q < blk; ++q)
                    for (int r = 0; r < n; ++r) Y[(size_t)r * blk + q] -= hs[((size_t)f * blk + q) * n + r].x;
            project(Y, blk);
            return Y;
        };
        std::vector<double> Q((size_t)n * blk);              // start block of this add step
        for (int r = 0; r < n; ++r)
            for (int j = 0; j < blk; ++j) Q[(size_t)r * blk + j] = X0all[(size_t)r * k * blk + step * blk + j];
        project(Q, blk);
        Q = orth_basis(Q, n, blk);
        DBuf<double2> FQ;
        std::vector<double> Y = applyK(Q, FQ);
        for (int t = 1; t < iters; ++t) {
            Q = orth_basis(Y, n, blk);
            Y = applyK(Q, FQ);
        }
        // Rayleigh-Ritz: H = Q^T Y, top eigenvector e, q = Q e
        std::vector<double> H((size_t)blk * blk, 0.0);
        for (int i = 0; i < blk; ++i)
            for (int j = 0; j < blk; ++j) {
                double d = 0;
                for (int r = 0; r < n; ++r) d += Q[(size_t)r * blk + i] * Y[(size_t)r * blk + j];
                H[(size_t)i * blk + j] = d;
            }
        for (int i = 0; i < blk; ++i)
            for (int j = i + 1; j < blk; ++j) H[(size_t)i * blk + j] = H[(size_t)j * blk + i] =
                0.5 * (H[(size_t)i * blk + j] + H[(size_t)j * blk + i]);
        std::vector<double> e = top(H, blk, 1);
        std::vector<double> q = matmul(Q, n, blk, e, 1);
        double nr = 0;
        int imax = 0;
        for (int r = 0; r < n; ++r) {
            nr += q[r] * q[r];
            if (std::fabs(q[r]) > std::fabs(q[imax])) imax = r;
        }
        nr = std::sqrt(nr);
        const double sgn = q[imax] >= 0 ? 1.0 : -1.0;              // largest entry positive (oracle rule)
        const double scale = sgn * std::sqrt((double)n) / nr;      // length sqrt(n) (reading R15)
        std::vector<double> out((size_t)n * (l + 1));
        for (int r = 0; r < n; ++r) {
            for (int j = 0; j < l; ++j) out[(size_t)r * (l + 1) + j] = M[(size_t)r * l + j];
            out[(size_t)r * (l + 1) + l] = scale * q[r];
        }
        M.swap(out);
        // fields of the new column from the last block's fields (no extra solve)
        std::vector<double> ge(blk);
        for (int j = 0; j < blk; ++j) ge[j] = scale * e[j];
        newfield = combine(FQ, blk, ge, 1);
    };
    auto append_field = [&](DBuf<double2>& Fm, int cols, const DBuf<double2>& nfld) {
        DBuf<double2> out(c.arena, (size_t)nf * (cols + 1) * K);
        for (int f = 0; f < nf; ++f) {
            DOT_CUDA_TRY(cudaMemcpyAsync(out.get() + (size_t)f * (cols + 1) * K, Fm.get() + (size_t)f * cols * K,
                                         (size_t)cols * K * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            DOT_CUDA_TRY(cudaMemcpyAsync(out.get() + ((size_t)f * (cols + 1) + cols) * K, nfld.get() + (size_t)f * K,
                                         (size_t)K * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        }
        sync();
        Fm = std::move(out);
    };
    // ---- phase two: add a source (Theorem 3.7), then a detector (Theorem 3.6)
    for (int step = 0; step < k; ++step) {
        DBuf<double2> nfz, nfy;
        add_step(0, W, a, YV, b, X0s, step, nfz);
        append_field(ZW, a, nfz);
        ++a;
        add_step(1, V, b, ZW, a, X0d, step, nfy);
        append_field(YV, b, nfy);
        ++b;
    }
    DBuf<double2> J = contract(YV.get(), b, ZW.get(), a);
    DBuf<double> d_obj(c.arena, 1);
    launch_sumsq(J.get(), (size_t)nf * b * a * n_p, d_obj.get(), s);
    *c.launches += 1;
    double obj = 0;
    DOT_CUDA_TRY(cudaMemcpyAsync(&obj, d_obj.get(), 8, cudaMemcpyDeviceToHost, s));
    sync();
    return obj;
}

}  // namespace dot
