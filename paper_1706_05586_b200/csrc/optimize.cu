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

// device helpers of the matrix-free add step (n x cols row-major real blocks) --------------
__device__ double block_sum(double v, double* red) {     // result valid in every thread
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0;
    for (int w = 0; w < nw; ++w) t += red[w];     // fixed order: every thread the same value
    return t;
}

// X[:, j] <- (I - QM QM^T) X[:, j] for every column j (QM: n x l orthonormal, l <= 32); one block
// per column
__global__ void __launch_bounds__(256) proj_complement_kernel(const double* QM, int n, int l, double* X, int cols) {
    __shared__ double red[8], d[32];
    const int j = blockIdx.x;
    for (int p = 0; p < l; ++p) {
        double v = 0;
        for (int r = threadIdx.x; r < n; r += blockDim.x) v += QM[(size_t)r * l + p] * X[(size_t)r * cols + j];
        v = block_sum(v, red);
        if (threadIdx.x == 0) d[p] = v;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double x = X[(size_t)r * cols + j];
        for (int p = 0; p < l; ++p) x -= d[p] * QM[(size_t)r * l + p];
        X[(size_t)r * cols + j] = x;
    }
}

// orthonormal basis of the columns of X in place: modified Gram-Schmidt, two passes (one block);
// *fail = 1 for a zero column
__global__ void __launch_bounds__(1024) mgs_kernel(double* X, int n, int cols, int* fail) {
    __shared__ double red[32];
    for (int j = 0; j < cols; ++j) {
        for (int pass = 0; pass < 2; ++pass)
            for (int i = 0; i < j; ++i) {
                double v = 0;
                for (int r = threadIdx.x; r < n; r += blockDim.x) v += X[(size_t)r * cols + i] * X[(size_t)r * cols + j];
                v = block_sum(v, red);
                for (int r = threadIdx.x; r < n; r += blockDim.x) X[(size_t)r * cols + j] -= v * X[(size_t)r * cols + i];
                __syncthreads();
            }
        double v = 0;
        for (int r = threadIdx.x; r < n; r += blockDim.x) v += X[(size_t)r * cols + j] * X[(size_t)r * cols + j];
        const double nr = sqrt(block_sum(v, red));
        if (nr == 0.0) {
            if (threadIdx.x == 0) *fail = 1;
            return;
        }
        for (int r = threadIdx.x; r < n; r += blockDim.x) X[(size_t)r * cols + j] /= nr;
        __syncthreads();
    }
}

// C[f][q][i][k] = conj(T) with T = J[f][i][q][k] (side 0: J = [nf][nF][blk][n_p]) or
// J[f][q][i][k] (side 1: J = [nf][blk][nF][n_p])
__global__ void conj_reorder_kernel(const double2* J, int nf, int blk, int nF, int n_p, int side, double2* C) {
    const size_t tot = (size_t)nf * blk * nF * n_p;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const int kk = (int)(e % n_p);
        size_t t = e / n_p;
        const int i = (int)(t % nF);
        t /= nF;
        const int q = (int)(t % blk);
        const int f = (int)(t / blk);
        const size_t src = side == 0 ? (((size_t)f * nF + i) * blk + q) * n_p + kk : (((size_t)f * blk + q) * nF + i) * n_p + kk;
        const double2 v = J[src];
        C[e] = make_double2(v.x, -v.y);
    }
}

// Y[r][q] = - sum_f Re(out[f][q][r])
__global__ void neg_re_sum_kernel(const double2* out, int nf, int blk, int n, double* Y) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * blk; e += gridDim.x * blockDim.x) {
        const int r = e / blk, q = e % blk;
        double v = 0;
        for (int f = 0; f < nf; ++f) v -= out[((size_t)f * blk + q) * n + r].x;
        Y[e] = v;
    }
}

// H[i][j] = sum_r A[r][i] B[r][j] (n x c blocks); one block per entry
__global__ void __launch_bounds__(256) small_atb_kernel(const double* A, const double* B, int n, int c, double* H) {
    __shared__ double red[8];
    const int i = blockIdx.x / c, j = blockIdx.x % c;
    double v = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) v += A[(size_t)r * c + i] * B[(size_t)r * c + j];
    v = block_sum(v, red);
    if (threadIdx.x == 0) H[blockIdx.x] = v;
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
        launch_contract(nf, K, b, a, n_p, lam, (size_t)b * K, u, (size_t)a * K, c.G, J.get(), s, c.gsp, &c.arena,
                        c.launches);
        *c.launches += 2;
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
    const int nf = c.nf, ns = c.ns, nd = c.nd, n_p = c.n_p, K = c.K, nP = c.nP;
    cudaStream_t s = c.stream;
    auto sync = [&]() { DOT_CUDA_TRY(cudaStreamSynchronize(s)); };
    // fields of device coefficients on S ([nf][ncols][K], returned) and on the samples P (outP)
    auto fields = [&](int side, const double* d_coeff, int ncols, DBuf<double2>& outP) {
        DBuf<double2> out(c.arena, std::max<size_t>((size_t)nf * ncols * K, 1));
        outP = DBuf<double2>(c.arena, std::max<size_t>((size_t)nf * ncols * nP, 1));
        ops.fields(side, d_coeff, ncols, out.get(), outP.get());
        return out;
    };
    // z fields of W and y fields of V on S [nf][cols][K] (contractions) and on the samples P
    // [nf][cols][nP] (kept in step, so that the final W, V leave their fields in the caches)
    DBuf<double2> ZW(c.arena, std::max<size_t>((size_t)nf * ls * K, 1)), YV(c.arena, std::max<size_t>((size_t)nf * ld * K, 1));
    DBuf<double2> ZWP(c.arena, std::max<size_t>((size_t)nf * ls * nP, 1)), YVP(c.arena, std::max<size_t>((size_t)nf * ld * nP, 1));
    ops.start_fields(W, ls, V, ld, ZW.get(), YV.get(), ZWP.get(), YVP.get());
    sync();
    int a = ls, b = ld;

    auto contract = [&](const double2* lam, int nl, const double2* u, int nu) {
        DBuf<double2> J(c.arena, std::max<size_t>((size_t)nf * nl * nu * n_p, 1));
        launch_contract(nf, K, nl, nu, n_p, lam, (size_t)nl * K, u, (size_t)nu * K, c.G, J.get(), s, c.gsp, &c.arena,
                        c.launches);
        return J;
    };
    // new fields F' [nf][m][L] = sum_j Gam[j][m] F[f][j][L]  (Gam host [ncols][m]; L = K or nP)
    auto combine = [&](const DBuf<double2>& F, int ncols, const std::vector<double>& Gam, int m, int L) {
        DBuf<double> dG(c.arena, Gam.size());
        DOT_CUDA_TRY(cudaMemcpyAsync(dG.get(), Gam.data(), Gam.size() * 8, cudaMemcpyHostToDevice, s));
        DBuf<double2> out(c.arena, std::max<size_t>((size_t)nf * m * L, 1));
        launch_rc_gemm(nf, m, L, ncols, dG.get(), m, F.get(), (size_t)ncols * L, L, 1, out.get(), (size_t)m * L, L, 1, s);
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
            ZW = combine(ZW, a, Gam, a - 1, K);
            ZWP = combine(ZWP, a, Gam, a - 1, nP);
            --a;
        }
        {
            DBuf<double2> J = contract(YV.get(), b, ZW.get(), a);
            std::vector<double> Gam = top(gram_of(J, nf, b, a * n_p), b, b - 1);
            V = matmul(V, nd, b, Gam, b - 1);
            YV = combine(YV, b, Gam, b - 1, K);
            YVP = combine(YVP, b, Gam, b - 1, nP);
            --b;
        }
    }

    // ---- one matrix-free add step.  side 0: new source (kept fields F = YV, b cols);
    // side 1: new detector (kept fields F = ZW, a cols).  M = current directions.  The block
    // Q, its image Y = K Q, the projection onto the complement of span(M) and the
    // orthonormalisation stay on the device; only the blk x blk Rayleigh-Ritz matrix and the
    // final block come to the host.
    DBuf<int> dfail(c.arena, 1);
    DOT_CUDA_TRY(cudaMemsetAsync(dfail.get(), 0, sizeof(int), s));
    auto add_step = [&](int side, std::vector<double>& M, int l, const DBuf<double2>& F, int nF,
                        const std::vector<double>& X0all, int step, DBuf<double2>& newfield,
                        DBuf<double2>& newfieldP) {
        const int n = side == 0 ? ns : nd;
        const std::vector<double> QMh = orth_basis(M, n, l);
        DBuf<double> QM(c.arena, QMh.size()), dQ(c.arena, (size_t)n * blk), dY(c.arena, (size_t)n * blk);
        DOT_CUDA_TRY(cudaMemcpyAsync(QM.get(), QMh.data(), QMh.size() * 8, cudaMemcpyHostToDevice, s));
        auto project = [&](double* X) {                            // X <- (I - QM QM^T) X
            proj_complement_kernel<<<blk, 256, 0, s>>>(QM.get(), n, l, X, blk);
            DOT_CUDA_TRY(cudaGetLastError());
            *c.launches += 1;
        };
        auto orth = [&](double* X) {
            mgs_kernel<<<1, 1024, 0, s>>>(X, n, blk, dfail.get());
            DOT_CUDA_TRY(cudaGetLastError());
            *c.launches += 1;
        };
        // Y = K Q (Q: n x blk in range(P)); FQ receives the fields of Q on S
        auto applyK = [&](DBuf<double2>& FQ, DBuf<double2>& FQP) {
            FQ = fields(side, dQ.get(), blk, FQP);                          // [nf][blk][K], [nf][blk][nP]
            // T[f][..] = Xr^T q in complex form; coefficients C[f][q][i][k] = conj(T)
            DBuf<double2> J = side == 0 ? contract(F.get(), nF, FQ.get(), blk)    // [nf][nF][blk][n_p]
                                        : contract(FQ.get(), blk, F.get(), nF);   // [nf][blk][nF][n_p]
            const size_t nC = (size_t)nf * blk * nF * n_p;
            DBuf<double2> dC(c.arena, std::max<size_t>(nC, 1)), w(c.arena, std::max<size_t>((size_t)nf * blk * K, 1));
            conj_reorder_kernel<<<(unsigned)std::min<size_t>((nC + 255) / 256, 1024), 256, 0, s>>>(J.get(), nf, blk,
                                                                                                nF, n_p, side, dC.get());
            DOT_CUDA_TRY(cudaGetLastError());
            launch_form_support_rhs(nf, blk, K, nF, n_p, dC.get(), F.get(), c.G, w.get(), s);
            DBuf<double2> out(c.arena, (size_t)nf * blk * n);
            ops.solve_support(w.get(), blk, side, out.get());
            neg_re_sum_kernel<<<(n * blk + 255) / 256, 256, 0, s>>>(out.get(), nf, blk, n, dY.get());
            DOT_CUDA_TRY(cudaGetLastError());
            *c.launches += 3;
            project(dY.get());
        };
        std::vector<double> Q0((size_t)n * blk);              // start block of this add step
        for (int r = 0; r < n; ++r)
            for (int j = 0; j < blk; ++j) Q0[(size_t)r * blk + j] = X0all[(size_t)r * k * blk + step * blk + j];
        DOT_CUDA_TRY(cudaMemcpyAsync(dQ.get(), Q0.data(), Q0.size() * 8, cudaMemcpyHostToDevice, s));
        project(dQ.get());
        orth(dQ.get());
        DBuf<double2> FQ, FQP;
        applyK(FQ, FQP);
        for (int t = 1; t < iters; ++t) {
            DOT_CUDA_TRY(cudaMemcpyAsync(dQ.get(), dY.get(), (size_t)n * blk * 8, cudaMemcpyDeviceToDevice, s));
            orth(dQ.get());
            applyK(FQ, FQP);
        }
        // Rayleigh-Ritz: H = Q^T Y (device), top eigenvector e (host), q = Q e
        DBuf<double> dH(c.arena, (size_t)blk * blk);
        small_atb_kernel<<<blk * blk, 256, 0, s>>>(dQ.get(), dY.get(), n, blk, dH.get());
        DOT_CUDA_TRY(cudaGetLastError());
        *c.launches += 1;
        std::vector<double> H((size_t)blk * blk), Q((size_t)n * blk);
        int failed = 0;
        DOT_CUDA_TRY(cudaMemcpyAsync(H.data(), dH.get(), H.size() * 8, cudaMemcpyDeviceToHost, s));
        DOT_CUDA_TRY(cudaMemcpyAsync(Q.data(), dQ.get(), Q.size() * 8, cudaMemcpyDeviceToHost, s));
        DOT_CUDA_TRY(cudaMemcpyAsync(&failed, dfail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        sync();
        if (failed) throw Error(DOT_ERR_ARG, "subspace block is rank deficient");
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
        std::vector<double> outM((size_t)n * (l + 1));
        for (int r = 0; r < n; ++r) {
            for (int j = 0; j < l; ++j) outM[(size_t)r * (l + 1) + j] = M[(size_t)r * l + j];
            outM[(size_t)r * (l + 1) + l] = scale * q[r];
        }
        M.swap(outM);
        // fields of the new column from the last block's fields (no extra solve)
        std::vector<double> ge(blk);
        for (int j = 0; j < blk; ++j) ge[j] = scale * e[j];
        newfield = combine(FQ, blk, ge, 1, K);
        newfieldP = combine(FQP, blk, ge, 1, nP);
    };
    auto append_field = [&](DBuf<double2>& Fm, int cols, const DBuf<double2>& nfld, int L) {
        DBuf<double2> out(c.arena, (size_t)nf * (cols + 1) * L);
        for (int f = 0; f < nf; ++f) {
            DOT_CUDA_TRY(cudaMemcpyAsync(out.get() + (size_t)f * (cols + 1) * L, Fm.get() + (size_t)f * cols * L,
                                         (size_t)cols * L * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            DOT_CUDA_TRY(cudaMemcpyAsync(out.get() + ((size_t)f * (cols + 1) + cols) * L, nfld.get() + (size_t)f * L,
                                         (size_t)L * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        }
        sync();
        Fm = std::move(out);
    };
    // ---- phase two: add a source (Theorem 3.7), then a detector (Theorem 3.6)
    for (int step = 0; step < k; ++step) {
        DBuf<double2> nfz, nfy, nfzP, nfyP;
        add_step(0, W, a, YV, b, X0s, step, nfz, nfzP);
        append_field(ZW, a, nfz, K);
        append_field(ZWP, a, nfzP, nP);
        ++a;
        add_step(1, V, b, ZW, a, X0d, step, nfy, nfyP);
        append_field(YV, b, nfy, K);
        append_field(YVP, b, nfyP, nP);
        ++b;
    }
    DBuf<double2> J = contract(YV.get(), b, ZW.get(), a);
    DBuf<double> d_obj(c.arena, 1);
    launch_sumsq(J.get(), (size_t)nf * b * a * n_p, d_obj.get(), s);
    *c.launches += 1;
    double obj = 0;
    DOT_CUDA_TRY(cudaMemcpyAsync(&obj, d_obj.get(), 8, cudaMemcpyDeviceToHost, s));
    sync();
    ops.finish(W, a, ZWP, V, b, YVP);      // the optimized W, V and their fields on P -> field caches
    return obj;
}

}  // namespace dot
