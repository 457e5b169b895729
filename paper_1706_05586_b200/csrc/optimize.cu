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
        launch_contract(nf, K, b, a, n_p, lam, (size_t)b * K, u, (size_t)a * K, c.G, J.get(), s);
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

}  // namespace dot
