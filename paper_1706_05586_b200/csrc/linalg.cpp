// Host dense symmetric eigensolver for the small SVD problems of PAPER.md
// Sec. 3.3.2 / Table 1 (left singular vectors of M = eigenvectors of M M^T,
// Lemma 3.2).  Householder reduction to tridiagonal form followed by the
// implicit QL iteration with Wilkinson-type shifts (the classical
// tred2 / tql2 pair, written out here from the textbook algorithm).
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <vector>

namespace dot {

void sym_eig(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& Z) {
    // A: row-major n x n symmetric.  On exit w[i] descending, Z[:, i] eigenvectors.
    if (n <= 0) {
        w.clear();
        Z.clear();
        return;
    }
    auto a = [&](int i, int j) -> double& { return A[(size_t)i * n + j]; };
    std::vector<double> d(n), e(n);
    // ---- Householder tridiagonalisation; A accumulates the orthogonal transform
    for (int i = n - 1; i > 0; --i) {
        const int l = i - 1;
        double h = 0.0, scale = 0.0;
        if (l > 0) {
            for (int k = 0; k <= l; ++k) scale += std::fabs(a(i, k));
            if (scale == 0.0) {
                e[i] = a(i, l);
            } else {
                for (int k = 0; k <= l; ++k) {
                    a(i, k) /= scale;
                    h += a(i, k) * a(i, k);
                }
                double f = a(i, l);
                double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
                e[i] = scale * g;
                h -= f * g;
                a(i, l) = f - g;
                f = 0.0;
                for (int j = 0; j <= l; ++j) {
                    a(j, i) = a(i, j) / h;
                    g = 0.0;
                    for (int k = 0; k <= j; ++k) g += a(j, k) * a(i, k);
                    for (int k = j + 1; k <= l; ++k) g += a(k, j) * a(i, k);
                    e[j] = g / h;
                    f += e[j] * a(i, j);
                }
                const double hh = f / (h + h);
                for (int j = 0; j <= l; ++j) {
                    f = a(i, j);
                    g = e[j] - hh * f;
                    e[j] = g;
                    for (int k = 0; k <= j; ++k) a(j, k) -= (f * e[k] + g * a(i, k));
                }
            }
        } else {
            e[i] = a(i, l);
        }
        d[i] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (int i = 0; i < n; ++i) {
        const int l = i - 1;
        if (d[i] != 0.0) {
            for (int j = 0; j <= l; ++j) {
                double g = 0.0;
                for (int k = 0; k <= l; ++k) g += a(i, k) * a(k, j);
                for (int k = 0; k <= l; ++k) a(k, j) -= g * a(k, i);
            }
        }
        d[i] = a(i, i);
        a(i, i) = 1.0;
        for (int j = 0; j <= l; ++j) a(j, i) = a(i, j) = 0.0;
    }
    // ---- implicit QL on the tridiagonal (d, e); rotations applied to A's columns
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    const double epsm = std::numeric_limits<double>::epsilon();
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= epsm * dd) break;
            }
            if (m != l) {
                if (iter++ == 200) throw std::runtime_error("sym_eig: QL iteration did not converge");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                bool underflow = false;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[i], b = c * e[i];
                    r = std::hypot(f, g);
                    e[i + 1] = r;
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        underflow = true;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    for (int k = 0; k < n; ++k) {
                        f = a(k, i + 1);
                        a(k, i + 1) = s * a(k, i) + c * f;
                        a(k, i) = c * a(k, i) - s * f;
                    }
                }
                if (underflow) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    // ---- sort descending
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return d[x] > d[y]; });
    w.resize(n);
    Z.assign((size_t)n * n, 0.0);
    for (int c = 0; c < n; ++c) {
        w[c] = d[idx[c]];
        for (int r = 0; r < n; ++r) Z[(size_t)r * n + c] = a(r, idx[c]);
    }
}

}  // namespace dot

extern "C" int dot_sym_eig(int n, const double* A, double* w, double* Z) {
    try {
        std::vector<double> a(A, A + (size_t)n * n), ww, zz;
        dot::sym_eig(n, a, ww, zz);
        std::copy(ww.begin(), ww.end(), w);
        std::copy(zz.begin(), zz.end(), Z);
        return 0;
    } catch (...) {
        return 1;
    }
}
