// Simultaneous optimized sources and detectors (Sec. 3.2, Sec. 3.3.2).
#pragma once
#include <vector>

#include "arena.h"
#include "kernels.h"

namespace dot {

struct OptContext {
    Arena& arena;
    cudaStream_t stream;
    int nf, ns, nd, n_p, K, nP;
    const double2* XU;        // full-data source fields on samples [nf][ns][nP]
    const double2* XL;        // full-data detector (adjoint) fields [nf][nd][nP]
    const int32_t* S_slot;    // [K] sample slot of each support node
    const double* G;          // [K][n_p]
    int64_t* launches;
};

// Two-phase alternating replacement of k directions; W (ns x ls) and V (nd x ld)
// row-major host matrices, updated in place.  Returns ||(W^T (x) V^T) J||_F^2.
double optimize_two_phase(OptContext& c, int k, std::vector<double>& W, int ls, std::vector<double>& V, int ld);

// Host symmetric eigen-decomposition (Householder tridiagonalisation + implicit
// QL); eigenvalues descending in w, eigenvectors as columns of Z (row-major n x n).
void sym_eig(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& Z);

// Device Gram matrix of a complex array X[o][r][i] (o < outer, r < R, i < inner):
// Gr[r][r'] = Re sum_{o,i} X[o][r][i] conj(X[o][r'][i]).
void launch_gram(const double2* X, int outer, int R, int inner, double* Gr, cudaStream_t s);

}  // namespace dot
