// Simultaneous optimized sources and detectors (Sec. 3.2, Sec. 3.3.2).
#pragma once
#include <functional>
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
    const GSparse* gsp = nullptr;   // block sparsity of G (null: dense contraction)
};

// Two-phase alternating replacement of k directions; W (ns x ls) and V (nd x ld)
// row-major host matrices, updated in place.  Returns ||(W^T (x) V^T) J||_F^2.
double optimize_two_phase(OptContext& c, int k, std::vector<double>& W, int ls, std::vector<double>& V, int ld);

// Solver callbacks of the matrix-free (subspace-iteration) variant, provided by the
// C-ABI layer (they run the batched multi-shift CG kernels; no host synchronisation needed):
struct SubspaceOps {
    // fields of point combinations on the support S: side 0 = B coeff (sources), 1 = C coeff
    // (detectors); coeff device [n_side][ncols] row-major; out device [nf][ncols][K], outP the
    // same fields on the samples P [nf][ncols][nP]
    std::function<void(int side, const double* d_coeff, int ncols, double2* out, double2* outP)> fields;
    // solve A_f x = w_f for nvec right-hand sides supported on S (w device [nf][nvec][K]) and
    // return b_s^T x (side 0, sources; b_s = theta e_s / cell volume) or c_d^T x (side 1):
    // out device [nf][nvec][n_side]
    std::function<void(const double2* w, int nvec, int side, double2* out)> solve_support;
    // fields of the starting W (ns x ls) and V (nd x ld) on S, zw [nf][ls][K], yv [nf][ld][K],
    // and on P, zwP [nf][ls][nP], yvP [nf][ld][nP]: from the library's field caches when the
    // preceding jacobian / misfit call solved them, else both sides in one joint batch
    std::function<void(const std::vector<double>& W, int ls, const std::vector<double>& V, int ld, double2* zw,
                       double2* yv, double2* zwP, double2* yvP)>
        start_fields;
    // hands the optimized W (ns x a), V (nd x b) and their fields on P (ownership moves) to the
    // library's field caches: a following jacobian / misfit with these W, V needs no solves
    std::function<void(const std::vector<double>& W, int a, DBuf<double2>& zwP, const std::vector<double>& V, int b,
                       DBuf<double2>& yvP)>
        finish;
};

// Two-phase replacement where the add steps (Theorems 3.7, 3.6) use `iters` steps of
// subspace iteration with a `blk`-vector block (reading R16) applied
// matrix-free (2 n_freq solves per block vector per step); the remove steps use the
// sketched Jacobian of the current W, V.  X0s [ns][k*blk], X0d [nd][k*blk]: add step t
// starts from columns t*blk .. (t+1)*blk - 1.
double optimize_two_phase_subspace(OptContext& c, SubspaceOps& ops, int k, int iters, int blk,
                                   std::vector<double>& W, int ls, std::vector<double>& V, int ld,
                                   const std::vector<double>& X0s, const std::vector<double>& X0d);

// Host symmetric eigen-decomposition (Householder tridiagonalisation + implicit
// QL); eigenvalues descending in w, eigenvectors as columns of Z (row-major n x n).
void sym_eig(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& Z);

// Device Gram matrix of a complex array X[o][r][i] (o < outer, r < R, i < inner):
// Gr[r][r'] = Re sum_{o,i} X[o][r][i] conj(X[o][r'][i]).
void launch_gram(const double2* X, int outer, int R, int inner, double* Gr, cudaStream_t s);

}  // namespace dot
