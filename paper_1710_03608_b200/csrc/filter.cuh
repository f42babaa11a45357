#pragma once
#include <vector>
#include "ctx.cuh"

namespace ctdgpu {

// FiberBasis (fiber_basis.hpp:21-61) resident in HBM: R (kept fibers, owned
// copies, CSC in acceptance order), a row index of R (per row, the kept
// columns containing it in ascending k — the order the reference's z scatter
// visits them), the first-appearance order of R's rows (the reference's
// `touched` order when every y_k != 0), and U = (R^T R)^-1 dense, leading
// dimension LD.  U is kept exactly symmetric, as the reference's is.
constexpr double kWPanelBytes = 8.0e9;  // largest W panel kept on the device

struct Basis {
  Ctx* ctx = nullptr;
  int64_t dim = 0;
  int64_t K = 0;     // kept columns
  int64_t LD = 0;    // U capacity (rows = cols)
  Buf<double> U;
  int64_t kcap = 0, rcap = 0, rnnz = 0;
  Buf<int64_t> rptr;  // [kcap+1]
  Buf<int32_t> rrow;  // [rcap]
  Buf<double> rval;   // [rcap]
  int64_t ricap = 0;
  Buf<int64_t> rowbase;  // [dim+1]
  Buf<int32_t> rowlen;   // [dim]
  Buf<int32_t> rek;      // [ricap] kept-column index
  Buf<double> rev;       // [ricap] value
  Buf<int32_t> sr_list;  // [dim] rows of R in first-appearance order
  Buf<int32_t> sr_pos;   // [dim] position in sr_list or -1
  Buf<int> sr_n;         // device count
  int64_t srn = 0;
  Buf<uint32_t> tag;     // [dim] candidate tag of the rows of the current x
  uint32_t tag_base = 0;
  Buf<double> zd;        // [dim]
  Buf<int32_t> kf;       // [dim] dynamic first k (slow path)
  // W = R T with U = T T^T: the orthonormal panel [dim][LD] (row-major) the
  // error pass gathers; Wok when it holds all K columns
  Buf<double> W;
  bool want_panel = false;  // maintain W (callers that will evaluate the error)
  bool Wok = false;
  std::vector<double> Wscale;  // 1/delta of each kept column (host)
  Buf<double> Wsc;             // the same on the device
  // Q: orthonormal basis of span(R) for the error pass (relerr.cu,
  // ortho_panel), cached for basis size Qk; Newton-Schulz iterations and the
  // starting defect |A^T A - I|_F of the last build
  // (Qcompl: the panel is (I - R U R^T)^T instead, Qcols = dim, for a basis
  // whose R U R^T is no projector)
  mutable Buf<double> Q;
  mutable int64_t Qk = -1, Qld = 0, Qcols = 0;
  mutable int Qiters = 0;
  mutable double Qdefect = 0.0;
  // P = Q E^T: the second-order correction panel of the error pass (relerr.cu
  // build_correction), kept when |E|_F^2 >= 1e-11
  mutable Buf<double> P;
  mutable bool Pok = false;
  mutable double Enorm = 0.0;
  mutable bool Qcompl = false;

  Basis(Ctx* c, int64_t d);
  // Copy R's host CSC and U (resume ctor, fiber_basis.cpp:13-19).
};

// Candidate fibers (device): candidate c = rows/vals [off[c], off[c]+len[c]).
struct Cands {
  int64_t n = 0;
  const int64_t* off = nullptr;
  const int32_t* len = nullptr;
  const int32_t* row = nullptr;
  const double* val = nullptr;
};

// Per-candidate outcome of try_append_fiber (fiber_basis.hpp:30-37).
struct BatchOut {
  std::vector<int32_t> accepted, degenerate;
  std::vector<double> delta, res_sq, x_sq;
  std::vector<int32_t> kept_cand;  // candidates accepted, in order
  std::vector<double> y_last;      // y of the last candidate (U R^T x)
  bool slow_path = false;
  int64_t n_spec = 0;              // rejections certified in batches (spec.cu)
};

// Runs the reference filter loop (ctd_static.cpp:40-44) over all candidates
// in order against the basis, appending the accepted ones.
void filter_batch(Basis& B, const Cands& c, double eps, BatchOut& out, bool want_y);

// Speculative rejection batches (spec.cu): evaluates candidates [pos, pos+b)
// against the current basis (K columns; Gram tables Gb [K0][n], Gc [n][n],
// kept_cand[k - K0] the candidate behind basis column k) and returns how many
// leading ones are certified rejections, writing their outcomes.
int64_t spec_certify(Basis& B, const Cands& c, const double* xsq, const double* Gb, const double* Gc,
                     const int* kept_cand, int64_t K0, int64_t K, int64_t pos, int64_t b, double eps, int32_t* acc,
                     int32_t* deg, double* dl, double* res_out);

// Loads a given R (host CSC: K columns over B.dim rows, rows ascending within
// a column) and optionally U (K x K row-major) into an empty basis, with R's
// row index: the operand form compute_core / chain_product read (read-only
// use; the filter's first-appearance bookkeeping is not rebuilt).
void basis_load(Basis& B, int64_t K, const int64_t* col_ptr, const int64_t* rows, const double* vals,
                const double* u);

// Host copies of the basis.
void basis_u(const Basis& B, double* u /* K*K row-major */);
void basis_r(const Basis& B, int64_t* col_ptr, int64_t* rows, double* vals);

}  // namespace ctdgpu
