// K5: QR-TEBD with controlled bond expansion (apply_gate_qr_cbe,
// proj/src/gates.cpp:388-450).
//
//   eta = expanded_dim (InputError beyond d*chi); Y0 = theta[:eta]
//   sweep (DMMA GEMMs + K3 QR/LQ)            -> Q_m, L = Rp^H, Q_n = Rp'^H
//   G = L^H L = Rp Rp^H                       (DMMA GEMM)
//   (w, V) = eigh(G), descending               (device block Jacobi, jacobi.cu)
//   s = sqrt(max(w, 0)); kk = choose_kept(s / |theta|)   (host: O(eta) scalars)
//   Z = Qp V_k  ->  B~n = Z^H (d, kk, chi_r), B~m = phiev Z (permuted store)
//   Xi~ = diag(s_k) / |kept|;  eps = |theta - Q_m (L V_k) Z^H|^2 / |theta|^2
// The only host round trip is the eta eigenvalues needed for the data-
// dependent kept width kk.
#include <cmath>
#include <cstring>
#include <vector>

#include "gate.cuh"

namespace qt {
namespace {

__global__ void diag_bond_kernel(const double* __restrict__ w, long long kk, double inv, double2* xi) {
  const long long total = kk * kk;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / kk, j = e % kk;
    double v = 0.0;
    if (i == j) v = (w[i] > 0.0 ? sqrt(w[i]) : 0.0) * inv;
    xi[e] = make_double2(v, 0.0);
  }
}

__global__ void cbe_zero_flag_kernel(int* f) { *f = 0; }

// choose_kept, proj/src/gates.cpp:226-240
long long choose_kept(const std::vector<double>& s_norm, const qt_policy& p) {
  size_t k = 0;
  while (k < s_norm.size() && s_norm[k] >= p.sv_cutoff) ++k;
  k = std::min<size_t>(k, p.chi_max);
  if (p.target_eps > 0.0) {
    std::vector<double> suffix(s_norm.size() + 1, 0.0);
    for (size_t i = s_norm.size(); i-- > 0;) suffix[i] = suffix[i + 1] + s_norm[i] * s_norm[i];
    size_t kt = 0;
    while (kt < s_norm.size() && suffix[kt] > p.target_eps) ++kt;
    k = std::min(k, kt);
  }
  return static_cast<long long>(std::max<size_t>(k, 1));
}

void gemm2(Engine& e, Op oa, Op ob, long long M, long long N, long long K, const double2* A, long long lda,
           const double2* B, long long ldb, double2* C, long long ldc) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.opA = oa;
  g.opB = ob;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.C = C;
  g.ldc = ldc;
  zgemm(g, e.gemm_scratch(), e.stream);
}

}  // namespace

CbeResult gate_cbe(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* u, const qt_policy& pol, const std::function<GateBuffers(long long)>& alloc) {
  const long long eta = cbe_eta(pol, D);
  const long long d = D.d, cl = D.chi_l, cm = D.chi_m, cr = D.chi_r;
  const long long rows = D.rows(), cols = D.cols();
  int* flag = reinterpret_cast<int*>(e.dscal + SC_TMP3);
  cbe_zero_flag_kernel<<<1, 1, 0, e.stream>>>(flag);
  QT_LAUNCHED();
  build_theta(e, D, xi, bm, bn, u, SC_THETA2);
  double2* phiev = e.cbuf(S_PHIEV, cm * d * d * cr);
  double2* theta = e.cbuf(S_THETA, cl * d * d * cr);
  double2* X = e.cbuf(S_X, rows * eta);
  double2* Qm = e.cbuf(S_QM, rows * eta);
  double2* Rm = e.cbuf(S_RM, eta * eta);
  double2* YH = e.cbuf(S_YH, cols * eta);
  double2* Qp = e.cbuf(S_QP, cols * eta);
  double2* Rp = e.cbuf(S_RP, eta * eta);

  // alternating sweep with Y0 = theta[:eta] (gates.cpp:403-404, :293-308)
  const int sweeps = std::max(1, static_cast<int>(pol.qr_sweeps));
  // Y = Q_m^H theta through the reflectors of QR(X) (see gate_qr_async); theta
  // becomes Q_full^H theta, Q_m is never formed (CBE keeps no left_iso)
  const bool qtheta = use_qtheta(e, pol, rows);
  const bool x_split = qtheta && use_qr_pair(rows, cols) && x_split_applies(e, eta);
  for (int it = 0; it < sweeps; ++it) {
    if (x_split) {
      x_gemm_split(e, rows, eta, cols, theta, it == 0 ? theta : Qp, it == 0, X, flag);
    } else {
      if (it == 0)
        gemm2(e, Op::N, Op::H, rows, eta, cols, theta, cols, theta, cols, X, eta);
      else
        gemm2(e, Op::N, Op::N, rows, eta, cols, theta, cols, Qp, eta, X, eta);
      check_finite(e, X, rows * eta, flag);
    }
    if (qtheta && use_qr_pair(rows, cols)) {
      qr_pair_pipelined(e, X, rows, eta, theta, cols, YH, Qp, Rp);
      check_finite(e, theta, eta * cols, flag);
      continue;
    }
    if (qtheta) {
      QrOpts o;
      o.capply = theta;
      o.ldc = cols;
      o.nc = cols;
      o.want_q = false;
      o.want_r = false;
      qr_inplace(e, X, rows, eta, eta, Qm, eta, Rm, eta, o);
      qtheta_yh(e, theta, cols, X, eta, YH);
    } else {
      qr_inplace(e, X, rows, eta, eta, Qm, eta, Rm, eta);
      gemm2(e, Op::H, Op::N, cols, eta, rows, theta, cols, Qm, eta, YH, eta);
    }
    check_finite(e, YH, cols * eta, flag);
    qr_inplace(e, YH, cols, eta, eta, Qp, eta, Rp, eta);
  }

  // G = L^H L = Rp Rp^H, eigh descending (gates.cpp:408-410)
  double2* gm = e.cbuf(S_GRAM, eta * eta);
  gemm2(e, Op::N, Op::H, eta, eta, eta, Rp, eta, Rp, eta, gm, eta);
  double* w = e.dbuf(S_EIG_W, eta + 8);
  double2* V = e.cbuf(S_MISC2, eta * eta);
  const EighStatus* esw = eigh_device(e, gm, eta, w, V);

  std::vector<double> wh(static_cast<size_t>(eta));
  EighStatus eig_status{1, 0, 0.0, 0.0};
  QT_CUDA(cudaMemcpyAsync(wh.data(), w, eta * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaMemcpyAsync(e.hscal, e.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  if (esw) QT_CUDA(cudaMemcpyAsync(&eig_status, esw, sizeof(EighStatus), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  require_eigh_converged(eig_status, eta);
  int fl = 0;
  std::memcpy(&fl, &e.hscal[SC_TMP3], sizeof(int));
  if (fl) throw Error(Err::input, "qr_reduced: non-finite entries");
  const double theta2 = e.hscal[SC_THETA2];
  const double theta_norm = std::sqrt(theta2);
  if (theta_norm <= 0.0) throw Error(Err::numeric, "evolved block has zero norm");  // gates.cpp:415-416

  // s = sqrt(max(w, 0)); kk = choose_kept(s / |theta|) (gates.cpp:411-419)
  std::vector<double> s_norm(static_cast<size_t>(eta));
  for (long long i = 0; i < eta; ++i) s_norm[i] = (wh[i] > 0.0 ? std::sqrt(wh[i]) : 0.0) / theta_norm;
  const long long kk = choose_kept(s_norm, pol);
  double kept2 = 0.0;
  for (long long i = 0; i < kk; ++i) {
    const double s = wh[i] > 0.0 ? std::sqrt(wh[i]) : 0.0;
    kept2 += s * s;
  }
  const double kept_norm = std::sqrt(kept2);
  const double den = pol.skip_renormalize ? theta_norm : kept_norm;

  const GateBuffers out = alloc(kk);
  // Z = Qp V_k (cols x kk): B~n rows = V_k^H Q_n = Z^H (gates.cpp:421-423)
  double2* Z = YH;  // consumed by the QR above
  gemm2(e, Op::N, Op::N, cols, kk, eta, Qp, eta, V, eta, Z, kk);
  {
    const long long shp[3] = {d, cr, kk};
    const int perm[3] = {0, 2, 1};
    permute(e, Z, 3, shp, perm, true, out.b_n);
  }
  {
    // B~m (i, beta, k) = (phiev (cm*d x cols) . Z)[(beta i), k]  (gates.cpp:186-190)
    GemmDesc g;
    g.M = cm * d;
    g.N = kk;
    g.K = cols;
    g.A = phiev;
    g.lda = cols;
    g.B = Z;
    g.ldb = kk;
    g.C = out.b_m;
    g.ldc = cm * kk;
    g.rsplit = d;
    g.ldc_hi = kk;
    zgemm(g, e.gemm_scratch(), e.stream);
  }
  diag_bond_kernel<<<static_cast<int>(std::min<long long>(ceil_div(kk * kk, 256), 1024)), 256, 0, e.stream>>>(
      w, kk, den > 0.0 ? 1.0 / den : 0.0, out.xi);
  QT_LAUNCHED();

  HostReport rep;
  rep.theta2 = theta2;
  rep.kept2 = kept2;
  rep.finite = true;
  if (pol.compute_explicit_error) {
    // center_kept = L V_k V_k^H (gates.cpp:441-444): eps = |theta - Q_m (L V_k) Z^H|^2 / |theta|^2
    // consumed by the QR above (with qtheta X still carries the gauge phases of
    // R on its diagonal and the unused Rm holds L V_k instead)
    double2* LV = qtheta ? Rm : X;
    gemm2(e, Op::H, Op::N, eta, kk, eta, Rp, eta, V, eta, LV, kk);
    double2* W = e.cbuf(S_W, eta * cols);
    gemm2(e, Op::N, Op::H, eta, cols, kk, LV, kk, Z, kk, W, cols);
    if (qtheta) {
      qtheta_resid(e, theta, rows, cols, X, eta, W, e.dscal + SC_RESID);
    } else {
    GemmDesc g;
    g.M = rows;
    g.N = cols;
    g.K = eta;
    g.A = Qm;
    g.lda = eta;
    g.B = W;
    g.ldb = cols;
    g.C = theta;
    g.ldc = cols;
    g.mode = GemmMode::resid;
    zgemm(g, e.gemm_scratch(), e.stream, e.dscal + SC_RESID);
    }
    double r = 0.0;
    QT_CUDA(cudaMemcpyAsync(&r, e.dscal + SC_RESID, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    rep.resid = r;
  }
  CbeResult res;
  res.eta = eta;
  res.kk = kk;
  res.rep = rep;
  return res;
}

}  // namespace qt
