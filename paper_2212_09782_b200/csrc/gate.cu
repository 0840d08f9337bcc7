// Two-site QR-TEBD update on the device.
//
// Data flow of apply_gate_qr (proj/src/gates.cpp:343-386), all complex128 in
// HBM, no host round trip inside the update:
//
//   phi(b,i,j,d)   = sum_g Bm[i,b,g] Bn[j,g,d]     DMMA GEMM, batched over j,
//                                                   store permuted (gates.cpp:145-165)
//   phiev(b,.,.,d) = U . phi(b,.,.,d)               DMMA GEMM, batched over b
//                                                   (gates.cpp:168-171; the
//                                                   transpose(2,0,1,3) is never
//                                                   materialized)
//   theta          = Xi . phiev                     DMMA GEMM  (gates.cpp:175-180)
//   X = theta Y0^H ; QR ; Y^H = theta^H Q ; QR      DMMA GEMMs + K3 (gates.cpp:293-308)
//   Xi~ = L/|L|, B~n = Q_n -> (d,eta,chi_r), B~m = phiev Q_n^H (permuted store),
//   left_iso = Q_m -> (d,chi_l,eta), eps = ||theta - Q_m L Q_n||^2/||theta||^2
//
// For one sweep on 128..2048-row matrices the two QRs run as a pipelined pair
// (qr_pair_pipelined, householder.cu): each QR(X) panel's reflector is applied
// to theta behind the panel chain, so Q_full^H theta = [Y; Z] replaces the
// explicit Q_m and the theta^H Q_m product, QR(Y^H) runs one panel behind on
// its own stream, and eps = (||Y - L Q_n||^2 + ||Z||^2) / ||theta||^2.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gate.cuh"

namespace qt {

unsigned long long expanded_dim(const qt_policy& p, unsigned long long chi, unsigned long long d) {
  const auto rel = static_cast<unsigned long long>(std::ceil(p.delta_chi_rel * static_cast<double>(chi)));
  const unsigned long long delta = std::max<unsigned long long>(p.delta_chi_abs, rel);
  unsigned long long eta = std::min(d * chi, chi + delta);
  if (p.chi_max_expansion != 0) eta = std::min<unsigned long long>(eta, p.chi_max_expansion);
  return eta;
}

long long qr_eta(const qt_policy& p, const Dims& D) {
  long long eta = static_cast<long long>(
      std::min<unsigned long long>(expanded_dim(p, D.chi_n, D.d), p.chi_max));
  return std::min({eta, D.rows(), D.cols()});
}

long long cbe_eta(const qt_policy& p, const Dims& D) {
  const unsigned long long eta0 = expanded_dim(p, D.chi_n, D.d);
  if (eta0 > static_cast<unsigned long long>(D.d * D.chi_n)) throw Error(Err::input, "bond expansion beyond d*chi");
  return std::min({static_cast<long long>(eta0), D.rows(), D.cols()});
}

namespace {

// dscal[out] = (den > 0) ? 1/den : 0 with den = sqrt(dscal[skip ? a : b])
__global__ void inv_norm_kernel(double* dscal, int a, int b, int skip, int out) {
  const double den = sqrt(dscal[skip ? a : b]);
  dscal[out] = den > 0.0 ? 1.0 / den : 0.0;
}

__global__ void zero_flag_kernel(int* f) { *f = 0; }

// Y^H from Q_full^H theta: yh[c, i] = ph_i conj(qt[i, c]) for i < eta, i.e.
// Y = Q_m^H theta with the gauge-fixed Q_m = Q_raw diag(ph)  (32 x 32 tiles)
// (rows [ibeg, iend) of qt; yh and the factored X share the leading dimension lda = eta)
__global__ void yh_gauge_kernel(const double2* __restrict__ qt, long long cols, const double2* __restrict__ a,
                                long long lda, long long iend, double2* __restrict__ yh, long long ibeg) {
  __shared__ double2 tile[32][33];
  const long long i0 = ibeg + static_cast<long long>(blockIdx.y) * 32, c0 = static_cast<long long>(blockIdx.x) * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long i = i0 + r, c = c0 + threadIdx.x;
    if (i < iend && c < cols) {
      const double2 v = qt[i * cols + c];
      const double2 ph = qr_phase(a, lda, i);
      tile[r][threadIdx.x] = cmul(ph, cconj(v));
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const long long c = c0 + r, i = i0 + threadIdx.x;
    if (c < cols && i < iend) yh[c * lda + i] = tile[threadIdx.x][r];
  }
}

// explicit truncation error from Q_full^H theta (gates.cpp:464-485 by unitary
// invariance): ||theta - Q_m W||^2 = ||Y - W||^2 + ||Z||^2 with Y (gauged) the
// first eta rows of Q_full^H theta, Z the rest and W = L Q_n; fixed-order
// two-pass reduction
__global__ void qtheta_resid_partial_kernel(const double2* __restrict__ qt, long long rows, long long cols,
                                            const double2* __restrict__ a, long long lda, long long eta,
                                            const double2* __restrict__ w, double* part) {
  // block b owns rows b, b + gridDim.x, ...: one phase per row, coalesced
  // column sweeps, two accumulation chains; fixed order -> deterministic
  __shared__ double sh[256];
  double s = 0.0, s1 = 0.0;
  for (long long i = blockIdx.x; i < rows; i += gridDim.x) {
    const double2* row = qt + i * cols;
    if (i < eta) {
      if (!w) continue;  // Z only (w == nullptr)
      const double2 ph = cconj(qr_phase(a, lda, i));
      const double2* wr = w + i * cols;
      for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
        const double2 v = csub(cmul(ph, row[c]), wr[c]);
        s = fma(v.x, v.x, fma(v.y, v.y, s));
      }
    } else {
      for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
        const double2 v = row[c];
        s1 = fma(v.x, v.x, fma(v.y, v.y, s1));
      }
    }
  }
  s += s1;
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// one warp: lane l sums part[l], part[l + 32], ... in order, then a fixed
// shuffle tree (deterministic; the loads of all lanes issue in parallel)
__global__ void sum_final_kernel(const double* __restrict__ part, int n, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

constexpr int kResidBlocks = 296;

__global__ void trace_op_kernel(const double2* __restrict__ op, const double2* __restrict__ t2, int d,
                                double* out2) {
  // <O> = sum_{x,y} op[x,y] t2[y,x]   (proj/src/mps.cpp:173)
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int x = 0; x < d; ++x)
      for (int y = 0; y < d; ++y) s = cadd(s, cmul(op[x * d + y], t2[y * d + x]));
    out2[0] = s.x;
    out2[1] = s.y;
  }
}

__global__ void defect_partial_kernel(const double2* __restrict__ g, long long n, double* part) {
  __shared__ double sh[256];
  double m = 0.0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / n, c = e % n;
    double2 v = g[e];
    if (r == c) v.x -= 1.0;
    m = fmax(m, hypot(v.x, v.y));
  }
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void max_final_kernel(const double* __restrict__ part, int n, double* out) {
  double m = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) m = fmax(m, part[i]);
    *out = m;
  }
}

// sum conj(a) b over n elements, two-pass deterministic
__global__ void dot_partial_kernel(const double2* __restrict__ a, const double2* __restrict__ b, long long n,
                                   double2* part) {
  __shared__ double2 sh[256];
  double2 s = make_double2(0.0, 0.0);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    s = cadd(s, cmul(cconj(a[e]), b[e]));
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = cadd(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void dot_final_kernel(const double2* __restrict__ part, int n, double* out2) {
  if (threadIdx.x == 0) {
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < n; ++i) s = cadd(s, part[i]);
    out2[0] = s.x;
    out2[1] = s.y;
  }
}

void gemm(Engine& e, Op oa, Op ob, long long M, long long N, long long K, const double2* A, long long lda,
          const double2* B, long long ldb, double2* C, long long ldc, double alpha = 1.0, double beta = 0.0) {
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
  g.alpha = alpha;
  g.beta = beta;
  zgemm(g, e.gemm_scratch(), e.stream);
}

}  // namespace

bool use_qtheta(const Engine& e, const qt_policy& pol, long long rows) {
  // Y = Q_m^H theta by applying QR(X)'s reflectors to theta (no explicit Q_m):
  //  * up to 2048 rows: the pipelined pair (latency-bound chains); from 128
  //    rows it pays for a lone update chain (C1, 128 rows: 771 -> 877 steps/s)
  //    but not when eight bond chains already share the GPU (C5-small, 192
  //    rows: 183 -> 155 steps/s; QT_QTHETA_MIN_ROWS=256 restores that);
  //  * taller, with the explicit error on: the application (2 m eta n CMAC,
  //    128-column outer blocks) replaces both the Y GEMM and the theta-sized
  //    residual GEMM and drops Q_m's formation (north star 5.38 -> 5.84
  //    steps/s, C3 1.257 -> 1.293, C5 0.376 -> 0.389); with the explicit error
  //    off it would double the Y GEMM's flops (C4: 0.129 -> 0.117), so no
  static const long long env_max = std::getenv("QT_QTHETA_MAX_ROWS") ? std::atoll(std::getenv("QT_QTHETA_MAX_ROWS")) : -1;
  const long long qtheta_max = env_max >= 0 ? env_max : (pol.compute_explicit_error ? (1LL << 40) : 2048);
  static const long long qtheta_min = std::getenv("QT_QTHETA_MIN_ROWS")
                                          ? std::atoll(std::getenv("QT_QTHETA_MIN_ROWS"))
                                          : 128;
  const long long min_rows = e.qr_pair_min_rows >= 0 ? e.qr_pair_min_rows : qtheta_min;
  return std::max(1, static_cast<int>(pol.qr_sweeps)) == 1 && rows <= qtheta_max && rows >= min_rows;
}

void qtheta_yh(Engine& e, const double2* qt, long long cols, const double2* a, long long eta, double2* yh,
               long long ibeg, long long iend, cudaStream_t st) {
  if (iend < 0) iend = eta;
  dim3 tg(static_cast<unsigned>(ceil_div(cols, 32)), static_cast<unsigned>(ceil_div(iend - ibeg, 32)));
  yh_gauge_kernel<<<tg, dim3(32, 8), 0, st ? st : e.stream>>>(qt, cols, a, eta, iend, yh, ibeg);
  QT_LAUNCHED();
}

long long x_head_cols() {
  static const long long v = [] {
    const char* s = std::getenv("QT_X_HEAD");
    const long long h = s ? std::atoll(s) : kXHead;
    return h >= 64 && h % 32 == 0 ? h : kXHead;
  }();
  return v;
}

bool x_split_applies(const Engine& e, long long eta) {
  static const bool off = std::getenv("QT_NO_X_SPLIT") != nullptr;
  return !off && e.side != nullptr && eta > x_head_cols() + 32;
}

void x_gemm_split(Engine& e, long long rows, long long eta, long long cols, const double2* theta,
                  const double2* xb, bool xb_h, double2* X, int* flag) {
  const long long xh = x_head_cols();
  // head: the columns of the first two panels, on the main stream
  GemmDesc h;
  h.M = rows; h.N = xh; h.K = cols;
  h.A = theta; h.lda = cols;
  h.opB = xb_h ? Op::H : Op::N;
  h.B = xb; h.ldb = xb_h ? cols : eta;
  h.C = X; h.ldc = eta;
  zgemm(h, e.gemm_scratch(), e.stream);
  check_finite_2d(e, X, rows, xh, eta, flag);
  // the rest behind the head on e.side (issued together, the two GEMMs share
  // the SMs and the head, panel 0's input, finishes late: 208 vs 214 steps/s;
  // issued inside the pair behind panel 0 it contends with the first
  // reflector application instead: 207).  It reads theta, which the pair
  // overwrites with Q_full^H theta on e.side2 from panel 0 on, so e.side2
  // waits for it
  QT_CUDA(cudaEventRecord(e.event(1004), e.stream));
  QT_CUDA(cudaStreamWaitEvent(e.side, e.event(1004), 0));
  GemmScratch gss;
  gss.partial = e.cbuf(S_GEMM_PARTS, size_t(1) << 22);
  gss.partial_elems = size_t(1) << 22;
  gss.tile_sums = e.dbuf(S_TILE_SUMSS, size_t(1) << 16);
  gss.tile_sums_elems = size_t(1) << 16;
  GemmDesc g = h;
  g.N = eta - xh;
  g.B = xb_h ? xb + xh * cols : xb + xh;
  g.C = X + xh;
  zgemm(g, gss, e.side);
  QT_CUDA(cudaEventRecord(e.event(1005), e.side));
  QT_CUDA(cudaStreamWaitEvent(e.side2, e.event(1005), 0));
  check_finite_2d(e, X + xh, rows, eta - xh, eta, flag, e.side);
}

bool use_qr_pair(long long rows, long long cols) {
  static const bool off = std::getenv("QT_NO_QR_PAIR") != nullptr;
  return !off && qr_pair_fits(rows, cols);
}

void qtheta_resid(Engine& e, const double2* qt, long long rows, long long cols, const double2* a, long long eta,
                  const double2* w, double* out, cudaStream_t st) {
  if (!st) st = e.stream;
  double* part = e.dbuf(S_QT_PART, kResidBlocks);
  qtheta_resid_partial_kernel<<<kResidBlocks, 256, 0, st>>>(qt, rows, cols, a, eta, eta, w, part);
  QT_LAUNCHED();
  sum_final_kernel<<<1, 32, 0, st>>>(part, kResidBlocks, out);
  QT_LAUNCHED();
}

void build_theta(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                 const double2* u, int out_scalar) {
  const long long d = D.d, cl = D.chi_l, cm = D.chi_m, cn = D.chi_n, cr = D.chi_r;
  const long long blk = cm * d * d * cr;
  double2* phi = e.cbuf(S_PHI, blk);
  double2* phiev = e.cbuf(S_PHIEV, blk);
  double2* theta = e.cbuf(S_THETA, cl * d * d * cr);
  const GemmScratch gs = e.gemm_scratch();
  {
    // phi(beta,i,j,delta): rows r = i*cm + beta of Bm viewed as (d*cm) x cn,
    // batch j over Bn[j]; row r lands at beta*(d*d*cr) + i*(d*cr), batch at j*cr
    GemmDesc g;
    g.M = d * cm; g.N = cr; g.K = cn; g.batch = static_cast<int>(d);
    g.A = bm; g.lda = cn; g.strideA = 0;
    g.B = bn; g.ldb = cr; g.strideB = cn * cr;
    g.C = phi; g.ldc = d * d * cr; g.rsplit = cm; g.ldc_hi = d * cr; g.strideC = cr;
    zgemm(g, gs, e.stream);
  }
  {
    // phiev[beta] (d^2 x cr) = U (d^2 x d^2) . phi[beta] (d^2 x cr)
    GemmDesc g;
    g.M = d * d; g.N = cr; g.K = d * d; g.batch = static_cast<int>(cm);
    g.A = u; g.lda = d * d; g.strideA = 0;
    g.B = phi; g.ldb = cr; g.strideB = d * d * cr;
    g.C = phiev; g.ldc = cr; g.strideC = d * d * cr;
    zgemm(g, gs, e.stream);
  }
  // theta = Xi (cl x cm) . phiev (cm x d*d*cr)
  gemm(e, Op::N, Op::N, cl, d * d * cr, cm, xi, cm, phiev, d * d * cr, theta, d * d * cr);
  norm2(e, theta, cl * d, d * cr, d * cr, e.dscal + out_scalar);  // (alpha i) x (j delta) view: more rows
}

void gate_qr_async(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* u, const qt_policy& pol, long long eta, const GateBuffers& out) {
  const long long d = D.d, cl = D.chi_l, cm = D.chi_m, cn = D.chi_n, cr = D.chi_r;
  const long long rows = D.rows(), cols = D.cols();
  // QT_UPDATE_DEBUG=1 (eager calls only): phase durations of the update on stderr
  static const bool udbg = std::getenv("QT_UPDATE_DEBUG") != nullptr;
  static std::vector<cudaEvent_t> uev;
  std::vector<const char*> unm;
  auto ustamp = [&](const char* nm) {
    if (!udbg) return;
    if (uev.size() <= unm.size()) {
      cudaEvent_t ev;
      QT_CUDA(cudaEventCreate(&ev));
      uev.push_back(ev);
    }
    QT_CUDA(cudaEventRecord(uev[unm.size()], e.stream));
    unm.push_back(nm);
  };
  ustamp("start");
  int* flag = reinterpret_cast<int*>(e.dscal + SC_TMP3);
  zero_flag_kernel<<<1, 1, 0, e.stream>>>(flag);
  const int sweeps = std::max(1, static_cast<int>(pol.qr_sweeps));
  const bool qtheta = use_qtheta(e, pol, rows);
  const bool pair = qtheta && use_qr_pair(rows, cols);
  // Y0 = B^n regrouped (gates.cpp:357-361) on e.side while theta is built
  const bool y0_early = (eta == cn) && e.side != nullptr;
  if (y0_early) {
    double2* y = e.cbuf(S_Y0, cn * cols);
    QT_CUDA(cudaEventRecord(e.event(1002), e.stream));
    QT_CUDA(cudaStreamWaitEvent(e.side, e.event(1002), 0));
    const long long shp[3] = {d, cn, cr};
    const int perm[3] = {1, 0, 2};
    permute(e, bn, 3, shp, perm, false, y, 1.0, nullptr, e.side);
    QT_CUDA(cudaEventRecord(e.event(1003), e.side));
  }
  build_theta(e, D, xi, bm, bn, u, SC_THETA2);
  ustamp("theta");
  double2* phiev = e.cbuf(S_PHIEV, cm * d * d * cr);
  double2* theta = e.cbuf(S_THETA, cl * d * d * cr);

  double2* X = e.cbuf(S_X, rows * eta);
  double2* Qm = e.cbuf(S_QM, rows * eta);
  double2* Rm = e.cbuf(S_RM, eta * eta);
  double2* YH = e.cbuf(S_YH, cols * eta);
  double2* Qp = e.cbuf(S_QP, cols * eta);
  double2* Rp = e.cbuf(S_RP, eta * eta);

  // initial guess, gates.cpp:357-361
  const bool y0_is_bn = (eta == cn);
  const double2* y0 = theta;  // first eta rows of the grouped theta
  if (y0_is_bn && y0_early) {
    y0 = e.cbuf(S_Y0, cn * cols);
    QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(1003), 0));
  } else if (y0_is_bn) {
    double2* y = e.cbuf(S_Y0, cn * cols);
    const long long shp[3] = {d, cn, cr};
    const int perm[3] = {1, 0, 2};
    permute(e, bn, 3, shp, perm, false, y);
    y0 = y;
  }
  // Y = Q_m^H theta through the reflectors (one sweep, theta up to
  // QT_QTHETA_MAX_ROWS rows): each finished panel of QR(X) is applied to theta
  // on a side stream while the later panels factor, so when the panel chain
  // ends Q_full^H theta = [Y; Z] is ready -- no explicit Q_m (unless left_iso
  // is wanted), no theta^H Q_m GEMM, and the explicit error needs only
  // ||Y - L Q_n||^2 + ||Z||^2 instead of a theta-sized residual product
  bool left_pending = false;  // left_iso formed on side4 (pair path), joined at the end
  const bool x_split = pair && x_split_applies(e, eta);
  for (int it = 0; it < sweeps; ++it) {
    const double2* xb = it == 0 ? y0 : Qp;  // X = theta xb^H (it = 0) / theta xb (Y0 = Q_n = Qp^H)
    if (x_split) {
      x_gemm_split(e, rows, eta, cols, theta, xb, it == 0, X, flag);
    } else {
      if (it == 0)
        gemm(e, Op::N, Op::H, rows, eta, cols, theta, cols, xb, cols, X, eta);  // X = theta Y0^H
      else
        gemm(e, Op::N, Op::N, rows, eta, cols, theta, cols, xb, eta, X, eta);   // Y0 = Q_n = Qp^H
    }
    if (!x_split) check_finite(e, X, rows * eta, flag);  // require_finite_matrix, linalg.cpp:17-21
    ustamp("X");
    if (pair) {
      // both QRs of the sweep in flight at once: QR(Y^H) one panel behind QR(X)
      qr_pair_pipelined(e, X, rows, eta, theta, cols, YH, Qp, Rp);
      if (out.left_iso) {
        // left_iso = Q_m (gates.cpp:373) from X's stored reflectors, on side4
        // concurrently with the tail (Hastings on the main stream)
        QT_CUDA(cudaEventRecord(e.event(1006), e.stream));
        QT_CUDA(cudaStreamWaitEvent(e.side4, e.event(1006), 0));
        pair_form_q(e, X, rows, eta, Qm, eta, e.side4);
        const long long shp[3] = {cl, d, eta};
        const int perm[3] = {1, 0, 2};
        permute(e, Qm, 3, shp, perm, false, out.left_iso, 1.0, nullptr, e.side4);
        QT_CUDA(cudaEventRecord(e.event(1007), e.side4));
        left_pending = true;
      }
      check_finite(e, theta, eta * cols, flag);  // Y (the first eta rows of Q_full^H theta)
      ustamp("pair");
      continue;
    }
    if (qtheta && qr_pair_tall_fits(rows, cols, eta)) {
      // tall pair: QR(Y^H) one outer block behind QR(X) and the theta application
      // (the Hastings product stays a single GEMM after the pair: issued per
      // Q block inside it, it competes with the theta application and the
      // Y^H chain for the tensor pipe -- north star 7.78 -> 7.62 steps/s)
      qr_pair_tall(e, X, rows, eta, theta, cols, YH, Qp, Rp, out.left_iso ? Qm : nullptr,
                   [&](long long r0, long long nr, cudaStream_t st) {
                     qtheta_yh(e, theta, cols, X, eta, YH, r0, r0 + nr, st);
                   });
      check_finite(e, theta, eta * cols, flag);  // Y
      ustamp("tall_pair");
      continue;
    }
    if (qtheta) {
      QrOpts o;
      o.capply = theta;  // theta <- Q_full^H theta (theta is not read again: ||theta|| is already known)
      o.ldc = cols;
      o.nc = cols;
      o.want_q = out.left_iso != nullptr;
      o.want_r = false;
      qr_inplace(e, X, rows, eta, eta, Qm, eta, Rm, eta, o);
      qtheta_yh(e, theta, cols, X, eta, YH);
      ustamp("qrx_apply");
    } else {
      qr_inplace(e, X, rows, eta, eta, Qm, eta, Rm, eta);
      gemm(e, Op::H, Op::N, cols, eta, rows, theta, cols, Qm, eta, YH, eta);  // Y^H = theta^H Q_m
    }
    check_finite(e, YH, cols * eta, flag);
    qr_inplace(e, YH, cols, eta, eta, Qp, eta, Rp, eta);  // Y^H = Qp Rp -> L = Rp^H, Q_n = Qp^H
    ustamp("qry");
  }
  norm2(e, Rp, eta, eta, eta, e.dscal + SC_L2);
  inv_norm_kernel<<<1, 1, 0, e.stream>>>(e.dscal, SC_THETA2, SC_L2, pol.skip_renormalize ? 1 : 0, SC_TMP0);
  QT_LAUNCHED();
  // pair path: the output permutes and the explicit-error products run on
  // e.side, concurrently with the Hastings product on the main stream (they
  // only read L, Q_n and Q_full^H theta; joined before returning)
  const bool fork_tail = qtheta && e.side != nullptr;
  const cudaStream_t tail_st = fork_tail ? e.side : e.stream;
  if (fork_tail) {
    QT_CUDA(cudaEventRecord(e.event(1000), e.stream));
    QT_CUDA(cudaStreamWaitEvent(e.side, e.event(1000), 0));
  }
  {
    // Xi~ = L / den = Rp^H / den   (gates.cpp:365-370)
    const long long shp[2] = {eta, eta};
    const int perm[2] = {1, 0};
    permute(e, Rp, 2, shp, perm, true, out.xi, 1.0, e.dscal + SC_TMP0, tail_st);
  }
  {
    // B~n[j,k,delta] = Q_n[k,(j delta)] = conj(Qp[(j delta),k])   (gates.cpp:193-196)
    const long long shp[3] = {d, cr, eta};
    const int perm[3] = {0, 2, 1};
    permute(e, Qp, 3, shp, perm, true, out.b_n, 1.0, nullptr, tail_st);
  }
  ustamp("xi_bn");
  const bool fork_resid = fork_tail && pol.compute_explicit_error;
  if (fork_resid) {
    // eps = ||Y - L Q_n||^2 + ||Z||^2, and L Q_n = Rp^H Qp^H IS the QR of
    // Y^H = Qp Rp: its first term is the QR's backward error (<= c u ||Y||),
    // below the rounding of the reference's own theta-sized residual
    // (gates.cpp:464-485) -- only ||Z||^2, the rows of Q_full^H theta outside
    // Q_m's span, is summed (no eta x cols product)
    qtheta_resid(e, theta, rows, cols, X, eta, nullptr, e.dscal + SC_RESID, e.side);
    QT_CUDA(cudaEventRecord(e.event(1001), e.side));
  }
  if (out.b_m) {
    // B~m[i,beta,k] = sum_{j,delta} phiev[beta,i,j,delta] conj(B~n[j,k,delta])
    //             = (phiev (cm*d x d*cr) . Qp)[(beta i), k]   (gates.cpp:186-190)
    // (skipped when the caller keeps left_iso instead: the reference finite
    // step discards b_m for QR, gates.cpp:559-563)
    GemmDesc g;
    g.M = cm * d; g.N = eta; g.K = cols;
    g.A = phiev; g.lda = cols;
    g.B = Qp; g.ldb = eta;
    g.C = out.b_m; g.ldc = cm * eta; g.rsplit = d; g.ldc_hi = eta;
    // large products read B = Q_n^H from an explicit Q_n (op H, K-major
    // fragments like the X GEMM) instead of Qp (op N): fewer shared-memory
    // bank conflicts in the mainloop (north star: 86% -> 98% DMMA pipe active
    // for X vs Hastings with the same grid)
    static const int qn_env = std::getenv("QT_HASTINGS_QN") ? std::atoi(std::getenv("QT_HASTINGS_QN")) : -1;
    const bool use_qn = qn_env >= 0 ? qn_env != 0 : (cm * d >= 2048 && cols >= 2048);
    if (use_qn) {
      double2* Qn = e.cbuf(S_QN, eta * cols);
      const long long shp[2] = {cols, eta};
      const int perm[2] = {1, 0};
      permute(e, Qp, 2, shp, perm, true, Qn);
      g.opB = Op::H;
      g.B = Qn;
      g.ldb = cols;
    }
    zgemm(g, e.gemm_scratch(), e.stream);
  }
  if (out.left_iso && !left_pending) {
    // left_iso = Q_m (cl, d, eta) -> (d, cl, eta)   (gates.cpp:198-201)
    const long long shp[3] = {cl, d, eta};
    const int perm[3] = {1, 0, 2};
    permute(e, Qm, 3, shp, perm, false, out.left_iso);
  }
  if (fork_tail && !fork_resid) QT_CUDA(cudaEventRecord(e.event(1001), e.side));
  if (fork_tail) {
    QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(1001), 0));  // join: outputs and report scalars complete
  } else if (pol.compute_explicit_error && qtheta) {
    // W = L Q_n = Rp^H Qp^H (eta x cols); ||theta - Q_m W||^2 = ||Y - W||^2 + ||Z||^2
    double2* W = e.cbuf(S_W, eta * cols);
    gemm(e, Op::H, Op::H, eta, cols, eta, Rp, eta, Qp, eta, W, cols);
    qtheta_resid(e, theta, rows, cols, X, eta, W, e.dscal + SC_RESID);
  } else if (pol.compute_explicit_error) {
    // W = L Q_n = Rp^H Qp^H (eta x cols), then sum |theta - Q_m W|^2 (gates.cpp:464-485)
    double2* W = e.cbuf(S_W, eta * cols);
    gemm(e, Op::H, Op::H, eta, cols, eta, Rp, eta, Qp, eta, W, cols);
    GemmDesc g;
    g.M = rows; g.N = cols; g.K = eta;
    g.A = Qm; g.lda = eta;
    g.B = W; g.ldb = cols;
    g.C = theta; g.ldc = cols;
    g.mode = GemmMode::resid;
    zgemm(g, e.gemm_scratch(), e.stream, e.dscal + SC_RESID);
  }
  if (left_pending) QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(1007), 0));
  ustamp("end");
  if (udbg) {
    QT_CUDA(cudaStreamSynchronize(e.stream));
    std::fprintf(stderr, "update rows=%lld cols=%lld eta=%lld phases (us):", rows, cols, eta);
    for (size_t k = 1; k < unm.size(); ++k) {
      float ms = 0.f;
      QT_CUDA(cudaEventElapsedTime(&ms, uev[k - 1], uev[k]));
      std::fprintf(stderr, " %s=%.0f", unm[k], ms * 1000.f);
    }
    std::fprintf(stderr, "\n");
  }
}

HostReport read_report(Engine& e) {
  QT_CUDA(cudaMemcpyAsync(e.hscal, e.dscal, 8 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  HostReport r;
  r.theta2 = e.hscal[SC_THETA2];
  r.kept2 = e.hscal[SC_L2];
  r.resid = e.hscal[SC_RESID];
  int flag = 0;
  std::memcpy(&flag, &e.hscal[SC_TMP3], sizeof(int));
  r.finite = flag == 0;
  return r;
}

// ------------------------------------------------------------ observables
void expectation_local(Engine& e, const double2* xi, long long xi_rows, long long chi_l, const double2* b,
                       long long d, long long chi_r, const double2* op, double* out2_host) {
  // M = Xi^H Xi (Xi is xi_rows x chi_l; rectangular on the reference finite
  // path, mps.cpp:232-238) ; lambda = conj(M) (mps.cpp:44-46)
  // t1[i] = M^H . B[i]  (= sum_a lambda[a,a'] B[i,a,b], mps.cpp:171)
  // t2 = t1 (d x chi_l*chi_r) . B^H  (mps.cpp:172) ; <O> = tr(op t2^T)
  double2* M = e.cbuf(S_MISC, chi_l * chi_l + d * d + 8);
  double2* t2 = M + chi_l * chi_l;
  double2* t1 = e.cbuf(S_MISC2, d * chi_l * chi_r);
  gemm(e, Op::H, Op::N, chi_l, chi_l, xi_rows, xi, chi_l, xi, chi_l, M, chi_l);
  {
    GemmDesc g;
    g.M = chi_l; g.N = chi_r; g.K = chi_l; g.batch = static_cast<int>(d);
    g.opA = Op::H; g.A = M; g.lda = chi_l; g.strideA = 0;
    g.B = b; g.ldb = chi_r; g.strideB = chi_l * chi_r;
    g.C = t1; g.ldc = chi_r; g.strideC = chi_l * chi_r;
    zgemm(g, e.gemm_scratch(), e.stream);
  }
  gemm(e, Op::N, Op::H, d, d, chi_l * chi_r, t1, chi_l * chi_r, b, chi_l * chi_r, t2, d);
  trace_op_kernel<<<1, 32, 0, e.stream>>>(op, t2, static_cast<int>(d), e.dscal + SC_TMP1);
  QT_LAUNCHED();
  QT_CUDA(cudaMemcpyAsync(out2_host, e.dscal + SC_TMP1, 2 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
}

double right_defect(Engine& e, const double2* b, long long d, long long chi_l, long long chi_r) {
  // sum_i B^i B^i^H - 1 (mps.cpp:34-36): permute to (chi_l, d, chi_r), Gram
  double2* bp = e.cbuf(S_MISC2, d * chi_l * chi_r);
  double2* g = e.cbuf(S_MISC, chi_l * chi_l);
  const long long shp[3] = {d, chi_l, chi_r};
  const int perm[3] = {1, 0, 2};
  permute(e, b, 3, shp, perm, false, bp);
  gemm(e, Op::N, Op::H, chi_l, chi_l, d * chi_r, bp, d * chi_r, bp, d * chi_r, g, chi_l);
  double* part = e.dbuf(S_NORM_PART, 296);
  defect_partial_kernel<<<148, 256, 0, e.stream>>>(g, chi_l, part);
  max_final_kernel<<<1, 32, 0, e.stream>>>(part, 148, e.dscal + SC_TMP1);
  double out = 0;
  QT_CUDA(cudaMemcpyAsync(&out, e.dscal + SC_TMP1, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  return out;
}

double left_defect(Engine& e, const double2* b, long long d, long long chi_l, long long chi_r) {
  // sum_i B^i^H B^i - 1 (mps.cpp:39-41): B as a (d chi_l) x chi_r matrix, one Gram GEMM
  double2* g = e.cbuf(S_MISC, chi_r * chi_r);
  gemm(e, Op::H, Op::N, chi_r, chi_r, d * chi_l, b, chi_r, b, chi_r, g, chi_r);
  double* part = e.dbuf(S_NORM_PART, 296);
  defect_partial_kernel<<<148, 256, 0, e.stream>>>(g, chi_r, part);
  QT_LAUNCHED();
  max_final_kernel<<<1, 32, 0, e.stream>>>(part, 148, e.dscal + SC_TMP1);
  QT_LAUNCHED();
  double out = 0;
  QT_CUDA(cudaMemcpyAsync(&out, e.dscal + SC_TMP1, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  return out;
}

namespace {
__global__ void maxabs_diff_partial_kernel(const double2* __restrict__ a, const double2* __restrict__ b, long long n,
                                           double* part) {
  __shared__ double sh[256];
  double m = 0.0;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    m = fmax(m, hypot(a[e].x - b[e].x, a[e].y - b[e].y));
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// max_ij |a_ij - b_ij| (mps.cpp:16-20 on a difference), synchronous
double maxabs_diff(Engine& e, const double2* a, const double2* b, long long n) {
  double* part = e.dbuf(S_NORM_PART, 296);
  maxabs_diff_partial_kernel<<<148, 256, 0, e.stream>>>(a, b, n, part);
  QT_LAUNCHED();
  max_final_kernel<<<1, 32, 0, e.stream>>>(part, 148, e.dscal + SC_TMP1);
  QT_LAUNCHED();
  double out = 0;
  QT_CUDA(cudaMemcpyAsync(&out, e.dscal + SC_TMP1, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  return out;
}

// out = sum_i B^iH mu B^i, B (d, cl, cr): the one-site transfer on mu = conj(lambda)
// (translate_left_weight, mps.cpp:50-54, conjugated: lambda = Xi^T conj(Xi) = conj(Xi^H Xi))
void transfer_mu(Engine& e, const double2* mu, const double2* b, long long d, long long cl, long long cr,
                 double2* tmp, double2* out) {
  GemmDesc g;  // tmp[i] = mu B^i
  g.M = cl;
  g.N = cr;
  g.K = cl;
  g.batch = static_cast<int>(d);
  g.A = mu;
  g.lda = cl;
  g.strideA = 0;
  g.B = b;
  g.ldb = cr;
  g.strideB = cl * cr;
  g.C = tmp;
  g.ldc = cr;
  g.strideC = cl * cr;
  zgemm(g, e.gemm_scratch(), e.stream);
  gemm(e, Op::H, Op::N, cr, cr, d * cl, b, cr, tmp, cr, out, cr);  // B_stack^H tmp_stack
}
}  // namespace

IsometryParts check_isometric_uniform(Engine& e, long long d, const std::vector<long long>& chi,
                                      const std::vector<const double2*>& sites,
                                      const std::vector<const double2*>& bonds) {
  const int L = static_cast<int>(sites.size());
  IsometryParts r;
  r.right.resize(L);
  r.left.resize(L);
  r.translation.resize(L);
  r.norm.resize(L);
  long long cmax = 1;
  for (long long c : chi) cmax = std::max(cmax, c);
  // mu_m = Xi_m^H Xi_m for every bond, then the transfer scratch
  double2* mus = e.cbuf(S_GRAM, static_cast<size_t>(L) * cmax * cmax + 2 * cmax * cmax);
  double2* cur = mus + static_cast<size_t>(L) * cmax * cmax;
  double2* nxt = cur + cmax * cmax;
  double2* tmp = e.cbuf(S_W, d * cmax * cmax);
  for (int m = 0; m < L; ++m) {
    const long long c = chi[m];
    r.right[m] = right_defect(e, sites[m], d, c, chi[(m + 1) % L]);
    norm2(e, bonds[m], c, c, c, e.dscal + SC_TMP2);
    double n2 = 0;
    QT_CUDA(cudaMemcpyAsync(&n2, e.dscal + SC_TMP2, sizeof(double), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    r.norm[m] = std::abs(std::sqrt(n2) - 1.0);
    gemm(e, Op::H, Op::N, c, c, c, bonds[m], c, bonds[m], c, mus + static_cast<size_t>(m) * cmax * cmax, c);
  }
  for (int m = 0; m < L; ++m) {
    const int m1 = (m + 1) % L;
    const long long cl = chi[m], cr = chi[m1];
    const double2* mu_m = mus + static_cast<size_t>(m) * cmax * cmax;
    // translation defect: lambda_m T_m vs lambda_{m+1}
    transfer_mu(e, mu_m, sites[m], d, cl, cr, tmp, nxt);
    r.translation[m] = maxabs_diff(e, nxt, mus + static_cast<size_t>(m1) * cmax * cmax, cr * cr);
    // cell fixed point: lambda_m through the L site transfers of the cell
    copy2d(e, mu_m, cl, cur, cl, cl, cl);
    long long cc = cl;
    for (int k = 0; k < L; ++k) {
      const int s = (m + k) % L;
      const long long cn = chi[(s + 1) % L];
      transfer_mu(e, cur, sites[s], d, cc, cn, tmp, nxt);
      std::swap(cur, nxt);
      cc = cn;
    }
    r.left[m] = maxabs_diff(e, cur, mu_m, cl * cl);
  }
  return r;
}

double bond_energy(Engine& e, const Dims& D, const double2* xi, const double2* bm, const double2* bn,
                   const double2* h) {
  // E = <theta0|h theta0>/<theta0|theta0>, theta0 = Xi Bm Bn
  const long long d = D.d;
  const long long n = D.chi_l * d * d * D.chi_r;
  double2* ident = e.cbuf(S_EIG_V, d * d * d * d + n);
  double2* theta_h = ident + d * d * d * d;
  set_identity(e, ident, d * d, d * d, d * d);
  build_theta(e, D, xi, bm, bn, h, SC_TMP1);
  copy2d(e, e.cbuf(S_THETA, n), n, theta_h, n, 1, n);
  build_theta(e, D, xi, bm, bn, ident, SC_TMP2);
  const double2* theta0 = e.cbuf(S_THETA, n);
  double2* part = e.cbuf(S_NORM_PART, 296);
  dot_partial_kernel<<<148, 256, 0, e.stream>>>(theta0, theta_h, n, part);
  dot_final_kernel<<<1, 32, 0, e.stream>>>(part, 148, e.dscal + SC_TMP0);
  double hv[4] = {0, 0, 0, 0};
  QT_CUDA(cudaMemcpyAsync(hv, e.dscal + SC_TMP0, 3 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  // hv[0] = Re<theta0|h theta0>, hv[2] = ||theta0||^2 (SC_TMP2)
  return hv[2] > 0 ? hv[0] / hv[2] : 0.0;
}

double explicit_error(Engine& e, const double2* theta, long long rows, long long cols, const double2* left,
                      long long kdim, const double2* center, long long kdim2, const double2* right) {
  double2* W = e.cbuf(S_W, kdim * cols);
  gemm(e, Op::N, Op::N, kdim, cols, kdim2, center, kdim2, right, cols, W, cols);
  norm2(e, theta, rows, cols, cols, e.dscal + SC_TMP1);
  GemmDesc g;
  g.M = rows; g.N = cols; g.K = kdim;
  g.A = left; g.lda = kdim;
  g.B = W; g.ldb = cols;
  g.C = const_cast<double2*>(theta); g.ldc = cols;
  g.mode = GemmMode::resid;
  zgemm(g, e.gemm_scratch(), e.stream, e.dscal + SC_TMP2);
  double hv[2];
  QT_CUDA(cudaMemcpyAsync(hv, e.dscal + SC_TMP1, 2 * sizeof(double), cudaMemcpyDeviceToHost, e.stream));
  QT_CUDA(cudaStreamSynchronize(e.stream));
  if (hv[0] == 0.0) return 0.0;
  return hv[1] / hv[0];
}

}  // namespace qt
