// K3: blocked Householder QR with explicit thin Q and the reference gauge.
//
// Replaces qr_reduced / fix_qr_gauge (proj/src/linalg.cpp:25-51, Eigen
// HouseholderQR + householderQ()*I).  LAPACK zgeqrf/zlarfg/zlarft/zungqr
// conventions: H_c = I - tau_c v_c v_c^H with v_c[c] = 1, beta real,
// tau = 0 for an exactly-zero column (rank-deficient blocks, e.g. product
// states, proj/tests/test_gates.cc:354-367); Q = H_0 ... H_{k-1}.
//
// Panel (32 columns): one cooperative kernel.  The panel rows are spread
// over up to 148 CTAs and kept in shared memory; each column needs ONE
// grid-wide reduction, because the norm of the column tail, the projections
// x^H a_k of the later columns and the T-factor products V^H v_c all come out
// of the same pass (lane k of every warp owns panel column k).  Partial sums
// are combined in a fixed order on every CTA, so the factorization is
// bitwise deterministic.
//
// Trailing update and Q formation: the compact-WY block reflector
// I - V T V^H applied with three DMMA GEMMs (V^H A, T^H W, A - V W2).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "engine.cuh"

namespace qt {
namespace {

constexpr int NB = 32;
constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;

__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct PanelArgs {
  double2* A;  // panel top-left, row-major, ld lda
  long long lda;
  long long mp;  // panel rows
  int nbp;       // panel columns (<= 32)
  int rpc;       // rows per CTA
  double2* V;    // V panel top-left, ld ldv (unit lower trapezoidal, written here)
  long long ldv;
  double2* T;      // 32 x 32 upper triangular T factor
  double2* part;   // [2][grid][32] partial sums
  double2* diag;   // [2][32] broadcast of the current diagonal row
  unsigned* bar;   // grid barrier words
  long long* dbg;  // optional per-column clock64 stamps (CTA 0, thread 0)
};

__global__ void __launch_bounds__(PANEL_THREADS, 1) panel_kernel(PanelArgs a) {
  extern __shared__ double2 psm[];
  double2* P = psm;                            // [rpc][32]
  double2* red = P + size_t(a.rpc) * NB;       // [8][32]
  double2* Ts = red + PANEL_WARPS * NB;        // [32][32]
  double2* ssum = Ts + NB * NB;                // [32]
  double2* zs = ssum + NB;                     // [32]

  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  const unsigned G = gridDim.x;
  const long long r0 = static_cast<long long>(blockIdx.x) * a.rpc;
  const int nloc = static_cast<int>(max(0LL, min(static_cast<long long>(a.rpc), a.mp - r0)));
  const int nbp = a.nbp;

  for (int lr = w; lr < a.rpc; lr += PANEL_WARPS)
    P[lr * NB + k] = (lr < nloc && k < nbp) ? a.A[(r0 + lr) * a.lda + k] : make_double2(0.0, 0.0);
  for (int e = threadIdx.x; e < NB * NB; e += PANEL_THREADS) Ts[e] = make_double2(0.0, 0.0);
  __syncthreads();

  for (int c = 0; c < nbp; ++c) {
    const int par = c & 1;
    // ---- phase 1: one pass over the local rows below the diagonal
    //   lane k >= c : g_k = sum conj(x_r) a_rk   (k == c gives ||x||^2)
    //   lane k <  c : h_k = sum conj(v_rk) x_r   (T-factor products)
    double2 acc = make_double2(0.0, 0.0);
    for (int lr = w; lr < nloc; lr += PANEL_WARPS) {
      if (r0 + lr <= c) continue;
      const double2 x = P[lr * NB + c];
      const double2 y = P[lr * NB + k];
      const double2 u = (k >= c) ? x : y;
      const double2 v = (k >= c) ? y : x;
      acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
      acc.y = fma(u.x, v.y, fma(-u.y, v.x, acc.y));
    }
    red[w * NB + k] = acc;
    __syncthreads();
    if (w == 0) {
      double2 s = red[k];
      for (int ww = 1; ww < PANEL_WARPS; ++ww) s = cadd(s, red[ww * NB + k]);
      a.part[(size_t(par) * G + blockIdx.x) * NB + k] = s;
    }
    if (blockIdx.x == 0 && w == 1) a.diag[par * NB + k] = P[c * NB + k];
    grid_sync(a.bar, G);

    // ---- phase 2: combine partials (fixed order) and form the reflector;
    // warp w sums the CTAs b = w (mod 8) with four independent chains (the
    // L2 loads of the G partial rows issue in parallel), then warp 0 adds the
    // eight warp sums in order
    {
      double2 s0 = make_double2(0.0, 0.0), s1 = s0, s2 = s0, s3 = s0;
      unsigned b = w;
      for (; b + 3 * PANEL_WARPS < G; b += 4 * PANEL_WARPS) {
        s0 = cadd(s0, __ldcg(&a.part[(size_t(par) * G + b) * NB + k]));
        s1 = cadd(s1, __ldcg(&a.part[(size_t(par) * G + b + PANEL_WARPS) * NB + k]));
        s2 = cadd(s2, __ldcg(&a.part[(size_t(par) * G + b + 2 * PANEL_WARPS) * NB + k]));
        s3 = cadd(s3, __ldcg(&a.part[(size_t(par) * G + b + 3 * PANEL_WARPS) * NB + k]));
      }
      for (; b < G; b += PANEL_WARPS) s0 = cadd(s0, __ldcg(&a.part[(size_t(par) * G + b) * NB + k]));
      red[w * NB + k] = cadd(cadd(s0, s1), cadd(s2, s3));
    }
    __syncthreads();
    if (w == 0) {
      double2 s = red[k];
      for (int ww = 1; ww < PANEL_WARPS; ++ww) s = cadd(s, red[ww * NB + k]);
      ssum[k] = s;
    }
    __syncthreads();
    const double2 alpha = __ldcg(&a.diag[par * NB + c]);
    const double xnorm2 = ssum[c].x;
    double2 tau, scale;
    double beta;
    if (xnorm2 == 0.0 && alpha.y == 0.0) {
      tau = make_double2(0.0, 0.0);
      beta = alpha.x;
      scale = make_double2(0.0, 0.0);
    } else {
      const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2);
      beta = alpha.x >= 0.0 ? -nrm : nrm;
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      // scale = 1 / (alpha - beta)
      const double2 den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    const double2 ctau = cconj(tau);
    // w_k = a_ck + conj(scale) g_k  for k > c
    const double2 a_ck = __ldcg(&a.diag[par * NB + k]);
    const double2 wk = cadd(a_ck, cmul(cconj(scale), ssum[k]));
    const double2 ctw = cmul(ctau, wk);  // conj(tau) w_k

    // T column c (zlarft, forward/columnwise): T[0:c,c] = T[0:c,0:c] z,
    // z_i = -tau (conj(v_c,i) + scale h_i)
    if (w == 0) {
      double2 z = make_double2(0.0, 0.0);
      if (k < c) z = cmul(make_double2(-tau.x, -tau.y), cadd(cconj(a_ck), cmul(scale, ssum[k])));
      zs[k] = z;
      __syncwarp();
      if (k < c) {
        double2 t = make_double2(0.0, 0.0);
        for (int l = k; l < c; ++l) t = cadd(t, cmul(Ts[k * NB + l], zs[l]));
        Ts[k * NB + c] = t;
      } else if (k == c) {
        Ts[c * NB + c] = tau;
      }
    }

    // ---- phase 3: apply H_c^H to the local rows, store v in column c
    for (int lr = w; lr < nloc; lr += PANEL_WARPS) {
      const long long gr = r0 + lr;
      if (gr < c) continue;
      if (gr == c) {
        if (k > c && k < nbp) P[lr * NB + k] = csub(P[lr * NB + k], ctw);
        __syncwarp();
        if (k == c) P[lr * NB + c] = make_double2(beta, 0.0);
      } else {
        const double2 vr = cmul(scale, P[lr * NB + c]);
        __syncwarp();
        if (k > c && k < nbp) P[lr * NB + k] = csub(P[lr * NB + k], cmul(vr, ctw));
        if (k == c) P[lr * NB + c] = vr;
      }
    }
    __syncthreads();
  }

  // ---- write back R/V to A, the dense unit-lower V panel, and T
  for (int lr = w; lr < nloc; lr += PANEL_WARPS) {
    const long long gr = r0 + lr;
    if (k < nbp) {
      const double2 v = P[lr * NB + k];
      a.A[gr * a.lda + k] = v;
      a.V[gr * a.ldv + k] =
          gr > k ? v : (gr == k ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0));
    } else {
      a.V[gr * a.ldv + k] = make_double2(0.0, 0.0);  // full 32-wide rows (bulk-copied by larfb)
    }
  }
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < NB * NB; e += PANEL_THREADS) a.T[e] = Ts[e];
}

// R_ii = |R_ii|, Q[:, i] *= ph_i, R[i, :] *= conj(ph_i), ph_i = R_ii/|R_ii|
__global__ void gauge_q_kernel(const double2* __restrict__ a, long long lda, double2* q, long long ldq,
                               long long m, long long k) {
  const long long total = m * k;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / k, c = e % k;
    const double2 d = a[c * lda + c];
    const double ad = hypot(d.x, d.y);
    if (ad == 0.0) continue;
    const double2 ph = make_double2(d.x / ad, d.y / ad);
    q[r * ldq + c] = cmul(q[r * ldq + c], ph);
  }
}

// gauge phases on columns [c0, c0 + nb) of q only (one Q block of the pair)
__global__ void gauge_q_cols_kernel(const double2* __restrict__ a, long long lda, double2* q, long long ldq,
                                    long long m, long long c0, long long nb) {
  const long long total = m * nb;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / nb, c = c0 + e % nb;
    const double2 d = a[c * lda + c];
    const double ad = hypot(d.x, d.y);
    if (ad == 0.0) continue;
    q[r * ldq + c] = cmul(q[r * ldq + c], make_double2(d.x / ad, d.y / ad));
  }
}

__global__ void gauge_r_kernel(const double2* __restrict__ a, long long lda, double2* r, long long ldr,
                               long long k, long long n) {
  const long long total = k * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / n, c = e % n;
    double2 v = make_double2(0.0, 0.0);
    if (c >= i) {
      const double2 d = a[i * lda + i];
      const double ad = hypot(d.x, d.y);
      if (c == i) {
        v = make_double2(ad, 0.0);
      } else {
        v = a[i * lda + c];
        if (ad != 0.0) v = cmul(v, make_double2(d.x / ad, -d.y / ad));
      }
    }
    r[i * ldr + c] = v;
  }
}

#include "qr_panel.cuh"
#include "larfb_cluster.cuh"

int grid_for(long long total) {
  const long long b = ceil_div(total, 256);
  return static_cast<int>(b < 16LL * kNumSMs ? (b > 0 ? b : 1) : 16LL * kNumSMs);
}

// returns false when the panel is too tall for one cluster's shared memory
template <int RPW>
void launch_panel_rpw(Engine& e, const PanelArgs& a, long long cs, cudaStream_t st) {
  auto kern = panel_cluster_kernel<RPW>;
  constexpr size_t smem_attr = panel_cluster_smem(RPW);
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_attr)));
  });
  const size_t smem = panel_cluster_smem(RPW);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs));
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  QT_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  QT_LAUNCHED();
}

bool launch_panel_cluster(Engine& e, const PanelArgs& base, long long mp, cudaStream_t st) {
  // probed once, thread-safe (magic static): concurrent first calls from the
  // chain's bond threads must agree on the path
  static const int max_cs = [] {
    auto kern = panel_cluster_kernel<CL_MAX_RPW>;
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const size_t smem_max = panel_cluster_smem(CL_MAX_RPW);
    QT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_max)));
    int found = 0;
    for (int cs : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(CL_THREADS);
      cfg.dynamicSmemBytes = smem_max;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n >= 1) {
        found = cs;
        break;
      }
      cudaGetLastError();
    }
    return found;
  }();
  if (max_cs == 0) return false;
  // as many CTAs as the cluster allows (short per-warp row loops), >= 32 rows
  // each so CTA 0 owns the whole diagonal block
  static const int cs_cap = std::getenv("QT_PANEL_CS") ? std::atoi(std::getenv("QT_PANEL_CS")) : 16;
  const long long cs_max = std::min(max_cs, std::max(1, cs_cap));
  // rows per warp held in registers: smallest instantiation that covers the
  // panel with <= cs_max CTAs (16 row warps each)
  const long long need = ceil_div(mp, cs_max * CL_WARPS);
  int rpw = 0;
  for (int r : {2, 3, 5, 8, 10, 14, CL_MAX_RPW})
    if (r >= need) {
      rpw = r;
      break;
    }
  if (rpw == 0) return false;
  const long long cs = ceil_div(mp, static_cast<long long>(rpw) * CL_WARPS);
  PanelArgs a = base;
  a.rpc = rpw * CL_WARPS;
  switch (rpw) {
    case 2: launch_panel_rpw<2>(e, a, cs, st); break;
    case 3: launch_panel_rpw<3>(e, a, cs, st); break;
    case 5: launch_panel_rpw<5>(e, a, cs, st); break;
    case 8: launch_panel_rpw<8>(e, a, cs, st); break;
    case 10: launch_panel_rpw<10>(e, a, cs, st); break;
    case 14: launch_panel_rpw<14>(e, a, cs, st); break;
    default: launch_panel_rpw<CL_MAX_RPW>(e, a, cs, st); break;
  }
  return true;
}

void launch_panel(Engine& e, const PanelArgs& base, long long mp, cudaStream_t st = nullptr) {
  if (!st) st = e.stream;
  if (launch_panel_cluster(e, base, mp, st)) return;
  // grid-wide fallback for very tall panels: ~128 rows per CTA, at most one
  // CTA per SM (co-residency for the grid barrier), at least 32 rows so CTA 0
  // owns the whole diagonal block
  long long G = std::min<long long>(e.num_sms, std::max<long long>(1, ceil_div(mp, 128)));
  long long rpc = std::max<long long>(NB, ceil_div(mp, G));
  rpc = ceil_div(rpc, 8) * 8;
  G = ceil_div(mp, rpc);
  if (rpc > 1024) throw Error(Err::capacity, "QR panel taller than 148 x 1024 rows");
  PanelArgs a = base;
  a.rpc = static_cast<int>(rpc);
  const size_t smem = (size_t(rpc) * NB + PANEL_WARPS * NB + NB * NB + 2 * NB) * sizeof(double2);
  // opt in once to the device's per-block maximum (thread-safe; every launch
  // below needs at most that much)
  static std::once_flag attr_once;
  static int smem_cap = 0;
  std::call_once(attr_once, [] {
    int dev = 0;
    QT_CUDA(cudaGetDevice(&dev));
    QT_CUDA(cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    QT_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap));
  });
  if (smem > static_cast<size_t>(smem_cap)) throw Error(Err::capacity, "QR panel exceeds the shared-memory capacity");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(G));
  cfg.blockDim = dim3(PANEL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  QT_CUDA(cudaLaunchKernelEx(&cfg, panel_kernel, a));
  QT_LAUNCHED();
}

// C <- (I - V T' V^H) C for a block of nbp reflectors, T' = T^H (Q^H C, the
// factorization) or T (Q C, Q formation); T has leading dimension ldt; three
// DMMA GEMMs on stream st (W/W2 and the split-K scratch belong to that stream)
void apply_block_reflector(const double2* Vp, long long ldv, const double2* Tp, double2* C, long long ldc,
                           long long mp, long long nc, int nbp, double2* W, double2* W2, const GemmScratch& gs,
                           cudaStream_t st, const std::function<void()>& after_top = nullptr, long long ldt = NB,
                           bool t_adjoint = true) {
  GemmDesc g;
  g.M = nbp; g.N = nc; g.K = mp;
  g.opA = Op::H; g.A = Vp; g.lda = ldv;
  g.opB = Op::N; g.B = C; g.ldb = ldc;
  g.C = W; g.ldc = nc;
  zgemm(g, gs, st);
  GemmDesc g2;
  g2.M = nbp; g2.N = nc; g2.K = nbp;
  g2.opA = t_adjoint ? Op::H : Op::N; g2.A = Tp; g2.lda = ldt;
  g2.opB = Op::N; g2.B = W; g2.ldb = nc;
  g2.C = W2; g2.ldc = nc;
  zgemm(g2, gs, st);
  // C -= V W2; with after_top: the first nbp rows first (the block the caller
  // publishes next), then the callback, then the remaining rows
  const long long top = after_top ? std::min<long long>(nbp, mp) : mp;
  GemmDesc g3;
  g3.M = top; g3.N = nc; g3.K = nbp;
  g3.opA = Op::N; g3.A = Vp; g3.lda = ldv;
  g3.opB = Op::N; g3.B = W2; g3.ldb = nc;
  g3.C = C; g3.ldc = ldc;
  g3.alpha = -1.0; g3.beta = 1.0;
  zgemm(g3, gs, st);
  if (!after_top) return;
  after_top();
  if (mp > top) {
    g3.M = mp - top;
    g3.A = Vp + top * ldv;
    g3.C = C + top * ldc;
    zgemm(g3, gs, st);
  }
}

}  // namespace

namespace {
// T_ob (ob x ob, ld ob) of an outer block of npb panels starting at column J:
// zero, with the panels' T factors (NB x NB each, the valid nbp x nbp part)
// on the diagonal blocks
__global__ void tob_init_kernel(const double2* __restrict__ T, long long J, long long k, int npb, double2* tob,
                                int ob) {
  const int total = ob * ob;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int i = t / ob, j = t % ob, p = i / NB;
    double2 v = make_double2(0.0, 0.0);
    if (j / NB == p && p < npb) {
      const long long nbp = std::min<long long>(NB, k - J - static_cast<long long>(p) * NB);
      const int ii = i % NB, jj = j % NB;
      if (ii < nbp && jj < nbp) v = T[(static_cast<long long>(J / NB) + p) * NB * NB + ii * NB + jj];
    }
    tob[t] = v;
  }
}

int qr_outer_width() {
  static const int ob = [] {
    const char* s = std::getenv("QT_QR_OB");
    const int v = s ? std::atoi(s) : 128;
    return v >= 64 && v % NB == 0 && v <= 512 ? v : (v == 0 ? 0 : 128);
  }();
  return ob;
}

}  // namespace

namespace {
// Outer block [J, J + w) of a tall QR: its 32-column panels, each panel's
// reflector reaching only the rest of the block (narrow GEMMs), on stream st.
// V's rows [J, J + w) x cols [J, J + w) are zeroed above each panel's own rows
// first (the panels write their unit-lower triangles and everything below).
void outer_block_factor(Engine& e, double2* a, long long lda, long long m, long long k, double2* V, long long kp,
                        double2* T, long long J, long long w, double2* W, double2* W2, const GemmScratch& gs,
                        const PanelArgs& base, cudaStream_t st) {
  const int npb = static_cast<int>(ceil_div(w, NB));
  QT_CUDA(cudaMemset2DAsync(V + J * kp + J, kp * sizeof(double2), 0, w * sizeof(double2), w, st));
  for (int c = 0; c < npb; ++c) {
    const long long j = J + static_cast<long long>(c) * NB;
    const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
    const long long mp = m - j;
    PanelArgs pa = base;
    pa.A = a + j * lda + j;
    pa.lda = lda;
    pa.ldv = kp;
    pa.mp = mp;
    pa.nbp = nbp;
    pa.V = V + j * kp + j;
    pa.T = T + (j / NB) * NB * NB;
    launch_panel(e, pa, mp, st);
    const long long ninner = J + w - (j + nbp);
    if (ninner > 0) apply_block_reflector(pa.V, kp, pa.T, a + j * lda + j + nbp, lda, mp, ninner, nbp, W, W2, gs, st);
  }
}

// T_ob (ld ob) of outer block [J, J + w): the panels' T factors on the
// diagonal, T_ob[0:c0, c0:c0+32] = -T_prev (V_prev^H V_c) T_c above it
void outer_block_tob(Engine& e, const double2* V, long long kp, const double2* T, long long J, long long w,
                     long long k, long long m, double2* Tb, int ob, double2* G, double2* Z, const GemmScratch& gs,
                     cudaStream_t st) {
  const int npb = static_cast<int>(ceil_div(w, NB));
  const double2* Vb = V + J * kp + J;
  tob_init_kernel<<<static_cast<int>(ceil_div(static_cast<long long>(ob) * ob, 256)), 256, 0, st>>>(T, J, k, npb, Tb,
                                                                                                      ob);
  QT_LAUNCHED();
  if (npb <= 1) return;
  GemmDesc gg;
  gg.M = w; gg.N = w; gg.K = m - J;
  gg.opA = Op::H; gg.A = Vb; gg.lda = kp;
  gg.opB = Op::N; gg.B = Vb; gg.ldb = kp;
  gg.C = G; gg.ldc = ob;
  zgemm(gg, gs, st);
  for (int c = 1; c < npb; ++c) {
    const long long c0 = static_cast<long long>(c) * NB;
    const long long nbc = std::min<long long>(NB, w - c0);
    GemmDesc gz;  // Z = (V_prev^H V_c) T_c
    gz.M = c0; gz.N = nbc; gz.K = nbc;
    gz.A = G + c0; gz.lda = ob;
    gz.B = T + (J / NB + c) * NB * NB; gz.ldb = NB;
    gz.C = Z; gz.ldc = NB;
    zgemm(gz, gs, st);
    GemmDesc gx;  // T_ob[0:c0, c0:c0+nbc] = -T_prev Z
    gx.M = c0; gx.N = nbc; gx.K = c0;
    gx.A = Tb; gx.lda = ob;
    gx.B = Z; gx.ldb = NB;
    gx.C = Tb + c0; gx.ldc = ob;
    gx.alpha = -1.0; gx.beta = 0.0;
    zgemm(gx, gs, st);
  }
}
}  // namespace

// Tall QR (panels beyond one block-reflector cluster, m > 2048): two-level
// blocking.  Panels of NB = 32 columns are factored inside outer blocks of OB
// columns (QT_QR_OB, default 128), each panel's reflector reaching only the
// rest of its outer block (narrow GEMMs); then the OB reflectors of the block
// are combined into one compact-WY pair (V_ob, T_ob):
//   T_ob = [[T_prev, -T_prev (V_prev^H V_c) T_c], [0, T_c]]   (panel by panel)
// and the trailing matrix -- and, in Q formation, Q -- is updated with K = OB
// DMMA GEMMs instead of K = 32 ones.  Look-ahead: the next outer block's
// columns are updated on the main stream, the rest on e.side while the next
// block's panels run; QrOpts::capply applies (V_ob, T_ob) to C on e.side2.
void qr_inplace_outer(Engine& e, double2* a, long long m, long long n, long long lda, double2* q, long long ldq,
                      double2* r, long long ldr, const QrOpts& opts) {
  const long long k = std::min(m, n);
  const int OB = qr_outer_width();
  const long long npan = ceil_div(k, NB);
  const long long kp = npan * NB;
  const long long nob = ceil_div(k, static_cast<long long>(OB));
  double2* V = e.cbuf(S_QR_V, static_cast<size_t>(m) * kp);
  double2* T = e.cbuf(S_QR_T, static_cast<size_t>(npan) * NB * NB);
  double2* TOB = e.cbuf(S_QR_TOB, static_cast<size_t>(nob) * OB * OB);
  double2* G = e.cbuf(S_QR_GRAM, static_cast<size_t>(OB) * OB + static_cast<size_t>(OB) * NB);
  double2* Z = G + static_cast<size_t>(OB) * OB;
  double2* W = e.cbuf(S_QR_W, static_cast<size_t>(OB) * n);
  double2* W2 = e.cbuf(S_QR_W2, static_cast<size_t>(OB) * n);
  double2* SW = e.cbuf(S_QR_WS, static_cast<size_t>(OB) * n);
  double2* SW2 = e.cbuf(S_QR_WS2, static_cast<size_t>(OB) * n);
  double2* part = e.cbuf(S_QR_PART, static_cast<size_t>(2) * kNumSMs * NB + 2 * NB);
  const GemmScratch gs = e.gemm_scratch();
  GemmScratch gss;
  gss.partial = e.cbuf(S_GEMM_PARTS, size_t(1) << 22);
  gss.partial_elems = size_t(1) << 22;
  gss.tile_sums = e.dbuf(S_TILE_SUMSS, size_t(1) << 16);
  gss.tile_sums_elems = size_t(1) << 16;
  const bool capply = opts.capply != nullptr && opts.nc > 0;
  double2 *CW = nullptr, *CW2 = nullptr;
  GemmScratch gs2;
  if (capply) {
    CW = e.cbuf(S_QA_W, static_cast<size_t>(OB) * opts.nc);
    CW2 = e.cbuf(S_QA_W2, static_cast<size_t>(OB) * opts.nc);
    gs2 = e.gemm_scratch2();
  }
  PanelArgs base{};
  base.lda = lda;
  base.ldv = kp;
  base.part = part;
  base.diag = part + 2 * kNumSMs * NB;
  base.bar = e.barrier;
  base.dbg = nullptr;

  // event ids: 3000 + 2b (T_ob(b) ready), 3001 + 2b (side update of block b done)
  const size_t ev0 = 3000;
  long long side_last = -1;
  for (long long b = 0; b < nob; ++b) {
    const long long J = b * OB;
    const long long w = std::min<long long>(OB, k - J);  // reflectors in this block
    const long long mb = m - J;
    const int npb = static_cast<int>(ceil_div(w, NB));
    outer_block_factor(e, a, lda, m, k, V, kp, T, J, w, W, W2, gs, base, e.stream);
    double2* Tb = TOB + b * OB * OB;
    const double2* Vb = V + J * kp + J;
    outer_block_tob(e, V, kp, T, J, w, k, m, Tb, OB, G, Z, gs, e.stream);
    if (capply) {  // C <- Q_ob^H C on side2, behind this block
      QT_CUDA(cudaEventRecord(e.event(ev0 + 2 * b), e.stream));
      QT_CUDA(cudaStreamWaitEvent(e.side2, e.event(ev0 + 2 * b), 0));
      apply_block_reflector(Vb, kp, Tb, opts.capply + J * opts.ldc, opts.ldc, mb, opts.nc, static_cast<int>(w), CW,
                            CW2, gs2, e.side2, nullptr, OB, true);
    }
    const long long ntr = n - (J + w);
    if (ntr <= 0) continue;
    // look-ahead: the next block's columns on the main stream (after the side
    // stream's update of the previous block reached them), the rest on e.side
    const long long nn = std::min<long long>(OB, ntr);
    if (side_last >= 0) QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(ev0 + 2 * side_last + 1), 0));
    if (ntr > nn) {
      if (!capply) QT_CUDA(cudaEventRecord(e.event(ev0 + 2 * b), e.stream));
      QT_CUDA(cudaStreamWaitEvent(e.side, e.event(ev0 + 2 * b), 0));
    }
    apply_block_reflector(Vb, kp, Tb, a + J * lda + J + w, lda, mb, nn, static_cast<int>(w), W, W2, gs, e.stream,
                          nullptr, OB, true);
    if (ntr > nn) {
      apply_block_reflector(Vb, kp, Tb, a + J * lda + J + w + nn, lda, mb, ntr - nn, static_cast<int>(w), SW, SW2,
                            gss, e.side, nullptr, OB, true);
      QT_CUDA(cudaEventRecord(e.event(ev0 + 2 * b + 1), e.side));
      side_last = b;
    }
  }
  if (side_last >= 0) QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(ev0 + 2 * side_last + 1), 0));
  if (capply) {  // join side2: Q^H C complete
    QT_CUDA(cudaEventRecord(e.event(ev0 + 2 * nob + 2), e.side2));
    QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(ev0 + 2 * nob + 2), 0));
  }
  if (opts.want_q) {
    // explicit thin Q = Q_ob(0) ... Q_ob(nob-1) I[:, :k], outer blocks backward
    set_identity(e, q, m, k, ldq);
    for (long long b = nob - 1; b >= 0; --b) {
      const long long J = b * OB;
      const long long w = std::min<long long>(OB, k - J);
      apply_block_reflector(V + J * kp + J, kp, TOB + b * OB * OB, q + J * ldq + J, ldq, m - J, k - J,
                            static_cast<int>(w), W, W2, gs, e.stream, nullptr, OB, false);
    }
    gauge_q_kernel<<<grid_for(m * k), 256, 0, e.stream>>>(a, lda, q, ldq, m, k);
    QT_LAUNCHED();
  }
  if (opts.want_r) {
    gauge_r_kernel<<<grid_for(k * n), 256, 0, e.stream>>>(a, lda, r, ldr, k, n);
    QT_LAUNCHED();
  }
}

namespace {
// q[(j0 + i) * ld + j0 + i] += 1, i < w (the identity part of a column block
// of Q = I - V T V^H)
__global__ void add_diag_kernel(double2* q, long long ld, long long j0, int w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < w) q[(j0 + i) * ld + j0 + i].x += 1.0;
}
}  // namespace

bool qr_pair_tall_fits(long long m, long long nc, long long k) {
  static const bool off = std::getenv("QT_NO_TALL_PAIR") != nullptr;
  // both chains on cluster panels (<= 5120 rows): two grid-barrier panels in
  // flight at once could each hold part of the GPU while waiting for the rest
  return !off && qr_outer_width() > 0 && !larfb_cluster_fits(m) && !larfb_cluster_fits(nc) && m <= 5120 &&
         nc <= 5120 && k > NB && k <= m && k <= nc;
}

void qr_pair_tall(Engine& e, double2* x, long long m, long long k, double2* c, long long nc, double2* yh,
                  double2* qy, double2* ry, double2* qx,
                  const std::function<void(long long, long long, cudaStream_t)>& extract) {
  const int OB = qr_outer_width();
  const long long npan = ceil_div(k, NB);
  const long long kp = npan * NB;
  const long long nob = ceil_div(k, static_cast<long long>(OB));
  const cudaStream_t sx = e.stream, sxw = e.side, sa = e.side2, sy = e.side3;
  // X chain (main + look-ahead side stream) and the theta application (side2)
  double2* V = e.cbuf(S_QR_V, static_cast<size_t>(m) * kp);
  double2* T = e.cbuf(S_QR_T, static_cast<size_t>(npan) * NB * NB);
  double2* TOB = e.cbuf(S_QR_TOB, static_cast<size_t>(nob) * OB * OB);
  double2* G = e.cbuf(S_QR_GRAM, static_cast<size_t>(OB) * OB + static_cast<size_t>(OB) * NB);
  double2* W = e.cbuf(S_QR_W, static_cast<size_t>(OB) * k);
  double2* W2 = e.cbuf(S_QR_W2, static_cast<size_t>(OB) * k);
  double2* SW = e.cbuf(S_QR_WS, static_cast<size_t>(OB) * k);
  double2* SW2 = e.cbuf(S_QR_WS2, static_cast<size_t>(OB) * k);
  double2* CW = e.cbuf(S_QA_W, static_cast<size_t>(OB) * nc);
  double2* CW2 = e.cbuf(S_QA_W2, static_cast<size_t>(OB) * nc);
  double2* part = e.cbuf(S_QR_PART, static_cast<size_t>(2) * kNumSMs * NB + 2 * NB);
  // Y^H chain (side3)
  double2* Vy = e.cbuf(S_QR_V2, static_cast<size_t>(nc) * kp);
  double2* Ty = e.cbuf(S_QR_T2, static_cast<size_t>(npan) * NB * NB);
  double2* TOBy = e.cbuf(S_QR_TOB2, static_cast<size_t>(nob) * OB * OB);
  double2* Gy = e.cbuf(S_QR_GRAM2, static_cast<size_t>(OB) * OB + static_cast<size_t>(OB) * NB);
  double2* YW = e.cbuf(S_QR_YW, static_cast<size_t>(k) * std::max(nc, k));
  double2* YW2 = e.cbuf(S_QR_YW2, static_cast<size_t>(k) * std::max(nc, k));
  double2* TALL = e.cbuf(S_QR_TALL, static_cast<size_t>(k) * k);
  double2* TZ = e.cbuf(S_QR_TALLZ, static_cast<size_t>(2) * k * OB);
  double2* party = e.cbuf(S_QR_PART2, static_cast<size_t>(2) * kNumSMs * NB + 2 * NB);
  // Q of Y^H, column block b, on sq right behind Y^H block b (T_all is
  // left-looking, so Q[:, J:J+w] = E - V[:, :J+w] (T_all[:J+w, :J+w]
  // V[J:J+w, :J+w]^H) is final once block b is factored)
  double2* QYM = e.cbuf(S_QR_QYM, static_cast<size_t>(k) * OB);
  const cudaStream_t sq = e.side5;
  const GemmScratch gs4 = e.gemm_scratch4();
  const GemmScratch gs = e.gemm_scratch();
  GemmScratch gss;
  gss.partial = e.cbuf(S_GEMM_PARTS, size_t(1) << 22);
  gss.partial_elems = size_t(1) << 22;
  gss.tile_sums = e.dbuf(S_TILE_SUMSS, size_t(1) << 16);
  gss.tile_sums_elems = size_t(1) << 16;
  const GemmScratch gs2 = e.gemm_scratch2(), gsy = e.gemm_scratch3();

  PanelArgs bx{};
  bx.part = part;
  bx.diag = part + 2 * kNumSMs * NB;
  bx.bar = e.barrier;
  bx.dbg = nullptr;
  PanelArgs by = bx;
  by.part = party;
  by.diag = party + 2 * kNumSMs * NB;
  by.bar = e.barrier + 16;

  // QT_PAIR_DEBUG=1 (eager calls only): timeline of the tall pair on stderr
  static const bool tdbg = std::getenv("QT_PAIR_DEBUG") != nullptr;
  static std::vector<cudaEvent_t> tev;
  std::vector<std::string> tname;
  auto stamp = [&](const std::string& nm, cudaStream_t st) {
    if (!tdbg) return;
    if (tev.size() <= tname.size()) {
      cudaEvent_t ev;
      QT_CUDA(cudaEventCreate(&ev));
      tev.push_back(ev);
    }
    QT_CUDA(cudaEventRecord(tev[tname.size()], st));
    tname.push_back(nm);
  };
  stamp("start", sx);

  // events: 4000 + 4b: X block b's T ready; +1: X side update done; +2: rows
  // of Y^H block b published; 4000 + 4 nob: start / joins; + 3 + b: Y^H block
  // b factored (Q column block b may start); + 3 + nob: Q complete
  const size_t ev0 = 4000, evs = ev0 + 4 * static_cast<size_t>(nob);
  QT_CUDA(cudaEventRecord(e.event(evs), sx));  // everything earlier on sx precedes both side chains
  QT_CUDA(cudaStreamWaitEvent(sy, e.event(evs), 0));
  QT_CUDA(cudaStreamWaitEvent(sa, e.event(evs), 0));
  QT_CUDA(cudaStreamWaitEvent(sq, e.event(evs), 0));
  QT_CUDA(cudaMemsetAsync(TALL, 0, static_cast<size_t>(k) * k * sizeof(double2), sy));
  // the combined reflector of the finished Y^H blocks is used from row 0: the
  // rows above each block's own diagonal block must be zero
  QT_CUDA(cudaMemsetAsync(Vy, 0, static_cast<size_t>(nc) * kp * sizeof(double2), sy));
  long long side_last = -1;
  for (long long b = 0; b < nob; ++b) {
    const long long J = b * OB;
    const long long w = std::min<long long>(OB, k - J);
    // ---- X block b (main stream), T_ob
    outer_block_factor(e, x, k, m, k, V, kp, T, J, w, W, W2, gs, bx, sx);
    double2* Tb = TOB + b * OB * OB;
    const double2* Vb = V + J * kp + J;
    outer_block_tob(e, V, kp, T, J, w, k, m, Tb, OB, G, G + static_cast<size_t>(OB) * OB, gs, sx);
    stamp("X" + std::to_string(b), sx);
    QT_CUDA(cudaEventRecord(e.event(ev0 + 4 * b), sx));
    // ---- theta side: C <- Q_ob^H C, then rows [J, J + w) of C are final:
    // published as columns [J, J + w) of Y^H
    QT_CUDA(cudaStreamWaitEvent(sa, e.event(ev0 + 4 * b), 0));
    apply_block_reflector(Vb, kp, Tb, c + J * nc, nc, m - J, nc, static_cast<int>(w), CW, CW2, gs2, sa,
                          [&] {
                            extract(J, w, sa);
                            stamp("ext" + std::to_string(b), sa);
                            // the Y^H chain needs only the published block, not
                            // the rest of C: release it here
                            QT_CUDA(cudaEventRecord(e.event(ev0 + 4 * b + 2), sa));
                          },
                          OB, true);
    stamp("th" + std::to_string(b), sa);
    // ---- X look-ahead: the next block's columns on sx, the rest on sxw
    const long long ntr = k - (J + w);
    if (ntr > 0) {
      const long long nn = std::min<long long>(OB, ntr);
      if (side_last >= 0) QT_CUDA(cudaStreamWaitEvent(sx, e.event(ev0 + 4 * side_last + 1), 0));
      if (ntr > nn) QT_CUDA(cudaStreamWaitEvent(sxw, e.event(ev0 + 4 * b), 0));
      apply_block_reflector(Vb, kp, Tb, x + J * k + J + w, k, m - J, nn, static_cast<int>(w), W, W2, gs, sx, nullptr,
                            OB, true);
      if (ntr > nn) {
        apply_block_reflector(Vb, kp, Tb, x + J * k + J + w + nn, k, m - J, ntr - nn, static_cast<int>(w), SW, SW2,
                              gss, sxw, nullptr, OB, true);
        QT_CUDA(cudaEventRecord(e.event(ev0 + 4 * b + 1), sxw));
        stamp("Xw" + std::to_string(b), sxw);
        side_last = b;
      }
    }
    // ---- Y^H block b (side3): the finished blocks' combined reflector
    // (left-looking), its panels, its T_ob, and T_all's new block column
    QT_CUDA(cudaStreamWaitEvent(sy, e.event(ev0 + 4 * b + 2), 0));
    stamp("Ys" + std::to_string(b), sy);
    if (b > 0)
      apply_block_reflector(Vy, kp, TALL, yh + J, k, nc, w, static_cast<int>(J), YW, YW2, gsy, sy, nullptr, k, true);
    stamp("Yl" + std::to_string(b), sy);
    outer_block_factor(e, yh, k, nc, k, Vy, kp, Ty, J, w, YW, YW2, gsy, by, sy);
    stamp("Yf" + std::to_string(b), sy);
    double2* Tyb = TOBy + b * OB * OB;
    outer_block_tob(e, Vy, kp, Ty, J, w, k, nc, Tyb, OB, Gy, Gy + static_cast<size_t>(OB) * OB, gsy, sy);
    stamp("Yt" + std::to_string(b), sy);
    copy2d(e, Tyb, OB, TALL + J * k + J, k, w, w, sy);
    if (b > 0) {
      GemmDesc gg;  // V_prev^H V_b (J x w), rows J.. of both (V_prev is zero above its own rows < J only)
      gg.M = J; gg.N = w; gg.K = nc - J;
      gg.opA = Op::H; gg.A = Vy + J * kp; gg.lda = kp;
      gg.B = Vy + J * kp + J; gg.ldb = kp;
      gg.C = TZ; gg.ldc = w;
      zgemm(gg, gsy, sy);
      GemmDesc gz;  // Z = (V_prev^H V_b) T_b
      gz.M = J; gz.N = w; gz.K = w;
      gz.A = TZ; gz.lda = w;
      gz.B = Tyb; gz.ldb = OB;
      gz.C = TZ + J * w; gz.ldc = w;
      zgemm(gz, gsy, sy);
      GemmDesc gx;  // T_all[0:J, J:J+w] = -T_all[0:J, 0:J] Z
      gx.M = J; gx.N = w; gx.K = J;
      gx.A = TALL; gx.lda = k;
      gx.B = TZ + J * w; gx.ldb = w;
      gx.C = TALL + J; gx.ldc = k;
      gx.alpha = -1.0; gx.beta = 0.0;
      zgemm(gx, gsy, sy);
    }
    stamp("Y" + std::to_string(b), sy);
    QT_CUDA(cudaEventRecord(e.event(evs + 3 + b), sy));
    QT_CUDA(cudaStreamWaitEvent(sq, e.event(evs + 3 + b), 0));
    {
      const long long jw = J + w;
      GemmDesc gm;  // QYM = T_all[:jw, :jw] V[J:jw, :jw]^H  (jw x w)
      gm.M = jw; gm.N = w; gm.K = jw;
      gm.A = TALL; gm.lda = k;
      gm.opB = Op::H; gm.B = Vy + J * kp; gm.ldb = kp;
      gm.C = QYM; gm.ldc = w;
      zgemm(gm, gs4, sq);
      GemmDesc gq;  // Q[:, J:jw] = -V[:, :jw] QYM, then + E
      gq.M = nc; gq.N = w; gq.K = jw;
      gq.A = Vy; gq.lda = kp;
      gq.B = QYM; gq.ldb = w;
      gq.C = qy + J; gq.ldc = k;
      gq.alpha = -1.0; gq.beta = 0.0;
      zgemm(gq, gs4, sq);
      add_diag_kernel<<<1, 256, 0, sq>>>(qy, k, J, static_cast<int>(w));
      QT_LAUNCHED();
      // gauge phases of columns [J, jw): R_ii of Y^H, final with block b
      gauge_q_kernel<<<grid_for(nc * w), 256, 0, sq>>>(yh + J * k + J, k, qy + J, k, nc, w);
      QT_LAUNCHED();
      stamp("Q" + std::to_string(b), sq);
    }
  }
  // ---- gauge-fixed Q (formed on sq) and R of Y^H (side3), X's Q if asked
  QT_CUDA(cudaEventRecord(e.event(evs + 3 + nob), sq));
  QT_CUDA(cudaStreamWaitEvent(sy, e.event(evs + 3 + nob), 0));
  gauge_r_kernel<<<grid_for(k * k), 256, 0, sy>>>(yh, k, ry, k, k, k);
  QT_LAUNCHED();
  if (side_last >= 0) QT_CUDA(cudaStreamWaitEvent(sx, e.event(ev0 + 4 * side_last + 1), 0));
  if (qx) {  // X's Q (left_iso), backward over X's outer blocks on sx after the factorization
    set_identity(e, qx, m, k, k, sx);
    for (long long b = nob - 1; b >= 0; --b) {
      const long long J = b * OB;
      const long long w = std::min<long long>(OB, k - J);
      apply_block_reflector(V + J * kp + J, kp, TOB + b * OB * OB, qx + J * k + J, k, m - J, k - J,
                            static_cast<int>(w), W, W2, gs, sx, nullptr, OB, false);
    }
    gauge_q_kernel<<<grid_for(m * k), 256, 0, sx>>>(x, k, qx, k, m, k);
    QT_LAUNCHED();
  }
  QT_CUDA(cudaEventRecord(e.event(evs + 1), sa));
  QT_CUDA(cudaStreamWaitEvent(sx, e.event(evs + 1), 0));
  QT_CUDA(cudaEventRecord(e.event(evs + 2), sy));
  QT_CUDA(cudaStreamWaitEvent(sx, e.event(evs + 2), 0));
  stamp("end", sx);
  if (tdbg) {
    QT_CUDA(cudaStreamSynchronize(sx));
    std::fprintf(stderr, "qr_pair_tall m=%lld k=%lld nc=%lld timeline (us from start):", m, k, nc);
    for (size_t i = 1; i < tname.size(); ++i) {
      float ms = 0.f;
      QT_CUDA(cudaEventElapsedTime(&ms, tev[0], tev[i]));
      std::fprintf(stderr, " %s=%.0f", tname[i].c_str(), ms * 1000.f);
    }
    std::fprintf(stderr, "\n");
  }
}

namespace {
bool use_outer_qr(long long m, long long k) {
  return qr_outer_width() > 0 && !larfb_cluster_fits(m) && k > NB;
}
}  // namespace

void qr_inplace(Engine& e, double2* a, long long m, long long n, long long lda, double2* q, long long ldq,
                double2* r, long long ldr, const QrOpts& opts) {
  const long long k = std::min(m, n);
  if (k == 0) return;
  if (use_outer_qr(m, k)) {
    qr_inplace_outer(e, a, m, n, lda, q, ldq, r, ldr, opts);
    return;
  }
  const long long npan = ceil_div(k, NB);
  const long long kp = npan * NB;
  double2* V = e.cbuf(S_QR_V, static_cast<size_t>(m) * kp);
  double2* T = e.cbuf(S_QR_T, static_cast<size_t>(npan) * NB * NB);
  double2* W = e.cbuf(S_QR_W, static_cast<size_t>(NB) * n);
  double2* W2 = e.cbuf(S_QR_W2, static_cast<size_t>(NB) * n);
  double2* part = e.cbuf(S_QR_PART, static_cast<size_t>(2) * kNumSMs * NB + 2 * NB);
  const GemmScratch gs = e.gemm_scratch();

  PanelArgs base{};
  base.lda = lda;
  base.ldv = kp;
  base.part = part;
  base.diag = part + 2 * kNumSMs * NB;
  base.bar = e.barrier;
  // QT_PANEL_DEBUG=1: per-column phase timings of the cluster panel (stderr)
  static const bool dbg_on = std::getenv("QT_PANEL_DEBUG") != nullptr;
  static long long* dbg_buf = nullptr;
  if (dbg_on && !dbg_buf) QT_CUDA(cudaMalloc(&dbg_buf, 8 * NB * sizeof(long long)));
  base.dbg = dbg_on ? dbg_buf : nullptr;

  // look-ahead of the trailing update (m <= 16 x 128: block reflectors in one
  // cluster launch): the next panel's columns on the main stream, the rest on
  // e.side behind the next panel; taller panels take qr_inplace_outer (or,
  // with QT_QR_OB=0, sequential three-GEMM updates); QT_QR_NO_LOOKAHEAD
  // disables it
  static const bool la_env = std::getenv("QT_QR_NO_LOOKAHEAD") == nullptr;
  const bool la_cluster = larfb_cluster_fits(m);
  const bool lookahead = la_env && npan >= 2 && e.side != nullptr && la_cluster;
  bool wide_pending = false;
  long long last_wide = -1;
  // QrOpts::capply: panel p's reflector reaches C on side2 once the panel is
  // factored (events 2 npan + p), concurrently with the later panels
  const bool capply = opts.capply != nullptr && opts.nc > 0;
  const size_t cev = static_cast<size_t>(2 * npan + 2);
  double2 *CW = nullptr, *CW2 = nullptr;
  GemmScratch gs2;
  if (capply) {
    CW = e.cbuf(S_QA_W, static_cast<size_t>(NB) * opts.nc);
    CW2 = e.cbuf(S_QA_W2, static_cast<size_t>(NB) * opts.nc);
    gs2 = e.gemm_scratch2();
  }
  for (long long p = 0; p < npan; ++p) {
    const long long j = p * NB;
    const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
    const long long mp = m - j;
    PanelArgs pa = base;
    pa.A = a + j * lda + j;
    pa.mp = mp;
    pa.nbp = nbp;
    pa.V = V + j * kp + p * NB;
    pa.T = T + p * NB * NB;
    launch_panel(e, pa, mp);
    if (capply) {
      QT_CUDA(cudaEventRecord(e.event(cev + p), e.stream));
      QT_CUDA(cudaStreamWaitEvent(e.side2, e.event(cev + p), 0));
      apply_block_reflector(pa.V, kp, pa.T, opts.capply + j * opts.ldc, opts.ldc, mp, opts.nc, nbp, CW, CW2, gs2,
                            e.side2);
    }
    if (dbg_on) {
      long long h[8 * NB];
      QT_CUDA(cudaMemcpyAsync(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost, e.stream));
      QT_CUDA(cudaStreamSynchronize(e.stream));
      // phases of CTA 0 / warp 0 per column: CTA reduce, push, DSMEM wait,
      // cluster combine, zlarfg, ctw/Z, barrier + broadcast, row pass
      static const char* names[8] = {"cta_red", "push", "wait", "combine", "refl", "ctwZ", "bcast", "rows"};
      double ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = 0; c + 1 < nbp; ++c) {
        for (int q = 0; q < 7; ++q) ph[q] += h[c * 8 + q + 1] - h[c * 8 + q];
        ph[7] += h[(c + 1) * 8 + 0] - h[c * 8 + 7];
      }
      std::fprintf(stderr, "panel m=%lld nbp=%d cycles/col:", mp, nbp);
      for (int q = 0; q < 8; ++q) std::fprintf(stderr, " %s %.0f", names[q], ph[q] / (nbp - 1));
      std::fprintf(stderr, "\n");
    }
    const long long ntr = n - j - nbp;
    if (lookahead && ntr > 0) {
      // look-ahead: H_p reaches the next panel's columns first (main stream,
      // after the side stream finished H_{p-1} on them); the rest of the
      // trailing matrix is updated on the side stream while panel p+1 runs
      const long long nn = std::min<long long>(NB, ntr);
      if (p > 0 && wide_pending) QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(2 * (p - 1) + 1), 0));
      if (ntr > nn) {
        QT_CUDA(cudaEventRecord(e.event(2 * p), e.stream));  // panel p done: V_p, T_p ready
        QT_CUDA(cudaStreamWaitEvent(e.side, e.event(2 * p), 0));
      }
      larfb_cluster(e, pa.V, kp, pa.T, a + j * lda + j + nbp, lda, mp, nn, nbp, true, e.stream);
      wide_pending = ntr > nn;
      if (wide_pending) {
        larfb_cluster(e, pa.V, kp, pa.T, a + j * lda + j + nbp + nn, lda, mp, ntr - nn, nbp, true, e.side);
        QT_CUDA(cudaEventRecord(e.event(2 * p + 1), e.side));
        last_wide = p;
      }
      continue;
    }
    if (ntr > 0 && !larfb_cluster(e, pa.V, kp, pa.T, a + j * lda + j + nbp, lda, mp, ntr, nbp, true)) {
      GemmDesc g;
      // W = V^H A_trail
      g.M = nbp; g.N = ntr; g.K = mp;
      g.opA = Op::H; g.A = pa.V; g.lda = kp;
      g.opB = Op::N; g.B = a + j * lda + j + nbp; g.ldb = lda;
      g.C = W; g.ldc = ntr;
      zgemm(g, gs, e.stream);
      // W2 = T^H W
      GemmDesc g2;
      g2.M = nbp; g2.N = ntr; g2.K = nbp;
      g2.opA = Op::H; g2.A = pa.T; g2.lda = NB;
      g2.opB = Op::N; g2.B = W; g2.ldb = ntr;
      g2.C = W2; g2.ldc = ntr;
      zgemm(g2, gs, e.stream);
      // A_trail -= V W2
      GemmDesc g3;
      g3.M = mp; g3.N = ntr; g3.K = nbp;
      g3.opA = Op::N; g3.A = pa.V; g3.lda = kp;
      g3.opB = Op::N; g3.B = W2; g3.ldb = ntr;
      g3.C = a + j * lda + j + nbp; g3.ldc = lda;
      g3.alpha = -1.0; g3.beta = 1.0;
      zgemm(g3, gs, e.stream);
    }
  }

  if (last_wide >= 0) QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(2 * last_wide + 1), 0));  // join the side stream
  if (capply) {  // join side2: Q^H C complete
    QT_CUDA(cudaEventRecord(e.event(cev + npan), e.side2));
    QT_CUDA(cudaStreamWaitEvent(e.stream, e.event(cev + npan), 0));
  }
  if (!opts.want_q) {
    if (opts.want_r) {
      gauge_r_kernel<<<grid_for(k * n), 256, 0, e.stream>>>(a, lda, r, ldr, k, n);
      QT_LAUNCHED();
    }
    return;
  }

  // explicit thin Q = H_0 ... H_{k-1} I[:, :k], block reflectors backward
  set_identity(e, q, m, k, ldq);
  for (long long p = npan - 1; p >= 0; --p) {
    const long long j = p * NB;
    const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
    const long long mp = m - j, nq = k - j;
    const double2* Vp = V + j * kp + p * NB;
    const double2* Tp = T + p * NB * NB;
    double2* Qs = q + j * ldq + j;
    if (larfb_cluster(e, Vp, kp, Tp, Qs, ldq, mp, nq, nbp, false)) continue;
    GemmDesc g;
    g.M = nbp; g.N = nq; g.K = mp;
    g.opA = Op::H; g.A = Vp; g.lda = kp;
    g.opB = Op::N; g.B = Qs; g.ldb = ldq;
    g.C = W; g.ldc = nq;
    zgemm(g, gs, e.stream);
    GemmDesc g2;
    g2.M = nbp; g2.N = nq; g2.K = nbp;
    g2.opA = Op::N; g2.A = Tp; g2.lda = NB;
    g2.opB = Op::N; g2.B = W; g2.ldb = nq;
    g2.C = W2; g2.ldc = nq;
    zgemm(g2, gs, e.stream);
    GemmDesc g3;
    g3.M = mp; g3.N = nq; g3.K = nbp;
    g3.opA = Op::N; g3.A = Vp; g3.lda = kp;
    g3.opB = Op::N; g3.B = W2; g3.ldb = nq;
    g3.C = Qs; g3.ldc = ldq;
    g3.alpha = -1.0; g3.beta = 1.0;
    zgemm(g3, gs, e.stream);
  }

  gauge_q_kernel<<<grid_for(m * k), 256, 0, e.stream>>>(a, lda, q, ldq, m, k);
  QT_LAUNCHED();
  if (opts.want_r) {
    gauge_r_kernel<<<grid_for(k * n), 256, 0, e.stream>>>(a, lda, r, ldr, k, n);
    QT_LAUNCHED();
  }
}


bool qr_pair_fits(long long m, long long nc) { return larfb_cluster_fits(m) && larfb_cluster_fits(nc); }

void pair_form_q(Engine& e, const double2* x, long long m, long long k, double2* q, long long ldq, cudaStream_t st) {
  // Q = H_0 ... H_{k-1} I[:, :k] from QR(X)'s reflectors as the pair left them
  // (S_QR_V / S_QR_T, leading dimension kp), block reflectors backward in one
  // cluster launch each, then the gauge phases of X's diagonal
  const long long npan = ceil_div(k, NB);
  const long long kp = npan * NB;
  const double2* V = e.cbuf(S_QR_V, static_cast<size_t>(m) * kp);
  const double2* T = e.cbuf(S_QR_T, static_cast<size_t>(npan) * NB * NB);
  set_identity(e, q, m, k, ldq, st);
  for (long long p = npan - 1; p >= 0; --p) {
    const long long j = p * NB;
    const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
    if (!larfb_cluster(e, V + j * kp + j, kp, T + p * NB * NB, q + j * ldq + j, ldq, m - j, k - j, nbp, false, st))
      throw Error(Err::internal, "pair_form_q: block reflector does not fit one cluster");
  }
  gauge_q_kernel<<<grid_for(m * k), 256, 0, st>>>(x, k, q, ldq, m, k);
  QT_LAUNCHED();
}

namespace {
// Rows [j, j + nbp) of H_p^H C and block p of Y^H in one pass over 32-column
// tiles (replaces three launches on the theta side's critical chain):
//   W2 = T^H W             (T upper triangular; W2 feeds the C_rest GEMM)
//   C_top -= V_top W2      (V_top unit lower triangular)
//   yh[c, j + r] = ph_{j+r} conj(C_top[r, c])   (Y = Q_m^H theta, Q_m gauged)
__global__ void __launch_bounds__(256) pair_top_kernel(const double2* __restrict__ W, const double2* __restrict__ T,
                                                       const double2* __restrict__ Vt, long long ldv,
                                                       double2* __restrict__ ct, long long nc, int nbp,
                                                       double2* __restrict__ W2, const double2* __restrict__ x,
                                                       long long k, double2* __restrict__ yh, long long j) {
  // T and V_top entries are warp-uniform (one row r per warp): broadcast
  // loads through the read-only path, only the column tiles in shared memory
  __shared__ double2 ws[NB][NB + 1], w2s[NB][NB + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const long long c0 = static_cast<long long>(blockIdx.x) * NB, c = c0 + tx;
  const double2 z = make_double2(0.0, 0.0);
  for (int r = ty; r < NB; r += 8) ws[r][tx] = (r < nbp && c < nc) ? W[r * nc + c] : z;
  __syncthreads();
  for (int r = ty; r < nbp; r += 8) {
    double2 acc = z;
    for (int q = 0; q <= r; ++q) {
      const double2 t = __ldg(&T[q * NB + r]), w = ws[q][tx];  // acc += conj(T[q][r]) W[q]
      acc.x = fma(t.x, w.x, fma(t.y, w.y, acc.x));
      acc.y = fma(t.x, w.y, fma(-t.y, w.x, acc.y));
    }
    w2s[r][tx] = acc;
    if (c < nc) W2[r * nc + c] = acc;
  }
  __syncthreads();
  for (int r = ty; r < nbp; r += 8) {
    if (c < nc) {
      double2 acc = ct[r * nc + c];
      for (int q = 0; q <= r; ++q) acc = csub(acc, cmul(__ldg(&Vt[r * ldv + q]), w2s[q][tx]));
      ct[r * nc + c] = acc;
      ws[r][tx] = cmul(qr_phase(x, k, j + r), cconj(acc));
    }
  }
  __syncthreads();
  for (int r = ty; r < NB; r += 8)
    if (c0 + r < nc && tx < nbp) yh[(c0 + r) * k + j + tx] = ws[tx][r];
}
}  // namespace

void qr_pair_pipelined(Engine& e, double2* x, long long m, long long k, double2* c, long long nc, double2* yh,
                       double2* qy, double2* ry) {
  if (k == 0) return;
  if (k > m || k > nc || !qr_pair_fits(m, nc)) throw Error(Err::internal, "qr_pair_pipelined: shape not supported");
  const long long npan = ceil_div(k, NB);
  const long long kp = npan * NB;
  // X: reflectors in S_QR_V / S_QR_T, Y^H: S_QR_V2 / S_QR_T2 (both QRs are in flight at once)
  double2* Vx = e.cbuf(S_QR_V, static_cast<size_t>(m) * kp);
  double2* Tx = e.cbuf(S_QR_T, static_cast<size_t>(npan) * NB * NB);
  double2* Vy = e.cbuf(S_QR_V2, static_cast<size_t>(nc) * kp);
  double2* Ty = e.cbuf(S_QR_T2, static_cast<size_t>(npan) * NB * NB);
  double2* part = e.cbuf(S_QR_PART, static_cast<size_t>(2) * kNumSMs * NB + 2 * NB);
  double2* CW = e.cbuf(S_QA_W, static_cast<size_t>(NB) * nc);
  double2* CW2 = e.cbuf(S_QA_W2, static_cast<size_t>(NB) * nc);
  const GemmScratch gs2 = e.gemm_scratch2();
  const cudaStream_t sx = e.stream, sxw = e.side, sa = e.side2, sy = e.side3;
  // events: X look-ahead 2p / 2p+1, panel done P0 + p, block extracted E0 + p, joins J0..
  const size_t P0 = static_cast<size_t>(2 * npan + 2), E0 = P0 + npan + 1, J0 = E0 + npan + 1;

  PanelArgs base{};
  base.part = part;
  base.diag = part + 2 * kNumSMs * NB;
  base.bar = e.barrier;
  base.dbg = nullptr;

  // the Y chain may only start after everything earlier on the caller's stream
  QT_CUDA(cudaEventRecord(e.event(J0), sx));
  QT_CUDA(cudaStreamWaitEvent(sy, e.event(J0), 0));
  // explicit Q of Y^H formed block by block on sq behind the Y chain: column
  // block b of Q = H'_0 ... H'_b [e_{32b} .. e_{32b+31}] (reflectors > b leave
  // those columns alone), one reverse multi-reflector launch per block
  static const bool qblocks = std::getenv("QT_NO_QBLOCKS") == nullptr;
  const cudaStream_t sq = e.side4, su = e.side5;
  const size_t Q0 = J0 + 8;         // events: Y panel b done
  const size_t U0 = Q0 + npan + 2;  // events: block p updated with reflectors 0..p-2
  if (qblocks) {
    set_identity(e, qy, nc, k, k, sy);
  }

  // QT_PAIR_DEBUG=1 (eager calls only): timeline of the pair on stderr
  static const bool tdbg = std::getenv("QT_PAIR_DEBUG") != nullptr;
  static std::vector<cudaEvent_t> tev;
  std::vector<std::string> tname;
  auto stamp = [&](const std::string& nm, cudaStream_t st) {
    if (!tdbg) return;
    if (tev.size() <= tname.size()) {
      cudaEvent_t ev;
      QT_CUDA(cudaEventCreate(&ev));
      tev.push_back(ev);
    }
    QT_CUDA(cudaEventRecord(tev[tname.size()], st));
    tname.push_back(nm);
  };
  stamp("start", sx);
  bool wide_pending = false;
  long long last_wide = -1;
  for (long long p = 0; p < npan; ++p) {
    const long long j = p * NB;
    const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
    // ---- X: panel p (look-ahead as in qr_inplace)
    PanelArgs pa = base;
    pa.A = x + j * k + j;
    pa.lda = k;
    pa.mp = m - j;
    pa.nbp = nbp;
    pa.V = Vx + j * kp + p * NB;
    pa.ldv = kp;
    pa.T = Tx + p * NB * NB;
    launch_panel(e, pa, m - j, sx);
    stamp("Xpanel" + std::to_string(p), sx);
    // ---- theta side: C <- H_p^H C, then rows [j, j + nbp) of C are final
    QT_CUDA(cudaEventRecord(e.event(P0 + p), sx));
    QT_CUDA(cudaStreamWaitEvent(sa, e.event(P0 + p), 0));
    // rows [j, j + nbp) of H_p^H C are final first: publish them as block p
    // of Y^H before the rest of C is updated
    {
      // C <- (I - V T V^H)^H C: W = V^H C, then rows of block p (W2 = T^H W,
      // C_top -= V_top W2, published as block p of Y^H) in one kernel, then
      // the rest of C (C_rest -= V_rest W2)
      const long long mp = m - j;
      GemmDesc g;
      g.M = nbp; g.N = nc; g.K = mp;
      g.opA = Op::H; g.A = pa.V; g.lda = kp;
      g.B = c + j * nc; g.ldb = nc;
      g.C = CW; g.ldc = nc;
      zgemm(g, gs2, sa);
      stamp("thW" + std::to_string(p), sa);
      pair_top_kernel<<<static_cast<unsigned>(ceil_div(nc, NB)), dim3(NB, 8), 0, sa>>>(
          CW, pa.T, pa.V, kp, c + j * nc, nc, nbp, CW2, x, k, yh, j);
      QT_LAUNCHED();
      stamp("extract" + std::to_string(p), sa);
      QT_CUDA(cudaEventRecord(e.event(E0 + p), sa));
      if (mp > nbp) {
        GemmDesc g3;
        g3.M = mp - nbp; g3.N = nc; g3.K = nbp;
        g3.A = pa.V + nbp * kp; g3.lda = kp;
        g3.B = CW2; g3.ldb = nc;
        g3.C = c + (j + nbp) * nc; g3.ldc = nc;
        g3.alpha = -1.0; g3.beta = 1.0;
        zgemm(g3, gs2, sa);
        stamp("threst" + std::to_string(p), sa);
      }
    }
    // ---- X trailing update (look-ahead: next panel's columns on sx, the rest on sxw)
    const long long ntr = k - j - nbp;
    if (ntr > 0) {
      const long long nn = std::min<long long>(NB, ntr);
      if (p > 0 && wide_pending) QT_CUDA(cudaStreamWaitEvent(sx, e.event(2 * (p - 1) + 1), 0));
      if (ntr > nn) {
        QT_CUDA(cudaEventRecord(e.event(2 * p), sx));
        QT_CUDA(cudaStreamWaitEvent(sxw, e.event(2 * p), 0));
      }
      larfb_cluster(e, pa.V, kp, pa.T, x + j * k + j + nbp, k, m - j, nn, nbp, true, sx);
      stamp("Xnarrow" + std::to_string(p), sx);
      wide_pending = ntr > nn;
      if (wide_pending) {
        larfb_cluster(e, pa.V, kp, pa.T, x + j * k + j + nbp + nn, k, m - j, ntr - nn, nbp, true, sxw);
        stamp("Xwide" + std::to_string(p), sxw);
        QT_CUDA(cudaEventRecord(e.event(2 * p + 1), sxw));
        last_wide = p;
      }
    }
    // ---- Y^H: block p receives the reflectors of Y panels < p, then panel p
    // block p receives reflectors 0..p-2 on su (concurrently with Y panel
    // p-1, once that panel's predecessor exists), then H'_{p-1} on sy right
    // after Y panel p-1: the Y chain carries only narrow updates
    if (p >= 2) {
      QT_CUDA(cudaStreamWaitEvent(su, e.event(E0 + p), 0));
      QT_CUDA(cudaStreamWaitEvent(su, e.event(Q0 + p - 2), 0));
      if (!larfb_multi(Vy, kp, Ty, yh + j, k, nc, nbp, static_cast<int>(p - 1), k, su))
        throw Error(Err::internal, "qr_pair_pipelined: block update does not fit a cluster");
      QT_CUDA(cudaEventRecord(e.event(U0 + p), su));
      QT_CUDA(cudaStreamWaitEvent(sy, e.event(U0 + p), 0));
    } else {
      QT_CUDA(cudaStreamWaitEvent(sy, e.event(E0 + p), 0));
    }
    stamp("Ystart" + std::to_string(p), sy);
    if (p >= 1) {
      const long long jq = (p - 1) * NB;
      larfb_cluster(e, Vy + jq * kp + (p - 1) * NB, kp, Ty + (p - 1) * NB * NB, yh + jq * k + j, k, nc - jq, nbp, NB,
                    true, sy);
    }
    PanelArgs py = base;
    py.A = yh + j * k + j;
    py.lda = k;
    py.mp = nc - j;
    py.nbp = nbp;
    py.V = Vy + j * kp + p * NB;
    py.ldv = kp;
    py.T = Ty + p * NB * NB;
    stamp("Yupdate" + std::to_string(p), sy);
    launch_panel(e, py, nc - j, sy);
    stamp("Ypanel" + std::to_string(p), sy);
    QT_CUDA(cudaEventRecord(e.event(Q0 + p), sy));  // Y panel p done: V'_p, T'_p exist
    if (qblocks) {
      QT_CUDA(cudaStreamWaitEvent(sq, e.event(Q0 + p), 0));
      // gauge-fixed on write-back (the phases of its R' diagonal are final after Y panel p)
      if (!larfb_multi(Vy, kp, Ty, qy + j, k, nc, nbp, static_cast<int>(p + 1), k, sq, true, false, yh, k, j))
        throw Error(Err::internal, "qr_pair_pipelined: Q block does not fit a cluster");
      stamp("Qblock" + std::to_string(p), sq);
    }
  }
  // join the X side streams (R of X is not needed; its diagonal carries the gauge phases)
  if (last_wide >= 0) QT_CUDA(cudaStreamWaitEvent(sx, e.event(2 * last_wide + 1), 0));
  QT_CUDA(cudaEventRecord(e.event(J0 + 1), sa));
  QT_CUDA(cudaStreamWaitEvent(sx, e.event(J0 + 1), 0));
  if (qblocks) {  // join sq: every column block of Q formed
    QT_CUDA(cudaEventRecord(e.event(Q0 + npan), sq));
    QT_CUDA(cudaStreamWaitEvent(sy, e.event(Q0 + npan), 0));
  } else {
    // explicit thin Q of Y^H = H'_0 ... H'_{k-1} I[:, :k] (backward block reflectors) on sy
    set_identity(e, qy, nc, k, k, sy);
    for (long long p = npan - 1; p >= 0; --p) {
      const long long j = p * NB;
      const int nbp = static_cast<int>(std::min<long long>(NB, k - j));
      if (!larfb_cluster(e, Vy + j * kp + p * NB, kp, Ty + p * NB * NB, qy + j * k + j, k, nc - j, k - j, nbp,
                         false, sy))
        throw Error(Err::internal, "qr_pair_pipelined: block reflector does not fit a cluster");
    }
  }
  if (!qblocks) {
    gauge_q_kernel<<<grid_for(nc * k), 256, 0, sy>>>(yh, k, qy, k, nc, k);
    QT_LAUNCHED();
  }
  gauge_r_kernel<<<grid_for(k * k), 256, 0, sy>>>(yh, k, ry, k, k, k);
  QT_LAUNCHED();
  QT_CUDA(cudaEventRecord(e.event(J0 + 2), sy));
  QT_CUDA(cudaStreamWaitEvent(sx, e.event(J0 + 2), 0));
  stamp("end", sx);
  if (tdbg) {
    QT_CUDA(cudaStreamSynchronize(sx));
    std::fprintf(stderr, "qr_pair m=%lld k=%lld nc=%lld timeline (us from start):", m, k, nc);
    for (size_t i = 1; i < tname.size(); ++i) {
      float ms = 0.f;
      QT_CUDA(cudaEventElapsedTime(&ms, tev[0], tev[i]));
      std::fprintf(stderr, " %s=%.0f", tname[i].c_str(), ms * 1000.f);
    }
    std::fprintf(stderr, "\n");
  }
}

}  // namespace qt
