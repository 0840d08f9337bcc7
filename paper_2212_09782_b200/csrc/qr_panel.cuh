// Cluster-resident Householder panel factorization (included by
// householder.cu inside its anonymous namespace).
//
// The panel rows are spread over one thread-block cluster (<= 16 CTAs) and
// live in REGISTERS: warp w of CTA r owns rows r*rpc + w + 16 i (i < RPW) and
// lane k holds column k of those rows.  Only the active column travels
// through shared memory (one 16-byte store by its owner lane, one broadcast
// load per row).  Per column c:
//   1. the 16 row warps reduce their partial sums (||x||^2, x^H a_k and the
//      T-factor products v_l^H x); warp 0 pushes the 32 CTA partials into every
//      CTA of the cluster with st.async + mbarrier complete_tx, and the warp
//      owning row c on CTA 0 pushes the diagonal row -- no cluster barrier, no
//      global memory;
//   2. warp 0 waits on its CTA's mbarrier, combines the 16 partials in a fixed
//      order (bitwise deterministic) and forms the reflector once (zlarfg:
//      beta real, tau = 0 for an exactly-zero column);
//   3. one fused pass applies H_c^H (y -= x * scale conj(tau) w_k), stores
//      v_c = scale x, and accumulates the partial sums of column c+1.
// A 17th warp on CTA 0 builds the T factor column by column (zlarft) while the
// row warps run the fused pass.
constexpr int CL_WARPS = 16;                    // row warps
constexpr int CL_THREADS = CL_WARPS * 32;       // 2 warps per SM sub-partition -> 128 registers
constexpr int CL_MAX_RPW = 20;                  // rows per warp (registers)
constexpr int CL_MAX_ROWS = CL_WARPS * CL_MAX_RPW;

__device__ __forceinline__ uint32_t cl_map(const void* p, unsigned rank) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_push(uint32_t remote_addr, double2 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   remote_addr),
               "d"(v.x), "d"(v.y), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void pmbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void pmbar_arm(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void pmbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "PW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra PW_DONE;\n\t"
      "bra PW_WAIT;\n"
      "PW_DONE:\n\t}" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

// acc += conj(u) v
__device__ __forceinline__ void cfma_conj(double2& acc, double2 u, double2 v) {
  acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
  acc.y = fma(u.x, v.y, fma(-u.y, v.x, acc.y));
}
// y -= u v
__device__ __forceinline__ void cfms(double2& y, double2 u, double2 v) {
  y.x = fma(-u.x, v.x, fma(u.y, v.y, y.x));
  y.y = fma(-u.x, v.y, fma(-u.y, v.x, y.y));
}

struct Reflector {
  double2 tau, scale;
  double beta, pad;
};

// zlarfg on (alpha, ||x||^2): beta real, tau = 0 for an exactly-zero column
__device__ __forceinline__ Reflector make_reflector(double2 alpha, double xnorm2) {
  Reflector r;
  r.pad = 0.0;
  if (xnorm2 == 0.0 && alpha.y == 0.0) {
    r.tau = make_double2(0.0, 0.0);
    r.beta = alpha.x;
    r.scale = make_double2(0.0, 0.0);
  } else {
    const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2);
    r.beta = alpha.x >= 0.0 ? -nrm : nrm;
    // two reciprocals instead of four divisions (FP64 divide ~114 cycles on B200)
    const double inv_b = 1.0 / r.beta;
    r.tau = make_double2((r.beta - alpha.x) * inv_b, -alpha.y * inv_b);
    const double2 den = make_double2(alpha.x - r.beta, alpha.y);
    const double inv_dd = 1.0 / (den.x * den.x + den.y * den.y);
    r.scale = make_double2(den.x * inv_dd, -den.y * inv_dd);
  }
  return r;
}

template <int RPW>
__global__ void __launch_bounds__(CL_THREADS, 1) panel_cluster_kernel(PanelArgs a) {
  constexpr int RPC = CL_WARPS * RPW;  // rows per CTA
  extern __shared__ __align__(16) double2 psm[];
  double2* colbuf = psm;                     // [2][RPC] active column (x of the pass, x1 of the next)
  double2* red = colbuf + 2 * RPC;           // [16][32]
  double2* recv = red + CL_WARPS * NB;       // [2][16][32] partials pushed by every CTA
  double2* rdiag = recv + 2 * 16 * NB;       // [2][32]    diagonal row pushed by CTA 0
  double2* drow = rdiag + 2 * NB;            // [2][32]    diagonal row staged by its owner warp
  double2* Ts = drow + 2 * NB;               // [32][32]   T factor (CTA 0)
  double2* Z = Ts + NB * NB;                 // [32][32]   z vectors of the T recurrence (CTA 0)
  double2* taus = Z + NB * NB;               // [32]
  double2* ssum = taus + NB;                 // [32]       combined partials of this column
  Reflector* refl = reinterpret_cast<Reflector*>(ssum + NB);   // (3 x double2)
  uint64_t* bars = reinterpret_cast<uint64_t*>(ssum + NB + 3);  // [2]

  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  constexpr bool twarp = false;  // T is assembled after the column loop
  const unsigned rank = cluster_rank();
  const int CS = static_cast<int>(gridDim.x);
  const int r0 = static_cast<int>(rank) * RPC;
  const int nloc = max(0, min(RPC, static_cast<int>(a.mp) - r0));
  const int nbp = a.nbp;
  const unsigned bytes_per_col = static_cast<unsigned>((CS * NB + NB) * sizeof(double2));

  if (threadIdx.x == 0) {
    pmbar_init(&bars[0], 1);
    pmbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pmbar_arm(&bars[0], bytes_per_col);
    if (nbp > 1) pmbar_arm(&bars[1], bytes_per_col);
  }
  double2 y[RPW];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int lr = w + CL_WARPS * i;
    y[i] = (!twarp && lr < nloc && k < nbp) ? a.A[(static_cast<long long>(r0) + lr) * a.lda + k]
                                             : make_double2(0.0, 0.0);
    if (!twarp && k == 0) colbuf[lr] = y[i];
    if (r0 + lr == 0) drow[k] = y[i];
  }
  if (twarp)
    for (int e = k; e < NB * NB; e += 32) Ts[e] = make_double2(0.0, 0.0);
  cluster_sync_all();  // barriers initialised and armed everywhere before any push

  // partials for column 0 (rows > 0)
  double2 acc = make_double2(0.0, 0.0);
  if (!twarp) {
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int lr = w + CL_WARPS * i;
      if (lr < nloc && r0 + lr > 0) cfma_conj(acc, colbuf[lr], y[i]);
    }
  }

  for (int c = 0; c < nbp; ++c) {
    const int par = c & 1;
    const double2* xcol = colbuf + par * RPC;     // column c of every local row
    double2* ncol = colbuf + (par ^ 1) * RPC;     // column c+1 after this pass
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 4 + 0] = clock64();
    if (!twarp) red[w * NB + k] = acc;
    __syncthreads();
    if (w == 0) {
      // four independent chains, then a fixed-order combine
      double2 s0 = red[k], s1 = red[NB + k], s2 = red[2 * NB + k], s3 = red[3 * NB + k];
#pragma unroll
      for (int ww = 4; ww < CL_WARPS; ww += 4) {
        s0 = cadd(s0, red[ww * NB + k]);
        s1 = cadd(s1, red[(ww + 1) * NB + k]);
        s2 = cadd(s2, red[(ww + 2) * NB + k]);
        s3 = cadd(s3, red[(ww + 3) * NB + k]);
      }
      const double2 s = cadd(cadd(s0, s1), cadd(s2, s3));
      double2* slot = &recv[(par * 16 + rank) * NB + k];
      for (int r = 0; r < CS; ++r) st_async_push(cl_map(slot, r), s, cl_map(&bars[par], r));
    }
    if (rank == 0 && w == 1) {
      // diagonal row c, staged in drow by its owner warp during pass c-1
      const double2 dv = drow[par * NB + k];
      for (int r = 0; r < CS; ++r) st_async_push(cl_map(&rdiag[par * NB + k], r), dv, cl_map(&bars[par], r));
    }
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 4 + 1] = clock64();
    if (w == 0) {
      pmbar_wait(&bars[par], (c >> 1) & 1);
      if (k == 0 && c + 2 < nbp) pmbar_arm(&bars[par], bytes_per_col);
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 4 + 2] = clock64();
      double2 sk = make_double2(0.0, 0.0);
      for (int r = 0; r < CS; ++r) sk = cadd(sk, recv[(par * 16 + r) * NB + k]);
      ssum[k] = sk;
      const double sc = __shfl_sync(0xffffffffu, sk.x, c);
      const Reflector Rw = make_reflector(rdiag[par * NB + c], sc);
      if (k == 0) *refl = Rw;
      // z vector of the T recurrence (zlarft): z_l = -tau (conj(v_c,l) + scale h_l), l < c
      if (rank == 0)
        Z[c * NB + k] = (k < c) ? cmul(make_double2(-Rw.tau.x, -Rw.tau.y),
                                       cadd(cconj(rdiag[par * NB + k]), cmul(Rw.scale, sk)))
                                : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const Reflector R = *refl;
    const double2 sk = ssum[k];
    const double2 a_ck = rdiag[par * NB + k];

    if (rank == 0 && threadIdx.x == 0) taus[c] = R.tau;
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 4 + 3] = clock64();

    // fused pass: y_k -= x (scale conj(tau) w_k); v_c = scale x; partials of c+1
    const double2 ctw = cmul(cconj(R.tau), cadd(a_ck, cmul(cconj(R.scale), sk)));  // conj(tau) w_k
    const double2 sctw = cmul(R.scale, ctw);
    const bool upd = (k > c) && (k < nbp);
    const int c1 = c + 1;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int lr = w + CL_WARPS * i;
      const int gr = r0 + lr;
      if (lr < nloc && gr >= c) {  // warp-uniform
        if (gr == c) {
          if (upd) y[i] = csub(y[i], ctw);
          if (k == c) y[i] = make_double2(R.beta, 0.0);
        } else {
          const double2 x = xcol[lr];
          if (upd) cfms(y[i], x, sctw);
          if (k == c) y[i] = cmul(R.scale, x);
        }
        if (k == c1) ncol[lr] = y[i];
        if (gr == c1) drow[(par ^ 1) * NB + k] = y[i];  // next diagonal row (CTA 0 only)
      }
    }
    __syncwarp();
    acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int lr = w + CL_WARPS * i;
      // the diagonal row (and rows above c+1) take no part in the next partials
      if (lr < nloc && r0 + lr > c1) {
        const double2 x1 = ncol[lr];
        if (k >= c1)
          cfma_conj(acc, x1, y[i]);
        else
          cfma_conj(acc, y[i], x1);
      }
    }
  }
  // all pushes into every CTA have landed (each CTA waited for all columns);
  // one barrier before retiring so no st.async targets an exited CTA
  cluster_sync_all();

  if (!twarp) {
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int lr = w + CL_WARPS * i;
      const long long gr = r0 + lr;
      if (lr < nloc && k < nbp) {
        a.A[gr * a.lda + k] = y[i];
        a.V[gr * a.ldv + k] = gr > k ? y[i] : (gr == k ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0));
      }
    }
  }
  if (rank != 0) return;
  // zlarft (forward, columnwise) on CTA 0: T[c,c] = tau_c, T[0:c,c] = T[0:c,0:c] z_c;
  // each column's triangular product is spread over the 16 warps
  for (int e = threadIdx.x; e < NB * NB; e += CL_THREADS) Ts[e] = make_double2(0.0, 0.0);
  __syncthreads();
  if (threadIdx.x < nbp) Ts[threadIdx.x * NB + threadIdx.x] = taus[threadIdx.x];
  __syncthreads();
  for (int c = 1; c < nbp; ++c) {
    double2 p = make_double2(0.0, 0.0);
    for (int l = w; l < c; l += CL_WARPS)
      if (l >= k) p = cadd(p, cmul(Ts[k * NB + l], Z[c * NB + l]));
    red[w * NB + k] = p;
    __syncthreads();
    if (w == 0 && k < c) {
      double2 s = red[k];
#pragma unroll
      for (int ww = 1; ww < CL_WARPS; ++ww) s = cadd(s, red[ww * NB + k]);
      Ts[k * NB + c] = s;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += CL_THREADS) a.T[e] = Ts[e];
}

constexpr size_t panel_cluster_smem(int rpw) {
  return (size_t(2 * CL_WARPS * rpw) + CL_WARPS * NB + 2 * 16 * NB + 4 * NB + 2 * NB * NB + 2 * NB + 3) *
             sizeof(double2) +
         2 * 8;
}
