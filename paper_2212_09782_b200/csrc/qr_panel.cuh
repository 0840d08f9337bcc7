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

// 1/x: hardware approximation + two Newton steps (full precision; the IEEE
// division's ~114-cycle latency sits on the per-column critical path)
__device__ __forceinline__ double prcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// zlarfg on (alpha, ||x||^2): beta real, tau = 0 for an exactly-zero column
__device__ __forceinline__ Reflector make_reflector(double2 alpha, double xnorm2) {
  Reflector r;
  r.pad = 0.0;
  if (xnorm2 == 0.0 && alpha.y == 0.0) {
    r.tau = make_double2(0.0, 0.0);
    r.beta = alpha.x;
    r.scale = make_double2(0.0, 0.0);
  } else {
    const double nrm = sqrt(fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xnorm2)));
    r.beta = alpha.x >= 0.0 ? -nrm : nrm;
    const double2 den = make_double2(alpha.x - r.beta, alpha.y);
    // the two reciprocals are independent: their latencies overlap
    const double inv_b = prcp(r.beta);
    const double inv_dd = prcp(fma(den.x, den.x, den.y * den.y));
    r.tau = make_double2((r.beta - alpha.x) * inv_b, -alpha.y * inv_b);
    r.scale = make_double2(den.x * inv_dd, -den.y * inv_dd);
  }
  return r;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// bulk DSMEM push: `bytes` from local shared memory into a peer CTA's shared
// memory, completing transaction bytes on the peer's mbarrier
__device__ __forceinline__ void bulk_push(uint32_t remote_dst, const void* src, unsigned bytes, uint32_t remote_bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(remote_dst),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes), "r"(remote_bar)
      : "memory");
}


// Per column c the critical path is: CTA reduction of the partials (warp 0)
// -> one bulk DSMEM push per peer CTA -> mbarrier wait -> fixed-order combine
// and zlarfg (warp 0) -> one CTA barrier -> the fused row pass.  The row pass
// is lean: the active column x (zero on rows <= c) is broadcast from shared
// memory and every lane applies y_k -= x (scale conj(tau) w_k) with a zero
// coefficient on lanes k <= c, so rows need no per-row predicates; only the
// diagonal row (CTA 0, first two register rows) is special.  The reflector
// vectors stay UNSCALED in registers (v_l = scale_l x^(l)) -- the scale is
// folded into the T-factor terms at combine time and applied once at the end.
template <int RPW>
__global__ void __launch_bounds__(CL_THREADS, 1) panel_cluster_kernel(PanelArgs a) {
  constexpr int RPC = CL_WARPS * RPW;  // rows per CTA
  extern __shared__ __align__(16) double2 psm[];
  double2* colbuf = psm;                     // [2][RPC] active column (x of the pass, x1 of the next)
  double2* red = colbuf + 2 * RPC;           // [16][32]
  double2* recv = red + CL_WARPS * NB;       // [2][16][32] partials pushed by every CTA
  double2* rdiag = recv + 2 * 16 * NB;       // [2][32]    diagonal row pushed by CTA 0
  double2* drow = rdiag + 2 * NB;            // [2][32]    diagonal row staged by its owner warp
  double2* mine = drow + 2 * NB;             // [2][32]    this CTA's combined partials (push source)
  double2* ctws = mine + 2 * NB;             // [32]       conj(tau) w_k of this column
  double2* Ts = ctws + NB;                   // [32][32]   T factor (CTA 0)
  double2* Z = Ts + NB * NB;                 // [32][32]   z vectors of the T recurrence (CTA 0)
  double2* taus = Z + NB * NB;               // [32]
  double2* scales = taus + NB;               // [32]       reflector scales (CTA 0)
  Reflector* refl = reinterpret_cast<Reflector*>(scales + NB);   // (3 x double2)
  __shared__ uint64_t bars[2];  // per-column partial exchange

  const int w = threadIdx.x >> 5, k = threadIdx.x & 31;
  const unsigned rank = cluster_rank();
  const int CS = static_cast<int>(gridDim.x);
  const int r0 = static_cast<int>(rank) * RPC;
  const int nloc = max(0, min(RPC, static_cast<int>(a.mp) - r0));
  const int nbp = a.nbp;
  constexpr unsigned PUSH = NB * sizeof(double2);  // one 32-lane row of double2
  const unsigned bytes_per_col = static_cast<unsigned>(CS + 1) * PUSH;

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
    const int gr = r0 + lr;
    y[i] = (lr < nloc && k < nbp) ? a.A[(static_cast<long long>(gr)) * a.lda + k] : make_double2(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < 2 * 16 * NB; e += CL_THREADS) recv[e] = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int lr = w + CL_WARPS * i;
    const int gr = r0 + lr;
    if (k == 0) colbuf[lr] = gr > 0 ? y[i] : make_double2(0.0, 0.0);
    if (gr == 0) drow[k] = y[i];
  }
  fence_proxy_async_smem();
  cluster_sync_all();  // barriers armed and inboxes zeroed everywhere before any push

  // partials for column 0: p_k = sum_{r > 0} conj(x_r) y_rk
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < RPW; ++i) cfma_conj(acc, colbuf[w + CL_WARPS * i], y[i]);
  double2 my_scale = make_double2(0.0, 0.0);  // scale of the reflector of column k (set at pass k)

  for (int c = 0; c < nbp; ++c) {
    const int par = c & 1;
    const double2* xcol = colbuf + par * RPC;     // column c of every local row (zero on rows <= c)
    double2* ncol = colbuf + (par ^ 1) * RPC;     // column c+1 after this pass
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 8 + 0] = clock64();
    red[w * NB + k] = acc;
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
      mine[par * NB + k] = cadd(cadd(s0, s1), cadd(s2, s3));
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 8 + 1] = clock64();
    }
    // warps 0..CS-1 each push this CTA's partials (and, on CTA 0, the diagonal
    // row) to one peer: the DSMEM stores of the 16 targets issue in parallel
    if (w < CS) {
      asm volatile("bar.sync 1, %0;" ::"r"(CS * 32) : "memory");
      const uint32_t bar_r = cl_map(&bars[par], w);
      st_async_push(cl_map(&recv[(par * 16 + rank) * NB + k], w), mine[par * NB + k], bar_r);
      if (rank == 0) st_async_push(cl_map(&rdiag[par * NB + k], w), drow[par * NB + k], bar_r);
    }
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 8 + 2] = clock64();
    if (w == 0) {
      pmbar_wait(&bars[par], (c >> 1) & 1);
      if (k == 0 && c + 2 < nbp) pmbar_arm(&bars[par], bytes_per_col);
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 8 + 3] = clock64();
      // all 16 slots (those of absent CTAs stay zero): loads issue back to
      // back, then a fixed pairwise tree
      double2 v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = recv[(par * 16 + r) * NB + k];
#pragma unroll
      for (int h = 8; h >= 2; h >>= 1)
#pragma unroll
        for (int r = 0; r < h; ++r) v[r] = cadd(v[r], v[r + h]);
      const double2 sk = cadd(v[0], v[1]);  // p_k: s_k for k >= c, conj(h_k / conj(scale_k)) for k < c
      const double2 dk = rdiag[par * NB + k];
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 8 + 4] = clock64() + static_cast<long long>(sk.x * 0.0);
      const Reflector Rw = make_reflector(rdiag[par * NB + c], __shfl_sync(0xffffffffu, sk.x, c));
      if (k == 0) *refl = Rw;
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 8 + 5] = clock64() + static_cast<long long>(Rw.tau.x * 0.0);
      // conj(tau) w_k, w_k = a_ck + conj(scale) s_k (zero on lanes that keep their column)
      ctws[k] = (k > c && k < nbp) ? cmul(cconj(Rw.tau), cadd(dk, cmul(cconj(Rw.scale), sk)))
                                   : make_double2(0.0, 0.0);
      // inputs of the z vector of the T recurrence, formed after the loop
      // (off the per-column chain): row c and the partials of column c
      if (rank == 0) {
        Z[c * NB + k] = dk;
        Ts[c * NB + k] = sk;
        if (k == 0) scales[c] = Rw.scale;
      }
      if (a.dbg && rank == 0 && k == 0) a.dbg[c * 8 + 6] = clock64();
    }
    __syncthreads();
    const Reflector R = *refl;
    const double2 ctw = ctws[k];
    const double2 sctw = cmul(R.scale, ctw);
    if (k == c) my_scale = R.scale;
    if (rank == 0 && threadIdx.x == 0) taus[c] = R.tau;
    if (a.dbg && rank == 0 && threadIdx.x == 0) a.dbg[c * 8 + 7] = clock64();

    const int c1 = c + 1;
    // rows in chunks whose column-c loads issue back to back (the compiler
    // cannot hoist a load of xcol above a store to ncol: same array)
    constexpr int CH = RPW < 6 ? RPW : 5;
#pragma unroll
    for (int i0 = 0; i0 < RPW; i0 += CH) {
      double2 xs[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (i0 + j < RPW) xs[j] = xcol[w + CL_WARPS * (i0 + j)];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int i = i0 + j;
        if (i >= RPW) break;
        const int lr = w + CL_WARPS * i;
        const int gr = r0 + lr;
        cfms(y[i], xs[j], sctw);  // x = 0 on rows <= c: R rows are left alone
        if (i < 2 && gr == c) {   // the diagonal row (CTA 0 only)
          y[i] = csub(y[i], ctw);
          if (k == c) y[i] = make_double2(R.beta, 0.0);
        }
        if (i < 2) {  // rows < 32 exist only on CTA 0: x1 = 0 on rows <= c+1, stage the next diagonal row
          if (k == c1) ncol[lr] = gr > c1 ? y[i] : make_double2(0.0, 0.0);
          if (gr == c1) drow[(par ^ 1) * NB + k] = y[i];  // pushed at the top of pass c+1
        } else if (k == c1) {
          ncol[lr] = y[i];
        }
      }
    }
    __syncwarp();
    // partials of column c+1, two interleaved chains (fixed order)
    double2 acc1 = make_double2(0.0, 0.0);
    acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < RPW; ++i) cfma_conj((i & 1) ? acc1 : acc, ncol[w + CL_WARPS * i], y[i]);
    acc = cadd(acc, acc1);
  }
  // all pushes into every CTA have landed (each CTA waited for all columns);
  // one barrier before retiring so no bulk copy targets an exited CTA
  cluster_sync_all();

#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int lr = w + CL_WARPS * i;
    const long long gr = r0 + lr;
    if (lr < nloc && k < nbp) {
      const double2 v = gr > k ? cmul(my_scale, y[i]) : y[i];  // v = scale x^(k) below the diagonal
      a.A[gr * a.lda + k] = v;
      a.V[gr * a.ldv + k] = gr > k ? v : (gr == k ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0));
    } else if (lr < nloc) {
      a.V[gr * a.ldv + k] = make_double2(0.0, 0.0);  // full 32-wide rows (bulk-copied by larfb)
    }
  }
  if (rank != 0) return;
  // T factor (zlarft, forward columnwise) on CTA 0 from the Gram entries of
  // the reflectors, M[l][c] = v_l^H v_c (l < c; all scales are final):
  //   v_c,l = scale_l x^(l)_c,  h_l = conj(scale_l) conj(p_l),  M = conj(v_c,l) + scale_c h_l
  // stored transposed (Z[c][l] = M[l][c]), zero on and below the diagonal and
  // past the panel width
  for (int c = w; c < NB; c += CL_WARPS) {
    double2 m = make_double2(0.0, 0.0);
    if (c < nbp && k < c) {
      const double2 dk = Z[c * NB + k], sk = Ts[c * NB + k], scl = scales[c];
      m = cadd(cconj(cmul(my_scale, dk)), cmul(scl, cmul(cconj(my_scale), cconj(sk))));
    }
    Z[c * NB + k] = m;
  }
  for (int e = threadIdx.x; e < NB * NB; e += CL_THREADS) {
    const int i = e / NB, j = e % NB;
    Ts[e] = (i == j && i < nbp) ? taus[i] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // recursive doubling instead of 31 dependent column steps: the T of two
  // adjacent reflector blocks B1, B2 is [[T11, T12], [0, T22]] with
  // T12 = -T11 (V1^H V2) T22; five levels of two small products each
  double2* P = red;  // [16 pairs x b x b] <= 256 entries
  for (int b = 1; b < NB; b <<= 1) {
    const int bb = b * b, nout = (NB / (2 * b)) * bb;
    for (int e = threadIdx.x; e < nout; e += CL_THREADS) {  // P = M[B1, B2] T22
      const int q = e / bb, r = (e % bb) / b, c = e % b, s0 = 2 * b * q;
      double2 acc = make_double2(0.0, 0.0);
      for (int l = 0; l <= c; ++l)
        acc = cadd(acc, cmul(Z[(s0 + b + l) * NB + s0 + r], Ts[(s0 + b + l) * NB + s0 + b + c]));
      P[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nout; e += CL_THREADS) {  // T12 = -T11 P
      const int q = e / bb, r = (e % bb) / b, c = e % b, s0 = 2 * b * q;
      double2 acc = make_double2(0.0, 0.0);
      for (int l = r; l < b; ++l) acc = cadd(acc, cmul(Ts[(s0 + r) * NB + s0 + l], P[q * bb + l * b + c]));
      Ts[(s0 + r) * NB + s0 + b + c] = make_double2(-acc.x, -acc.y);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += CL_THREADS) a.T[e] = Ts[e];
}

constexpr size_t panel_cluster_smem(int rpw) {
  return (size_t(2 * CL_WARPS * rpw) + CL_WARPS * NB + 2 * 16 * NB + 6 * NB + NB + 2 * NB * NB + 2 * NB + 3) *
             sizeof(double2) +
         2 * 8;
}
