// Fused block-reflector application for short panels (included by
// householder.cu inside its anonymous namespace; uses qr_panel.cuh helpers).
//
//   A <- (I - V T' V^H) A,   T' = T^H (trailing update of zgeqrf, zlarfb 'C')
//                            T' = T   (explicit Q, zungqr / zlarfb 'N')
//
// replaces the four launches W = V^H A (split-K + reduce), W2 = T' W,
// A -= V W2 when the panel is short (m <= 16 x 128 rows): one thread-block
// cluster per 32-column block of A, the cluster's CTAs split the rows.  Each
// CTA forms its partial W = V_r^H A_r in shared memory; the partials are
// reduce-scattered (row i of W summed on CTA i % CS in a fixed source order)
// and all-gathered through distributed shared memory with st.async +
// mbarrier complete_tx; every CTA then applies A_r -= V_r (T' W) to its rows.
// One launch, no global scratch, bitwise deterministic.
constexpr int LB_THREADS = 256;
constexpr int LB_MAX_RPC = 128;

__device__ __forceinline__ void lb_cp16(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "r"(pred ? 16 : 0)
               : "memory");
}

// One cluster per CW-column block of A (CW = 32, 16 or 8: narrow blocks put
// more SMs on short updates); the cluster's CTAs split the rows (rpc each).
// Thread t owns column j = t % CW and W rows ib + RS q (RS = 256 / CW).
template <int CW>
__global__ void __launch_bounds__(LB_THREADS, 1)
    larfb_cluster_kernel(const double2* __restrict__ V, long long ldv, const double2* __restrict__ T, double2* A,
                         long long lda, int mp, int ncols, int nbp, int rpc, int use_th, long long* dbg) {
  constexpr int RS = LB_THREADS / CW;     // 8, 16, 32
  constexpr int EW = (NB * CW) / LB_THREADS;  // W entries per thread: 4, 2, 1
  const bool stamp = dbg && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0;
  if (stamp) dbg[0] = clock64();
  extern __shared__ __align__(16) double2 lsm[];
  double2* Vs = lsm;                 // [rpc][32]
  double2* As = Vs + rpc * NB;       // [rpc][CW]
  double2* Wp = As + rpc * CW;       // [32][CW] W2 = T' W
  double2* Wf = Wp + NB * CW;        // [32][CW] reduced W (all-gathered)
  double2* Tp = Wf + NB * CW;        // [32][32] T'
  double2* rs = Tp + NB * NB;        // [CS][rows_owned][CW] reduce-scatter inbox
  __shared__ uint64_t bars[2];       // reduce-scatter, all-gather

  const int tid = threadIdx.x, j = tid % CW, ib = tid / CW;
  const unsigned rank = cluster_rank();
  const int CS = static_cast<int>(gridDim.x);
  const int rows_owned = (NB + CS - 1) / CS;  // W rows i with i % CS == rank
  const int my_rows = (NB - static_cast<int>(rank) + CS - 1) / CS;
  const long long c0 = static_cast<long long>(blockIdx.y) * CW;
  const int nc = static_cast<int>(min(static_cast<long long>(CW), ncols - c0));
  const int r0 = static_cast<int>(rank) * rpc;
  const int nloc = max(0, min(rpc, mp - r0));

  if (tid == 0) {
    pmbar_init(&bars[0], 1);
    pmbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pmbar_arm(&bars[0], static_cast<unsigned>(CS * my_rows * CW * sizeof(double2)));
    pmbar_arm(&bars[1], static_cast<unsigned>(NB * CW * sizeof(double2)));
  }
  // stage V rows (full 32-wide, zero-padded by the panel) and the A row
  // slices with asynchronous 16-byte copies, all in flight at once; zero-fill
  // past the panel and past A's edge
  for (int e = tid; e < rpc * NB; e += LB_THREADS) {
    const int r = e / NB, c = e % NB;
    const bool ok = r < nloc;
    lb_cp16(&Vs[e], ok ? &V[static_cast<long long>(r0 + r) * ldv + c] : V, ok);
  }
  for (int e = tid; e < rpc * CW; e += LB_THREADS) {
    const int r = e / CW, c = e % CW;
    const bool ok = r < nloc && c < nc;
    lb_cp16(&As[e], ok ? &A[static_cast<long long>(r0 + r) * lda + c0 + c] : A, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = tid; e < NB * NB; e += LB_THREADS) {
    const int i = e / NB, k = e % NB;
    Tp[e] = (i < nbp && k < nbp) ? (use_th ? cconj(T[k * NB + i]) : T[i * NB + k]) : make_double2(0.0, 0.0);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (stamp) dbg[1] = clock64();
  cluster_sync_all();  // inputs staged, barriers armed everywhere before any push
  if (stamp) dbg[2] = clock64();

  // partial W[i][j] = sum_r conj(V[r][i]) A[r][j] over the zero-padded rows
  // (rpc even), two interleaved chains per entry
  double2 acc[EW];
  {
    double2 a2[EW][2];
#pragma unroll
    for (int q = 0; q < EW; ++q) a2[q][0] = a2[q][1] = make_double2(0.0, 0.0);
#pragma unroll 2
    for (int r = 0; r < rpc; r += 2) {
      const double2 a0 = As[r * CW + j], a1 = As[(r + 1) * CW + j];
#pragma unroll
      for (int q = 0; q < EW; ++q) {
        cfma_conj(a2[q][0], Vs[r * NB + ib + RS * q], a0);
        cfma_conj(a2[q][1], Vs[(r + 1) * NB + ib + RS * q], a1);
      }
    }
#pragma unroll
    for (int q = 0; q < EW; ++q) acc[q] = cadd(a2[q][0], a2[q][1]);
  }
  if (stamp) dbg[3] = clock64() + static_cast<long long>(acc[0].x * 0.0);
  // reduce-scatter: row i -> CTA i % CS, slot (source rank, i / CS)
#pragma unroll
  for (int q = 0; q < EW; ++q) {
    const int i = ib + RS * q;
    const unsigned owner = static_cast<unsigned>(i % CS);
    double2* slot = &rs[(static_cast<int>(rank) * rows_owned + i / CS) * CW + j];
    st_async_push(cl_map(slot, owner), acc[q], cl_map(&bars[0], owner));
  }
  pmbar_wait(&bars[0], 0);
  if (stamp) dbg[4] = clock64();
  // owned rows: fixed-order sum over sources, then the all-gather; threads
  // split as (entry, group of destinations)
  {
    const int nent = my_rows * CW;
    const int groups = max(1, min(CS, LB_THREADS / max(1, nent)));
    for (int e = tid; e < nent * groups; e += LB_THREADS) {
      const int ent = e / groups, g = e % groups;
      const int li = ent / CW, jj = ent % CW;
      const int i = static_cast<int>(rank) + li * CS;
      double2 s = make_double2(0.0, 0.0);
      for (int src = 0; src < CS; ++src) s = cadd(s, rs[(src * rows_owned + li) * CW + jj]);
      for (int dst = g; dst < CS; dst += groups)
        st_async_push(cl_map(&Wf[i * CW + jj], dst), s, cl_map(&bars[1], dst));
    }
  }
  pmbar_wait(&bars[1], 0);
  if (stamp) dbg[5] = clock64();
  // W2 = T' W  (into Wp), two chains per entry
#pragma unroll
  for (int q = 0; q < EW; ++q) {
    const int i = ib + RS * q;
    double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
#pragma unroll 8
    for (int k = 0; k < NB; k += 2) {
      s0 = cadd(s0, cmul(Tp[i * NB + k], Wf[k * CW + j]));
      s1 = cadd(s1, cmul(Tp[i * NB + k + 1], Wf[(k + 1) * CW + j]));
    }
    Wp[i * CW + j] = cadd(s0, s1);
  }
  __syncthreads();
  if (stamp) dbg[6] = clock64();
  // A_r -= V_r W2: rows r = ib + RS t, column j, two chains per row
  double2 w2[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) w2[k] = Wp[k * CW + j];
#pragma unroll 2
  for (int r = ib; r < nloc; r += RS) {
    double2 s0 = As[r * CW + j], s1 = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < NB; k += 2) {
      cfms(s0, Vs[r * NB + k], w2[k]);
      cfms(s1, Vs[r * NB + k + 1], w2[k + 1]);
    }
    if (j < nc) A[static_cast<long long>(r0 + r) * lda + c0 + j] = cadd(s0, s1);
  }
  if (stamp) dbg[7] = clock64();
  cluster_sync_all();  // no CTA retires while a peer may still push into it
  if (stamp) dbg[8] = clock64();
}

constexpr size_t larfb_cluster_smem(int rpc, int cs, int cw) {
  return (size_t(rpc) * (NB + cw) + 2 * NB * cw + NB * NB + size_t(cs) * ((NB + cs - 1) / cs) * cw) * sizeof(double2);
}

template <int CW>
void larfb_launch(cudaLaunchConfig_t& cfg, const double2* V, long long ldv, const double2* T, double2* A,
                  long long lda, long long mp, long long ncols, int nbp, long long rpc, bool use_th, long long* dbg) {
  static bool attr = false;
  if (!attr) {
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<CW>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_cluster_smem(LB_MAX_RPC, 16, 32))));
    attr = true;
  }
  QT_CUDA(cudaLaunchKernelEx(&cfg, larfb_cluster_kernel<CW>, V, ldv, T, A, lda, static_cast<int>(mp),
                             static_cast<int>(ncols), nbp, static_cast<int>(rpc), use_th ? 1 : 0, dbg));
}

// A (mp x ncols, ld lda) <- (I - V T' V^H) A for a panel of nbp <= 32
// reflectors; returns false when the panel is too tall for one cluster.
bool larfb_cluster(Engine& e, const double2* V, long long ldv, const double2* T, double2* A, long long lda,
                   long long mp, long long ncols, int nbp, bool use_th) {
  static int max_cs = -1;
  if (max_cs < 0) {
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_cluster_smem(LB_MAX_RPC, 16, 32))));
    max_cs = 0;
    for (int cs : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1);
      cfg.blockDim = dim3(LB_THREADS);
      cfg.dynamicSmemBytes = larfb_cluster_smem(LB_MAX_RPC, cs, 32);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, larfb_cluster_kernel<32>, &cfg) == cudaSuccess && n >= 1) {
        max_cs = cs;
        break;
      }
      cudaGetLastError();
    }
  }
  static const bool disabled = std::getenv("QT_NO_LARFB_CLUSTER") != nullptr;
  if (disabled || max_cs == 0 || ncols <= 0) return ncols <= 0 && !disabled && max_cs > 0;
  long long rpc = std::max<long long>(8, ceil_div(mp, max_cs));
  rpc = ceil_div(rpc, 8) * 8;
  if (rpc > LB_MAX_RPC) return false;
  const long long cs = ceil_div(mp, rpc);
  // narrowest column block that keeps <= 8 clusters (one per GPC) in flight
  int cw = 32;
  if (ceil_div(ncols, 8) <= 8)
    cw = 8;
  else if (ceil_div(ncols, 16) <= 8)
    cw = 16;
  static const bool dbg_on = std::getenv("QT_LARFB_DEBUG") != nullptr;
  static long long* dbg = nullptr;
  if (dbg_on && !dbg) QT_CUDA(cudaMalloc(&dbg, 16 * sizeof(long long)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs), static_cast<unsigned>(ceil_div(ncols, cw)));
  cfg.blockDim = dim3(LB_THREADS);
  cfg.dynamicSmemBytes = larfb_cluster_smem(static_cast<int>(rpc), static_cast<int>(cs), cw);
  cfg.stream = e.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cw == 8)
    larfb_launch<8>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  else if (cw == 16)
    larfb_launch<16>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  else
    larfb_launch<32>(cfg, V, ldv, T, A, lda, mp, ncols, nbp, rpc, use_th, dbg);
  QT_LAUNCHED();
  if (dbg) {  // QT_LARFB_DEBUG=1: phase timings of CTA (0,0) on stderr
    long long h[9];
    QT_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, e.stream));
    QT_CUDA(cudaStreamSynchronize(e.stream));
    std::fprintf(stderr,
                 "larfb mp=%lld ncols=%lld cs=%lld rpc=%lld cw=%d cycles: stage %lld csync %lld W %lld rs %lld ag %lld "
                 "W2 %lld upd %lld exit %lld\n",
                 mp, ncols, cs, rpc, cw, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4],
                 h[6] - h[5], h[7] - h[6], h[8] - h[7]);
  }
  return true;
}
