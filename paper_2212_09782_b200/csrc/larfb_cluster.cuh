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

__global__ void __launch_bounds__(LB_THREADS, 1)
    larfb_cluster_kernel(const double2* __restrict__ V, long long ldv, const double2* __restrict__ T, double2* A,
                         long long lda, int mp, int ncols, int nbp, int rpc, int use_th) {
  extern __shared__ __align__(16) double2 lsm[];
  double2* Vs = lsm;                        // [rpc][32]
  double2* As = Vs + rpc * NB;              // [rpc][32]
  double2* Wp = As + rpc * NB;              // [32][32] partial W, later W2
  double2* Wf = Wp + NB * NB;               // [32][32] reduced W (all-gathered)
  double2* Tp = Wf + NB * NB;               // [32][32] T'
  double2* rs = Tp + NB * NB;               // [CS][rows_owned][32] reduce-scatter inbox
  __shared__ uint64_t bars[2];

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const unsigned rank = cluster_rank();
  const int CS = static_cast<int>(gridDim.x);
  const int rows_owned = (NB + CS - 1) / CS;  // W rows i with i % CS == rank
  const int my_rows = (NB - static_cast<int>(rank) + CS - 1) / CS;
  const long long c0 = static_cast<long long>(blockIdx.y) * NB;
  const int nc = static_cast<int>(min(static_cast<long long>(NB), ncols - c0));
  const int r0 = static_cast<int>(rank) * rpc;
  const int nloc = max(0, min(rpc, mp - r0));

  if (tid == 0) {
    pmbar_init(&bars[0], 1);
    pmbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pmbar_arm(&bars[0], static_cast<unsigned>(CS * my_rows * NB * sizeof(double2)));
    pmbar_arm(&bars[1], static_cast<unsigned>(NB * NB * sizeof(double2)));
  }
  for (int e = tid; e < rpc * NB; e += LB_THREADS) {
    const int r = e / NB, c = e % NB;
    const bool ok = r < nloc;
    Vs[e] = (ok && c < nbp) ? V[static_cast<long long>(r0 + r) * ldv + c] : make_double2(0.0, 0.0);
    As[e] = (ok && c < nc) ? A[static_cast<long long>(r0 + r) * lda + c0 + c] : make_double2(0.0, 0.0);
  }
  for (int e = tid; e < NB * NB; e += LB_THREADS) {
    const int i = e / NB, k = e % NB;
    Tp[e] = (i < nbp && k < nbp) ? (use_th ? cconj(T[k * NB + i]) : T[i * NB + k]) : make_double2(0.0, 0.0);
  }
  cluster_sync_all();  // inputs staged, barriers armed everywhere before any push

  // partial W[i][j] = sum_r conj(V[r][i]) A[r][j]; thread: column j = lane, rows i = w + 8q
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int r = 0; r < nloc; ++r) {
    const double2 a = As[r * NB + lane];
#pragma unroll
    for (int q = 0; q < 4; ++q) cfma_conj(acc[q], Vs[r * NB + w + 8 * q], a);
  }
  // reduce-scatter: row i -> CTA i % CS, slot (source rank, i / CS)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = w + 8 * q;
    const unsigned owner = static_cast<unsigned>(i % CS);
    double2* slot = &rs[(static_cast<int>(rank) * rows_owned + i / CS) * NB + lane];
    st_async_push(cl_map(slot, owner), acc[q], cl_map(&bars[0], owner));
  }
  pmbar_wait(&bars[0], 0);
  // owned rows: fixed-order sum over sources, then all-gather into every Wf
  for (int e = tid; e < my_rows * NB; e += LB_THREADS) {
    const int li = e / NB, j = e % NB;
    const int i = static_cast<int>(rank) + li * CS;
    double2 s = make_double2(0.0, 0.0);
    for (int src = 0; src < CS; ++src) s = cadd(s, rs[(src * rows_owned + li) * NB + j]);
    for (int dst = 0; dst < CS; ++dst) st_async_push(cl_map(&Wf[i * NB + j], dst), s, cl_map(&bars[1], dst));
  }
  pmbar_wait(&bars[1], 0);
  // W2 = T' W  (into Wp)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = w + 8 * q;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < NB; ++k) s = cadd(s, cmul(Tp[i * NB + k], Wf[k * NB + lane]));
    Wp[i * NB + lane] = s;
  }
  __syncthreads();
  // A_r -= V_r W2: thread column j = lane, rows r = w + 8 t
  double2 w2[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) w2[k] = Wp[k * NB + lane];
  for (int r = w; r < nloc; r += LB_THREADS / 32) {
    double2 s = As[r * NB + lane];
#pragma unroll
    for (int k = 0; k < NB; ++k) cfms(s, Vs[r * NB + k], w2[k]);
    if (lane < nc) A[static_cast<long long>(r0 + r) * lda + c0 + lane] = s;
  }
  cluster_sync_all();  // no CTA retires while a peer may still push into it
}

constexpr size_t larfb_cluster_smem(int rpc, int cs) {
  return (size_t(2) * rpc * NB + 3 * NB * NB + size_t(cs) * ((NB + cs - 1) / cs) * NB) * sizeof(double2);
}

// A (mp x ncols, ld lda) <- (I - V T' V^H) A for a panel of nbp <= 32
// reflectors; returns false when the panel is too tall for one cluster.
bool larfb_cluster(Engine& e, const double2* V, long long ldv, const double2* T, double2* A, long long lda,
                   long long mp, long long ncols, int nbp, bool use_th) {
  static int max_cs = -1;
  if (max_cs < 0) {
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    QT_CUDA(cudaFuncSetAttribute(larfb_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(larfb_cluster_smem(LB_MAX_RPC, 1))));
    max_cs = 0;
    for (int cs : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1);
      cfg.blockDim = dim3(LB_THREADS);
      cfg.dynamicSmemBytes = larfb_cluster_smem(LB_MAX_RPC, 1);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, larfb_cluster_kernel, &cfg) == cudaSuccess && n >= 1) {
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs), static_cast<unsigned>(ceil_div(ncols, NB)));
  cfg.blockDim = dim3(LB_THREADS);
  cfg.dynamicSmemBytes = larfb_cluster_smem(static_cast<int>(rpc), static_cast<int>(cs));
  cfg.stream = e.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  QT_CUDA(cudaLaunchKernelEx(&cfg, larfb_cluster_kernel, V, ldv, T, A, lda, static_cast<int>(mp),
                             static_cast<int>(ncols), nbp, static_cast<int>(rpc), use_th ? 1 : 0));
  QT_LAUNCHED();
  return true;
}
