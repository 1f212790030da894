// C ABI of libqcpgrad (include/qcpgrad.h): batch preparation, jvp / vjp
// pipelines and the LSMR driver loop.
//
// Pipelines (reference solution_map.py:325-385):
//   jvp: rhs = -D_theta Q(Pi z)[dtheta]/|z_N| -> LSMR(F, rhs) -> D phi(z)[dz]
//   vjp: dz = D phi(z)'[delta] -> LSMR(F', -dz) -> D_theta Q(Pi z)'[w] on patterns
// The loop runs in CUDA graphs of 4/16/64 iterations; every kernel reads a
// per-problem active flag so converged problems cost no memory traffic.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "operator.h"

namespace qg {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(int, const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
void count_launch(int n) { g_launches += n; }

cudaStream_t &alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

void *pinned_staging(size_t bytes, int slot) {
  struct Buf {
    void *p = nullptr;
    size_t n = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local Buf bufs[4];
  Buf &b = bufs[slot];
  if (bytes > b.n) {
    if (b.p) QG_CUDA(cudaFreeHost(b.p));
    b.p = nullptr;
    b.n = 0;
    QG_CUDA(cudaMallocHost(&b.p, bytes));
    b.n = bytes;
  }
  return b.p;
}

void init_pool() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
}

void Workspace::release() {
  dev_free(u); dev_free(v); dev_free(h); dev_free(hb); dev_free(x);
  dev_free(dpu); dev_free(dpv); dev_free(tY); dev_free(tY2); dev_free(part);
  dev_free(st); dev_free(d_nactive); dev_free(d_claim); dev_free(d_loop); dev_free(part2); dev_free(df); dev_free(rk1);
  h_nactive = nullptr;  // thread-local pinned word, owned by pinned_word()
}

// Captured (not instantiated) LSMR graphs per handle, keyed by (jvp, iters).
struct GraphCache {
  std::map<std::pair<int, int>, cudaGraph_t> graph;
  ~GraphCache() {
    for (auto &kv : graph) cudaGraphDestroy(kv.second);
  }
};
// One executable graph per (stream, jvp, iters) shared by all handles used
// on that stream: switching handles re-points its kernel nodes with
// cudaGraphExecUpdate (same topology, new arguments / grid sizes) instead of
// re-instantiating -- a new batch per training step pays one capture, not an
// instantiation.  Launches of one exec are serialised by CUDA, so keying by
// stream keeps independent streams (host threads) concurrent.
struct SharedExec {
  cudaGraphExec_t exec = nullptr;
  const Handle *owner = nullptr;
};
using ExecKey = std::tuple<cudaStream_t, int, int>;
static std::map<const Handle *, GraphCache *> g_graphs;
static std::map<ExecKey, SharedExec> g_exec;
static std::mutex g_graph_mu;

void Handle::loop_events() {
  if (!ev_loop[0]) {
    QG_CUDA(cudaEventCreate(&ev_loop[0]));
    QG_CUDA(cudaEventCreate(&ev_loop[1]));
  }
}

Handle::~Handle() {
  if (ev_loop[0]) cudaEventDestroy(ev_loop[0]);
  if (ev_loop[1]) cudaEventDestroy(ev_loop[1]);
  P.release(); Pc.release(); A.release(); AT.release();
  sP.release(); sAT.release(); sA.release();
  dev_free(x_rowof); dev_free(y_rowof);
  dev_free(c16P); dev_free(c16AT); dev_free(c16A); dev_free(eng_blob); dev_free(eng_prof);
  dev_free(d_xunits); dev_free(d_ft_order); dev_free(d_xoff); dev_free(d_yoff); dev_free(d_xunit_ptr); dev_free(d_yunit_ptr);
  dev_free(q); dev_free(b); dev_free(xbar); dev_free(ybar); dev_free(sbar); dev_free(Pxbar); dev_free(emb);
  dev_free(xred); dev_free(psum); dev_free(d_iota);
  ws.release();
  std::lock_guard<std::mutex> g(g_graph_mu);
  auto it = g_graphs.find(this);
  if (it != g_graphs.end()) {
    delete it->second;
    g_graphs.erase(it);
  }
  for (auto &kv : g_exec)
    if (kv.second.owner == this) kv.second.owner = nullptr;  // must be re-pointed before next use
}

// ------------------------------------------------------------ create ----
// QG_TRACE: per-stage wall time of the batch preparation (syncs the stream at
// every point; diagnostics only).  what == nullptr resets the clock.
void trace_point(const char *what, cudaStream_t st) {
  static const bool on = std::getenv("QG_TRACE") != nullptr;
  static thread_local std::chrono::steady_clock::time_point t0;
  if (!on) return;
  cudaStreamSynchronize(st);
  const auto t1 = std::chrono::steady_clock::now();
  if (what) std::fprintf(stderr, "[qg] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
  t0 = t1;
}

struct Tracer {
  cudaStream_t st;
  explicit Tracer(cudaStream_t s) : st(s) { trace_point(nullptr, st); }
  void operator()(const char *what) { trace_point(what, st); }
};

// The deferred-finalize loop (kFeatDF) is wanted for one problem, no row
// partition, whose
// operator step streams >= 1e5 stored entries (P, A', A): there the SpMV
// hides CTA 0's finalize (c3: 70.5 -> 47.6 us per LSMR iteration; c2 with
// 1024-entry units: 35.3 -> 30.0).  QG_DEFER_FIN=0|1 forces it off / on
// (where eligible).
static bool defer_fin_intent(const Handle &H, const qg_batch_desc &d) {
  if (H.B != 1 || H.comm) return false;
  const char *e = std::getenv("QG_DEFER_FIN");
  if (e) return std::atoi(e) != 0;
  return H.noffP[1] + 2 * H.noffA[1] >= 100000;
}

static void build_handle(Handle &H, const qg_batch_desc &d, cudaStream_t st) {
  NvtxRange nv("qg:prepare");
  Tracer trace(st);
  const int B = (int)d.nprob;
  if (B <= 0) throw Error{QG_ERR_VALIDATION, "batch must hold at least one problem"};
  H.B = B;
  H.n.assign(d.n, d.n + B);
  H.m.assign(d.m, d.m + B);
  H.nnzP.assign(d.P_nnz, d.P_nnz + B);
  H.nnzA.assign(d.A_nnz, d.A_nnz + B);
  H.xoff.assign(B + 1, 0);
  H.yoff.assign(B + 1, 0);
  H.noffP.assign(B + 1, 0);
  H.noffA.assign(B + 1, 0);
  for (int p = 0; p < B; ++p) {
    if (H.n[p] < 0 || H.m[p] < 0) throw Error{QG_ERR_VALIDATION, "negative problem dimension"};
    H.xoff[p + 1] = H.xoff[p] + H.n[p];
    H.yoff[p + 1] = H.yoff[p] + H.m[p];
    H.noffP[p + 1] = H.noffP[p] + H.nnzP[p];
    H.noffA[p + 1] = H.noffA[p] + H.nnzA[p];
  }
  H.NX = H.xoff[B];
  H.NY = H.yoff[B];
  H.NE = H.NX + H.NY + B;

  // sparse structures
  CscBatch cp{d.P_colptr, d.P_rowidx, d.P_vals, H.n, H.n, H.nnzP};
  csc_to_csr(cp, H.P, &H.Pc, true, st);
  trace("transpose P");
  CscBatch ca{d.A_colptr, d.A_rowidx, d.A_vals, H.n, H.m, H.nnzA};
  csc_to_csr(ca, H.A, &H.AT, true, st);
  H.AT.val = dev_alloc<double>(H.noffA[B]);
  if (H.noffA[B])
    QG_CUDA(cudaMemcpyAsync(H.AT.val, d.A_vals, sizeof(double) * H.noffA[B], cudaMemcpyDeviceToDevice, st));
  trace("transpose A");

  // Unit sizes from host-known totals (the descriptor's nnz counts): the cone
  // table's host passes then run while the transposes above are still on the
  // GPU, before the row-pointer download synchronises the stream.
  const int64_t nnzX = H.noffP[B] + H.noffA[B], nnzY = H.noffA[B];
  // aim for >= 4 CTAs per SM when the batch is large enough, 2k..16k entries per unit
  const int64_t total = nnzX + nnzY + H.NX + H.NY;
  // small problems get small units (all SMs busy, short per-warp chains),
  // large batches amortise per-CTA work over up to 16k entries
  // (a single problem caps units at 8k entries: c5b's dense LASSO rows run
  // 542 -> 502 us per LSMR iteration with 4k..10k-entry units vs 16k)
  const int64_t cap_nnz = B == 1 ? 8192 : 16384;
  int64_t target_nnz = std::max<int64_t>(256, std::min<int64_t>(cap_nnz, total / (8 * 148) + 1));
  // a single problem on the deferred-finalize loop (below): CTA 0 sums 4
  // partials per unit, so units of >= 1024 entries (c2: 914 -> ~230 units,
  // 35.3 -> 30.0 us per LSMR iteration)
  const bool df_intent = defer_fin_intent(H, d);
  if (df_intent) target_nnz = std::max<int64_t>(target_nnz, 1024);
  if (const char *e = std::getenv("QG_TARGET_NNZ")) target_nnz = std::max<int64_t>(64, std::atoll(e));  // A/B
  const double avg_y = H.NY ? (double)nnzY / H.NY + 1.0 : 1.0;
  const int64_t target_rows_y = std::max<int64_t>(8, std::min<int64_t>(4096, (int64_t)(target_nnz / avg_y)));

  // cones and Y units
  H.cones.build(d.blocks, d.nblocks, H.yoff, target_rows_y, st);
  trace("cone table");

  // row-length statistics for the unit partition (pinned staging: DMA speed)
  int32_t *rpP = static_cast<int32_t *>(pinned_staging(sizeof(int32_t) * (2 * (H.NX + 1) + H.NY + 1), 0));
  int32_t *rpAT = rpP + (H.NX + 1), *rpA = rpAT + (H.NX + 1);
  QG_CUDA(cudaMemcpyAsync(rpP, H.P.rp, sizeof(int32_t) * (H.NX + 1), cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaMemcpyAsync(rpAT, H.AT.rp, sizeof(int32_t) * (H.NX + 1), cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaMemcpyAsync(rpA, H.A.rp, sizeof(int32_t) * (H.NY + 1), cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  trace("rowptr D2H");
  if ((int64_t)rpP[H.NX] + rpAT[H.NX] != nnzX || rpA[H.NY] != nnzY)
    throw Error{QG_ERR_VALIDATION, "sparse structure does not match the declared nnz counts"};

  // X units: nnz-balanced row ranges within each problem (problems in
  // parallel host chunks, concatenated in problem order)
  H.xunit_ptr.assign(B + 1, 0);
  {
    const int64_t nchunk = std::min<int64_t>(B, 64);
    std::vector<std::vector<Unit>> part(nchunk);
    host_parallel(nchunk, 1, [&](int64_t c0, int64_t c1) {
      for (int64_t c = c0; c < c1; ++c) {
        std::vector<Unit> &out = part[c];
        for (int p = (int)(B * c / nchunk); p < (int)(B * (c + 1) / nchunk); ++p) {
          H.xunit_ptr[p + 1] = 0;
          int64_t r = H.xoff[p];
          const int64_t end = H.xoff[p + 1];
          while (r < end) {
            int64_t e = r, w = 0;
            while (e < end && (e == r || (w < target_nnz && e - r < 4096))) {
              w += (int64_t)(rpP[e + 1] - rpP[e]) + (rpAT[e + 1] - rpAT[e]) + 1;
              ++e;
            }
            out.push_back(Unit{p, (int32_t)r, (int32_t)e, 0, 0, CLS_ELEM});
            ++H.xunit_ptr[p + 1];
            r = e;
          }
        }
      }
    });
    for (int p = 0; p < B; ++p) H.xunit_ptr[p + 1] += H.xunit_ptr[p];
    H.xunits.reserve(H.xunit_ptr[B]);
    for (auto &v : part) H.xunits.insert(H.xunits.end(), v.begin(), v.end());
  }
  H.d_xunits = dev_alloc<Unit>(H.xunits.size());  // uploaded by build_sell with the modes
  trace("x units");

  H.engine = engine_candidate(H);
  build_sell(H, rpP, rpAT, rpA, H.engine, st);
  H.engine = H.engine && engine_units_ok(H);
  trace("sell layout");
  H.d_xoff = dev_alloc<int64_t>(B + 1);
  H.d_yoff = dev_alloc<int64_t>(B + 1);
  QG_CUDA(cudaMemcpyAsync(H.d_xoff, H.xoff.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(H.d_yoff, H.yoff.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
  H.d_xunit_ptr = dev_alloc<int64_t>(B + 1);
  H.d_yunit_ptr = dev_alloc<int64_t>(B + 1);
  QG_CUDA(cudaMemcpyAsync(H.d_xunit_ptr, H.xunit_ptr.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(H.d_yunit_ptr, H.cones.unit_ptr.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
  if (H.engine) {
    build_engine_layout(H, st);
    trace("engine layout");
  }
  if (H.cones.max_psd_order > 0) {
    // F' launch order: PSD units first (k_step), then every other unit
    std::vector<int32_t> order;
    order.reserve(H.nxu() + H.nyu());
    for (int u = 0; u < H.nyu(); ++u)
      if (H.cones.units[u].cls == CLS_PSD) order.push_back(H.nxu() + u);
    H.n_psd_units = (int)order.size();
    const char *split_env = std::getenv("QG_PSD_SPLIT");
    H.psd_split = !split_env || std::atoi(split_env) != 0;
    for (int u = 0; u < H.nxu(); ++u) order.push_back(u);
    for (int u = 0; u < H.nyu(); ++u)
      if (H.cones.units[u].cls != CLS_PSD) order.push_back(H.nxu() + u);
    H.d_ft_order = dev_alloc<int32_t>(order.size());
    QG_CUDA(cudaMemcpyAsync(H.d_ft_order, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, st));
    QG_CUDA(cudaStreamSynchronize(st));  // host vector
  }

  // problem vectors
  H.q = dev_alloc<double>(H.NX);
  H.b = dev_alloc<double>(H.NY);
  H.xbar = dev_alloc<double>(H.NX);
  H.ybar = dev_alloc<double>(H.NY);
  H.sbar = dev_alloc<double>(H.NY);
  H.Pxbar = dev_alloc<double>(H.NX);
  H.emb = dev_alloc<Embed>(B);
  if (H.NX) {
    QG_CUDA(cudaMemcpyAsync(H.q, d.q, sizeof(double) * H.NX, cudaMemcpyDeviceToDevice, st));
    QG_CUDA(cudaMemcpyAsync(H.xbar, d.x, sizeof(double) * H.NX, cudaMemcpyDeviceToDevice, st));
  }
  if (H.NY) QG_CUDA(cudaMemcpyAsync(H.b, d.b, sizeof(double) * H.NY, cudaMemcpyDeviceToDevice, st));

  // workspace
  Workspace &W = H.ws;
  W.u = dev_alloc<double>(H.NE); W.v = dev_alloc<double>(H.NE); W.h = dev_alloc<double>(H.NE);
  W.hb = dev_alloc<double>(H.NE); W.x = dev_alloc<double>(H.NE);
  W.dpu = dev_alloc<double>(H.NY); W.dpv = dev_alloc<double>(H.NY);
  W.tY = dev_alloc<double>(H.NY); W.tY2 = dev_alloc<double>(H.NY);
  W.part = dev_alloc<double>((size_t)(H.nxu() + H.nyu() + 1) * kSlots);
  W.st = dev_alloc<Lsmr>(B);
  W.d_nactive = dev_alloc<int>(1);
  W.d_claim = dev_alloc<int>(1);
  W.d_loop = dev_alloc<long long>(2);
  W.h_nactive = nullptr;
  // deferred finalize (kFeatDF): one problem on the graph loop, no PSD blocks
  // (their F' units run as a second kernel), no row partition; the unit rows
  // are staged in shared memory (<= 2048 rows: 32 KB).  QG_DEFER_FIN=0: the
  // finalize kernels of round 1 (A/B).
  {
    for (const Unit &u : H.xunits) H.max_unit_rows = std::max(H.max_unit_rows, u.row1 - u.row0);
    for (const Unit &u : H.cones.units) H.max_unit_rows = std::max(H.max_unit_rows, u.row1 - u.row0);
    // <= 4096 work units: CTA 0 sums 4 partials per unit (c5b's 5004+ units:
    // neutral)
    // (no CTA-per-row units: that path is not exercised by any eligible config)
    // PSD blocks: only with their F' units in k_step_psd, and then only the F
    // step defers (mixed loop: the F' step is the split launch, its finalize
    // runs in the next F step's CTA 0, the F step's own in a k_fin_cta)
    const bool psd = H.cones.max_psd_order > 0;
    H.defer_fin = defer_fin_intent(H, d) && !H.engine && !H.has_wide && H.nxu() + H.nyu() > 0 &&
                  H.nxu() + H.nyu() <= 4096 && H.max_unit_rows <= 2048 && (!psd || psd_split(H));
    H.df_mixed = H.defer_fin && psd;
    if (H.defer_fin) {
      W.part2 = dev_alloc<double>((size_t)(H.nxu() + H.nyu() + 1) * kSlots);
      W.df = dev_alloc<DfCtl>(1);
      QG_CUDA(cudaMemsetAsync(W.df, 0, sizeof(DfCtl), st));
    }
  }
  if (H.comm) {
    H.xred = dev_alloc<double>(H.NX);
    H.psum = dev_alloc<double>(2 * (size_t)B * kSlots);
    std::vector<int64_t> iota(B + 1);
    for (int p = 0; p <= B; ++p) iota[p] = p;
    H.d_iota = dev_alloc<int64_t>(B + 1);
    QG_CUDA(cudaMemcpyAsync(H.d_iota, iota.data(), sizeof(int64_t) * (B + 1), cudaMemcpyHostToDevice, st));
    QG_CUDA(cudaStreamSynchronize(st));  // iota is a stack vector
  }
  trace("workspace");

  // embedding: z = (x, y - s, 1); Pi z; D Pi prep; P xbar, xbar'P xbar
  double *zmid = H.cones.d_zmid;
  launch_embed_prep(H, d.x, d.y, d.s, zmid, st);
  H.cones.prepare(zmid, H.ybar, 1, true, st);
  H.cones.check_errors(st);
  trace("cone prep");
  Mats M = make_mats(H);
  launch_embed_consts(H, M, W.part, st);
  trace("embedding consts");
}

}  // namespace qg

// sbar = ybar - zmid (solution_map.py:223): tiny kernel kept local
namespace qg {
__global__ void k_sub(const double *a, const double *b, double *out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}
static void launch_sub(const double *a, const double *b, double *out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_sub<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, b, out, n);
  QG_LAUNCHED();
}

// ----------------------------------------------------------- LSMR loop --
// Deferred finalize (kFeatDF launches) for this handle's loop steps: not
// with the refine rank-one term (its steps use the all-features kernels).
static bool host_loop() {  // QG_HOST_LOOP=1: the host-polled chunk loop (chunks of 1..64 iterations)
  static const char *env = std::getenv("QG_HOST_LOOP");
  return env && std::atoi(env) != 0;
}
// (not on the host-polled loop: its odd chunk lengths would break the mixed
// loop's alternating publication slots)
static bool defer_fin(const Handle &H) { return H.defer_fin && !H.use_rk1 && !host_loop(); }

// Step / finalize arguments of one LSMR iteration (u-step with the deferred
// update of the previous iteration, v-step), shared by the graph and the
// persistent paths.
static void iter_args(Handle &H, bool jvp, StepArgs &su, StepArgs &sv, FinArgs &fu, FinArgs &fv) {
  Workspace &W = H.ws;
  const int ku = jvp ? STEP_F : STEP_FT, kv = jvp ? STEP_FT : STEP_F;
  const double *rk1 = H.use_rk1 ? W.rk1 : nullptr;
  su = StepArgs{W.v, W.dpv, W.u, W.u, ku == STEP_FT ? W.dpu : nullptr, W.tY, W.tY2, W.st, 0, W.part};
  su.upd_h = W.h;
  su.upd_hb = W.hb;
  su.upd_x = W.x;
  su.rk1 = rk1;
  fu = FinArgs{H.B, PH_STEP_U, ku, W.st, W.part, W.v, W.u, W.u, W.h, W.hb, W.x, W.v};
  fu.rk1 = rk1;
  sv = StepArgs{W.u, W.dpu, W.v, W.v, kv == STEP_FT ? W.dpv : nullptr, W.tY, W.tY2, W.st, 1, W.part};
  sv.rk1 = rk1;
  fv = FinArgs{H.B, PH_STEP_V, kv, W.st, W.part, W.u, W.v, W.v, W.h, W.hb, W.x, W.v};
  fv.rk1 = rk1;
  // each follows a step kernel, which never writes the LSMR state or T entries
  fu.early = fv.early = 1;
  if (defer_fin(H) && !H.df_mixed) {
    // each step's CTA 0 runs the finalize the previous step owes: the u-step
    // finalizes the last v-step (partials in part2), the v-step the u-step
    su.df = sv.df = W.df;
    su.df_par = 0;
    sv.df_par = 1;
    su.df_next = PH_STEP_U;
    sv.df_next = PH_STEP_V;
    sv.part = W.part2;
    sv.fin = fu;
    fin_ptrs(H, sv.fin);  // (reads part: the u-step's partials)
    su.fin = fv;
    su.fin.part = W.part2;
    fin_ptrs(H, su.fin);
  } else if (defer_fin(H)) {
    // mixed (PSD blocks): the F step's CTA 0 runs the finalize of the F' step
    // before it (partials in part); the F step writes part2, finalized by a
    // k_fin_cta after it.  df_par alternates per iteration (capture_iters).
    StepArgs &sF = jvp ? su : sv;
    FinArgs &fFT = jvp ? fv : fu, &fF = jvp ? fu : fv;
    sF.df = W.df;
    sF.df_next = fFT.phase;
    sF.part = W.part2;
    sF.fin = fFT;
    fin_ptrs(H, sF.fin);
    fF.part = W.part2;
  }
}

static void capture_iters(Handle &H, const Mats &M, bool jvp, int iters, cudaStream_t st) {
  const int ku = jvp ? STEP_F : STEP_FT, kv = jvp ? STEP_FT : STEP_F;
  // The vector update of iteration k (hbar, x, h) runs fused into the u-step
  // kernel of iteration k+1 (which streams v_k anyway), and its stopping
  // test runs at the head of that iteration's PH_STEP_U finalize; the last
  // iteration's update is flushed by lsmr_flush().  4 launches / iteration.
  StepArgs su, sv;
  FinArgs fu, fv;
  iter_args(H, jvp, su, sv, fu, fv);
  const bool df = su.df != nullptr && sv.df != nullptr;  // finalizes run inside the next step (CTA 0)
  const bool mixed = !df && (su.df != nullptr || sv.df != nullptr);  // only the F step defers
  for (int i = 0; i < iters; ++i) {
    if (mixed) (jvp ? su : sv).df_par = i & 1;  // successive F steps alternate slots (chunks are even)
    launch_step(H, M, ku, su, st);
    if (!df && !(mixed && !jvp)) launch_fin(H, M, fu, st);  // (vjp: fin U runs in the F step's CTA 0)
    launch_step(H, M, kv, sv, st);
    if (!df && !(mixed && jvp)) launch_fin(H, M, fv, st);   // (jvp: fin V runs in the next F step's CTA 0)
  }
}

// Apply the pending update of the last completed iteration and its stopping
// test (problems that hit the cap are the only ones still active here).
static void lsmr_flush(Handle &H, const Mats &M, bool jvp, cudaStream_t st) {
  Workspace &W = H.ws;
  const int kv = jvp ? STEP_FT : STEP_F;
  UpdArgs ua{W.h, W.hb, W.x, W.v, W.st, W.part};
  launch_update(H, M, ua, st);
  FinArgs fx{H.B, PH_STEP_X, kv, W.st, W.part, W.u, W.v, W.v, W.h, W.hb, W.x, W.v};
  launch_fin(H, M, fx, st);
}

static cudaGraph_t capture_graph(Handle &H, const Mats &M, bool jvp, int iters) {
  cudaStream_t cs;
  QG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t graph;
  QG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const long long before = g_launches.load();
  try {
    capture_iters(H, M, jvp, iters, cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    throw;
  }
  g_launches = before;  // captured launches are counted when the graph runs
  QG_CUDA(cudaStreamEndCapture(cs, &graph));
  cudaStreamDestroy(cs);
  return graph;
}

// The whole LSMR loop as ONE graph: a conditional WHILE node whose body is
// `chunk` iterations plus k_loop_cond, which re-arms the node while a
// problem is active and the cap (W.d_loop[1]) is not reached.  No host
// round trip between chunks (the host-polled loop counted active problems
// and synchronised the stream before every chunk).
constexpr int kWhileChunk = 4;

static cudaGraph_t capture_while_graph(Handle &H, const Mats &M, bool jvp, int chunk) {
  cudaGraph_t g;
  QG_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  QG_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  QG_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStream_t cs;
  QG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  QG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const long long before = g_launches.load();
  cudaGraph_t out;
  try {
    capture_iters(H, M, jvp, chunk, cs);
    launch_loop_cond(H, h, chunk, cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &out);
    cudaStreamDestroy(cs);
    cudaGraphDestroy(g);
    throw;
  }
  g_launches = before;  // counted from the iterations actually run (lsmr_finish)
  QG_CUDA(cudaStreamEndCapture(cs, &out));
  cudaStreamDestroy(cs);
  return g;
}

// Launch `iters` LSMR iterations of handle H as one graph on `st`
// (iters = -kWhileChunk: the device-terminated WHILE graph).
static void launch_iters(Handle &H, const Mats &M, bool jvp, int iters, cudaStream_t st) {
  if (H.comm && !H.comm->capturable()) {  // host-synchronised exchange: plain launches
    capture_iters(H, M, jvp, iters, st);
    return;
  }
  // partitioned graphs carry the exchange nodes: a different topology
  const auto key = std::make_pair((jvp ? 1 : 0) + (H.comm ? 2 : 0) + (H.use_rk1 ? 4 : 0), iters);
  std::lock_guard<std::mutex> lock(g_graph_mu);
  auto git = g_graphs.find(&H);
  if (git == g_graphs.end()) git = g_graphs.emplace(&H, new GraphCache()).first;
  GraphCache *gc = git->second;
  auto cit = gc->graph.find(key);
  if (cit == gc->graph.end())
    cit = gc->graph.emplace(key, iters < 0 ? capture_while_graph(H, M, jvp, -iters) : capture_graph(H, M, jvp, iters))
              .first;
  SharedExec &se = g_exec[ExecKey{st, key.first, key.second}];
  if (se.exec == nullptr) {
    QG_CUDA(cudaGraphInstantiate(&se.exec, cit->second, 0));
  } else if (se.owner != &H) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(se.exec, cit->second, &info) != cudaSuccess) {
      cudaGetLastError();  // clear the sticky-free update error, fall back to a fresh instantiation
      cudaGraphExecDestroy(se.exec);
      se.exec = nullptr;
      QG_CUDA(cudaGraphInstantiate(&se.exec, cit->second, 0));
    }
  }
  se.owner = &H;
  QG_CUDA(cudaGraphLaunch(se.exec, st));
}

// One pinned word per host thread for the active-problem count (pinned
// allocation is expensive; never per handle).
static int *pinned_word() {
  static thread_local int *p = nullptr;
  if (!p) QG_CUDA(cudaMallocHost(&p, sizeof(int)));
  return p;
}

static int kernels_per_iter(const Handle &H) {
  // k_step<F>, k_step<F'> (one carries the deferred update), 2 x k_fin;
  // row-partitioned: each step is X_PARTIAL + X_FINISH and each finalize is
  // k_part_reduce + k_fin (the NCCL kernels are not ours)
  // (+1: the F' step's PSD units as k_step_psd)
  const int psd = psd_split(H) ? 1 : 0;
  if (H.comm) return 8 + psd - (H.nxu() + H.nyu() == 0 ? 2 : 0) - (H.nxu() == 0 ? 2 : 0);
  if (defer_fin(H)) return H.df_mixed ? 3 + psd : 2;
  return 4 + psd - (H.nxu() + H.nyu() == 0 ? 2 : 0);
}

static void run_lsmr_loop(Handle &H, const Mats &M, bool jvp, long long cap, cudaStream_t st) {
  Workspace &W = H.ws;
  // deferred finalize: nothing owed at the start, except in a mixed vjp loop,
  // whose first F' step's finalize runs in the first F step
  if (defer_fin(H)) launch_init_df(H, H.df_mixed && !jvp ? PH_STEP_U : 0, st);
  if ((!H.comm || H.comm->capturable()) && !host_loop()) {
    // W.d_loop = [0, cap] was armed by k_init_state
    if (cap > 0) launch_iters(H, M, jvp, -kWhileChunk, st);
    H.while_pending = true;
    return;
  }
  long long done = 0;
  while (true) {
    launch_count_active(H, st);
    int *pinned = pinned_word();
    QG_CUDA(cudaMemcpyAsync(pinned, W.d_nactive, sizeof(int), cudaMemcpyDeviceToHost, st));
    QG_CUDA(cudaStreamSynchronize(st));
    if (*pinned == 0 || done >= cap) break;
    const long long rem = cap - done;
    // 16 first (early convergence wastes little), then chunks of 64
    const long long want = done == 0 ? std::min<long long>(rem, 16) : rem;
    const int g = want >= 64 ? 64 : (want >= 16 ? 16 : (want >= 4 ? 4 : 1));
    launch_iters(H, M, jvp, g, st);
    if (!H.comm || H.comm->capturable()) count_launch(g * kernels_per_iter(H));  // else counted as launched
    done += g;
  }
}

static void lsmr_begin(Handle &H, const qg_lsmr_opts &o, cudaStream_t st, long long &cap) {
  cap = 0;
  for (int p = 0; p < H.B; ++p) {
    const long long N = H.n[p] + H.m[p] + 1;
    // lsmr.py:69-70: None -> 10 * (in + out); the ABI encodes None as 0 and an
    // explicit cap of zero as a negative value (k_init_state applies the same
    // rule per problem on the device)
    cap = std::max(cap, (o.max_iter > 0) ? (long long)o.max_iter : (o.max_iter < 0 ? 0LL : 20 * N));
  }
  launch_init_state(H, o.atol, o.btol, o.max_iter, cap, st);
  Workspace &W = H.ws;
  QG_CUDA(cudaMemsetAsync(W.x, 0, sizeof(double) * H.NE, st));
  QG_CUDA(cudaMemsetAsync(W.h, 0, sizeof(double) * H.NE, st));
  QG_CUDA(cudaMemsetAsync(W.hb, 0, sizeof(double) * H.NE, st));
}

static void lsmr_finish(Handle &H, qg_diag *diag, cudaStream_t st) {
  std::vector<Lsmr> L(H.B);
  QG_CUDA(cudaMemcpyAsync(L.data(), H.ws.st, sizeof(Lsmr) * H.B, cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  if (H.while_pending) {
    long long run[2] = {0, 0};
    QG_CUDA(cudaMemcpyAsync(run, H.ws.d_loop, sizeof(run), cudaMemcpyDeviceToHost, st));
    QG_CUDA(cudaStreamSynchronize(st));
    count_launch((run[0] / kWhileChunk) * (kWhileChunk * kernels_per_iter(H) + 1));
    H.while_pending = false;
  }
  if (H.loop_pending) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, H.ev_loop[0], H.ev_loop[1]) == cudaSuccess) H.loop_ms[H.loop_pending - 1] = ms;
    H.loop_pending = 0;
  }
  for (int p = 0; p < H.B; ++p) {
    if (L[p].status) {
      throw Error{QG_ERR_NUMERICAL, (H.B > 1 ? "problem " + std::to_string(p) + ": " : std::string()) +
                                        "non-finite quantity in LSMR at iteration " + std::to_string(L[p].itn)};
    }
    if (diag) {
      diag[p].iterations = L[p].itn;
      diag[p].converged = L[p].converged;
      diag[p].residual_norm = L[p].normr;
      diag[p].atr_norm = L[p].normar;
      diag[p].rhs_norm = L[p].normb;
      diag[p].derivative_unreliable = L[p].normr > 1e-6 * L[p].normb;   // solution_map.py:314
    }
  }
}

// After the rhs is in W.u (and, for vjp, D Pi(u_Y) in W.dpu): initial
// v = OP'(u)/beta, alpha, h = v, hbar = x = 0 (lsmr.py:72-103), then loop.
static void lsmr_solve(Handle &H, const Mats &M, bool jvp, int rhs_kind, long long cap, cudaStream_t st) {
  NvtxRange nv(jvp ? "qg:lsmr(F)" : "qg:lsmr(F')");
  Workspace &W = H.ws;
  FinArgs fr{H.B, PH_RHS, rhs_kind, W.st, W.part, W.u, nullptr, W.u, W.h, W.hb, W.x, W.v};
  launch_fin(H, M, fr, st);
  const int kv = jvp ? STEP_FT : STEP_F;
  StepArgs s0{W.u, W.dpu, nullptr, W.v, kv == STEP_FT ? W.dpv : nullptr, W.tY, W.tY2, W.st, 0, W.part};
  s0.rk1 = H.use_rk1 ? W.rk1 : nullptr;
  launch_step(H, M, kv, s0, st);
  FinArgs f0{H.B, PH_INIT_V, kv, W.st, W.part, W.u, nullptr, W.v, W.h, W.hb, W.x, W.v};
  f0.rk1 = s0.rk1;
  launch_fin(H, M, f0, st);
  UpdArgs ua{W.h, W.hb, W.x, W.v, W.st, W.part};
  launch_update(H, M, ua, st);
  // the loop is bracketed by events on the call's stream (qg_loop_time; read
  // back after lsmr_finish's synchronisation)
  H.loop_events();
  QG_CUDA(cudaEventRecord(H.ev_loop[0], st));
  if (H.engine && !H.use_rk1) {
    launch_engine(H, M, jvp, st);  // the whole loop, problem-resident (engine.cu)
  } else {
    run_lsmr_loop(H, M, jvp, cap, st);
    if (defer_fin(H) && (!H.df_mixed || jvp)) {
      // the finalize the loop's last v-step still owes (full: its partials in
      // part2; mixed jvp: the last F' step's, in part; mixed vjp owes none)
      StepArgs su, sv;
      FinArgs fu, fv;
      iter_args(H, jvp, su, sv, fu, fv);
      fv.part = H.df_mixed ? W.part : W.part2;
      fin_ptrs(H, fv);
      launch_df_tail(H, M, fv, st);
    }
    lsmr_flush(H, M, jvp, st);
  }
  QG_CUDA(cudaEventRecord(H.ev_loop[1], st));
  H.loop_pending = jvp ? 1 : 2;
}

}  // namespace qg

using namespace qg;

#define QG_API_BEGIN_NS try {
#define QG_API_BEGIN \
  try {              \
    qg::StreamScope _scope((cudaStream_t)stream);
#define QG_API_END                                                     \
  return QG_OK;                                                        \
  }                                                                    \
  catch (const qg::Error &e) { return qg::fail(e.code, e.msg); }        \
  catch (const std::exception &e) { return qg::fail(QG_ERR_CUDA, e.what()); }

extern "C" {

const char *qg_last_error(void) { return g_last_error.c_str(); }
const char *qg_version(void) { return "qcpgrad 0.1.0 (sm_100a)"; }
int64_t qg_kernel_launches(void) { return g_launches.load(); }

static int create_batch(qg_handle **out, const qg_batch_desc *desc, qg_comm *comm, void *stream) {
  QG_API_BEGIN
  cudaStream_t st = (cudaStream_t)stream;
  auto *H = new Handle();
  H->comm = reinterpret_cast<Comm *>(comm);
  try {
    build_handle(*H, *desc, st);
    launch_sub(H->ybar, H->cones.d_zmid, H->sbar, H->NY, st);
    // host fence before any PDL chain (operator.cu, launch_pdl invariant)
    QG_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    delete H;
    throw;
  }
  *out = reinterpret_cast<qg_handle *>(H);
  QG_API_END
}

int qg_create_batch(qg_handle **out, const qg_batch_desc *desc, void *stream) {
  return create_batch(out, desc, nullptr, stream);
}

int qg_create_batch_dist(qg_handle **out, const qg_batch_desc *desc, qg_comm *comm, void *stream) {
  if (!comm) return fail(QG_ERR_VALIDATION, "qg_create_batch_dist needs a communicator");
  return create_batch(out, desc, comm, stream);
}

int qg_destroy(qg_handle *h) {
  QG_API_BEGIN_NS
  delete reinterpret_cast<Handle *>(h);
  QG_API_END
}

int qg_handle_sizes(const qg_handle *h, int64_t *nprob, int64_t *total_n, int64_t *total_m) {
  QG_API_BEGIN_NS
  const Handle *H = reinterpret_cast<const Handle *>(h);
  *nprob = H->B;
  *total_n = H->NX;
  *total_m = H->NY;
  QG_API_END
}

int qg_handle_layout(const qg_handle *h, int64_t *sell_slices_x, int64_t *sell_slices_y) {
  QG_API_BEGIN_NS
  const Handle *H = reinterpret_cast<const Handle *>(h);
  *sell_slices_x = H->nslice_x;
  *sell_slices_y = H->nslice_y;
  QG_API_END
}

int qg_handle_engine(const qg_handle *h, int32_t *resident) {
  QG_API_BEGIN_NS
  *resident = reinterpret_cast<const Handle *>(h)->engine ? 1 : 0;
  QG_API_END
}

int qg_loop_time(const qg_handle *h, double *jvp_ms, double *vjp_ms) {
  QG_API_BEGIN_NS
  const Handle *H = reinterpret_cast<const Handle *>(h);
  *jvp_ms = H->loop_ms[0];
  *vjp_ms = H->loop_ms[1];
  QG_API_END
}

int qg_embedding_point(qg_handle *h, double *pz, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  cudaStream_t st = (cudaStream_t)stream;
  if (H.NX) QG_CUDA(cudaMemcpyAsync(pz, H.xbar, sizeof(double) * H.NX, cudaMemcpyDeviceToDevice, st));
  if (H.NY) QG_CUDA(cudaMemcpyAsync(pz + H.NX, H.ybar, sizeof(double) * H.NY, cudaMemcpyDeviceToDevice, st));
  std::vector<Embed> E(H.B);
  QG_CUDA(cudaMemcpyAsync(E.data(), H.emb, sizeof(Embed) * H.B, cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  std::vector<double> t(H.B);
  for (int p = 0; p < H.B; ++p) t[p] = E[p].tau;
  QG_CUDA(cudaMemcpyAsync(pz + H.NX + H.NY, t.data(), sizeof(double) * H.B, cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

int qg_apply_F(qg_handle *h, int transpose, const double *w, double *out, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  if (!H.deriv_ready) throw Error{QG_ERR_VALIDATION, "projection derivative not prepared at the current point"};
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  if (!transpose) H.cones.apply(w + H.NX, W.dpv, st);
  StepArgs a{w, W.dpv, nullptr, out, nullptr, W.tY, W.tY2, nullptr, 0, W.part};
  launch_step(H, M, transpose ? STEP_FT : STEP_F, a, st);
  FinArgs f{H.B, PH_APPLY, transpose ? STEP_FT : STEP_F, nullptr, W.part, w, nullptr, out,
            nullptr, nullptr, nullptr, nullptr};
  launch_fin(H, M, f, st);
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

// jvp / vjp formulas hold at a normalized embedding (solution_map.py:197-203)
static void require_normalized(const Handle &H) {
  if (!H.normalized)
    throw Error{QG_ERR_DOMAIN, "derivative formulas require the normalized embedding z_N = 1"};
  if (!H.deriv_ready) throw Error{QG_ERR_VALIDATION, "projection derivative not prepared at the current point"};
}

// Move the handle to the embedding point z = [X | Y | T] (refine, testkit.py
// :410-470): x part, middle block, z_N per problem; Pi z, P xbar, x'Px and
// (want_deriv) D Pi at the new point.  z_N <= 0 is a DomainError
// (embedding.py:384-387, 413-414).
static void set_point(Handle &H, const double *z, bool want_deriv, cudaStream_t st) {
  std::vector<double> zt(H.B);
  QG_CUDA(cudaMemcpyAsync(zt.data(), z + H.NX + H.NY, sizeof(double) * H.B, cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  bool norm = true;
  for (int p = 0; p < H.B; ++p) {
    if (!(zt[p] > 0.0))
      throw Error{QG_ERR_DOMAIN, (H.B > 1 ? "problem " + std::to_string(p) + ": " : std::string()) +
                                     "the point needs z_N > 0, got z_N = " + std::to_string(zt[p])};
    norm = norm && zt[p] == 1.0;
  }
  H.normalized = false;  // until the new point is fully in place
  H.deriv_ready = false;
  if (H.NX) QG_CUDA(cudaMemcpyAsync(H.xbar, z, sizeof(double) * H.NX, cudaMemcpyDeviceToDevice, st));
  double *zmid = H.cones.d_zmid;
  if (H.NY) QG_CUDA(cudaMemcpyAsync(zmid, z + H.NX, sizeof(double) * H.NY, cudaMemcpyDeviceToDevice, st));
  H.cones.prepare(zmid, H.ybar, 1, want_deriv, st);
  H.cones.check_errors(st);
  Mats M = make_mats(H);
  launch_embed_consts(H, M, H.ws.part, st, z + H.NX + H.NY);
  launch_sub(H.ybar, zmid, H.sbar, H.NY, st);
  // host fence: emb and the D Pi data are read before griddepcontrol.wait by
  // the PDL-launched step kernels (operator.cu, launch_pdl invariant)
  QG_CUDA(cudaStreamSynchronize(st));
  H.normalized = norm;
  H.deriv_ready = want_deriv;
}

int qg_jvp(qg_handle *h, const qg_perturbation *d, const qg_lsmr_opts *opts, double *dx, double *dy, double *ds,
           qg_diag *diag, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  require_normalized(H);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  PertDev pd{};
  DevCsr tP, tA, tAT;
  double *vP = nullptr, *vA = nullptr;
  if (d->same_pattern) {
    vP = dev_alloc<double>(H.P.nnz);
    vA = dev_alloc<double>(H.A.nnz);
    launch_gather(H.P.perm, d->dP_vals, vP, H.P.nnz, st);
    launch_gather(H.A.perm, d->dA_vals, vA, H.A.nnz, st);
    pd.dP_rp = H.P.rp; pd.dP_col = H.P.col; pd.dP_val = vP;
    pd.dA_rp = H.A.rp; pd.dA_col = H.A.col; pd.dA_val = vA;
    pd.dAT_rp = H.AT.rp; pd.dAT_col = H.AT.col; pd.dAT_val = d->dA_vals;
  } else {
    std::vector<int64_t> pn(d->dP_nnz, d->dP_nnz + H.B), an(d->dA_nnz, d->dA_nnz + H.B);
    CscBatch cp{d->dP_colptr, d->dP_rowidx, d->dP_vals, H.n, H.n, pn};
    csc_to_csr(cp, tP, nullptr, false, st);
    CscBatch ca{d->dA_colptr, d->dA_rowidx, d->dA_vals, H.n, H.m, an};
    csc_to_csr(ca, tA, &tAT, false, st);
    pd.dP_rp = tP.rp; pd.dP_col = tP.col; pd.dP_val = tP.val;
    pd.dA_rp = tA.rp; pd.dA_col = tA.col; pd.dA_val = tA.val;
    pd.dAT_rp = tAT.rp; pd.dAT_col = tAT.col; pd.dAT_val = d->dA_vals;
  }
  pd.dq = d->dq;
  pd.db = d->db;
  try {
    long long cap;
    lsmr_begin(H, *opts, st, cap);
    {
      NvtxRange nv("qg:jvp rhs");
      launch_jvp_rhs(H, M, pd, W.u, W.part, st);
    }
    lsmr_solve(H, M, true, RHS_JVP, cap, st);
    lsmr_finish(H, diag, st);
    // D phi: dy/ds need D Pi(dz_mid)
    NvtxRange nv("qg:jvp assembly");
    H.cones.apply(W.x + H.NX, W.tY, st);
    launch_dphi(H, M, W.x, W.tY, dx, dy, ds, st);
    QG_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    dev_free(vP); dev_free(vA); tP.release(); tA.release(); tAT.release();
    throw;
  }
  dev_free(vP); dev_free(vA); tP.release(); tA.release(); tAT.release();
  QG_API_END
}

int qg_vjp(qg_handle *h, const double *dx, const double *dy, const double *ds, const qg_lsmr_opts *opts,
           double *dP_vals, double *dA_vals, double *dq, double *db, qg_diag *diag, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  require_normalized(H);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  long long cap;
  lsmr_begin(H, *opts, st, cap);
  // dz = D phi'(delta): D Pi(dy + ds) - ds ; rhs = -dz ; D Pi(rhs_Y) for the first F
  {
    NvtxRange nv("qg:vjp rhs");
    launch_add(H, dy, ds, W.tY2, H.NY, st);
    H.cones.apply(W.tY2, W.tY, st);
    launch_vjp_rhs(H, M, dx, dy, ds, W.tY, W.u, W.part, st);
    H.cones.apply(W.u + H.NX, W.dpu, st);
  }
  lsmr_solve(H, M, false, RHS_VJP, cap, st);
  lsmr_finish(H, diag, st);
  NvtxRange nv("qg:vjp assembly");
  launch_vjp_grad(H, M, W.x, dP_vals, dA_vals, dq, db, st);
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

int qg_set_point(qg_handle *h, const double *z, int want_deriv, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  if (H.comm) throw Error{QG_ERR_VALIDATION, "qg_set_point is not available on a row-partitioned handle"};
  set_point(H, z, want_deriv != 0, (cudaStream_t)stream);
  QG_API_END
}

int qg_residual(qg_handle *h, double *out, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  if (H.comm) throw Error{QG_ERR_VALIDATION, "qg_residual is not available on a row-partitioned handle"};
  cudaStream_t st = (cudaStream_t)stream;
  Mats M = make_mats(H);
  launch_residual(H, M, out, H.ws.part, st);
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

// LSMR on J = F - r e_N' (r = rank1, or F alone when rank1 is null) from the
// right-hand side rhs; the solution (embedding layout) goes to sol.
// testkit.refine's Gauss-Newton model (testkit.py:439-454).
int qg_lsmr_jacobian(qg_handle *h, const double *rhs, const double *rank1, const qg_lsmr_opts *opts, double *sol,
                     qg_diag *diag, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  if (!H.deriv_ready) throw Error{QG_ERR_VALIDATION, "projection derivative not prepared at the current point"};
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  if (rank1) {
    if (!W.rk1) W.rk1 = dev_alloc<double>(H.NE);
    QG_CUDA(cudaMemcpyAsync(W.rk1, rank1, sizeof(double) * H.NE, cudaMemcpyDeviceToDevice, st));
  }
  struct Rk1Scope {
    Handle &H;
    Rk1Scope(Handle &h, bool on) : H(h) { H.use_rk1 = on; }
    ~Rk1Scope() { H.use_rk1 = false; }
  } scope(H, rank1 != nullptr);
  long long cap;
  lsmr_begin(H, *opts, st, cap);
  QG_CUDA(cudaMemcpyAsync(W.u, rhs, sizeof(double) * H.NE, cudaMemcpyDeviceToDevice, st));
  launch_vec_rhs(H, M, W.u, W.u, W.part, st);
  lsmr_solve(H, M, true, RHS_VEC, cap, st);
  lsmr_finish(H, diag, st);
  QG_CUDA(cudaMemcpyAsync(sol, W.x, sizeof(double) * H.NE, cudaMemcpyDeviceToDevice, st));
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

int qg_check(qg_handle *h, const double *x, const double *y, const double *s, double *report, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  if (H.comm) throw Error{QG_ERR_VALIDATION, "qg_check is not available on a row-partitioned handle"};
  std::lock_guard<std::mutex> lock(H.mu);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  // projections of s onto K and y onto K* (cones.py:926-941); the prepared
  // derivative at the embedding point is left untouched
  H.cones.prepare(s, W.tY, 0, false, st);
  H.cones.check_errors(st);
  H.cones.prepare(y, W.tY2, 1, false, st);
  H.cones.check_errors(st);
  double *rep = dev_alloc<double>(5 * (size_t)H.B);
  launch_kkt(H, M, x, y, s, W.tY, W.tY2, W.part, rep, st);
  QG_CUDA(cudaMemcpyAsync(report, rep, sizeof(double) * 5 * H.B, cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  dev_free(rep);
  QG_API_END
}

int qg_spmv_csc(int64_t nrows, int64_t ncols, const int64_t *col_ptr, const int64_t *row_idx, const double *values,
                int64_t nnz, int adjoint, const double *x, double *out, void *stream) {
  QG_API_BEGIN
  cudaStream_t st = (cudaStream_t)stream;
  DevCsr t, tc;
  CscBatch c{col_ptr, row_idx, values, {ncols}, {nrows}, {nnz}};
  csc_to_csr(c, t, &tc, false, st);
  if (adjoint) {
    tc.val = dev_alloc<double>(nnz);
    if (nnz) QG_CUDA(cudaMemcpyAsync(tc.val, values, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st));
    launch_csr_spmv(tc.rp, tc.col, tc.val, ncols, x, out, st);
  } else {
    launch_csr_spmv(t.rp, t.col, t.val, nrows, x, out, st);
  }
  QG_CUDA(cudaStreamSynchronize(st));
  t.release();
  tc.release();
  QG_API_END
}

int qg_time_kernel(qg_handle *h, int which, int reps, double *avg_ms, void *stream) {
  QG_API_BEGIN
  Handle &H = *reinterpret_cast<Handle *>(h);
  std::lock_guard<std::mutex> lock(H.mu);
  cudaStream_t st = (cudaStream_t)stream;
  Workspace &W = H.ws;
  Mats M = make_mats(H);
  // deterministic finite inputs: v = 1/sqrt(NE), u = v (D Pi v from the prepared derivative)
  std::vector<double> ones(H.NE, 1.0 / std::sqrt((double)std::max<int64_t>(H.NE, 1)));
  QG_CUDA(cudaMemcpyAsync(W.v, ones.data(), sizeof(double) * H.NE, cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(W.u, ones.data(), sizeof(double) * H.NE, cudaMemcpyHostToDevice, st));
  QG_CUDA(cudaMemcpyAsync(W.h, ones.data(), sizeof(double) * H.NE, cudaMemcpyHostToDevice, st));
  H.cones.apply(W.v + H.NX, W.dpv, st);
  // a state in which every problem is active with unit coefficients
  std::vector<Lsmr> L(H.B);
  for (auto &l : L) {
    l = Lsmr{};
    l.active = 1;
    l.s_in = 1.0; l.c_out = 0.5; l.s_v = 1.0;
    l.c_hbar = 0.25; l.c_x = 0.5; l.c_h = 0.125;
  }
  QG_CUDA(cudaMemcpyAsync(W.st, L.data(), sizeof(Lsmr) * H.B, cudaMemcpyHostToDevice, st));
  auto launch = [&]() {
    if (which == 0) {
      StepArgs a{W.v, W.dpv, W.u, W.u, nullptr, W.tY, W.tY2, W.st, 0, W.part};
      launch_step(H, M, STEP_F, a, st);
    } else if (which == 1) {
      StepArgs a{W.u, W.dpu, W.v, W.v, W.dpv, W.tY, W.tY2, W.st, 0, W.part};
      launch_step(H, M, STEP_FT, a, st);
    } else if (which == 3) {
      if (!psd_split(H)) throw Error{QG_ERR_VALIDATION, "qg_time_kernel: which = 3 needs PSD blocks"};
      StepArgs a{W.u, W.dpu, W.v, W.v, W.dpv, W.tY, W.tY2, W.st, 0, W.part};
      launch_step_psd(H, M, a, st);
    } else {
      UpdArgs ua{W.h, W.hb, W.x, W.v, W.st, W.part};
      launch_update(H, M, ua, st);
    }
  };
  QG_CUDA(cudaMemsetAsync(W.hb, 0, sizeof(double) * H.NE, st));
  QG_CUDA(cudaMemsetAsync(W.x, 0, sizeof(double) * H.NE, st));
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t e0, e1;
  QG_CUDA(cudaEventCreate(&e0));
  QG_CUDA(cudaEventCreate(&e1));
  QG_CUDA(cudaEventRecord(e0, st));
  for (int i = 0; i < reps; ++i) launch();
  QG_CUDA(cudaEventRecord(e1, st));
  QG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  QG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *avg_ms = (double)ms / std::max(reps, 1);
  if (which == 1 && H.cones.max_psd_order > 0 && std::getenv("QG_PSD_PROF")) {
    // one more F' launch with the PSD units' phase clocks (diagnostics)
    unsigned long long *d = dev_alloc<unsigned long long>(5), h5[5];
    QG_CUDA(cudaMemsetAsync(d, 0, sizeof(h5), st));
    StepArgs a{W.u, W.dpu, W.v, W.v, W.dpv, W.tY, W.tY2, W.st, 0, W.part};
    a.prof = d;
    launch_step(H, M, STEP_FT, a, st);
    QG_CUDA(cudaMemcpyAsync(h5, d, sizeof(h5), cudaMemcpyDeviceToHost, st));
    QG_CUDA(cudaStreamSynchronize(st));
    dev_free(d);
    const double u = (double)std::max<unsigned long long>(h5[0], 1);
    std::fprintf(stderr, "[qg psd] %llu PSD units, cycles per unit: SpMV pass %.0f | D Pi t %.0f | rows %.0f | "
                 "D Pi o %.0f\n", h5[0], h5[1] / u, h5[2] / u, h5[3] / u, h5[4] / u);
  }
  QG_API_END
}

// ----------------------------------------------------- cone calculus ----
struct ConesHandle {
  ConeTable t;
};

int qg_cones_create(qg_cones **out, const qg_cone_block *blocks, int64_t nblocks, void *stream) {
  QG_API_BEGIN
  auto *c = new ConesHandle();
  try {
    int64_t m = 0;
    for (int64_t i = 0; i < nblocks; ++i) m += blocks[i].dim;
    std::vector<int64_t> yoff{0, m};
    c->t.build(blocks, &nblocks, yoff, 1024, (cudaStream_t)stream);
  } catch (...) {
    delete c;
    throw;
  }
  *out = reinterpret_cast<qg_cones *>(c);
  QG_API_END
}

int qg_cones_destroy(qg_cones *c) {
  QG_API_BEGIN_NS
  delete reinterpret_cast<ConesHandle *>(c);
  QG_API_END
}

int qg_cones_project(qg_cones *c, int dual, const double *z, double *out, void *stream) {
  QG_API_BEGIN
  ConeTable &t = reinterpret_cast<ConesHandle *>(c)->t;
  cudaStream_t st = (cudaStream_t)stream;
  t.prepare(z, out, dual, false, st);
  t.check_errors(st);
  QG_API_END
}

int qg_cones_prepare(qg_cones *c, int dual, const double *z, void *stream) {
  QG_API_BEGIN
  ConeTable &t = reinterpret_cast<ConesHandle *>(c)->t;
  cudaStream_t st = (cudaStream_t)stream;
  t.prepare(z, nullptr, dual, true, st);
  t.check_errors(st);
  QG_API_END
}

int qg_cones_apply(qg_cones *c, const double *dz, double *out, void *stream) {
  QG_API_BEGIN
  ConeTable &t = reinterpret_cast<ConesHandle *>(c)->t;
  cudaStream_t st = (cudaStream_t)stream;
  t.apply(dz, out, st);
  QG_CUDA(cudaStreamSynchronize(st));
  QG_API_END
}

}  // extern "C"
