// Cone preparation and application kernels.
//
// k_cone_prep: one pass over the Y work units computing, per block, the
//   projection (primal or dual) and the prepared derivative parameters
//   (cones.py:730-795 soc/psd, 414-480 exp, 647-722 pow, 803-883 dispatch).
// k_dpi_apply: standalone blockwise D Pi application (cones.py:899-906).
#include "cone_table.h"
#include "dpi_dev.cuh"

namespace qg {

__device__ __forceinline__ void record_error(unsigned long long *err, int phase, int blk, int code) {
  const unsigned long long key = ((unsigned long long)phase << 60) | ((unsigned long long)blk << 4) |
                                 (unsigned long long)code;
  atomicMin(err, key);
}

struct PrepArgs {
  const BlockInfo *blk;
  const Unit *units;
  const double *z;      // Y layout
  double *proj;         // Y layout or null
  double *soc_nu;
  int32_t *soc_code;
  double *psd;
  double *tri_D;
  int32_t *tri_flip;
  int dual;
  int want_deriv;
  unsigned long long *err;
};

__global__ void __launch_bounds__(kThreads) k_cone_prep(PrepArgs a) {
  extern __shared__ double sm[];
  const Unit u = a.units[blockIdx.x];
  if (u.cls == CLS_ELEM) {
    const int kind = a.blk[u.blk0].kind;
    if (a.proj)
      for (int r = u.row0 + threadIdx.x; r < u.row1; r += blockDim.x) {
        const double z = a.z[r];
        a.proj[r] = (kind == QG_CONE_ZERO) ? (a.dual ? z : 0.0) : fmax(z, 0.0);
      }
    return;
  }
  if (u.cls == CLS_SOC) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = u.blk0 + warp; k < u.blk1; k += (blockDim.x >> 5)) {
      const BlockInfo b = a.blk[k];
      const double *z = a.z + b.row;
      double part = 0.0;
      for (int i = 1 + lane; i < b.dim; i += 32) part += z[i] * z[i];
      const double nu = sqrt(warp_sum(part));
      const double t = z[0];
      if (a.want_deriv && lane == 0) {
        int code;
        if (nu == 0.0 && t == 0.0) code = 2;
        else if (nu < -t) code = 0;
        else if (nu < t) code = 1;
        else code = 3;
        a.soc_nu[b.param] = nu;
        a.soc_code[b.param] = code;
      }
      if (a.proj) {
        double *o = a.proj + b.row;
        if (nu <= -t) {
          for (int i = lane; i < b.dim; i += 32) o[i] = 0.0;
        } else if (nu <= t) {
          for (int i = lane; i < b.dim; i += 32) o[i] = z[i];
        } else {
          const double f = 0.5 * (1.0 + t / nu);
          for (int i = lane; i < b.dim; i += 32) o[i] = f * (i == 0 ? nu : z[i]);
        }
      }
    }
    return;
  }
  if (u.cls == CLS_PSD) {
    const BlockInfo b = a.blk[u.blk0];
    const int d = b.order, dd = d * d;
    double *A = sm, *V = sm + dd, *lam = sm + 2 * dd, *rot = lam + d;
    int *flag = (int *)(rot + 4 * 33);
    const double *z = a.z + b.row;
    for (int idx = threadIdx.x; idx < dd; idx += blockDim.x) {
      const int i = idx % d, j = idx / d;
      const int p = i >= j ? i : j, q = i >= j ? j : i;
      const double v = z[svec_index(p, q, d)];
      A[idx] = (p == q) ? v : v / kSqrt2;
    }
    __syncthreads();
    jacobi_eigh_cta(A, V, lam, d, rot, flag);
    if (a.want_deriv) {
      double *Vg = a.psd + b.param, *Bg = Vg + dd;
      __shared__ double s_tol;
      if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int i = 0; i < d; ++i) mx = fmax(mx, fabs(lam[i]));
        s_tol = 1e-12 * mx;
      }
      __syncthreads();
      const double tol = s_tol;
      for (int idx = threadIdx.x; idx < dd; idx += blockDim.x) {
        const int i = idx % d, j = idx / d;
        Vg[idx] = V[idx];
        const bool pi = lam[i] >= -tol, pj = lam[j] >= -tol;
        double bij;
        if (pi && pj) bij = 1.0;
        else if (pi && !pj) bij = lam[i] / (lam[i] - lam[j]);
        else if (!pi && pj) bij = lam[j] / (lam[j] - lam[i]);
        else bij = 0.0;
        Bg[idx] = bij;  // cones.py:782-789
      }
    }
    if (a.proj) {
      double *o = a.proj + b.row;
      for (int idx = threadIdx.x; idx < dd; idx += blockDim.x) {
        const int i = idx % d, j = idx / d;
        if (i < j) continue;
        double s = 0.0;
        for (int k = 0; k < d; ++k) s += (V[i + k * d] * fmax(lam[k], 0.0)) * V[j + k * d];
        o[svec_index(i, j, d)] = (i == j) ? s : s * kSqrt2;
      }
    }
    return;
  }
  // CLS_TRI: one thread per 3-dimensional block
  for (int k = u.blk0 + (int)threadIdx.x; k < u.blk1; k += blockDim.x) {
    const BlockInfo b = a.blk[k];
    const double z3[3] = {a.z[b.row], a.z[b.row + 1], a.z[b.row + 2]};
    if (a.proj) {
      double o[3];
      const int st = tri_project(b.kind, b.alpha, a.dual, z3, o);
      if (st != QG_OK) {
        record_error(a.err, 0, k, st);
        o[0] = o[1] = o[2] = 0.0;
      }
      a.proj[b.row] = o[0]; a.proj[b.row + 1] = o[1]; a.proj[b.row + 2] = o[2];
    }
    if (a.want_deriv) {
      double D[9];
      int flip = 0;
      const int st = tri_deriv(b.kind, b.alpha, a.dual, z3, D, flip);
      if (st != QG_OK) {
        record_error(a.err, 1, k, st);
        for (int i = 0; i < 9; ++i) D[i] = 0.0;
      }
      for (int i = 0; i < 9; ++i) a.tri_D[9 * b.param + i] = D[i];
      a.tri_flip[b.param] = flip;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_dpi_apply(DpiView dv, const Unit *units, const double *in,
                                                        double *out) {
  extern __shared__ double sm[];
  const Unit u = units[blockIdx.x];
  dpi_apply_unit(dv, u, in + u.row0, out + u.row0, sm);
}

// ------------------------------------------------------------- host side --

size_t ConeTable::psd_smem_prep() const {
  if (max_psd_order == 0) return 0;
  const int d = max_psd_order;
  return (size_t)(2 * d * d + d + 4 * 33 + 2) * sizeof(double);
}

size_t ConeTable::psd_smem_apply() const {
#if QG_PSD_DMMA
  const int dp = (max_psd_order + 7) & ~7, ld = dp + 4;  // psd_pad / psd_ld (dpi_dev.cuh)
#else
  const int dp = (max_psd_order + 3) & ~3, ld = dp + 1;
#endif
  return (size_t)3 * dp * ld * sizeof(double);  // V, S (= W), T: psd_apply_cta
}

void ConeTable::prepare(const double *z, double *proj, int dual_mode, bool want_deriv, cudaStream_t st) {
  if (units.empty()) return;
  if (want_deriv) dual = dual_mode;
  QG_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), st));
  PrepArgs a{d_blk, d_units, z, proj, d_soc_nu, d_soc_code, d_psd, d_tri_D, d_tri_flip, dual_mode,
             want_deriv ? 1 : 0, d_err};
  const size_t smem = psd_smem_prep();
  if (smem > 48 * 1024)
    raise_dynamic_smem(reinterpret_cast<const void *>(k_cone_prep), smem);
  k_cone_prep<<<(unsigned)units.size(), kThreads, smem, st>>>(a);
  QG_LAUNCHED();
  if (want_deriv && z != d_zmid)
    QG_CUDA(cudaMemcpyAsync(d_zmid, z, sizeof(double) * (size_t)ny, cudaMemcpyDeviceToDevice, st));
}

void ConeTable::check_errors(cudaStream_t st) {
  if (units.empty()) return;  // nothing was prepared (empty cone)
  unsigned long long key = 0;
  QG_CUDA(cudaMemcpyAsync(&key, d_err, sizeof(key), cudaMemcpyDeviceToHost, st));
  QG_CUDA(cudaStreamSynchronize(st));
  if (key == ~0ull) return;
  const int code = (int)(key & 0xf);
  const long long blk = (long long)((key >> 4) & ((1ull << 56) - 1));
  if (blk < 0 || blk >= (long long)h_blk.size())
    throw Error{QG_ERR_CUDA, "corrupt cone error record (block " + std::to_string(blk) + ")"};
  const BlockInfo &b = h_blk[blk];
  static const char *names[] = {"zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow"};
  std::string what;
  if (code == QG_ERR_NOT_DIFFERENTIABLE)
    what = "power cone projection is not differentiable at z = 0 with x = 0 or y = 0";
  else if (b.kind == QG_CONE_EXP || b.kind == QG_CONE_DEXP)
    what = (key >> 60) ? "exponential cone projection derivative failed (root-finding or overflow)"
                       : "exponential cone projection root-finding did not converge";
  else
    what = "cone computation failed";
  std::string prefix = nprob > 1 ? "problem " + std::to_string(b.prob) + ": " : std::string();
  throw Error{code, prefix + "cone block " + std::to_string(b.local) + " (" + names[b.kind] + "): " + what};
}

DpiView ConeTable::view() const {
  return DpiView{d_blk, d_zmid, d_soc_nu, d_soc_code, d_psd, d_tri_D, d_tri_flip, dual};
}

void ConeTable::apply(const double *in, double *out, cudaStream_t st) {
  if (units.empty()) return;
  const size_t smem = psd_smem_apply();
  if (smem > 48 * 1024)
    raise_dynamic_smem(reinterpret_cast<const void *>(k_dpi_apply), smem);
  k_dpi_apply<<<(unsigned)units.size(), kThreads, smem, st>>>(view(), d_units, in, out);
  QG_LAUNCHED();
}

void ConeTable::build(const qg_cone_block *blocks, const int64_t *nblocks, const std::vector<int64_t> &yoff,
                      int64_t target_rows, cudaStream_t st) {
  nprob = (int)yoff.size() - 1;
  ny = yoff.back();
  // serial pass: validation and per-problem parameter offsets
  std::vector<int64_t> boff(nprob + 1, 0), soc_off(nprob + 1, 0), tri_off(nprob + 1, 0), psd_off(nprob + 1, 0);
  for (int p = 0; p < nprob; ++p) {
    boff[p + 1] = boff[p] + nblocks[p];
    int64_t rows = 0, ns = 0, nt = 0, np = 0;
    for (int64_t i = boff[p]; i < boff[p + 1]; ++i) {
      const qg_cone_block &c = blocks[i];
      rows += c.dim;
      if (c.kind == QG_CONE_SOC) ++ns;
      else if (c.kind == QG_CONE_PSD) {
        if (c.order > kMaxPsdOrder)
          throw Error{QG_ERR_UNSUPPORTED, "psd block order " + std::to_string(c.order) +
                                              " exceeds this build's limit " + std::to_string(kMaxPsdOrder)};
        np += 2LL * c.order * c.order;
        max_psd_order = std::max(max_psd_order, (int)c.order);
      } else if (c.kind >= QG_CONE_EXP) ++nt;
    }
    if (rows != yoff[p + 1] - yoff[p]) throw Error{QG_ERR_VALIDATION, "cone dimension does not match m"};
    soc_off[p + 1] = soc_off[p] + ns;
    tri_off[p + 1] = tri_off[p] + nt;
    psd_off[p + 1] = psd_off[p] + np;
  }
  const int64_t nsoc = soc_off[nprob], ntri = tri_off[nprob], psd_total = psd_off[nprob];
  h_blk.resize(boff[nprob]);
  // parallel pass over problem chunks: block records and work units (never
  // crossing problems or classes), concatenated in problem order
  unit_ptr.assign(nprob + 1, 0);
  const int64_t nchunk = std::min<int64_t>(nprob, 64);
  std::vector<std::vector<Unit>> part(nchunk);
  host_parallel(nchunk, 1, [&](int64_t c0, int64_t c1) {
    for (int64_t c = c0; c < c1; ++c) {
      std::vector<Unit> &out = part[c];
      for (int p = (int)(nprob * c / nchunk); p < (int)(nprob * (c + 1) / nchunk); ++p) {
        int64_t row = yoff[p], isoc = soc_off[p], itri = tri_off[p], ipsd = psd_off[p];
        for (int64_t i = boff[p]; i < boff[p + 1]; ++i) {
          const qg_cone_block &cb = blocks[i];
          BlockInfo b{};
          b.kind = cb.kind;
          b.row = (int32_t)row;
          b.dim = cb.dim;
          b.order = cb.order;
          b.alpha = cb.alpha;
          b.prob = p;
          b.local = (int32_t)(i - boff[p]);
          b.param = -1;
          if (cb.kind == QG_CONE_SOC) b.param = isoc++;
          else if (cb.kind == QG_CONE_PSD) {
            b.param = ipsd;
            ipsd += 2LL * cb.order * cb.order;
          } else if (cb.kind >= QG_CONE_EXP) b.param = itri++;
          h_blk[i] = b;
          row += cb.dim;
        }
        const size_t before = out.size();
        int64_t bi = boff[p];
        const int64_t bend = boff[p + 1];
        while (bi < bend) {
          const BlockInfo &b = h_blk[bi];
          if (b.kind == QG_CONE_ZERO || b.kind == QG_CONE_NONNEG) {
            for (int64_t r = b.row; r < b.row + b.dim; r += target_rows)
              out.push_back(Unit{p, (int32_t)r, (int32_t)std::min<int64_t>(r + target_rows, b.row + b.dim),
                                 (int32_t)bi, (int32_t)bi + 1, CLS_ELEM});
            ++bi;
          } else if (b.kind == QG_CONE_PSD) {
            out.push_back(Unit{p, b.row, b.row + b.dim, (int32_t)bi, (int32_t)bi + 1, CLS_PSD});
            ++bi;
          } else {
            const int cls = (b.kind == QG_CONE_SOC) ? CLS_SOC : CLS_TRI;
            const int64_t maxblk = (cls == CLS_SOC) ? 16 * kWarps : kThreads;
            int64_t e = bi, rows = 0;
            while (e < bend && e - bi < maxblk) {
              const BlockInfo &cc = h_blk[e];
              const int ccls = (cc.kind == QG_CONE_SOC) ? CLS_SOC : (cc.kind >= QG_CONE_EXP ? CLS_TRI : -1);
              if (ccls != cls) break;
              if (rows > 0 && rows + cc.dim > target_rows) break;
              rows += cc.dim;
              ++e;
            }
            Unit un{p, b.row, (int32_t)(b.row + rows), (int32_t)bi, (int32_t)e, cls};
            if (cls == CLS_SOC) {  // thread-per-block fused epilogue for small SOC blocks
              int maxdim = 0;
              for (int64_t k = bi; k < e; ++k) maxdim = std::max(maxdim, (int)h_blk[k].dim);
              // lanes per block of the engine's group epilogue (power of two >= dim)
              int g = 1;
              while (g < maxdim) g <<= 1;
              un.group = maxdim <= 32 ? g : 0;
            }
            out.push_back(un);
            bi = e;
          }
        }
        unit_ptr[p + 1] = (int64_t)(out.size() - before);
      }
    }
  });
  for (int p = 0; p < nprob; ++p) unit_ptr[p + 1] += unit_ptr[p];
  units.reserve(unit_ptr[nprob]);
  for (auto &v : part) units.insert(units.end(), v.begin(), v.end());
  nblk = (int64_t)h_blk.size();
  trace_point("  cone table: host passes", st);
  d_blk = dev_alloc<BlockInfo>(h_blk.size());
  QG_CUDA(cudaMemcpyAsync(d_blk, h_blk.data(), sizeof(BlockInfo) * h_blk.size(), cudaMemcpyHostToDevice, st));
  d_units = dev_alloc<Unit>(units.size());
  QG_CUDA(cudaMemcpyAsync(d_units, units.data(), sizeof(Unit) * units.size(), cudaMemcpyHostToDevice, st));
  d_zmid = dev_alloc<double>(ny);
  d_soc_nu = dev_alloc<double>(nsoc);
  d_soc_code = dev_alloc<int32_t>(nsoc);
  d_psd = dev_alloc<double>(psd_total);
  d_tri_D = dev_alloc<double>(9 * ntri);
  d_tri_flip = dev_alloc<int32_t>(ntri);
  d_err = dev_alloc<unsigned long long>(1);
  QG_CUDA(cudaMemsetAsync(d_err, 0xff, sizeof(unsigned long long), st));
  QG_CUDA(cudaStreamSynchronize(st));  // host vectors above are sources of async copies
}

ConeTable::~ConeTable() {
  dev_free(d_blk);
  dev_free(d_units);
  dev_free(d_zmid);
  dev_free(d_soc_nu);
  dev_free(d_soc_code);
  dev_free(d_psd);
  dev_free(d_tri_D);
  dev_free(d_tri_flip);
  dev_free(d_err);
}

}  // namespace qg
