// Host-side owner of a batch's cone structure: block table, Y work units and
// the prepared projection-derivative parameters in HBM.
#pragma once

#include <algorithm>
#include <vector>

#include "qg_common.cuh"

namespace qg {

struct ConeTable {
  int nprob = 0;
  int64_t ny = 0, nblk = 0;
  int max_psd_order = 0;
  int dual = 1;
  std::vector<BlockInfo> h_blk;
  std::vector<Unit> units;          // Y work units, problem-major
  std::vector<int64_t> unit_ptr;    // [nprob+1] unit ranges per problem
  BlockInfo *d_blk = nullptr;
  Unit *d_units = nullptr;
  double *d_zmid = nullptr, *d_soc_nu = nullptr, *d_psd = nullptr, *d_tri_D = nullptr;
  int32_t *d_soc_code = nullptr, *d_tri_flip = nullptr;
  unsigned long long *d_err = nullptr;

  ConeTable() = default;
  ConeTable(const ConeTable &) = delete;
  ConeTable &operator=(const ConeTable &) = delete;
  ~ConeTable();

  // blocks: concatenated per problem, nblocks[p] of problem p (yoff: [nprob+1])
  void build(const qg_cone_block *blocks, const int64_t *nblocks, const std::vector<int64_t> &yoff,
             int64_t target_rows, cudaStream_t st);
  // Projection of z (primal or dual) into proj (may be null) and, when
  // want_deriv, the derivative parameters at z (z is kept as zmid).
  void prepare(const double *z, double *proj, int dual_mode, bool want_deriv, cudaStream_t st);
  void check_errors(cudaStream_t st);  // throws the first failing block
  void apply(const double *in, double *out, cudaStream_t st);
  DpiView view() const;
  size_t psd_smem_prep() const;
  size_t psd_smem_apply() const;
};

}  // namespace qg
