// Communicators of the row-partitioned mode: the Y rows
// of A (with b, y, s and whole cone blocks) are split over ranks; X, T and
// the LSMR scalars are replicated.  Each operator step has ONE exchange: the
// sum over ranks of the A_r' partial products on the X rows, plus the
// per-problem partial sums of the finalize.  Both are sum-allreduces issued
// on the compute stream between kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qg {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // in-place sum over ranks, stream-ordered; identical bits on every rank
  virtual void allreduce(double *buf, int64_t n, cudaStream_t st) = 0;
  // may the allreduce be recorded into a CUDA graph?
  virtual bool capturable() const = 0;
};

}  // namespace qg
