// Device kernels of the data operations beside the GEMM:
// precision conversion, reshape remap, row/column partial sums and folds.
// Precision codes follow the reference (precision.hpp:14): 0 Half16,
// 1 Single32, 2 Double64.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dm {

inline int precision_bytes(int p) { return p == 0 ? 2 : p == 1 ? 4 : 8; }

// dst[i] = convert(src[i]) for i < count with the reference's scalar rules:
// widen exactly, narrow once with round-to-nearest-even (half.hpp:17-77,
// precision.hpp:74-89).  src may be a peer pointer.
cudaError_t convert_copy(const void* src, int src_prec, void* dst, int dst_prec, int64_t count,
                         cudaStream_t stream);

// Reshape remap (ReshapeExec, ops.hpp:772-944): element (i, j) of the
// destination block whose top-left global coordinate is (r0, c0) in a
// destination matrix with `dst_gcols` columns takes the source element with
// the same row-major linear index.  `src_blocks` is a device array of
// n_block_rows * n_block_cols source block pointers (peer pointers allowed).
struct RemapGeometry {
  int64_t dst_rows, dst_cols;  // destination block extent
  int64_t r0, c0;              // its global origin
  int64_t dst_gcols;           // destination global columns
  int64_t src_grows, src_gcols, src_brows, src_bcols;
  int32_t src_nbc;
};
cudaError_t remap_gather(const void* const* src_blocks, int src_prec, void* dst, int dst_prec,
                         const RemapGeometry& g, cudaStream_t stream);

// One worker's partial for one row (axis 0) or column (axis 1) segment
// (RowColSumExec::local_partial, ops.hpp:1039-1068): for each i < len,
// acc = 0; for lane in the given blocks (ascending): for k: acc += widen(x);
// accumulation at float (double for Double64), stored at the matrix precision.
// `blocks` is a device array of `nlanes` block pointers, `inner` the
// per-lane inner extent (device array), `pitch` each block's row pitch.
cudaError_t segment_partial(const void* const* blocks, const int64_t* inner, const int64_t* pitch,
                            int nlanes, int axis, int prec, int64_t len, void* out,
                            cudaStream_t stream);

// out[i] = fold of parts[0..nparts) in the given order at the accumulation
// precision (RowColSumExec::reduce_segment, ops.hpp:1077-1110).
cudaError_t fold_partials(const void* const* parts, int nparts, int prec, int64_t len, void* out,
                          cudaStream_t stream);

}  // namespace dm
