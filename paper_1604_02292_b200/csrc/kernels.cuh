// kernels.cuh -- sm_100a kernels of the local tomography hot path (common.cuh,
// projectors.cuh, fgp.cuh, support.cuh).
//
// Notation follows PAPER.md (arXiv 1604.02292) and DESIGN.md:
//   W   Joseph projector, W[(a,d),(i,j)] = hat((t_d - t_ij)/c_a)/c_a      (V2)
//   "tile"  = a square block of pixels processed as one unit: the extended
//             ROI L' of one local reconstruction, or the
//             whole N x N grid for the global operators (Alg. 1, a10).
//   "window" = the contiguous run of detector bins that a tile can reach at
//             one angle (V4); W_{L'} is evaluated only there.
//
// Layouts (DESIGN.md §Data layout):
//   padded tile image  [tile][T][TP], data at columns PADL..PADL+T-1, two-sided
//                      zero padding so Joseph taps never need bounds checks.
//                      Every padded image has a transposed twin (lines = columns)
//                      so column-driven angles march contiguous memory too.
//   plain tile image   [tile][T][T]
//   window sinogram    [tile][N_theta][Wwin]
//   sinogram           [N_theta][N_d]
#pragma once

#include "common.cuh"
#include "projectors.cuh"
#include "fgp.cuh"
#include "support.cuh"
