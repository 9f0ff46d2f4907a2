// Sparse coupling of the factorized hex8 element operator, shared by the tile
// kernel (hex8_apply.cu) and the fused coarse-tail kernel (tail.cu).
#pragma once
#include "vt_device.cuh"

namespace vt {

// Sparse coupling in the (S,D)^3 basis: O = s * M C.  Pattern bit0 = x,
// bit1 = y, bit2 = z (1 = D / W).  Derived from the closed-form K0
// [ref: element.py:61-99]; see DESIGN.md for the table.
__device__ __forceinline__ void couple(const double C[3][8], double s, const double* kc,
                                       double O[3][8]) {
  const double a1 = s * kc[0], a2 = s * kc[1], a3 = s * kc[2], a4 = s * kc[3], a5 = s * kc[4],
               a6 = s * kc[5];
  const double d0 = C[0][1] + C[1][2] + C[2][4];
  const double ld = a1 * d0;
  O[0][1] = fma(a2, C[0][1], ld);
  O[1][2] = fma(a2, C[1][2], ld);
  O[2][4] = fma(a2, C[2][4], ld);
  const double t01 = a3 * (C[0][2] + C[1][1]);
  const double t02 = a3 * (C[0][4] + C[2][1]);
  const double t12 = a3 * (C[1][4] + C[2][2]);
  O[0][2] = t01; O[1][1] = t01;
  O[0][4] = t02; O[2][1] = t02;
  O[1][4] = t12; O[2][2] = t12;
  double w = a4 * (C[0][3] + C[2][6]);
  O[0][3] = fma(a3, C[0][3], w);
  O[2][6] = fma(a3, C[2][6], w);
  w = a4 * (C[0][5] + C[1][6]);
  O[0][5] = fma(a3, C[0][5], w);
  O[1][6] = fma(a3, C[1][6], w);
  w = a4 * (C[1][3] + C[2][5]);
  O[1][3] = fma(a3, C[1][3], w);
  O[2][5] = fma(a3, C[2][5], w);
  const double tt = C[0][6] + C[1][5] + C[2][3];
  O[0][6] = a5 * (tt + C[0][6]);
  O[1][5] = a5 * (tt + C[1][5]);
  O[2][3] = a5 * (tt + C[2][3]);
  O[0][7] = a6 * C[0][7];
  O[1][7] = a6 * C[1][7];
  O[2][7] = a6 * C[2][7];
}

}  // namespace vt
