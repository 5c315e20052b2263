// h3d_device.cuh -- device-side primitives shared by every hull kernel.
//
// Semantics follow the reference kernels (pkg/src/hull3d/_ckernels.pyx):
//   evtime  :34-46   act :49-60   find_bridge :63-83
// fp64 throughout with explicit round-to-nearest intrinsics, so no FMA can be
// contracted into the event-time arithmetic (the reference builds with
// -ffp-contract=off, pkg/setup.py:51-54); the library is additionally built
// with -fmad=false.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hull3d_b200.h"

namespace h3d {

constexpr int NIL = -1;
constexpr double INF = __builtin_huge_val();

// error word: first error wins (0 = ok); codes are the reference's negatives
__device__ __forceinline__ void raise_err(long long *err, long long code) {
  atomicCAS(reinterpret_cast<unsigned long long *>(err), 0ull,
            static_cast<unsigned long long>(code));
}

// Kinetic collinearity time of (a, b, c) given their coordinates; base
// point a, xy-determinant tested against 0 before the xz one is formed.
__device__ __forceinline__ double evtime_xyz(double ax, double ay, double az,
                                             double bx, double by, double bz,
                                             double cx, double cy, double cz) {
  const double dbx = __dsub_rn(bx, ax);
  const double dcx = __dsub_rn(cx, ax);
  const double den = __dsub_rn(__dmul_rn(dbx, __dsub_rn(cy, ay)),
                               __dmul_rn(dcx, __dsub_rn(by, ay)));
  if (den == 0.0) return INF;
  const double num = __dsub_rn(__dmul_rn(dbx, __dsub_rn(cz, az)),
                               __dmul_rn(dcx, __dsub_rn(bz, az)));
  return __ddiv_rn(num, den);
}

// xy turn of (p, q, r) as the bridge walk evaluates it (_ckernels.pyx:71,75)
__device__ __forceinline__ double turn_xy(double px, double py, double qx,
                                          double qy, double rx, double ry) {
  return __dsub_rn(__dmul_rn(__dsub_rn(qx, px), __dsub_rn(ry, py)),
                   __dmul_rn(__dsub_rn(rx, px), __dsub_rn(qy, py)));
}

// Reference-layout point access: pts is (n,3) row-major f64; the upper pass
// negates z on load (IEEE negation is exact and rounding is sign-symmetric,
// so every derived time is bit-identical to the reference's negated copy,
// pkg/src/hull3d/api.py:215-216).
struct RowPts {
  const double *__restrict__ p;
  double zs;  // +1.0 lower pass, -1.0 upper pass
  __device__ __forceinline__ double x(long long i) const { return p[3 * i]; }
  __device__ __forceinline__ double y(long long i) const { return p[3 * i + 1]; }
  __device__ __forceinline__ double z(long long i) const { return zs * p[3 * i + 2]; }
  __device__ __forceinline__ double evt(long long a, long long b, long long c) const {
    if (a == NIL || b == NIL || c == NIL) return INF;
    return evtime_xyz(x(a), y(a), z(a), x(b), y(b), z(b), x(c), y(c), z(c));
  }
};

}  // namespace h3d
