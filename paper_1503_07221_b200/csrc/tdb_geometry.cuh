// Geometry primitives shared by the assembly (tdb_assembly.cu) and the
// potential (tdb_potential.cu).  Every operation is an explicitly rounded IEEE
// op in the evaluation order numpy uses in the reference (mesh.py:286-354), so
// distances are bitwise identical to the reference's.
#pragma once

#include <cuda_runtime.h>

namespace tdb {

struct V3 {
  double x, y, z;
};
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {sub_(a.x, b.x), sub_(a.y, b.y), sub_(a.z, b.z)}; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {add_(a.x, b.x), add_(a.y, b.y), add_(a.z, b.z)}; }
__device__ __forceinline__ V3 vscale(double s, V3 a) { return {mul_(s, a.x), mul_(s, a.y), mul_(s, a.z)}; }
// numpy einsum('ij,ij->i') order
__device__ __forceinline__ double edot(V3 a, V3 b) {
  return add_(add_(mul_(a.x, b.x), mul_(a.z, b.z)), mul_(a.y, b.y));
}
// numpy linalg.norm(axis=-1) order
__device__ __forceinline__ double enorm(V3 d) {
  return sqrt(add_(add_(mul_(d.x, d.x), mul_(d.y, d.y)), mul_(d.z, d.z)));
}
__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
__device__ __forceinline__ V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }

__device__ inline double seg_seg(V3 p0, V3 p1, V3 q0, V3 q1) {
  V3 d1 = vsub(p1, p0), d2 = vsub(q1, q0), r = vsub(p0, q0);
  double a = edot(d1, d1), e = edot(d2, d2), b = edot(d1, d2), c = edot(d1, r), f = edot(d2, r);
  double den = sub_(mul_(a, e), mul_(b, b));
  double as = a > 0 ? a : 1.0, es = e > 0 ? e : 1.0;
  double s = den > 0.0 ? clip01(sub_(mul_(b, f), mul_(c, e)) / den) : 0.0;
  double t = add_(mul_(b, s), f) / es;
  if (t < 0.0) s = clip01(-c / as);
  if (t > 1.0) s = clip01(sub_(b, c) / as);
  t = e > 0.0 ? clip01(t) : 0.0;
  s = a > 0.0 ? s : 0.0;
  return enorm(vsub(vadd(p0, vscale(s, d1)), vadd(q0, vscale(t, d2))));
}

__device__ inline double pt_seg(V3 p, V3 a, V3 b) {
  V3 ab = vsub(b, a);
  double den = edot(ab, ab);
  double t = edot(vsub(p, a), ab) / (den > 0 ? den : 1.0);
  t = den > 0.0 ? clip01(t) : 0.0;
  return enorm(vsub(vsub(p, a), vscale(t, ab)));
}

__device__ inline double pt_tri(V3 p, V3 v0, V3 v1, V3 v2) {
  V3 e0 = vsub(v1, v0), e1 = vsub(v2, v0);
  V3 n = {sub_(mul_(e0.y, e1.z), mul_(e0.z, e1.y)), sub_(mul_(e0.z, e1.x), mul_(e0.x, e1.z)),
          sub_(mul_(e0.x, e1.y), mul_(e0.y, e1.x))};
  double nn = edot(n, n);
  V3 w = vsub(p, v0);
  double dplane = fabs(edot(w, n)) / sqrt(nn > 0 ? nn : 1.0);
  double d00 = edot(e0, e0), d01 = edot(e0, e1), d11 = edot(e1, e1), d20 = edot(w, e0), d21 = edot(w, e1);
  double den = sub_(mul_(d00, d11), mul_(d01, d01));
  double dens = den > 0 ? den : 1.0;
  double u = sub_(mul_(d11, d20), mul_(d01, d21)) / dens;
  double v = sub_(mul_(d00, d21), mul_(d01, d20)) / dens;
  bool inside = u >= 0.0 && v >= 0.0 && add_(u, v) <= 1.0 && den > 0.0 && nn > 0.0;
  if (inside) return dplane;
  return fmin(fmin(pt_seg(p, v0, v1), pt_seg(p, v1, v2)), pt_seg(p, v2, v0));
}

__device__ __forceinline__ V3 corner(const double* __restrict__ corners, int e, int a) {
  const double* c = corners + 9 * (long long)e + 3 * a;
  return {c[0], c[1], c[2]};
}

}  // namespace tdb
