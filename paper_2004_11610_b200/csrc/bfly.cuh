// bfly.cuh -- fp64 complex butterflies of the inverse-direction (+) DFT, radices 2, 3, 4, 5, 6, 8, 9
// (shared by the C2R passes, c2r.cu, and the small-operator fused apply, small.cu).
#pragma once
#include <cuda_runtime.h>

namespace xcb {

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_ip(double2 a) { return make_double2(-a.y, a.x); }  // +i a

// Inverse-direction (+) butterflies
__device__ __forceinline__ void bf2(double2* v) {
  double2 t = c_sub(v[0], v[1]);
  v[0] = c_add(v[0], v[1]);
  v[1] = t;
}
__device__ __forceinline__ void bf4(double2& v0, double2& v1, double2& v2, double2& v3) {
  double2 a = c_add(v0, v2), b = c_sub(v0, v2), c = c_add(v1, v3), d = c_ip(c_sub(v1, v3));
  v0 = c_add(a, c);
  v2 = c_sub(a, c);
  v1 = c_add(b, d);
  v3 = c_sub(b, d);
}
__device__ __forceinline__ void bf8(double2* v) {
  const double R2 = 0.70710678118654752440;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  bf4(e0, e1, e2, e3);
  bf4(o0, o1, o2, o3);
  o1 = make_double2(R2 * (o1.x - o1.y), R2 * (o1.y + o1.x));
  o2 = c_ip(o2);
  o3 = make_double2(R2 * (-o3.x - o3.y), R2 * (-o3.y + o3.x));
  v[0] = c_add(e0, o0);
  v[4] = c_sub(e0, o0);
  v[1] = c_add(e1, o1);
  v[5] = c_sub(e1, o1);
  v[2] = c_add(e2, o2);
  v[6] = c_sub(e2, o2);
  v[3] = c_add(e3, o3);
  v[7] = c_sub(e3, o3);
}
__device__ __forceinline__ void bf3(double2* v) {
  const double C = -0.5, SN = 0.86602540378443864676;
  double2 a = c_add(v[1], v[2]), b = c_sub(v[1], v[2]);
  double2 m = make_double2(v[0].x + C * a.x, v[0].y + C * a.y);
  double2 ib = make_double2(-SN * b.y, SN * b.x);
  v[0] = c_add(v[0], a);
  v[1] = c_add(m, ib);
  v[2] = c_sub(m, ib);
}
__device__ __forceinline__ void bf5(double2* v) {
  const double C1 = 0.30901699437494742410, C2 = -0.80901699437494742410;
  const double S1 = 0.95105651629515357212, S2 = 0.58778525229247312917;
  double2 a1 = c_add(v[1], v[4]), b1 = c_sub(v[1], v[4]);
  double2 a2 = c_add(v[2], v[3]), b2 = c_sub(v[2], v[3]);
  double2 x0 = v[0];
  double2 m1 = make_double2(x0.x + C1 * a1.x + C2 * a2.x, x0.y + C1 * a1.y + C2 * a2.y);
  double2 m2 = make_double2(x0.x + C2 * a1.x + C1 * a2.x, x0.y + C2 * a1.y + C1 * a2.y);
  double2 t1 = make_double2(S1 * b1.x + S2 * b2.x, S1 * b1.y + S2 * b2.y);
  double2 t2 = make_double2(S2 * b1.x - S1 * b2.x, S2 * b1.y - S1 * b2.y);
  v[0] = make_double2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
  v[1] = make_double2(m1.x - t1.y, m1.y + t1.x);
  v[4] = make_double2(m1.x + t1.y, m1.y - t1.x);
  v[2] = make_double2(m2.x - t2.y, m2.y + t2.x);
  v[3] = make_double2(m2.x + t2.y, m2.y - t2.x);
}
// 6 = 2 x 3: DFT3 of the even and odd points, odd ones times e^{+i pi k/3}, then radix 2.
__device__ __forceinline__ void bf6(double2* v) {
  const double C = 0.5, SN = 0.86602540378443864676;
  double2 a[3] = {v[0], v[2], v[4]}, b[3] = {v[1], v[3], v[5]};
  bf3(a);
  bf3(b);
  b[1] = make_double2(C * b[1].x - SN * b[1].y, C * b[1].y + SN * b[1].x);     // e^{i pi/3}
  b[2] = make_double2(-C * b[2].x - SN * b[2].y, -C * b[2].y + SN * b[2].x);   // e^{2 i pi/3}
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[k] = c_add(a[k], b[k]);
    v[k + 3] = c_sub(a[k], b[k]);
  }
}
// 9 = 3 x 3: inner DFT3 over m (x[j + 3m]), twiddle e^{+2 pi i j k1 / 9}, outer DFT3 over j,
// output k1 + 3 k2.
__device__ __forceinline__ void bf9(double2* v) {
  const double C1 = 0.76604444311897803520, S1 = 0.64278760968653932632;   // 40 deg
  const double C2 = 0.17364817766693034885, S2 = 0.98480775301220805936;   // 80 deg
  const double C4 = -0.93969262078590838405, S4 = 0.34202014332566873304;  // 160 deg
  double2 A[3][3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    A[j][0] = v[j];
    A[j][1] = v[j + 3];
    A[j][2] = v[j + 6];
    bf3(A[j]);
  }
  A[1][1] = c_mul(A[1][1], make_double2(C1, S1));
  A[1][2] = c_mul(A[1][2], make_double2(C2, S2));
  A[2][1] = c_mul(A[2][1], make_double2(C2, S2));
  A[2][2] = c_mul(A[2][2], make_double2(C4, S4));
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    double2 t[3] = {A[0][k1], A[1][k1], A[2][k1]};
    bf3(t);
    v[k1] = t[0];
    v[k1 + 3] = t[1];
    v[k1 + 6] = t[2];
  }
}
template <int r>
__device__ __forceinline__ void bfly(double2* v) {
  if (r == 2) bf2(v);
  else if (r == 3) bf3(v);
  else if (r == 4) bf4(v[0], v[1], v[2], v[3]);
  else if (r == 5) bf5(v);
  else if (r == 6) bf6(v);
  else if (r == 9) bf9(v);
  else bf8(v);
}


}  // namespace xcb
