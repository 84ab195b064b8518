// Length-4096 complex transform in three radix-16 passes (four-step, 4096 = 16 x 16 x 16) for 256
// threads, with the data in registers at entry and exit.
//
// Thread t holds x[t + 256 m], m = 0..15, on entry and X[t + 256 m] on exit (the same
// distribution), so a transform can start from global loads or a gather's registers, and an
// inverse transform can follow a forward one's consumer without a shared-memory round trip. The
// passes exchange through one shared buffer of kFFT16Buf complex values (two exchanges, against
// five read-write rounds -- bit reversal plus four radix-8 passes -- of fft_block):
//
//   n = 256 n1 + 16 a + b,  k = k1 + 16 c1 + 256 c2
//   A: thread t = 16 a + b: DFT16 over n1 of x[t + 256 n1] -> k1; times w4096^{t k1};
//      Y[k1][t]                                            (k1-major, contiguous in t)
//   B: thread (k1, b) = (t >> 4, t & 15): DFT16 over a of Y[k1][16 a + b] -> c1; times
//      w256^{b c1}; U[c1][k1][b] at c1 * 272 + k1 * 17 + b (pitch 17: conflict-free in C)
//   C: thread (c1, k1) = (t >> 4, t & 15): DFT16 over b of U[c1][k1][b] -> c2; X[k1 + 16 c1 + 256 c2]
//      = X[t + 256 c2]
//
// Every shared access of a warp covers contiguous runs of 16 complex values (A, B) or a 17-pitch
// column (C), i.e. the minimum four wavefronts per 512 bytes. Twiddles: one root-table load per pass
// and thread, powers by repeated multiplication (<= 15 products: a few ulp, far inside the 1e-10
// parity bar). Unnormalised; INV uses the conjugate roots, like fft_block. `bar` is the named
// barrier the 256 participating threads synchronise on (two transforms can run side by side in one
// CTA on two halves, each with its own buffer and barrier id).
#pragma once
#include "fft.cuh"

namespace apx {

constexpr int kFFT16Buf = 16 * 16 * 17;  // complex values of the exchange buffer (68 KB)

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// 4-point DFT in place: forward w4 = -i, inverse +i
template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = csub(x1, x3);
  // -i * d13 (forward) / +i * d13 (inverse)
  const double2 r13 = INV ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, r13);
  x3 = csub(d02, r13);
}

// 16-point DFT in place, natural order in and out (radix 4 x 4: j = 4 j1 + j2, k = k1 + 4 k2)
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;  // cos, sin(pi / 8)
  constexpr double r2 = 0.70710678118654752440;
  constexpr double sg = INV ? 1.0 : -1.0;  // w16^m = cos(2 pi m / 16) + sg i sin(2 pi m / 16)
#pragma unroll
  for (int j2 = 0; j2 < 4; ++j2) dft4<INV>(v[j2], v[4 + j2], v[8 + j2], v[12 + j2]);  // over j1 -> k1
  // twiddles w16^{j2 k1}: v[4 k1 + j2] now holds a[j2][k1]
  auto tw = [&](double2& x, double c, double s) { x = make_double2(x.x * c - x.y * s, x.x * s + x.y * c); };
  // m = 1: (c1, sg s1), 2: (r2, sg r2), 3: (s1, sg c1), 4: (0, sg), 6: (-r2, sg r2), 9: (-c1, -sg s1)
  tw(v[4 + 1], c1, sg * s1);   // k1 = 1, j2 = 1: m = 1
  tw(v[4 + 2], r2, sg * r2);   // k1 = 1, j2 = 2: m = 2
  tw(v[4 + 3], s1, sg * c1);   // k1 = 1, j2 = 3: m = 3
  tw(v[8 + 1], r2, sg * r2);   // k1 = 2, j2 = 1: m = 2
  v[8 + 2] = INV ? make_double2(-v[8 + 2].y, v[8 + 2].x) : make_double2(v[8 + 2].y, -v[8 + 2].x);  // m = 4
  tw(v[8 + 3], -r2, sg * r2);  // k1 = 2, j2 = 3: m = 6
  tw(v[12 + 1], s1, sg * c1);  // k1 = 3, j2 = 1: m = 3
  tw(v[12 + 2], -r2, sg * r2); // k1 = 3, j2 = 2: m = 6
  tw(v[12 + 3], -c1, -sg * s1);  // k1 = 3, j2 = 3: m = 9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);  // over j2
  // v[4 k1 + k2] holds X[k1 + 4 k2]: transpose the 4 x 4 index grid
  double2 t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[4 * k1 + k2];
}

// 8-point DFT in place, natural order in and out (even/odd split into two 4-point DFTs)
template <bool INV>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  constexpr double r2 = 0.70710678118654752440;
  constexpr double sg = INV ? 1.0 : -1.0;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  // o_k *= w8^k: w8 = (r2, sg r2), w8^2 = (0, sg), w8^3 = (-r2, sg r2)
  o1 = make_double2(r2 * (o1.x - sg * o1.y), r2 * (sg * o1.x + o1.y));
  o2 = INV ? make_double2(-o2.y, o2.x) : make_double2(o2.y, -o2.x);
  o3 = make_double2(r2 * (-o3.x - sg * o3.y), r2 * (sg * o3.x - o3.y));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3);
  v[7] = csub(e3, o3);
}

// v[i] *= w^i, i = 0..15, w = roots[idx] (conjugated for INV)
template <bool INV, int N = 16>
__device__ __forceinline__ void twiddle_powers(double2 (&v)[N], const double2* __restrict__ roots, int idx) {
  double2 w = __ldg(roots + idx);
  if (INV) w.y = -w.y;
  double2 p = w;
#pragma unroll
  for (int i = 1; i < N; ++i) {
    v[i] = cmul(v[i], p);
    if (i < N - 1) p = cmul(p, w);
  }
}

template <bool INV>
__device__ __forceinline__ void fft4096_r16(double2 (&v)[16], double2* __restrict__ buf,
                                            const double2* __restrict__ roots, int t, int bar) {
  // pass A
  dft16<INV>(v);
  twiddle_powers<INV>(v, roots, t);  // w4096^{t k1}
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + t] = v[k1];
  named_bar(bar, 256);
  // pass B
  const int hi = t >> 4, lo = t & 15;
#pragma unroll
  for (int a = 0; a < 16; ++a) v[a] = buf[hi * 256 + 16 * a + lo];
  named_bar(bar, 256);  // every Y read done before U overwrites the buffer
  dft16<INV>(v);
  twiddle_powers<INV>(v, roots, 16 * lo);  // w256^{b c1}, b = lo
#pragma unroll
  for (int c1 = 0; c1 < 16; ++c1) buf[c1 * 272 + hi * 17 + lo] = v[c1];
  named_bar(bar, 256);
  // pass C: thread t = (c1, k1) = (hi, lo)
#pragma unroll
  for (int b = 0; b < 16; ++b) v[b] = buf[hi * 272 + lo * 17 + b];
  dft16<INV>(v);
  named_bar(bar, 256);  // the buffer may be reused by the caller
}

}  // namespace apx
