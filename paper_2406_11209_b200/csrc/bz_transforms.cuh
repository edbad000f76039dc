// bz_transforms.cuh -- factored per-line orthonormal transforms in f64 registers.
//
// Same bases as transforms.py:67-81 (DCT-II entries sqrt((1+(k>0))/s) cos(pi k
// (2n+1)/(2s)); coarse-to-fine Haar), evaluated with even/odd butterflies
// instead of dense s*s products: 36 flops per 8-point DCT instead of 64.
// Results agree with the dense products to a few f64 ulps (different
// rounding order), which SURVEY.md §7.2-1 shows leaves indices bit-exact.
//
// Every function works on v[off + i*stride], i = 0..E-1, with compile-time
// offsets after unrolling, so arrays stay in registers.
#pragma once

namespace bz {

constexpr int DCT = 0, HAAR = 1;

namespace c {
constexpr double R2 = 0.7071067811865475244008444;   // 1/sqrt(2)
constexpr double C4_1 = 0.6532814824381882639283216; // cos(pi/8)/sqrt(2)
constexpr double C4_3 = 0.2705980500730984921998616; // cos(3pi/8)/sqrt(2)
constexpr double K0 = 0.3535533905932737622004222;   // 1/sqrt(8)
constexpr double K1 = 0.4903926402016152245630911;   // cos(k pi/16)/2
constexpr double K2 = 0.4619397662556433780640916;
constexpr double K3 = 0.4157348061512726185393942;
constexpr double K5 = 0.2777851165098011123714154;
constexpr double K6 = 0.19134171618254488586423;
constexpr double K7 = 0.09754516100806413392414243;
}  // namespace c

// ----------------------------------------------------------------- DCT ----
template <int E, int S>
__device__ __forceinline__ void fdct(double* v) {
  if constexpr (E == 1) {
  } else if constexpr (E == 2) {
    double a = v[0], b = v[S];
    v[0] = (a + b) * c::R2;
    v[S] = (a - b) * c::R2;
  } else if constexpr (E == 4) {
    double x0 = v[0], x1 = v[S], x2 = v[2 * S], x3 = v[3 * S];
    double a = x0 + x3, b = x1 + x2, d0 = x0 - x3, d1 = x1 - x2;
    v[0] = (a + b) * 0.5;
    v[2 * S] = (a - b) * 0.5;
    v[S] = __fma_rn(c::C4_1, d0, c::C4_3 * d1);
    v[3 * S] = __fma_rn(c::C4_3, d0, -(c::C4_1 * d1));
  } else if constexpr (E == 8) {
    double e0 = v[0] + v[7 * S], o0 = v[0] - v[7 * S];
    double e1 = v[S] + v[6 * S], o1 = v[S] - v[6 * S];
    double e2 = v[2 * S] + v[5 * S], o2 = v[2 * S] - v[5 * S];
    double e3 = v[3 * S] + v[4 * S], o3 = v[3 * S] - v[4 * S];
    double ee0 = e0 + e3, ee1 = e1 + e2, eo0 = e0 - e3, eo1 = e1 - e2;
    v[0] = (ee0 + ee1) * c::K0;
    v[4 * S] = (ee0 - ee1) * c::K0;
    v[2 * S] = __fma_rn(c::K2, eo0, c::K6 * eo1);
    v[6 * S] = __fma_rn(c::K6, eo0, -(c::K2 * eo1));
    v[S] = __fma_rn(c::K1, o0, __fma_rn(c::K3, o1, __fma_rn(c::K5, o2, c::K7 * o3)));
    v[3 * S] = __fma_rn(c::K3, o0, -__fma_rn(c::K7, o1, __fma_rn(c::K1, o2, c::K5 * o3)));
    v[5 * S] = __fma_rn(c::K5, o0, __fma_rn(-c::K1, o1, __fma_rn(c::K7, o2, c::K3 * o3)));
    v[7 * S] = __fma_rn(c::K7, o0, __fma_rn(-c::K5, o1, __fma_rn(c::K3, o2, -(c::K1 * o3))));
  }
}

template <int E, int S>
__device__ __forceinline__ void idct(double* v) {
  if constexpr (E == 1) {
  } else if constexpr (E == 2) {
    double a = v[0], b = v[S];
    v[0] = (a + b) * c::R2;
    v[S] = (a - b) * c::R2;
  } else if constexpr (E == 4) {
    double X0 = v[0], X1 = v[S], X2 = v[2 * S], X3 = v[3 * S];
    double p = (X0 + X2) * 0.5, q = (X0 - X2) * 0.5;
    double u = __fma_rn(c::C4_1, X1, c::C4_3 * X3);
    double w = __fma_rn(c::C4_3, X1, -(c::C4_1 * X3));
    v[0] = p + u;
    v[3 * S] = p - u;
    v[S] = q + w;
    v[2 * S] = q - w;
  } else if constexpr (E == 8) {
    double X0 = v[0], X1 = v[S], X2 = v[2 * S], X3 = v[3 * S];
    double X4 = v[4 * S], X5 = v[5 * S], X6 = v[6 * S], X7 = v[7 * S];
    double a = (X0 + X4) * c::K0, b = (X0 - X4) * c::K0;
    double p = __fma_rn(c::K2, X2, c::K6 * X6);
    double q = __fma_rn(c::K6, X2, -(c::K2 * X6));
    double E0 = a + p, E3 = a - p, E1 = b + q, E2 = b - q;
    double O0 = __fma_rn(c::K1, X1, __fma_rn(c::K3, X3, __fma_rn(c::K5, X5, c::K7 * X7)));
    double O1 = __fma_rn(c::K3, X1, -__fma_rn(c::K7, X3, __fma_rn(c::K1, X5, c::K5 * X7)));
    double O2 = __fma_rn(c::K5, X1, __fma_rn(-c::K1, X3, __fma_rn(c::K7, X5, c::K3 * X7)));
    double O3 = __fma_rn(c::K7, X1, __fma_rn(-c::K5, X3, __fma_rn(c::K3, X5, -(c::K1 * X7))));
    v[0] = E0 + O0; v[7 * S] = E0 - O0;
    v[S] = E1 + O1; v[6 * S] = E1 - O1;
    v[2 * S] = E2 + O2; v[5 * S] = E2 - O2;
    v[3 * S] = E3 + O3; v[4 * S] = E3 - O3;
  }
}

// ---------------------------------------------------------------- Haar ----
// coarse-to-fine ordering (transforms.py:74-81): C[0] scaling, then levels
// from coarsest to finest; finest wavelets occupy C[E/2 .. E-1].
template <int E, int S>
__device__ __forceinline__ void fhaar(double* v) {
  if constexpr (E > 1) {
    double cur[E], out[E];
#pragma unroll
    for (int i = 0; i < E; ++i) cur[i] = v[i * S];
#pragma unroll
    for (int m = E; m > 1; m >>= 1) {
#pragma unroll
      for (int j = 0; j < m / 2; ++j) {
        double a = cur[2 * j], b = cur[2 * j + 1];
        out[m / 2 + j] = (a - b) * c::R2;
        cur[j] = (a + b) * c::R2;
      }
    }
    out[0] = cur[0];
#pragma unroll
    for (int i = 0; i < E; ++i) v[i * S] = out[i];
  }
}

template <int E, int S>
__device__ __forceinline__ void ihaar(double* v) {
  if constexpr (E > 1) {
    double in[E], cur[E];
#pragma unroll
    for (int i = 0; i < E; ++i) in[i] = v[i * S];
    cur[0] = in[0];
#pragma unroll
    for (int m = 2; m <= E; m <<= 1) {
      double nxt[E];
#pragma unroll
      for (int j = 0; j < m / 2; ++j) {
        double s = cur[j], d = in[m / 2 + j];
        nxt[2 * j] = (s + d) * c::R2;
        nxt[2 * j + 1] = (s - d) * c::R2;
      }
#pragma unroll
      for (int j = 0; j < m; ++j) cur[j] = nxt[j];
    }
#pragma unroll
    for (int i = 0; i < E; ++i) v[i * S] = cur[i];
  }
}

template <int FAM, int E, int S>
__device__ __forceinline__ void fline(double* v) {
  if constexpr (FAM == DCT) fdct<E, S>(v); else fhaar<E, S>(v);
}
template <int FAM, int E, int S>
__device__ __forceinline__ void iline(double* v) {
  if constexpr (FAM == DCT) idct<E, S>(v); else ihaar<E, S>(v);
}

// Transform an E x E plane p[r*E + c] (rows along the slower axis): rows
// first?  The reference contracts axis 0 first (transforms.py:120-125); the
// result is order independent up to rounding, we do the fast axis first.
template <int FAM, int E, bool INV>
__device__ __forceinline__ void plane(double* p) {
#pragma unroll
  for (int r = 0; r < E; ++r) {
    if constexpr (INV) iline<FAM, E, 1>(p + r * E); else fline<FAM, E, 1>(p + r * E);
  }
#pragma unroll
  for (int col = 0; col < E; ++col) {
    if constexpr (INV) iline<FAM, E, E>(p + col); else fline<FAM, E, E>(p + col);
  }
}

}  // namespace bz
