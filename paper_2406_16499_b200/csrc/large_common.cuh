// Scalar abstraction of the large-problem path: real binary32/binary64 and
// complex64/complex128 (interleaved re, im) with the conjugate of a real
// being the identity, so every kernel is written once with Hermitian
// transposes (the reference's transposes for real data).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mlsb {
namespace lg {

struct cf {
  float x, y;
};
struct cd {
  double x, y;
};

template <class T> struct tr;
template <> struct tr<float> {
  using real = float;
  using wide = double;  // u_r precision twin
  static constexpr bool cplx = false;
};
template <> struct tr<double> {
  using real = double;
  using wide = double;
  static constexpr bool cplx = false;
};
template <> struct tr<cf> {
  using real = float;
  using wide = cd;
  static constexpr bool cplx = true;
};
template <> struct tr<cd> {
  using real = double;
  using wide = cd;
  static constexpr bool cplx = true;
};

__host__ __device__ __forceinline__ float conj_(float a) { return a; }
__host__ __device__ __forceinline__ double conj_(double a) { return a; }
__host__ __device__ __forceinline__ cf conj_(cf a) { return cf{a.x, -a.y}; }
__host__ __device__ __forceinline__ cd conj_(cd a) { return cd{a.x, -a.y}; }

template <class T> __host__ __device__ __forceinline__ T zero() { return T{}; }
template <class T> __host__ __device__ __forceinline__ T one();
template <> __host__ __device__ __forceinline__ float one<float>() { return 1.f; }
template <> __host__ __device__ __forceinline__ double one<double>() { return 1.0; }
template <> __host__ __device__ __forceinline__ cf one<cf>() { return cf{1.f, 0.f}; }
template <> __host__ __device__ __forceinline__ cd one<cd>() { return cd{1.0, 0.0}; }

__host__ __device__ __forceinline__ cf operator+(cf a, cf b) { return cf{a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ cf operator-(cf a, cf b) { return cf{a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ cf operator-(cf a) { return cf{-a.x, -a.y}; }
__host__ __device__ __forceinline__ cf operator*(cf a, cf b) {
  return cf{fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x)};
}
__host__ __device__ __forceinline__ cf operator*(float s, cf b) { return cf{s * b.x, s * b.y}; }
__host__ __device__ __forceinline__ bool operator==(cf a, cf b) { return a.x == b.x && a.y == b.y; }
__host__ __device__ __forceinline__ bool operator!=(cf a, cf b) { return !(a == b); }
__host__ __device__ __forceinline__ cd operator+(cd a, cd b) { return cd{a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ cd operator-(cd a, cd b) { return cd{a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ cd operator-(cd a) { return cd{-a.x, -a.y}; }
__host__ __device__ __forceinline__ cd operator*(cd a, cd b) {
  return cd{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__host__ __device__ __forceinline__ cd operator*(double s, cd b) { return cd{s * b.x, s * b.y}; }
__host__ __device__ __forceinline__ bool operator==(cd a, cd b) { return a.x == b.x && a.y == b.y; }
__host__ __device__ __forceinline__ bool operator!=(cd a, cd b) { return !(a == b); }

// acc += a * b  (one FFMA / DFMA, four for complex)
__device__ __forceinline__ void mac(float& acc, float a, float b) { acc = fmaf(a, b, acc); }
__device__ __forceinline__ void mac(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void mac(cf& acc, cf a, cf b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
__device__ __forceinline__ void mac(cd& acc, cd a, cd b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// |a|^2 in binary64
__device__ __forceinline__ double abs2d(float a) { return double(a) * double(a); }
__device__ __forceinline__ double abs2d(double a) { return a * a; }
__device__ __forceinline__ double abs2d(cf a) { return double(a.x) * a.x + double(a.y) * a.y; }
__device__ __forceinline__ double abs2d(cd a) { return a.x * a.x + a.y * a.y; }

// widening / narrowing
__device__ __forceinline__ double widen(float a) { return double(a); }
__device__ __forceinline__ double widen(double a) { return a; }
__device__ __forceinline__ cd widen(cf a) { return cd{double(a.x), double(a.y)}; }
__device__ __forceinline__ cd widen(cd a) { return a; }
template <class T> __device__ __forceinline__ T narrow(double a);
template <> __device__ __forceinline__ float narrow<float>(double a) { return float(a); }
template <> __device__ __forceinline__ double narrow<double>(double a) { return a; }
template <class T> __device__ __forceinline__ T narrow(cd a);
template <> __device__ __forceinline__ cf narrow<cf>(cd a) { return cf{float(a.x), float(a.y)}; }
template <> __device__ __forceinline__ cd narrow<cd>(cd a) { return a; }

template <class T> __device__ __forceinline__ T scale(typename tr<T>::real s, T a);
template <> __device__ __forceinline__ float scale<float>(float s, float a) { return s * a; }
template <> __device__ __forceinline__ double scale<double>(double s, double a) { return s * a; }
template <> __device__ __forceinline__ cf scale<cf>(float s, cf a) { return cf{s * a.x, s * a.y}; }
template <> __device__ __forceinline__ cd scale<cd>(double s, cd a) { return cd{s * a.x, s * a.y}; }

__device__ __forceinline__ bool finite_(double a) { return isfinite(a); }
__device__ __forceinline__ bool finite_(cd a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ double mag(double a) { return fabs(a); }
__device__ __forceinline__ double mag(cd a) { return hypot(a.x, a.y); }

__device__ __forceinline__ float shfl_xor(float v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ double shfl_xor(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ cf shfl_xor(cf v, int o) {
  return cf{__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o)};
}
__device__ __forceinline__ cd shfl_xor(cd v, int o) {
  return cd{__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o)};
}
// conversions between the factor (FT) and compute (CT) scalars
__device__ __forceinline__ void cvt(float a, float& o) { o = a; }
__device__ __forceinline__ void cvt(float a, double& o) { o = double(a); }
__device__ __forceinline__ void cvt(double a, double& o) { o = a; }
__device__ __forceinline__ void cvt(double a, float& o) { o = float(a); }
__device__ __forceinline__ void cvt(cf a, cf& o) { o = a; }
__device__ __forceinline__ void cvt(cf a, cd& o) { o = cd{double(a.x), double(a.y)}; }
__device__ __forceinline__ void cvt(cd a, cd& o) { o = a; }
__device__ __forceinline__ void cvt(cd a, cf& o) { o = cf{float(a.x), float(a.y)}; }
template <class To, class From> __device__ __forceinline__ To widen_to(From a) {
  To o;
  cvt(a, o);
  return o;
}

__device__ __forceinline__ float cdiv(float a, float b) { return a / b; }
__device__ __forceinline__ double cdiv(double a, double b) { return a / b; }
__device__ __forceinline__ cf cdiv(cf a, cf b) {
  const float den = b.x * b.x + b.y * b.y;
  return cf{(a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den};
}
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  const double den = b.x * b.x + b.y * b.y;
  return cd{(a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den};
}

__device__ __forceinline__ float shfl_idx(float v, int s) { return __shfl_sync(0xffffffffu, v, s); }
__device__ __forceinline__ double shfl_idx(double v, int s) { return __shfl_sync(0xffffffffu, v, s); }
__device__ __forceinline__ cf shfl_idx(cf v, int s) {
  return cf{__shfl_sync(0xffffffffu, v.x, s), __shfl_sync(0xffffffffu, v.y, s)};
}
__device__ __forceinline__ cd shfl_idx(cd v, int s) {
  return cd{__shfl_sync(0xffffffffu, v.x, s), __shfl_sync(0xffffffffu, v.y, s)};
}

template <class T> __device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = v + shfl_xor(v, o);
  return v;
}

}  // namespace lg
}  // namespace mlsb
