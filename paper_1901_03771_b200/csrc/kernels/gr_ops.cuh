// gr_ops.cuh — hand-written device-function templates for the point program.
//
// One function per ElemCode with NumPy's
// semantics, so a fused region computes what the eager NumPy baseline computes
// ("semantics ... match the corresponding numpy operations"):
//   * IEEE +,-,*,/ and sqrt, never contracted (NVRTC --fmad=false) and never
//     flushed (no fast-math): bit-identical to NumPy on x86;
//   * maximum/minimum propagate NaN and return the second operand on ties
//     (np.maximum(-0.,0.) == 0., np.maximum(0.,-0.) == -0.);
//   * integer +,-,* wrap (two's complement); // and % follow Python floor
//     semantics with x//0 == x%0 == 0 as NumPy does;
//   * float->int casts reproduce x86 cvtt*: NaN/out-of-range -> INT_MIN;
//   * transcendentals use CUDA's accurate (non-intrinsic) libm: within a few
//     ulp of NumPy/SciPy, not bit-identical (tolerances in DESIGN.md).
// Compiled by NVRTC together with the generated region source; no system
// headers are used so compilation stays fast.
#pragma once

namespace gr {

typedef long long i64;
typedef unsigned long long u64;

template <class T> struct is_float { static constexpr bool value = false; };
template <> struct is_float<float> { static constexpr bool value = true; };
template <> struct is_float<double> { static constexpr bool value = true; };

// ---- casts (Op CAST, ufunc loop casts) ------------------------------------
template <class To, class From> struct Cast {
  static __device__ __forceinline__ To run(From x) { return (To)x; }
};
template <class From> struct Cast<bool, From> {
  static __device__ __forceinline__ bool run(From x) { return x != From(0); }
};
template <> struct Cast<bool, bool> {
  static __device__ __forceinline__ bool run(bool x) { return x; }
};
#define GR_F2I(FT, IT, MINV)                                                \
  template <> struct Cast<IT, FT> {                                         \
    static __device__ __forceinline__ IT run(FT x) {                        \
      FT t = trunc(x);                                                      \
      const FT lo = (FT)(MINV);                                             \
      return (t >= lo && t < -lo) ? (IT)t : (IT)(MINV);                     \
    }                                                                       \
  };
GR_F2I(float, int, (-2147483647 - 1))
GR_F2I(double, int, (-2147483647 - 1))
GR_F2I(float, i64, (-9223372036854775807LL - 1))
GR_F2I(double, i64, (-9223372036854775807LL - 1))
#undef GR_F2I
template <class To, class From> __device__ __forceinline__ To cast(From x) { return Cast<To, From>::run(x); }

// ---- arithmetic -----------------------------------------------------------
template <class T> __device__ __forceinline__ T add(T a, T b) { return a + b; }
template <> __device__ __forceinline__ int add(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
template <> __device__ __forceinline__ i64 add(i64 a, i64 b) { return (i64)((u64)a + (u64)b); }
template <> __device__ __forceinline__ bool add(bool a, bool b) { return a || b; }

template <class T> __device__ __forceinline__ T sub(T a, T b) { return a - b; }
template <> __device__ __forceinline__ int sub(int a, int b) { return (int)((unsigned)a - (unsigned)b); }
template <> __device__ __forceinline__ i64 sub(i64 a, i64 b) { return (i64)((u64)a - (u64)b); }

template <class T> __device__ __forceinline__ T mul(T a, T b) { return a * b; }
template <> __device__ __forceinline__ int mul(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
template <> __device__ __forceinline__ i64 mul(i64 a, i64 b) { return (i64)((u64)a * (u64)b); }
template <> __device__ __forceinline__ bool mul(bool a, bool b) { return a && b; }

template <class T> __device__ __forceinline__ T div(T a, T b) { return a / b; }

// Division by a divisor shared by many dividends (a row's std, a constant):
// r = RN(1/s) once, then per element Markstein's correction
//   q0 = RN(x*r); e = x - q0*s (exact with FMA); q = RN(q0 + e*r)
// which is the correctly rounded x/s whenever no intermediate leaves the
// normal range (Markstein 1990).  Outside a conservative exponent window (and
// for zeros, inf, NaN) the IEEE division is used, so the result is always
// bit-identical to x / s.
template <class T> struct DivWin;
template <> struct DivWin<float> {
  static __device__ __forceinline__ float lo() { return 7.8886091e-31f; }   // 2^-100
  static __device__ __forceinline__ float hi() { return 1.2676506e+30f; }   // 2^100
};
template <> struct DivWin<double> {
  static __device__ __forceinline__ double lo() { return 1.4916681462400413e-154; }  // 2^-510
  static __device__ __forceinline__ double hi() { return 6.7039039649712985e+153; }  // 2^510
};
template <class T> struct DivShared {
  T s, r, xlo, xhi;   // |x| in [xlo, xhi]  =>  x, q and the residual stay normal
};
template <class T> __device__ __forceinline__ DivShared<T> div_prep(T s) {
  DivShared<T> d;
  const T as = s < T(0) ? -s : s;
  d.s = s;
  if (as >= DivWin<T>::lo() && as <= DivWin<T>::hi()) {
    d.r = T(1) / s;
    const T a = DivWin<T>::lo() * as * T(4), b = DivWin<T>::hi() * as * T(0.25);
    d.xlo = a > DivWin<T>::lo() ? a : DivWin<T>::lo();
    d.xhi = b < DivWin<T>::hi() ? b : DivWin<T>::hi();
  } else {
    d.r = T(0);
    d.xlo = T(1);
    d.xhi = T(0);  // empty window: always the IEEE path
  }
  return d;
}
__device__ __noinline__ float div_slow(float x, float s) { return x / s; }
__device__ __noinline__ double div_slow(double x, double s) { return x / s; }
template <class T> __device__ __forceinline__ T div_shared(T x, const DivShared<T>& d) {
  const T q0 = x * d.r;
  const T e = fma(-q0, d.s, x);
  const T q = fma(e, d.r, q0);
  const T ax = fabs(x);
  return (ax >= d.xlo && ax <= d.xhi) ? q : div_slow(x, d.s);
}
// Two-pass form for kernels that can redo a work item: the FAST pass returns
// the Markstein quotient and only records (branch-free) whether any dividend
// fell outside the window; the caller then re-runs the whole item with
// FAST=false (exact per-element IEEE fallback) when any thread saw one.  No
// per-element branch or call in the hot pass.
template <bool FAST, class T>
__device__ __forceinline__ T div_sh(T x, const DivShared<T>& d, bool& bad) {
  if constexpr (FAST) {
    const T q0 = x * d.r;
    const T e = fma(-q0, d.s, x);
    const T q = fma(e, d.r, q0);
#ifndef GR_DIVSH_NOCHECK   // experiments only (tools/variant_bench.py)
    const T ax = fabs(x);
    bad |= !(ax >= d.xlo && ax <= d.xhi);
#endif
    return q;
  } else {
    (void)bad;
    return div_shared<T>(x, d);
  }
}

// Per-row accumulator of the fast pass's dividend range: two FMNMX per
// element instead of a two-sided window test; the row is flagged once at the
// end if any |dividend| left [xlo, xhi].  (NaN dividends give NaN quotients
// either way.)
template <class T> struct DivRange {
  T amin, amax;
};
template <class T> __device__ __forceinline__ DivRange<T> div_range_init() {
  return {T(__int_as_float(0x7f800000)), T(0)};
}
template <bool FAST, class T>
__device__ __forceinline__ T div_shr(T x, const DivShared<T>& d, DivRange<T>& w) {
  if constexpr (FAST) {
    const T q0 = x * d.r;
    const T e = fma(-q0, d.s, x);
    const T q = fma(e, d.r, q0);
    const T ax = fabs(x);
    w.amin = fmin(w.amin, ax);
    w.amax = fmax(w.amax, ax);
    return q;
  } else {
    (void)w;
    return div_shared<T>(x, d);
  }
}
template <class T> __device__ __forceinline__ bool div_range_bad(const DivRange<T>& w, const DivShared<T>& d) {
  return !(w.amin >= d.xlo && w.amax <= d.xhi);
}

// fused multiply-add for inexact regions (codegen.inexact_region): one
// rounding of a*b+c where NumPy rounds the product and the sum separately
__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }

template <class T> __device__ __forceinline__ T neg(T a) { return -a; }
template <> __device__ __forceinline__ int neg(int a) { return (int)(0u - (unsigned)a); }
template <> __device__ __forceinline__ i64 neg(i64 a) { return (i64)(0ull - (u64)a); }

template <class T> __device__ __forceinline__ T square(T a) { return mul<T>(a, a); }

__device__ __forceinline__ float abs_(float a) { return fabsf(a); }
__device__ __forceinline__ double abs_(double a) { return fabs(a); }
__device__ __forceinline__ int abs_(int a) { return a < 0 ? neg<int>(a) : a; }
__device__ __forceinline__ i64 abs_(i64 a) { return a < 0 ? neg<i64>(a) : a; }
__device__ __forceinline__ bool abs_(bool a) { return a; }

// npy_divmod (numpy/_core/src/npymath/npy_math_internal.h.src)
template <class T> __device__ __forceinline__ T fdivmod(T a, T b, T* modulus) {
  T mod = fmod(a, b);
  if (b == T(0)) {
    *modulus = mod;
    return a / b;
  }
  T dv = (a - mod) / b;
  if (mod != T(0)) {
    if ((b < T(0)) != (mod < T(0))) {
      mod += b;
      dv -= T(1);
    }
  } else {
    mod = copysign(T(0), b);
  }
  T fl;
  if (dv != T(0)) {
    fl = floor(dv);
    if (dv - fl > T(0.5)) fl += T(1);
  } else {
    fl = copysign(T(0), a / b);
  }
  *modulus = mod;
  return fl;
}
template <class T> __device__ __forceinline__ T floordiv(T a, T b) {
  // integers: Python floor division, x // 0 == 0, INT_MIN // -1 wraps
  if (b == T(0)) return T(0);
  if (b == T(-1)) return neg<T>(a);
  T q = a / b;
  if ((a % b != T(0)) && ((a < T(0)) != (b < T(0)))) q -= T(1);
  return q;
}
template <> __device__ __forceinline__ float floordiv(float a, float b) { float m; return fdivmod<float>(a, b, &m); }
template <> __device__ __forceinline__ double floordiv(double a, double b) { double m; return fdivmod<double>(a, b, &m); }

template <class T> __device__ __forceinline__ T mod(T a, T b) {
  if (b == T(0) || b == T(-1)) return T(0);
  T r = a % b;
  if (r != T(0) && ((r < T(0)) != (b < T(0)))) r += b;
  return r;
}
template <> __device__ __forceinline__ float mod(float a, float b) { float m; fdivmod<float>(a, b, &m); return m; }
template <> __device__ __forceinline__ double mod(double a, double b) { double m; fdivmod<double>(a, b, &m); return m; }

template <class T> __device__ __forceinline__ T pow_(T a, T b) {
  // integer power by squaring (wraps); negative exponents give 0 (NumPy raises)
  if (b < T(0)) return T(0);
  T r = T(1), base = a;
  u64 e = (u64)b;
  while (e) {
    if (e & 1) r = mul<T>(r, base);
    base = mul<T>(base, base);
    e >>= 1;
  }
  return r;
}
template <> __device__ __forceinline__ float pow_(float a, float b) { return powf(a, b); }
template <> __device__ __forceinline__ double pow_(double a, double b) { return pow(a, b); }

// NaN-propagating, second-operand-on-tie (np.maximum / np.minimum)
template <class T> __device__ __forceinline__ T maximum(T a, T b) { return (a > b || a != a) ? a : b; }
template <class T> __device__ __forceinline__ T minimum(T a, T b) { return (a < b || a != a) ? a : b; }

// ---- transcendentals (accurate libm; not intrinsics) ------------------------
__device__ __forceinline__ float exp_(float a) { return expf(a); }
__device__ __forceinline__ double exp_(double a) { return exp(a); }
__device__ __forceinline__ float log_(float a) { return logf(a); }
__device__ __forceinline__ double log_(double a) { return log(a); }
__device__ __forceinline__ float sqrt_(float a) { return sqrtf(a); }  // IEEE (prec-sqrt)
// inexact regions (codegen.inexact_region, FAST_DIV): full-range 2-ulp
// division (div.full.f32: MUFU.RCP + scaling, no Newton steps, no FCHK
// slow path) and the MUFU square root (sqrt.approx.f32, ~1 ulp, subnormals
// kept) — error of the same class as the libm transcendentals the region
// already carries
// Debug runs (GRUMPY_DEBUG_BOUNDS=1): a leaf read outside [0, n) prints the
// leaf slot and offset and traps ("bounds-checked in debug runs").
__device__ __noinline__ bool bounds_ok(long long off, long long n, int leaf) {
  if ((unsigned long long)off >= (unsigned long long)n) {
    printf("grumpy: leaf %d read at %lld, outside [0, %lld)\n", leaf, off, n);
    __trap();
  }
  return true;
}

__device__ __forceinline__ float div_full(float a, float b) {
  float r;
  asm("div.full.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float a) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double sqrt_(double a) { return sqrt(a); }
__device__ __forceinline__ float sin_(float a) { return sinf(a); }
__device__ __forceinline__ double sin_(double a) { return sin(a); }
__device__ __forceinline__ float cos_(float a) { return cosf(a); }
__device__ __forceinline__ double cos_(double a) { return cos(a); }
__device__ __forceinline__ float tanh_(float a) { return tanhf(a); }
__device__ __forceinline__ double tanh_(double a) { return tanh(a); }
__device__ __forceinline__ float erf_(float a) { return erff(a); }
__device__ __forceinline__ double erf_(double a) { return erf(a); }
__device__ __forceinline__ float floor_(float a) { return floorf(a); }
__device__ __forceinline__ double floor_(double a) { return floor(a); }
__device__ __forceinline__ float ceil_(float a) { return ceilf(a); }
__device__ __forceinline__ double ceil_(double a) { return ceil(a); }
template <class T> __device__ __forceinline__ T floor_(T a) { return a; }
template <class T> __device__ __forceinline__ T ceil_(T a) { return a; }
template <class T> __device__ __forceinline__ bool isnan_(T a) { return a != a; }

// ---- comparisons / logic ----------------------------------------------------
template <class T> __device__ __forceinline__ bool lt(T a, T b) { return a < b; }
template <class T> __device__ __forceinline__ bool gt(T a, T b) { return a > b; }
template <class T> __device__ __forceinline__ bool le(T a, T b) { return a <= b; }
template <class T> __device__ __forceinline__ bool ge(T a, T b) { return a >= b; }
template <class T> __device__ __forceinline__ bool eq(T a, T b) { return a == b; }
template <class T> __device__ __forceinline__ bool ne(T a, T b) { return a != b; }
template <class T> __device__ __forceinline__ bool land(T a, T b) { return (a != T(0)) && (b != T(0)); }
template <class T> __device__ __forceinline__ bool lor(T a, T b) { return (a != T(0)) || (b != T(0)); }
template <class T> __device__ __forceinline__ bool lxor(T a, T b) { return (a != T(0)) != (b != T(0)); }
template <class T> __device__ __forceinline__ bool lnot(T a) { return !(a != T(0)); }
template <class T> __device__ __forceinline__ T select(bool c, T a, T b) { return c ? a : b; }

// clamp an index into [0, hi] (slice-assign value branch stays in bounds)
__device__ __forceinline__ long long clampll(long long x, long long hi) { return x < 0 ? 0 : (x > hi ? hi : x); }

// ---- bit-exact constants ----------------------------------------------------
__device__ __forceinline__ float f32_bits(unsigned u) { return __uint_as_float(u); }
__device__ __forceinline__ double f64_bits(u64 u) { return __longlong_as_double((i64)u); }

}  // namespace gr
