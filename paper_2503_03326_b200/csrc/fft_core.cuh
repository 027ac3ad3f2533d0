// fft_core.cuh — register/shared-memory Stockham FFT for one CTA (sm_100a).
//
// Synthesis direction, unnormalized: X[k] = sum_n x[n] exp(+2 pi i n k / N)
// (fft.hpp:10-17; the reference's radix-2 loop fft.cpp:17-37 computes the
// same transform, so results agree to fp32 rounding).
//
// Plan for length N (power of two, 2..16384): E = min(N, 32) elements per
// thread, T = N / E threads per transform, passes of radix E and a last pass
// of radix N / E^(P-1). Pass 0 loads straight from the caller's source
// (coalesced: thread t takes n = t + r T), middle passes exchange through
// padded shared memory, the last pass stores straight to the caller's sink
// (again coalesced: index b + r Ns). Inner DFTs are radix-2 DIF networks in
// registers with compile-time twiddles; the inter-pass twiddles come from a
// per-N table laid out [r][b mod Ns] so a warp reads consecutive entries.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>
#include <utility>

namespace ocn {
namespace fft {

// ---------------------------------------------------------------- compile-time helpers
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

constexpr int clog2(int n) { return n <= 1 ? 0 : 1 + clog2(n / 2); }
constexpr int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// constexpr sin/cos for compile-time twiddles (Taylor series after reduction
// to [0, pi/4]; exact to < 1e-17 which is far below fp32 rounding).
constexpr double c_sin_small(double x) {
  double x2 = x * x, term = x, sum = x;
  for (int n = 1; n < 14; ++n) {
    term *= -x2 / ((2 * n) * (2 * n + 1));
    sum += term;
  }
  return sum;
}
constexpr double c_cos_small(double x) {
  double x2 = x * x, term = 1.0, sum = 1.0;
  for (int n = 1; n < 14; ++n) {
    term *= -x2 / ((2 * n - 1) * (2 * n));
    sum += term;
  }
  return sum;
}
// cos / sin of 2 pi k / n for integers (exact octant reduction)
constexpr double c_cospi2(int k, int n) {
  k %= n;
  if (k < 0) k += n;
  // angle = 2 pi k / n; reduce by octants using integer arithmetic on 8k / n
  const double pi = 3.14159265358979323846264338327950288;
  // map to [0, 2pi): use symmetries
  if (8 * k <= n) return c_cos_small(2 * pi * k / n);
  if (4 * k <= n) return c_sin_small(2 * pi * (n - 4 * k) / (4.0 * n));  // cos(pi/2 - a)
  if (2 * k <= n) return -c_cospi2(n - 2 * k, 2 * n);                    // cos(pi - a)
  return c_cospi2(n - k, n);                                             // cos(2pi - a)
}
constexpr double c_sinpi2(int k, int n) {
  k %= n;
  if (k < 0) k += n;
  const double pi = 3.14159265358979323846264338327950288;
  if (8 * k <= n) return c_sin_small(2 * pi * k / n);
  if (4 * k <= n) return c_cos_small(2 * pi * (n - 4 * k) / (4.0 * n));
  if (2 * k <= n) return c_sinpi2(n - 2 * k, 2 * n);
  return -c_sinpi2(n - k, n);
}

template <int LEN, int K>
struct Tw {
  static constexpr float c = (float)c_cospi2(K, LEN);
  static constexpr float s = (float)c_sinpi2(K, LEN);
};

// Complex arithmetic on the packed fp32x2 pipe of sm_100 (FADD2 / FMUL2 /
// FFMA2: one instruction per complex add, two per complex multiply; operand
// broadcast, swap and per-half negation are free modifiers). The rounding of
// cmul and the general twiddle matches the scalar fmaf forms exactly.
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(OCN_SCALAR_COMPLEX)
#define OCN_F32X2 1
#endif

__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#ifdef OCN_F32X2
  return __fadd2_rn(a, b);
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
#ifdef OCN_F32X2
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
#ifdef OCN_F32X2
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
#else
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
#endif
}

// x * exp(+2 pi i K / LEN) with the trivial angles special-cased
template <int LEN, int K>
__device__ __forceinline__ float2 twiddle_c(float2 x) {
  constexpr int k = K % LEN;
  if constexpr (k == 0) {
    return x;
  } else if constexpr (4 * k == LEN) {  // *i
    return make_float2(-x.y, x.x);
  } else if constexpr (2 * k == LEN) {  // *-1
    return make_float2(-x.x, -x.y);
  } else if constexpr (4 * k == 3 * LEN) {  // *-i
    return make_float2(x.y, -x.x);
  } else if constexpr (8 * k == LEN) {  // *(1+i)/sqrt2
    constexpr float h = 0.70710678118654752440f;
#ifdef OCN_F32X2
    return __fmul2_rn(__fadd2_rn(make_float2(x.x, x.x), make_float2(-x.y, x.y)), make_float2(h, h));
#else
    return make_float2((x.x - x.y) * h, (x.x + x.y) * h);
#endif
  } else if constexpr (8 * k == 3 * LEN) {  // *(-1+i)/sqrt2
    constexpr float h = 0.70710678118654752440f;
#ifdef OCN_F32X2
    return __fmul2_rn(__fadd2_rn(make_float2(x.y, x.x), make_float2(x.x, -x.y)), make_float2(-h, h));
#else
    return make_float2(-(x.x + x.y) * h, (x.x - x.y) * h);
#endif
  } else {
    constexpr float c = Tw<LEN, k>::c, s = Tw<LEN, k>::s;
#ifdef OCN_F32X2
    return __ffma2_rn(make_float2(x.x, x.x), make_float2(c, s), __fmul2_rn(make_float2(x.y, x.y), make_float2(-s, c)));
#else
    return make_float2(fmaf(x.x, c, -x.y * s), fmaf(x.x, s, x.y * c));
#endif
  }
}

// In-place radix-2 DIF DFT of length R on v[OFF .. OFF+R): natural input,
// output X[m] left in v[OFF + bitrev(m)].
template <int R, int OFF = 0>
__device__ __forceinline__ void dft_dif(float2* v) {
  constexpr int L = clog2(R);
  static_for<0, L>([&](auto si) {
    constexpr int len = R >> decltype(si)::value;
    constexpr int half = len / 2;
    static_for<0, R / len>([&](auto bi) {
      static_for<0, half>([&](auto ki) {
        constexpr int k = decltype(ki)::value;
        constexpr int i0 = OFF + decltype(bi)::value * len + k;
        constexpr int i1 = i0 + half;
        float2 a = v[i0], b = v[i1];
        v[i0] = cadd(a, b);
        v[i1] = twiddle_c<len, k>(csub(a, b));
      });
    });
  });
}

// ---------------------------------------------------------------- plan
template <int N>
struct Plan {
  static_assert(N >= 2 && (N & (N - 1)) == 0, "N must be a power of two");
  static constexpr int E = N >= 32 ? 32 : N;
  static constexpr int T = N / E;
  static constexpr int LOGN = clog2(N), LOGE = clog2(E);
  static constexpr int P = 1 + (LOGN - LOGE + LOGE - 1) / LOGE;  // passes
  static constexpr int radix(int p) {
    return p < P - 1 ? E : N / ipow(E, P - 1);
  }
  static constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
  static constexpr int ns(int p) { return ipow(E, p); }
  // offset of pass p's twiddles in the table (passes 1..P-1)
  static constexpr int tw_offset(int p) {
    int off = 0;
    for (int q = 1; q < p; ++q) off += ns(q) * radix(q);
    return off;
  }
  static constexpr int tw_size() { return tw_offset(P); }
  // padded shared-memory slots per transform
  static constexpr int SMEM = N + N / 32;
};

__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

// Shared stride (float2) between the buffers of the transforms one CTA runs
// side by side, chosen so no half-warp of 64-bit shared accesses has a bank
// conflict in any pass (checked by brute-force simulation of the access
// pattern, tools/fft_banks.py):
//  * transform-major lanes (t fastest, the row kernels): Plan::SMEM itself;
//  * column-major lanes (PC columns per CTA, column index fastest, the column
//    kernels): a half-warp spans min(PC, 16) buffers, so the stride must
//    spread them over distinct bank pairs: odd when PC >= 16, else
//    == 16 / PC (mod 32 / PC).
constexpr int col_stride(int smem, int pc) {
  if (pc >= 16) return smem | 1;
  if (pc <= 1) return smem;
  int s = smem;
  while (s % (32 / pc) != 16 / pc) ++s;
  return s;
}

template <int N, int MIN_THREADS = 256>
struct CtaLaunch {
  using PL = Plan<N>;
  static constexpr int T = PL::T;
  static constexpr int THREADS = T > MIN_THREADS ? T : MIN_THREADS;
  static constexpr int PER_CTA = THREADS / T;  // transforms per CTA
  static constexpr int ROW_STRIDE = PL::SMEM;
  static constexpr int COL_STRIDE = col_stride(PL::SMEM, PER_CTA);
  static constexpr size_t ROW_SMEM_BYTES = PL::P > 1 ? (size_t)PER_CTA * ROW_STRIDE * 8 : 0;
  static constexpr size_t COL_SMEM_BYTES = PL::P > 1 ? (size_t)PER_CTA * COL_STRIDE * 8 : 0;
  static constexpr size_t SMEM_BYTES = ROW_SMEM_BYTES > COL_SMEM_BYTES ? ROW_SMEM_BYTES : COL_SMEM_BYTES;
};

// One CTA-cooperative transform. t in [0, T). `load(n)` returns input element
// n, `store(k, x)` consumes output element k. `sm` = this transform's padded
// shared buffer (Plan<N>::SMEM float2). `tw` = the per-N twiddle table.
// Every thread of the CTA must call this the same number of times (it
// contains __syncthreads when P > 1).
//   WARP     : the T threads of a transform are inside one warp (T <= 32):
//              exchanges synchronise with __syncwarp instead of __syncthreads
//   LOAD_SM  : `load` reads `sm` itself (adds a sync before pass 0 overwrites it)
//   STORE_SM : `store` writes `sm` itself (adds a sync before the last stores)
template <bool WARP, int BAR = 0, int BAR_THREADS = 0>
__device__ __forceinline__ void fft_sync() {
  if constexpr (WARP) __syncwarp();
  else if constexpr (BAR > 0) asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(BAR_THREADS) : "memory");
  else __syncthreads();
}

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// `on_free()` (optional) is called by every thread right after the last
// shared-memory reads of the transform, before the final DFT and stores: from
// then on `sm` may be reused (e.g. refilled by TMA for the next tile).
//   TW_SM    : `tw` points to shared memory (plain loads instead of __ldg)
//   BAR, BAR_THREADS : (!WARP) synchronise on named barrier BAR of BAR_THREADS
//              threads instead of __syncthreads (warp-specialised kernels)
//   SPARSE   : (P > 1) with `edge_only` set at run time, only inputs n < T
//              and n >= N - T (r = 0 and r = E - 1 of every thread) may be
//              nonzero: pass 0 is then the 2-term DFT x_0 + x_{E-1} w^{-m}
//              (a band-limited column: rows [0, R) and (N - R, N), R <= T)
//   on_mid   : (optional, P > 1) called by every thread right after the
//              barrier that follows pass 0 (every thread's pass-0 loads and
//              exchange stores are done)
template <int N, bool WARP = false, bool LOAD_SM = false, bool STORE_SM = false, bool TW_SM = false,
          int BAR = 0, int BAR_THREADS = 0, bool SPARSE = false, class Load, class Store,
          class Free = NoHook, class Mid = NoHook>
__device__ __forceinline__ void cta_fft(int t, float2* sm, const float2* __restrict__ tw,
                                        Load&& load, Store&& store, Free&& on_free = Free{},
                                        bool edge_only = false, Mid&& on_mid = Mid{}) {
  using PL = Plan<N>;
  constexpr int E = PL::E, T = PL::T, P = PL::P;
  static_assert(!WARP || T <= 32, "warp-synchronous FFT needs T <= 32");
  static_assert(!SPARSE || P > 1, "the sparse pass 0 writes the exchange buffer");
  float2 v[E];
  bool pass0_done = false;
  if constexpr (SPARSE) {
    if (edge_only) {
      const float2 x0 = load(t), xl = load(t + (E - 1) * T);
      if constexpr (LOAD_SM) fft_sync<WARP, BAR, BAR_THREADS>();
      static_for<0, E>([&](auto mi) {
        constexpr int m = decltype(mi)::value;
        sm[pad32(t * E + m)] = cadd(x0, twiddle_c<E, ((E - 1) * m) % E>(xl));
      });
      pass0_done = true;
    }
  }
  if (!pass0_done) {
  // ---- pass 0: radix E, Ns = 1, no twiddles
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = load(t + r * T);
  if constexpr (LOAD_SM) fft_sync<WARP, BAR, BAR_THREADS>();
  dft_dif<E>(v);
  }
  if constexpr (P == 1) {
    if constexpr (STORE_SM && !LOAD_SM) fft_sync<WARP, BAR, BAR_THREADS>();
    static_for<0, E>([&](auto ri) {
      constexpr int r = decltype(ri)::value;
      store(r, v[bitrev(r, PL::LOGE)]);
    });
  } else {
    if (!pass0_done)
      static_for<0, E>([&](auto ri) {
        constexpr int r = decltype(ri)::value;
        sm[pad32(t * E + r)] = v[bitrev(r, PL::LOGE)];
      });
    fft_sync<WARP, BAR, BAR_THREADS>();
    on_mid();
    static_for<1, P>([&](auto pi) {
      constexpr int p = decltype(pi)::value;
      constexpr int R = PL::radix(p);
      constexpr int NS = PL::ns(p);
      constexpr int Q = E / R;  // butterflies per thread
      constexpr int LOGR = clog2(R);
      const float2* twp = tw + PL::tw_offset(p);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int b = t + q * T;
        const int bm = b & (NS - 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 x = sm[pad32(b + r * (N / R))];
          if (r > 0) {
            if constexpr (TW_SM) x = cmul(x, twp[r * NS + bm]);
            else x = cmul(x, __ldg(twp + r * NS + bm));
          }
          v[q * R + r] = x;
        }
      }
      if constexpr (p == P - 1) on_free();
      static_for<0, Q>([&](auto qi) {
        constexpr int q = decltype(qi)::value;
        dft_dif<R, q * R>(v);
      });
      if constexpr (p == P - 1) {
        if constexpr (STORE_SM) fft_sync<WARP, BAR, BAR_THREADS>();
        static_for<0, Q>([&](auto qi) {
          constexpr int q = decltype(qi)::value;
          const int b = t + q * T;
          static_for<0, R>([&](auto ri) {
            constexpr int r = decltype(ri)::value;
            store(b + r * NS, v[q * R + bitrev(r, LOGR)]);
          });
        });
      } else {
        fft_sync<WARP, BAR, BAR_THREADS>();
        static_for<0, Q>([&](auto qi) {
          constexpr int q = decltype(qi)::value;
          const int b = t + q * T;
          const int base = (b / NS) * NS * R + (b & (NS - 1));
          static_for<0, R>([&](auto ri) {
            constexpr int r = decltype(ri)::value;
            sm[pad32(base + r * NS)] = v[q * R + bitrev(r, LOGR)];
          });
        });
        fft_sync<WARP, BAR, BAR_THREADS>();
      }
    });
  }
}

}  // namespace fft
}  // namespace ocn
