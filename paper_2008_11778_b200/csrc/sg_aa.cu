// sg_aa.cu -- Anderson-acceleration window (seisopt/optim/anderson.py:55-148,
// seisopt/optim/qr.py:22-104) and the device vector helpers of the optimizer
// loop (anderson.py:283-376).
//
// B200 design: the reference keeps an explicit thin QR (Q: N x m) and updates
// it by CGS2 appends and Givens drops, ~6 m N words of traffic per iteration.
// Here the window is a ring of m residual-difference columns DF and G
// differences DG, plus an fp64 Gram matrix DF^T DF that one fused pass per
// push extends (new row + projections of f_k), reading each stored column once
// with fp64 accumulation.  The m x m problem (Cholesky, rank safeguard,
// least-squares solve, alpha recovery) runs on the host in fp64 and reproduces
// the reference's window decisions; the recombination is one more fused pass.
// Per iteration: (m+4) reads + 4 writes (push) and (m+1) reads + 1 write
// (step) of N-vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "seisgpu.h"
#include "sg_common.cuh"

using namespace sg;

namespace {

constexpr int kMaxMem = 32;  // largest supported AA memory
constexpr int kThreads = 256;
constexpr int kBlocks = 148 * 8;

struct Slots {
  int s[kMaxMem];
};
struct Coefs {
  double c[kMaxMem];
};

// 16-byte vectors: 4 floats or 2 doubles per load
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int W = 4;
  __device__ __forceinline__ static float get(const float4& v, int l) {
    return l == 0 ? v.x : l == 1 ? v.y : l == 2 ? v.z : v.w;
  }
  __device__ __forceinline__ static void set(float4& v, int l, float x) {
    if (l == 0) v.x = x; else if (l == 1) v.y = x; else if (l == 2) v.z = x; else v.w = x;
  }
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int W = 2;
  __device__ __forceinline__ static double get(const double2& v, int l) { return l == 0 ? v.x : v.y; }
  __device__ __forceinline__ static void set(double2& v, int l, double x) {
    if (l == 0) v.x = x; else v.y = x;
  }
};

// fused push: f_k = g - p; df = f_k - f_prev; dg = g - g_prev; store df, dg
// into slot `snew`; f_prev <- f_k, g_prev <- g; partial dots
//   [0..nw)   <df, DF_i>
//   nw        <df, df>
//   nw + 1    <f_k, df>
//   nw + 2    <f_k, f_k>
// The projections <f_k, DF_i> of the surviving columns follow on the host
// from <f_{k-1}, DF_i> + <df, DF_i>, so one accumulator per column suffices.
// first != 0: only f_prev/g_prev are written and <f_k, f_k> reduced.
// Element k of the vectorised loop covers elements [k*W, k*W + W); the tail
// n % W (and every element when VEC is false) runs the scalar loop.
// Windows of up to 12 columns load every column of an element before the
// stores (kHoist, 2 CTAs/SM for the registers): C2 push 0.70 -> 0.55 ms
// (5.1 -> 6.5 TB/s); wider windows keep the load-after-store order at 4 CTAs/SM.
// Windows wider than 12 columns keep 4 CTAs/SM: 2 CTAs/SM removes their
// accumulator spills but was slower (m = 20 push 2.01 vs 1.27 ms,
// profiles/r01e_ab_aa_wide.log).
#ifndef SG_AA_WIDE_MINB
#define SG_AA_WIDE_MINB 4
#endif
template <int MW, bool VEC>
struct PushCfg {
  static constexpr bool kHoist = VEC && MW <= 12;
  static constexpr int kMinBlocks = kHoist ? 2 : (MW > 12 ? SG_AA_WIDE_MINB : 4);
};

template <typename T, int MW, bool VEC>
__global__ void __launch_bounds__(kThreads, (PushCfg<MW, VEC>::kMinBlocks))
    k_aa_push(const T* __restrict__ p, const T* __restrict__ g, T* __restrict__ fprev,
              T* __restrict__ gprev, T* __restrict__ DF, T* __restrict__ DG, int64_t n,
              int64_t ld, const Slots slots, int nw, int snew, int first,
              double* __restrict__ part) {
  using VT = Vec<T>;
  using V = typename VT::type;
  constexpr int W = VEC ? VT::W : 1;
  constexpr bool kHoist = PushCfg<MW, VEC>::kHoist;
  double a_dd[MW];
#pragma unroll
  for (int i = 0; i < MW; ++i) a_dd[i] = 0.0;
  double dd = 0.0, fd = 0.0, ff = 0.0;
  T* dfn = DF + (int64_t)snew * ld;
  T* dgn = DG + (int64_t)snew * ld;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = n / W;
  auto body = [&](T gv, T pv, T fpv, T gpv, T& df_out, T& dg_out, T& fk_out) {
    const T fk = gv - pv;  // seisopt/optim/anderson.py:84
    const T df = fk - fpv; // anderson.py:89
    df_out = df;
    dg_out = gv - gpv;     // anderson.py:90
    fk_out = fk;
  };
  if (VEC) {
    for (int64_t e = gtid; e < nv; e += gstride) {
      const V gv = reinterpret_cast<const V*>(g)[e];
      const V pv = reinterpret_cast<const V*>(p)[e];
      V fpv = reinterpret_cast<const V*>(fprev)[e];
      V gpv = reinterpret_cast<const V*>(gprev)[e];
      V dfv, dgv, fkv;
      // every column load of this element issued before the stores below:
      // the new column's slot lies in DF too, so loads written after its
      // store could not be hoisted above it (two memory round trips per
      // iteration instead of one)
      V cols[kHoist ? MW : 1];
      if (kHoist && !first) {
#pragma unroll
        for (int i = 0; i < MW; ++i)
          if (i < nw) cols[i] = reinterpret_cast<const V*>(DF + (int64_t)slots.s[i] * ld)[e];
      }
#pragma unroll
      for (int l = 0; l < W; ++l) {
        T df, dg, fk;
        body(VT::get(gv, l), VT::get(pv, l), VT::get(fpv, l), VT::get(gpv, l), df, dg, fk);
        VT::set(dfv, l, df);
        VT::set(dgv, l, dg);
        VT::set(fkv, l, fk);
        ff += (double)fk * (double)fk;
        if (!first) {
          dd += (double)df * (double)df;
          fd += (double)fk * (double)df;
        }
      }
      if (kHoist && !first) {
#pragma unroll
        for (int i = 0; i < MW; ++i)
          if (i < nw) {
#pragma unroll
            for (int l = 0; l < W; ++l)
              a_dd[i] += (double)VT::get(dfv, l) * (double)VT::get(cols[kHoist ? i : 0], l);
          }
      }
      reinterpret_cast<V*>(fprev)[e] = fkv;
      reinterpret_cast<V*>(gprev)[e] = gv;
      if (first) continue;
      reinterpret_cast<V*>(dfn)[e] = dfv;
      reinterpret_cast<V*>(dgn)[e] = dgv;
#pragma unroll
      for (int i = 0; i < MW; ++i) {
        if (!kHoist && i < nw) {
          const V c = reinterpret_cast<const V*>(DF + (int64_t)slots.s[i] * ld)[e];
#pragma unroll
          for (int l = 0; l < W; ++l)
            a_dd[i] += (double)VT::get(dfv, l) * (double)VT::get(c, l);
        }
      }
    }
  }
  for (int64_t e = nv * W + gtid; e < n; e += gstride) {
    T df, dg, fk;
    body(g[e], p[e], fprev[e], gprev[e], df, dg, fk);
    fprev[e] = fk;
    gprev[e] = g[e];
    ff += (double)fk * (double)fk;
    if (first) continue;
    dfn[e] = df;
    dgn[e] = dg;
    dd += (double)df * (double)df;
    fd += (double)fk * (double)df;
#pragma unroll
    for (int i = 0; i < MW; ++i) {
      if (i < nw) {
        a_dd[i] += (double)df * (double)DF[(int64_t)slots.s[i] * ld + e];
      }
    }
  }
  // block reduction of nw + 3 accumulators, written as this block's partials
  const int na = nw + 3;
  __shared__ double red[kThreads / 32][2 * kMaxMem + 3];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto warp_put = [&](int idx, double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][idx] = v;
  };
#pragma unroll
  for (int i = 0; i < MW; ++i)
    if (i < nw) warp_put(i, a_dd[i]);
  warp_put(nw, dd);
  warp_put(nw + 1, fd);
  warp_put(nw + 2, ff);
  __syncthreads();
  for (int k = threadIdx.x; k < na; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w][k];
    part[(int64_t)blockIdx.x * na + k] = s;
  }
}

// sum partials over blocks in fixed order: out[k] = sum_b part[b*na + k]
__global__ void k_sum_cols(const double* __restrict__ part, int nb, int na,
                           double* __restrict__ out) {
  const int k = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(int64_t)b * na + k];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) out[k] = s;
}

// recombination (anderson.py:140-148):
//   beta == 1: out = G_k - sum_i gamma_i dG_i
//   else     : out = (1-beta) (p_k - sum gamma_i (dG_i - dF_i)) + beta (G_k - sum gamma_i dG_i)
//              (sum_i alpha_i x_i = x_k - sum_i gamma_i dx_i, p = G - f)
template <typename T, int MW, bool VEC>
__global__ void __launch_bounds__(kThreads)
    k_aa_step(const T* __restrict__ gk, const T* __restrict__ fk, const T* __restrict__ DF,
              const T* __restrict__ DG, int64_t n, int64_t ld, const Slots slots, int nw,
              const Coefs gam, double beta, T* __restrict__ out) {
  using VT = Vec<T>;
  using V = typename VT::type;
  constexpr int W = VEC ? VT::W : 1;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = n / W;
  if (VEC) {
    for (int64_t e = gtid; e < nv; e += gstride) {
      const V gv = reinterpret_cast<const V*>(gk)[e];
      double acc[W], cp[W];
#pragma unroll
      for (int l = 0; l < W; ++l) acc[l] = (double)VT::get(gv, l);
      if (beta != 1.0) {
        const V fv = reinterpret_cast<const V*>(fk)[e];
#pragma unroll
        for (int l = 0; l < W; ++l) cp[l] = acc[l] - (double)VT::get(fv, l);
      }
#pragma unroll
      for (int i = 0; i < MW; ++i) {
        if (i < nw) {
          const V dg = reinterpret_cast<const V*>(DG + (int64_t)slots.s[i] * ld)[e];
#pragma unroll
          for (int l = 0; l < W; ++l) acc[l] -= gam.c[i] * (double)VT::get(dg, l);
          if (beta != 1.0) {
            const V df = reinterpret_cast<const V*>(DF + (int64_t)slots.s[i] * ld)[e];
#pragma unroll
            for (int l = 0; l < W; ++l)
              cp[l] -= gam.c[i] * ((double)VT::get(dg, l) - (double)VT::get(df, l));
          }
        }
      }
      V o;
#pragma unroll
      for (int l = 0; l < W; ++l)
        VT::set(o, l, (T)(beta == 1.0 ? acc[l] : (1.0 - beta) * cp[l] + beta * acc[l]));
      reinterpret_cast<V*>(out)[e] = o;
    }
  }
  for (int64_t e = nv * W + gtid; e < n; e += gstride) {
    double acc = (double)gk[e];
    double cp = acc - (double)fk[e];
#pragma unroll
    for (int i = 0; i < MW; ++i)
      if (i < nw) {
        const double dg = (double)DG[(int64_t)slots.s[i] * ld + e];
        const double df = (double)DF[(int64_t)slots.s[i] * ld + e];
        acc -= gam.c[i] * dg;
        cp -= gam.c[i] * (dg - df);
      }
    out[e] = (T)(beta == 1.0 ? acc : (1.0 - beta) * cp + beta * acc);
  }
}

// Device thin-QR passes (the fallback for windows the fp64 Gram cannot
// resolve; reproduces SlidingQR.append_column's CGS2, seisopt/optim/qr.py:34-60):
//   mode 0: x = a (cast to fp64)           -> w = x; partials <q_i, x>, <x, x>
//   mode 1: x = w - sum_i h_i q_i          -> w = x; partials <q_i, x>, <x, x>
//   mode 2: q_nq = h_0 > 0 ? w / h_0 : 0   (normalise into basis column nq)
// q_i = Q + i ld (fp64).  Partials: nq + 1 per block.
template <typename T, int MW>
__global__ void __launch_bounds__(kThreads)
    k_qr_pass(const T* __restrict__ a, double* __restrict__ w, double* __restrict__ Q,
              int64_t n, int64_t ld, int nq, const Coefs h, int mode,
              double* __restrict__ part) {
  double acc[MW];
#pragma unroll
  for (int i = 0; i < MW; ++i) acc[i] = 0.0;
  double xx = 0.0;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = gtid; e < n; e += gstride) {
    if (mode == 2) {
      Q[(int64_t)nq * ld + e] = h.c[0] > 0.0 ? w[e] / h.c[0] : 0.0;
      continue;
    }
    double x;
    if (mode == 0) {
      x = (double)a[e];
    } else {
      x = w[e];
#pragma unroll
      for (int i = 0; i < MW; ++i)
        if (i < nq) x -= h.c[i] * Q[(int64_t)i * ld + e];
    }
    w[e] = x;
#pragma unroll
    for (int i = 0; i < MW; ++i)
      if (i < nq) acc[i] += Q[(int64_t)i * ld + e] * x;
    xx += x * x;
  }
  if (mode == 2) return;
  const int na = nq + 1;
  __shared__ double red[kThreads / 32][kMaxMem + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto warp_put = [&](int idx, double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][idx] = v;
  };
#pragma unroll
  for (int i = 0; i < MW; ++i)
    if (i < nq) warp_put(i, acc[i]);
  warp_put(nq, xx);
  __syncthreads();
  for (int k = threadIdx.x; k < na; k += blockDim.x) {
    double sum = 0.0;
    for (int w2 = 0; w2 < kThreads / 32; ++w2) sum += red[w2][k];
    part[(int64_t)blockIdx.x * na + k] = sum;
  }
}

// ---- vector helpers ------------------------------------------------------------

template <typename T>
__global__ void k_axpby(int64_t n, double a, const T* __restrict__ x, double b,
                        const T* __restrict__ y, T* __restrict__ z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (a == 1.0) z[e] = x[e] + (T)b * y[e];  // p - eta g  (anderson.py:322)
    else z[e] = (T)a * x[e] + (T)b * y[e];
  }
}

template <typename T>
__global__ void k_lerp(int64_t n, const T* __restrict__ x, const T* __restrict__ y, double lam,
                       T* __restrict__ z) {
  // z = x + lam (y - x)   (anderson.py:362, 369)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    z[e] = x[e] + (T)lam * (y[e] - x[e]);
}

// <g, pbar - p>, <g, ptil - pbar> partials (anderson.py:362-364)
template <typename T>
__global__ void k_blend_dots(int64_t n, const T* __restrict__ g, const T* __restrict__ p,
                             const T* __restrict__ pb, const T* __restrict__ pt,
                             double* __restrict__ part) {
  double s0 = 0.0, s1 = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double gv = (double)g[e];
    const double b = (double)pb[e];
    s0 += gv * (b - (double)p[e]);
    s1 += gv * ((double)pt[e] - b);
  }
  const double r0 = block_sum(s0);
  __syncthreads();
  const double r1 = block_sum(s1);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r0;
    part[2 * blockIdx.x + 1] = r1;
  }
}

// {min, max, max|x|, sum x^2, nonfinite} partials
template <typename T>
__global__ void k_stats(int64_t n, const T* __restrict__ x, double* __restrict__ part) {
  double mn = INFINITY, mx = -INFINITY, ma = 0.0, s2 = 0.0, bad = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)x[e];
    if (!isfinite(v)) {
      bad += 1.0;
      continue;
    }
    mn = fmin(mn, v);
    mx = fmax(mx, v);
    ma = fmax(ma, fabs(v));
    s2 += v * v;
  }
  __shared__ double r[3][kThreads];
  r[0][threadIdx.x] = mn;
  r[1][threadIdx.x] = mx;
  r[2][threadIdx.x] = ma;
  const double t2 = block_sum(s2);
  __syncthreads();
  const double tb = block_sum(bad);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      r[0][threadIdx.x] = fmin(r[0][threadIdx.x], r[0][threadIdx.x + s]);
      r[1][threadIdx.x] = fmax(r[1][threadIdx.x], r[1][threadIdx.x + s]);
      r[2][threadIdx.x] = fmax(r[2][threadIdx.x], r[2][threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = part + 5 * blockIdx.x;
    o[0] = r[0][0];
    o[1] = r[1][0];
    o[2] = r[2][0];
    o[3] = t2;
    o[4] = tb;
  }
}

// Krylov / quasi-Newton vector kernels (seisopt/krylov.py:130-190,
// seisopt/optim/quasi_newton.py:36-55): one pass over k vectors x_i and y.
struct Ptrs {
  const void* p[kMaxMem];
};

// partials per block: <x_i, y> (i < k), then <y, y>; fp64 accumulation
template <typename T, int MW>
__global__ void __launch_bounds__(kThreads)
    k_multi_dot(int64_t n, int k, const Ptrs xs, const T* __restrict__ y,
                double* __restrict__ part) {
  double acc[MW];
#pragma unroll
  for (int i = 0; i < MW; ++i) acc[i] = 0.0;
  double yy = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double yv = (double)y[e];
#pragma unroll
    for (int i = 0; i < MW; ++i)
      if (i < k) acc[i] += (double)reinterpret_cast<const T*>(xs.p[i])[e] * yv;
    yy += yv * yv;
  }
  const int na = k + 1;
  __shared__ double red[kThreads / 32][kMaxMem + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto warp_put = [&](int idx, double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][idx] = v;
  };
#pragma unroll
  for (int i = 0; i < MW; ++i)
    if (i < k) warp_put(i, acc[i]);
  warp_put(k, yy);
  __syncthreads();
  for (int q = threadIdx.x; q < na; q += blockDim.x) {
    double sum = 0.0;
    for (int w2 = 0; w2 < kThreads / 32; ++w2) sum += red[w2][q];
    part[(int64_t)blockIdx.x * na + q] = sum;
  }
}

// z = y + sum_i c_i x_i (y == nullptr: z = sum_i c_i x_i), fp64 arithmetic
// per element, in the order y, x_0, x_1, ... (krylov.py:189, quasi_newton.py:44-54)
template <typename T, int MW>
__global__ void __launch_bounds__(kThreads)
    k_multi_axpy(int64_t n, int k, const Coefs c, const Ptrs xs, const T* y, T* z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double acc = y ? (double)y[e] : 0.0;
#pragma unroll
    for (int i = 0; i < MW; ++i)
      if (i < k) acc += c.c[i] * (double)reinterpret_cast<const T*>(xs.p[i])[e];
    z[e] = (T)acc;
  }
}

// ||f_k - sum_i gamma_i DF_i||^2 partials (the explicit combined residual of
// qr.py:89-95 for Gram-solved windows), fp64 per element
template <typename T, int MW>
__global__ void __launch_bounds__(kThreads)
    k_aa_resid(const T* __restrict__ fk, const T* __restrict__ DF, int64_t n, int64_t ld,
               const Slots slots, int nw, const Coefs gam, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double r = (double)fk[e];
#pragma unroll
    for (int i = 0; i < MW; ++i)
      if (i < nw) r -= gam.c[i] * (double)DF[(int64_t)slots.s[i] * ld + e];
    acc += r * r;
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(kBlocks, (n + kThreads - 1) / kThreads)); }

// exactly rounded sum (Shewchuk partials, as Python's math.fsum)
double fsum(const std::vector<double>& xs) {
  std::vector<double> parts;
  for (double x : xs) {
    size_t i = 0;
    for (double y : parts) {
      if (std::fabs(x) < std::fabs(y)) std::swap(x, y);
      const double hi = x + y;
      const double lo = y - (hi - x);
      if (lo != 0.0) parts[i++] = lo;
      x = hi;
    }
    parts.resize(i);
    parts.push_back(x);
  }
  // sum partials from the top with correct rounding of the final result
  if (parts.empty()) return 0.0;
  int n = (int)parts.size() - 1;
  double hi = parts[n], lo = 0.0;
  while (n > 0) {
    const double x = hi;
    const double y = parts[--n];
    hi = x + y;
    const double yr = hi - x;
    lo = y - yr;
    if (lo != 0.0) break;
  }
  if (n > 0 && ((lo < 0 && parts[n - 1] < 0) || (lo > 0 && parts[n - 1] > 0))) {
    const double y = lo * 2.0;
    const double x = hi + y;
    const double yr = x - hi;
    if (y == yr) hi = x;
  }
  return hi;
}

}  // namespace

struct sg_aa {
  int64_t n = 0;
  int64_t ld = 0;  // slot stride (n rounded up to 64 elements, keeps columns 256-B aligned)
  int memory = 0;
  int esz = 8;
  int device = 0;
  cudaStream_t stream = 0;
  void* DF = nullptr;  // memory slots
  void* DG = nullptr;
  void* fk = nullptr;  // f_k (after push) = previous f for the next push
  void* gk = nullptr;  // G_k
  double* part = nullptr;
  double* out = nullptr;
  // window bookkeeping (oldest first)
  int head = 0;    // ring index of the oldest column
  int ncols = 0;   // columns in the window
  int pushes = 0;  // entries in fs (reference len(fs)), capped semantics below
  std::vector<double> gram;  // memory x memory, window order
  std::vector<double> bvec;  // <DF_i, f_k>
  double fk2 = 0.0;
  // device QR fallback (windows the Gram cannot resolve, or mode 1 = always):
  // fp64 basis Q (memory columns + one scratch column) and R of the current
  // window, valid while qr_active
  int qr_mode = 0;
  double* Qd = nullptr;
  bool qr_active = false;
  std::vector<double> Rq;
  int64_t qr_passes = 0;  // device QR passes run (diagnostics)
  // N-sharded windows: sums every device inner product over the ranks
  sg_reduce_fn reduce = nullptr;
  void* reduce_ctx = nullptr;
  // cached weights of the current window
  bool have_w = false;
  std::vector<double> gamma, alpha;
  double resid = 0.0;
};

namespace {

int slot_of(const sg_aa* a, int pos) { return (a->head + pos) % std::max(1, a->memory); }

// Every quantity the window reads back from the device is a plain sum over
// the N entries (Gram rows, projections, squared norms), so an N-sharded
// window only has to sum these few doubles over the ranks (sg_aa_set_reducer)
int reduce_sums(sg_aa* a, double* buf, int n) {
  if (a->reduce && a->reduce(buf, n, a->reduce_ctx) != 0)
    return fail(SG_ERR_STATE, "AA window reducer callback failed");
  return SG_OK;
}

double& G(sg_aa* a, int i, int j) { return a->gram[(size_t)i * a->memory + j]; }

void drop_oldest(sg_aa* a) {
  const int m = a->memory;
  std::vector<double> g2(a->gram.size(), 0.0);
  for (int i = 1; i < a->ncols; ++i)
    for (int j = 1; j < a->ncols; ++j) g2[(size_t)(i - 1) * m + (j - 1)] = a->gram[(size_t)i * m + j];
  a->gram.swap(g2);
  for (int i = 1; i < a->ncols; ++i) a->bvec[i - 1] = a->bvec[i];
  a->head = (a->head + 1) % m;
  a->ncols -= 1;
  a->pushes -= 1;  // ps/gs/fs/dgs all pop(0) in the reference (anderson.py:98-103)
}

// Cholesky R (upper, R^T R = Gram) with the reference's dependence rule: a
// pivot is zero when rho < 1e-15 max(||a||, 1) (qr.py:47-53) or when it is
// below the Gram formulation's resolution (rho^2 <= 1e-14 ||a||^2).
// Returns true when a pivot is below what the fp64 Gram resolves reliably
// (rho^2 <= 1e-10 ||a||^2, i.e. rho / ||a|| <= 1e-5): the window then takes the
// device QR instead.
bool cholesky(const sg_aa* a, std::vector<double>& R, std::vector<double>& diag) {
  const int k = a->ncols, m = a->memory;
  // fp64 (parity) windows leave the Gram path already at rho / ||a|| <= 1e-3:
  // the normal equations carry ~cond^2 eps error, and the reference solves
  // through its QR (qr.py:82-87); fp32 windows keep the Gram down to 1e-5
  const double unres = a->esz == 8 ? 1e-6 : 1e-10;
  R.assign((size_t)k * k, 0.0);
  diag.assign(k, 0.0);
  bool unresolved = false;
  for (int j = 0; j < k; ++j) {
    const double ajj = a->gram[(size_t)j * m + j];
    for (int i = 0; i < j; ++i) {
      double s = a->gram[(size_t)i * m + j];
      for (int l = 0; l < i; ++l) s -= R[(size_t)l * k + i] * R[(size_t)l * k + j];
      R[(size_t)i * k + j] = diag[i] > 0.0 ? s / diag[i] : 0.0;
    }
    double s = ajj;
    for (int l = 0; l < j; ++l) s -= R[(size_t)l * k + j] * R[(size_t)l * k + j];
    const double nrm = std::sqrt(std::max(ajj, 0.0));
    double rho = s > 0.0 ? std::sqrt(s) : 0.0;
    if (s <= unres * ajj) unresolved = true;
    if (rho <= 1e-300 || rho < 1e-15 * std::max(nrm, 1.0) || s <= 1e-14 * ajj) rho = 0.0;
    diag[j] = rho;
    R[(size_t)j * k + j] = rho;
  }
  return unresolved;
}

// one k_qr_pass launch + fixed-order partial sums -> host (nq + 1 values)
template <typename T>
int qr_pass(sg_aa* a, const T* col, int nq, const double* h, int mode, std::vector<double>* o) {
  const int nb = grid_for(a->n);
  Coefs cf{};
  for (int i = 0; i < (mode == 2 ? 1 : nq); ++i) cf.c[i] = h ? h[i] : 0.0;
  double* w = a->Qd + (int64_t)a->memory * a->ld;  // scratch column
  const int mw = std::max(nq, 1);
#define QRP(MW) k_qr_pass<T, MW><<<nb, kThreads, 0, a->stream>>>(col, w, a->Qd, a->n, a->ld, nq, cf, mode, a->part)
  if (mw <= 4) QRP(4);
  else if (mw <= 8) QRP(8);
  else if (mw <= 16) QRP(16);
  else QRP(32);
#undef QRP
  count_launch();
  a->qr_passes++;
  if (mode == 2) return SG_OK;
  const int na = nq + 1;
  k_sum_cols<<<na, 256, 0, a->stream>>>(a->part, nb, na, a->out);
  count_launch();
  SG_CK(cudaGetLastError());
  o->resize(na);
  SG_CK(cudaMemcpyAsync(o->data(), a->out, na * sizeof(double), cudaMemcpyDeviceToHost, a->stream));
  SG_CK(cudaStreamSynchronize(a->stream));
  return reduce_sums(a, o->data(), na);
}

// Thin QR of the current window (oldest column first) by CGS2 appends, the
// reference's append_column (seisopt/optim/qr.py:34-60): h = Q^T a,
// w = a - Q h, h2 = Q^T w, w -= Q h2, rho = ||w|| (zero basis when
// rho < 1e-15 max(||a||, 1)).  R (k x k, row-major) into a->Rq.
template <typename T>
int device_qr(sg_aa* a) {
  const int k = a->ncols;
  if (!a->Qd) {
    const size_t bytes = (size_t)(a->memory + 1) * a->ld * sizeof(double);
    cudaError_t e = rz_malloc((void**)&a->Qd, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      a->Qd = nullptr;
      return fail(SG_ERR_OOM, std::string("AA QR basis allocation failed: ") + cudaGetErrorString(e));
    }
  }
  a->Rq.assign((size_t)k * k, 0.0);
  const T* DF = reinterpret_cast<const T*>(a->DF);
  std::vector<double> o0, o1, o2;
  for (int j = 0; j < k; ++j) {
    const T* col = DF + (int64_t)slot_of(a, j) * a->ld;
    SG_TRY(qr_pass<T>(a, col, j, nullptr, 0, &o0));            // h = Q^T a, ||a||^2
    SG_TRY(qr_pass<T>(a, (const T*)nullptr, j, o0.data(), 1, &o1));  // w = a - Q h; h2
    SG_TRY(qr_pass<T>(a, (const T*)nullptr, j, o1.data(), 1, &o2));  // w -= Q h2; ||w||^2
    for (int i = 0; i < j; ++i) a->Rq[(size_t)i * k + j] = o0[i] + o1[i];
    double rho = std::sqrt(std::max(o2[j], 0.0));
    const double scale = std::max(std::sqrt(std::max(o0[j], 0.0)), 1.0);
    if (rho <= 1e-300 || rho < 1e-15 * scale) rho = 0.0;
    a->Rq[(size_t)j * k + j] = rho;
    SG_TRY(qr_pass<T>(a, (const T*)nullptr, j, &rho, 2, nullptr));  // q_j = w / rho
  }
  a->qr_active = true;
  return SG_OK;
}

// R of the current window: Cholesky of the Gram, or the device QR when the
// Gram cannot resolve it (or qr_mode == 1)
int window_r(sg_aa* a, std::vector<double>& R, std::vector<double>& d) {
  const bool unresolved = cholesky(a, R, d);
  a->qr_active = false;
  if (!unresolved && a->qr_mode != 1) return SG_OK;
  SG_TRY(a->esz == 4 ? device_qr<float>(a) : device_qr<double>(a));
  R = a->Rq;
  const int k = a->ncols;
  for (int j = 0; j < k; ++j) d[j] = std::fabs(R[(size_t)j * k + j]);
  return SG_OK;
}

// safeguard (anderson.py:105-112): shed oldest columns while
// min|diag R| <= 1e-12 ||R||_F
int safeguard(sg_aa* a) {
  std::vector<double> R, d;
  while (a->ncols > 0) {
    SG_TRY(window_r(a, R, d));
    double fro2 = 0.0;
    for (double v : R) fro2 += v * v;
    const double tol = 1e-12 * std::max(std::sqrt(fro2), 1e-300);
    if (*std::min_element(d.begin(), d.end()) > tol) break;
    drop_oldest(a);
    a->qr_active = false;
  }
  return SG_OK;
}

// gamma = solve_triangular(R, Q^T f) and ||f - Q Q^T f|| with the device basis
// (seisopt/optim/qr.py:82-95)
template <typename T>
int qr_solve(sg_aa* a, std::vector<double>& gmm, double& resid) {
  const int k = a->ncols;
  std::vector<double> qf, rr;
  SG_TRY(qr_pass<T>(a, reinterpret_cast<const T*>(a->fk), k, nullptr, 0, &qf));  // Q^T f, ||f||^2
  SG_TRY(qr_pass<T>(a, (const T*)nullptr, k, qf.data(), 1, &rr));               // ||f - Q Q^T f||^2
  gmm.assign(k, 0.0);
  const std::vector<double>& R = a->Rq;
  for (int i = k - 1; i >= 0; --i) {
    double s = qf[i];
    for (int l = i + 1; l < k; ++l) s -= R[(size_t)i * k + l] * gmm[l];
    gmm[i] = s / R[(size_t)i * k + i];
  }
  resid = std::min(std::sqrt(std::max(rr[k], 0.0)), std::sqrt(std::max(qf[k], 0.0)));
  return SG_OK;
}

// ||f_k - DF gamma|| by one device pass over the window (fp64 accumulation)
template <typename T>
int explicit_resid(sg_aa* a, const std::vector<double>& gmm, double& out) {
  const int k = a->ncols;
  const int nb = grid_for(a->n);
  Slots sl{};
  Coefs cf{};
  for (int i = 0; i < k; ++i) {
    sl.s[i] = slot_of(a, i);
    cf.c[i] = gmm[i];
  }
  const T* fk = reinterpret_cast<const T*>(a->fk);
  const T* DF = reinterpret_cast<const T*>(a->DF);
#define RES(MW) k_aa_resid<T, MW><<<nb, kThreads, 0, a->stream>>>(fk, DF, a->n, a->ld, sl, k, cf, a->part)
  if (k <= 4) RES(4);
  else if (k <= 8) RES(8);
  else if (k <= 16) RES(16);
  else RES(32);
#undef RES
  k_sum_cols<<<1, 256, 0, a->stream>>>(a->part, nb, 1, a->out);
  count_launch(2);
  SG_CK(cudaGetLastError());
  double r2 = 0.0;
  SG_CK(cudaMemcpyAsync(&r2, a->out, sizeof(double), cudaMemcpyDeviceToHost, a->stream));
  SG_CK(cudaStreamSynchronize(a->stream));
  SG_TRY(reduce_sums(a, &r2, 1));
  out = std::sqrt(std::max(r2, 0.0));
  return SG_OK;
}

int compute_weights(sg_aa* a) {
  const int k = a->ncols;
  if (k == 0 || a->pushes < 2) return fail(SG_ERR_EMPTY, "aa_weights needs at least one stored difference");
  std::vector<double> R, d, gmm(k);
  if (!a->qr_active) SG_TRY(window_r(a, R, d));
  if (a->qr_active) {
    SG_TRY(a->esz == 4 ? qr_solve<float>(a, gmm, a->resid) : qr_solve<double>(a, gmm, a->resid));
  } else {
    // forward solve R^T y = b, back solve R gamma = y  (== solve_triangular(R, Q^T f))
    std::vector<double> y(k);
    for (int i = 0; i < k; ++i) {
      double s = a->bvec[i];
      for (int l = 0; l < i; ++l) s -= R[(size_t)l * k + i] * y[l];
      y[i] = s / R[(size_t)i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
      double s = y[i];
      for (int l = i + 1; l < k; ++l) s -= R[(size_t)i * k + l] * gmm[l];
      gmm[i] = s / R[(size_t)i * k + i];
    }
    // residual ||f - A gamma||^2 = ||f||^2 - ||y||^2, clipped to [0, ||f||^2]
    double y2 = 0.0;
    for (double v : y) y2 += v * v;
    const double r2 = std::max(a->fk2 - y2, 0.0);
    a->resid = std::min(std::sqrt(r2), std::sqrt(a->fk2));
    // fp64 (parity) mode: the explicit ||f - A gamma|| instead of the
    // cancellation-prone sqrt(||f||^2 - ||y||^2) (accurate to ~sqrt(eps) ||f||)
    if (a->esz == 8) {
      double r = 0.0;
      SG_TRY(explicit_resid<double>(a, gmm, r));
      a->resid = std::min(r, std::sqrt(a->fk2));
    }
  }
  // alpha recovery with fsum fix-up (anderson.py:41-52)
  std::vector<double> al(k + 1);
  al[0] = gmm[0];
  for (int i = 1; i < k; ++i) al[i] = gmm[i] - gmm[i - 1];
  al[k] = 1.0 - gmm[k - 1];
  for (int it = 0; it < 3; ++it) {
    const double gap = 1.0 - fsum(al);
    if (gap == 0.0) break;
    int arg = 0;
    for (int i = 1; i <= k; ++i)
      if (std::fabs(al[i]) > std::fabs(al[arg])) arg = i;
    al[arg] += gap;
  }
  a->gamma = gmm;
  a->alpha = al;
  a->have_w = true;
  return SG_OK;
}

template <typename T>
int push_t(sg_aa* a, const void* p, const void* g) {
  const int first = (a->pushes == 0 || a->memory == 0) ? 1 : 0;
  Slots sl{};
  int nw = 0, snew = 0;
  if (!first) {
    // a full window drops its oldest column now; the new difference takes its slot
    if (a->ncols == a->memory) drop_oldest(a);
    a->qr_active = false;
    nw = a->ncols;
    for (int i = 0; i < nw; ++i) sl.s[i] = slot_of(a, i);
    snew = slot_of(a, nw);
  }
  const int nb = grid_for(a->n);
  const int na = nw + 3;
  T* DF = reinterpret_cast<T*>(a->DF);
  T* DG = reinterpret_cast<T*>(a->DG);
  const T* pp = reinterpret_cast<const T*>(p);
  const T* gg = reinterpret_cast<const T*>(g);
  T* fk = reinterpret_cast<T*>(a->fk);
  T* gk = reinterpret_cast<T*>(a->gk);
  const int mw = std::max(nw, 1);
  const bool vec = aligned16(pp) && aligned16(gg);
#define PUSH(MW)                                                                              \
  do {                                                                                        \
    if (vec)                                                                                  \
      k_aa_push<T, MW, true><<<nb, kThreads, 0, a->stream>>>(pp, gg, fk, gk, DF, DG, a->n, \
                                                              a->ld, sl, nw, snew, first,    \
                                                              a->part);                      \
    else                                                                                      \
      k_aa_push<T, MW, false><<<nb, kThreads, 0, a->stream>>>(pp, gg, fk, gk, DF, DG, a->n, \
                                                               a->ld, sl, nw, snew, first,   \
                                                               a->part);                     \
  } while (0)
  if (mw <= 4) PUSH(4);
  else if (mw <= 8) PUSH(8);
  else if (mw <= 12) PUSH(12);
  else if (mw <= 16) PUSH(16);
  else if (mw <= 20) PUSH(20);  // BASELINE C5 window (m = 20)
  else PUSH(32);
#undef PUSH
  k_sum_cols<<<na, 256, 0, a->stream>>>(a->part, nb, na, a->out);
  count_launch(2);
  SG_CK(cudaGetLastError());
  std::vector<double> o(na);
  SG_CK(cudaMemcpyAsync(o.data(), a->out, na * sizeof(double), cudaMemcpyDeviceToHost, a->stream));
  SG_CK(cudaStreamSynchronize(a->stream));
  SG_TRY(reduce_sums(a, o.data(), na));
  a->have_w = false;
  if (first) {
    // memory 0 keeps only the latest entry; otherwise this is fs[0]
    a->fk2 = o[nw + 2];
    a->pushes = 1;
    a->ncols = 0;
    a->head = 0;
    return SG_OK;
  }
  // oldest-first layout: window positions 0..nw-1 then the new column at nw
  const int m = a->memory;
  for (int i = 0; i < nw; ++i) {
    G(a, i, nw) = o[i];
    G(a, nw, i) = o[i];
    a->bvec[i] += o[i];  // <f_k, dF_i> = <f_{k-1}, dF_i> + <df, dF_i>
  }
  G(a, nw, nw) = o[nw];
  a->bvec[nw] = o[nw + 1];
  a->fk2 = o[nw + 2];
  a->ncols = nw + 1;
  a->pushes += 1;
  (void)m;
  a->qr_active = false;
  return safeguard(a);
}

template <typename T>
int step_t(sg_aa* a, double beta, const double* gamma, void* out) {
  const int k = a->ncols;
  Slots sl{};
  Coefs cf{};
  for (int i = 0; i < k; ++i) {
    sl.s[i] = slot_of(a, i);
    cf.c[i] = gamma ? gamma[i] : a->gamma[i];
  }
  const int nb = grid_for(a->n);
  const T* gk = reinterpret_cast<const T*>(a->gk);
  const T* fk = reinterpret_cast<const T*>(a->fk);
  const T* DF = reinterpret_cast<const T*>(a->DF);
  const T* DG = reinterpret_cast<const T*>(a->DG);
  T* o = reinterpret_cast<T*>(out);
  const int mw = std::max(k, 1);
  const bool vec = aligned16(o);
#define STEP(MW)                                                                               \
  do {                                                                                         \
    if (vec)                                                                                   \
      k_aa_step<T, MW, true><<<nb, kThreads, 0, a->stream>>>(gk, fk, DF, DG, a->n, a->ld, sl, \
                                                              k, cf, beta, o);                \
    else                                                                                       \
      k_aa_step<T, MW, false><<<nb, kThreads, 0, a->stream>>>(gk, fk, DF, DG, a->n, a->ld,   \
                                                               sl, k, cf, beta, o);           \
  } while (0)
  if (mw <= 4) STEP(4);
  else if (mw <= 8) STEP(8);
  else if (mw <= 12) STEP(12);
  else if (mw <= 16) STEP(16);
  else if (mw <= 20) STEP(20);
  else STEP(32);
#undef STEP
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

}  // namespace

extern "C" {

int sg_aa_create(int64_t n, int32_t memory, int32_t dtype, int32_t device, sg_aa** out) {
  if (!out) return fail(SG_ERR_ARG, "null argument");
  *out = nullptr;
  if (n < 1) return fail(SG_ERR_ARG, "rows must be positive");
  if (memory < 0) return fail(SG_ERR_ARG, "memory must be non-negative");
  if (memory > kMaxMem) return fail(SG_ERR_ARG, "memory above " + std::to_string(kMaxMem));
  if (dtype != SG_F32 && dtype != SG_F64) return fail(SG_ERR_ARG, "dtype must be 4 or 8");
  SG_CK(cudaSetDevice(device));
  sg_aa* a = new sg_aa();
  a->n = n;
  a->memory = memory;
  a->esz = dtype;
  a->device = device;
  a->ld = (n + 63) / 64 * 64;
  const size_t vb = (size_t)a->ld * dtype;
  const int slots = std::max(memory, 1);
  cudaError_t e = rz_malloc(&a->DF, vb * slots);
  if (e == cudaSuccess) e = rz_malloc(&a->DG, vb * slots);
  if (e == cudaSuccess) e = rz_malloc(&a->fk, vb);
  if (e == cudaSuccess) e = rz_malloc(&a->gk, vb);
  if (e == cudaSuccess) e = rz_malloc((void**)&a->part, sizeof(double) * kBlocks * (2 * kMaxMem + 3));
  if (e == cudaSuccess) e = rz_malloc((void**)&a->out, sizeof(double) * (2 * kMaxMem + 8));
  if (e != cudaSuccess) {
    sg_aa_destroy(a);
    cudaGetLastError();
    return fail(SG_ERR_OOM, std::string("AA window allocation failed: ") + cudaGetErrorString(e));
  }
  a->gram.assign((size_t)slots * slots, 0.0);
  a->bvec.assign(slots + 1, 0.0);
  *out = a;
  return SG_OK;
}

int sg_aa_destroy(sg_aa* a) {
  if (!a) return SG_OK;
  cudaSetDevice(a->device);
  for (void* p : {a->DF, a->DG, a->fk, a->gk, (void*)a->part, (void*)a->out, (void*)a->Qd})
    if (p) rz_free(p);
  delete a;
  return SG_OK;
}

int sg_aa_set_stream(sg_aa* a, void* s) {
  if (!a) return fail(SG_ERR_ARG, "null window");
  a->stream = reinterpret_cast<cudaStream_t>(s);
  return SG_OK;
}

int sg_aa_set_reducer(sg_aa* a, sg_reduce_fn fn, void* ctx) {
  if (!a) return fail(SG_ERR_ARG, "null window");
  a->reduce = fn;
  a->reduce_ctx = ctx;
  return SG_OK;
}

int sg_aa_clear(sg_aa* a) {
  if (!a) return fail(SG_ERR_ARG, "null window");
  a->head = a->ncols = a->pushes = 0;
  std::fill(a->gram.begin(), a->gram.end(), 0.0);
  a->have_w = false;
  a->qr_active = false;
  return SG_OK;
}

int sg_aa_push(sg_aa* a, const void* p, const void* g) {
  sg::Trace trace_("sg_aa_push");
  if (!a || !p || !g) return fail(SG_ERR_ARG, "null argument");
  SG_CK(cudaSetDevice(a->device));
  return a->esz == 4 ? push_t<float>(a, p, g) : push_t<double>(a, p, g);
}

int sg_aa_set_qr(sg_aa* a, int32_t mode) {
  if (!a) return fail(SG_ERR_ARG, "null window");
  if (mode != 0 && mode != 1) return fail(SG_ERR_ARG, "qr mode must be 0 (auto) or 1 (always)");
  a->qr_mode = mode;
  a->qr_active = false;
  a->have_w = false;
  return SG_OK;
}

int sg_aa_qr_info(sg_aa* a, int32_t* active, int64_t* passes) {
  if (!a) return fail(SG_ERR_ARG, "null window");
  if (active) *active = a->qr_active ? 1 : 0;
  if (passes) *passes = a->qr_passes;
  return SG_OK;
}

int sg_aa_m_k(sg_aa* a) {
  if (!a) return 0;
  return a->memory == 0 ? 0 : std::max(0, a->pushes - 1);
}

int sg_aa_weights(sg_aa* a, double* gamma, double* alpha, double* resid, int32_t* m_k) {
  sg::Trace trace_("sg_aa_weights");
  if (!a) return fail(SG_ERR_ARG, "null window");
  if (sg_aa_m_k(a) == 0) return fail(SG_ERR_EMPTY, "aa_weights needs at least one stored difference");
  if (!a->have_w) SG_TRY(compute_weights(a));
  const int k = a->ncols;
  if (gamma) std::memcpy(gamma, a->gamma.data(), k * sizeof(double));
  if (alpha) std::memcpy(alpha, a->alpha.data(), (k + 1) * sizeof(double));
  if (resid) *resid = a->resid;
  if (m_k) *m_k = k;
  return SG_OK;
}

int sg_aa_step(sg_aa* a, double beta, const double* gamma, const double* alpha, void* out) {
  sg::Trace trace_("sg_aa_step");
  (void)alpha;
  if (!a || !out) return fail(SG_ERR_ARG, "null argument");
  if (a->pushes == 0) return fail(SG_ERR_EMPTY, "aa_step on an empty window");
  SG_CK(cudaSetDevice(a->device));
  if (sg_aa_m_k(a) == 0) {
    // Picard: G_k (anderson.py:136-137)
    SG_CK(cudaMemcpyAsync(out, a->gk, (size_t)a->n * a->esz, cudaMemcpyDeviceToDevice, a->stream));
    return SG_OK;
  }
  if (!gamma && !a->have_w) SG_TRY(compute_weights(a));
  return a->esz == 4 ? step_t<float>(a, beta, gamma, out) : step_t<double>(a, beta, gamma, out);
}

int sg_aa_fk_norm(sg_aa* a, double* out) {
  if (!a || !out) return fail(SG_ERR_ARG, "null argument");
  if (a->pushes == 0) return fail(SG_ERR_EMPTY, "empty window");
  *out = std::sqrt(a->fk2);
  return SG_OK;
}

int sg_vec_axpby(int64_t n, int32_t dtype, double a, const void* x, double b, const void* y,
                 void* z, void* stream) {
  if (n < 0 || !x || !y || !z) return fail(SG_ERR_ARG, "bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == SG_F32) k_axpby<float><<<grid_for(n), kThreads, 0, s>>>(n, a, (const float*)x, b, (const float*)y, (float*)z);
  else k_axpby<double><<<grid_for(n), kThreads, 0, s>>>(n, a, (const double*)x, b, (const double*)y, (double*)z);
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

int sg_vec_lerp(int64_t n, int32_t dtype, const void* x, const void* y, double lam, void* z,
                void* stream) {
  if (n < 0 || !x || !y || !z) return fail(SG_ERR_ARG, "bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == SG_F32) k_lerp<float><<<grid_for(n), kThreads, 0, s>>>(n, (const float*)x, (const float*)y, lam, (float*)z);
  else k_lerp<double><<<grid_for(n), kThreads, 0, s>>>(n, (const double*)x, (const double*)y, lam, (double*)z);
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

int sg_vec_blend_dots(int64_t n, int32_t dtype, const void* g, const void* p, const void* pbar,
                      const void* ptil, double* out, void* stream) {
  if (n < 1 || !g || !p || !pbar || !ptil || !out) return fail(SG_ERR_ARG, "bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = grid_for(n);
  double* part = nullptr;
  SG_CK(cudaMallocAsync((void**)&part, sizeof(double) * 2 * nb, s));
  if (dtype == SG_F32) k_blend_dots<float><<<nb, kThreads, 0, s>>>(n, (const float*)g, (const float*)p, (const float*)pbar, (const float*)ptil, part);
  else k_blend_dots<double><<<nb, kThreads, 0, s>>>(n, (const double*)g, (const double*)p, (const double*)pbar, (const double*)ptil, part);
  count_launch();
  std::vector<double> h(2 * nb);
  SG_CK(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CK(cudaFreeAsync(part, s));
  SG_CK(cudaStreamSynchronize(s));
  double s0 = 0.0, s1 = 0.0;
  for (int b = 0; b < nb; ++b) {
    s0 += h[2 * b];
    s1 += h[2 * b + 1];
  }
  out[0] = s0;
  out[1] = s1;
  return SG_OK;
}

int sg_vec_multi_dot(int64_t n, int32_t dtype, int32_t k, const void* const* xs, const void* y,
                     double* out, void* stream) {
  if (n < 1 || k < 0 || k > kMaxMem || (k > 0 && !xs) || !y || !out)
    return fail(SG_ERR_ARG, "bad arguments");
  if (dtype != SG_F32 && dtype != SG_F64) return fail(SG_ERR_ARG, "dtype must be SG_F32 or SG_F64");
  Ptrs px{};
  for (int i = 0; i < k; ++i) {
    if (!xs[i]) return fail(SG_ERR_ARG, "null vector");
    px.p[i] = xs[i];
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = grid_for(n), na = k + 1;
  double* part = nullptr;
  SG_CK(cudaMallocAsync((void**)&part, sizeof(double) * ((size_t)na * nb + na), s));
  double* dout = part + (size_t)na * nb;
#define MD(TT, MW) k_multi_dot<TT, MW><<<nb, kThreads, 0, s>>>(n, k, px, (const TT*)y, part)
#define MDT(TT)                  \
  do {                           \
    if (k <= 1) MD(TT, 1);       \
    else if (k <= 4) MD(TT, 4);  \
    else if (k <= 8) MD(TT, 8);  \
    else if (k <= 16) MD(TT, 16); \
    else MD(TT, 32);             \
  } while (0)
  if (dtype == SG_F32) MDT(float);
  else MDT(double);
#undef MDT
#undef MD
  k_sum_cols<<<na, 256, 0, s>>>(part, nb, na, dout);
  count_launch(2);
  SG_CK(cudaGetLastError());
  SG_CK(cudaMemcpyAsync(out, dout, na * sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CK(cudaFreeAsync(part, s));
  SG_CK(cudaStreamSynchronize(s));
  return SG_OK;
}

int sg_vec_multi_axpy(int64_t n, int32_t dtype, int32_t k, const double* coef,
                      const void* const* xs, const void* y, void* z, void* stream) {
  if (n < 0 || k < 0 || k > kMaxMem || (k > 0 && (!xs || !coef)) || !z)
    return fail(SG_ERR_ARG, "bad arguments");
  if (dtype != SG_F32 && dtype != SG_F64) return fail(SG_ERR_ARG, "dtype must be SG_F32 or SG_F64");
  if (n == 0) return SG_OK;
  Ptrs px{};
  Coefs cf{};
  for (int i = 0; i < k; ++i) {
    if (!xs[i]) return fail(SG_ERR_ARG, "null vector");
    px.p[i] = xs[i];
    cf.c[i] = coef[i];
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = grid_for(n);
#define MA(TT, MW) k_multi_axpy<TT, MW><<<nb, kThreads, 0, s>>>(n, k, cf, px, (const TT*)y, (TT*)z)
#define MAT(TT)                  \
  do {                           \
    if (k <= 1) MA(TT, 1);       \
    else if (k <= 4) MA(TT, 4);  \
    else if (k <= 8) MA(TT, 8);  \
    else if (k <= 16) MA(TT, 16); \
    else MA(TT, 32);             \
  } while (0)
  if (dtype == SG_F32) MAT(float);
  else MAT(double);
#undef MAT
#undef MA
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

int sg_vec_stats(int64_t n, int32_t dtype, const void* x, double* out, void* stream) {
  if (n < 1 || !x || !out) return fail(SG_ERR_ARG, "bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nb = grid_for(n);
  double* part = nullptr;
  SG_CK(cudaMallocAsync((void**)&part, sizeof(double) * 5 * nb, s));
  if (dtype == SG_F32) k_stats<float><<<nb, kThreads, 0, s>>>(n, (const float*)x, part);
  else k_stats<double><<<nb, kThreads, 0, s>>>(n, (const double*)x, part);
  count_launch();
  std::vector<double> h(5 * nb);
  SG_CK(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CK(cudaFreeAsync(part, s));
  SG_CK(cudaStreamSynchronize(s));
  double mn = INFINITY, mx = -INFINITY, ma = 0.0, s2 = 0.0, bad = 0.0;
  for (int b = 0; b < nb; ++b) {
    mn = std::min(mn, h[5 * b]);
    mx = std::max(mx, h[5 * b + 1]);
    ma = std::max(ma, h[5 * b + 2]);
    s2 += h[5 * b + 3];
    bad += h[5 * b + 4];
  }
  out[0] = mn;
  out[1] = mx;
  out[2] = ma;
  out[3] = std::sqrt(s2);
  out[4] = bad;
  return SG_OK;
}

}  // extern "C"
