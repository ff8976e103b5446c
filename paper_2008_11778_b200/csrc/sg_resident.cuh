// sg_resident.cuh -- cluster-resident whole-sweep kernels for grids whose
// shot fits on the shared memory of one thread-block cluster (C1/C3/C4-sized
// grids, seisopt/wavesim.py:259-346).
//
// The one-step kernel (sg_kernels.cuh) streams every field through L2 at every
// step: ~43 KB of L2 traffic per 64x32 tile-shot and one launch per step.  At
// C3 (241 x 641 padded, 30 shots) the fields are L2-resident and the step is
// bound by L2 throughput and launch latency, not by HBM.  Here one cluster of
// CL CTAs owns one shot for the WHOLE sweep:
//
//   * CTA `rank` owns padded columns [rank W, rank W + W) and every row; its
//     field (u forward, V adjoint) lives in shared memory as two ping-pong
//     planes with 4 halo columns each side and 4 zero guard rows top/bottom
//     (zero-Dirichlet exterior, seisopt/wavesim.py:216-223).
//   * The pointwise state (inc forward, w adjoint) and the adjoint's image
//     accumulator live in registers for the whole sweep.
//   * After a step, the threads owning the first/last column quad also store
//     their new values into the neighbouring CTAs' halo columns through
//     distributed shared memory (st.shared::cluster); one cluster barrier
//     (arrive.release / wait.acquire) per step publishes them.  Ping-pong
//     planes make that single barrier sufficient: step n reads plane n&1 and
//     writes plane (n+1)&1 (own cells and the neighbours' halos).
//   * HBM traffic is only what must leave the chip: the forward's
//     acceleration history a_n (FULL reconstruction), gathers; the adjoint's
//     history reads (TMA, one plane per CTA per step, double-buffered one step
//     ahead) and its band injection rows.
//
// The arithmetic per cell is the one-step kernel's (difference-form
// Laplacian, increment-form leapfrog, V-form adjoint) in the same operation
// order, so sweeps are bitwise those of the one-step kernel.
#pragma once
#include "sg_kernels.cuh"

namespace sg {

constexpr int kResHW = 4;  // halo columns / guard rows in shared memory (any order)
#ifndef SG_RES_NR
#define SG_RES_NR 8
#endif
constexpr int kResNR = SG_RES_NR;  // rows per thread run (z-marching inside the run)
constexpr int kResMaxThreads = 384;
constexpr int kResRec = 128;  // receivers per CTA staged in shared memory

template <typename T>
struct ResArgs {
  CUtensorMap h_map;        // ADJ: history {ldx, nzp, planes}, box {W, hrows, 1}
  const T* inv_m;           // 1/m, row 0 col 0, row pitch ldx
  const T* pz;              // sponge profiles (rows / cols)
  const T* px;
  int nzp, nxp, ldx;
  int W, CL, Q, runs;       // columns per CTA, CTAs per cluster, quads per CTA, row runs
  int SR;                   // shared rows per plane (runs NR + 2 HW; HW zero guard rows each end)
  int hrows, hboxes;        // ADJ: TMA box rows (<= 256) and boxes per plane
  int n0, n1;               // steps [n0, n1): forward ascending, adjoint n1-1 .. n0
  int s0;                   // first batch shot of this launch
  T dt2;
  T cz[5], cx[5];
  // forward
  const int* src_rc;        // (shots, 4, 2) tap rows / cols of the batch
  const T* src_w;           // (shots, 4) weights * src_scale
  const T* wav;             // wavelet amplitudes (nt)
  T* hist;                  // FWD: acceleration history (nullptr: none)
  int64_t hplane;           // history plane (nzp * ldx)
  int hist_steps, hist_n0;  // plane of shot b at step n: b * hist_steps + n - hist_n0
  const T* rec_w;           // (4, nrec) receiver tap weights
  const int* rec_off;       // (4, nrec) shared-plane offsets relative to the owner CTA
  const int* rec_list;      // receivers sorted by owner rank
  const int* rec_start;     // (CL + 1) ranges into rec_list
  int nrec;
  T* gather;                // gathers (+ b * gather_stride + n * nrec + r); nullptr: none
  int64_t gather_stride;
  // adjoint
  const T* inj_dense;       // R^T y: (+ b * inj_stride + n * inj_nrows * nxp + rr * nxp + j)
  int64_t inj_stride;
  int inj_row0, inj_nrows;
  T* image;                 // per-shot image planes (+ b * image_stride + i * ldx + j)
  int64_t image_stride;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

// a column quad as two packed pairs (cols 0-1, cols 2-3)
template <typename T>
struct Quad {
  V2<T> a, b;
};

template <typename T>
__device__ __forceinline__ Quad<T> lds4(const T* p) {
  Quad<T> q;
  q.a = lds2(p);
  q.b = lds2(p + 2);
  return q;
}

template <>
__device__ __forceinline__ Quad<float> lds4<float>(const float* p) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  Quad<float> q;
  q.a = V2<float>::make(v.x, v.y);
  q.b = V2<float>::make(v.z, v.w);
  return q;
}

template <typename T>
__device__ __forceinline__ void st4(T* p, V2<T> a, V2<T> b) {
  st2(p, a);
  st2(p + 2, b);
}

template <>
__device__ __forceinline__ void st4<float>(float* p, V2<float> a, V2<float> b) {
  float4 v;
  a.split(v.x, v.y);
  b.split(v.z, v.w);
  *reinterpret_cast<float4*>(p) = v;
}

template <typename T>
__host__ __device__ constexpr int res_align(int n) {
  return ((n * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
}

// Shared-memory plan of a resident CTA (element offsets, 128-B aligned):
//   two own-column planes  SR x W           (ping-pong, rows -HW .. SR-HW-1)
//   three halo slots       2 x SR x 4       (left | right neighbour columns)
//   ADJ: two history planes hboxes*hrows x W (TMA staging)
template <typename T>
struct ResSmem {
  int plane, halo, hist, bytes;
  __host__ __device__ ResSmem(bool adj, int SR, int W, int hrows, int hboxes) {
    plane = res_align<T>(SR * W);
    halo = res_align<T>(2 * SR * 4);
    hist = res_align<T>(hrows * hboxes * W);
    bytes = (2 * plane + 3 * halo + (adj ? 2 * hist : 0)) * (int)sizeof(T);
  }
};

// 16-byte asynchronous store into another CTA's shared memory, completing
// `bytes` on that CTA's mbarrier (both addresses already mapped)
__device__ __forceinline__ void st_async4(uint32_t raddr, uint32_t rbar, float v0, float v1,
                                          float v2, float v3) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          raddr),
      "f"(v0), "f"(v1), "f"(v2), "f"(v3), "r"(rbar)
      : "memory");
}

// Laplacian of the quad at window row `c` (a register window of quads) in
// difference form, horizontal neighbours from the quads left (L) and right
// (Rt) of it -- the one-step kernel's lap2 per pair, same operation order.
template <typename T, int R>
__device__ __forceinline__ void res_lap(const Quad<T>* w, int c, const Quad<T>& L,
                                        const Quad<T>& Rt, const T* cz, const T* cx, V2<T>& la,
                                        V2<T>& lb) {
  using P = V2<T>;
  const P ua = w[c].a, ub = w[c].b;
  T l0, l1, l2, l3, c0, c1, c2, c3, r0, r1, r2, r3;
  L.a.split(l0, l1);
  L.b.split(l2, l3);
  ua.split(c0, c1);
  ub.split(c2, c3);
  Rt.a.split(r0, r1);
  Rt.b.split(r2, r3);
  P xma[5], xpa[5], xmb[5], xpb[5];
  xma[1] = P::make(l3, c0);
  xpa[1] = P::make(c1, c2);
  xmb[1] = P::make(c1, c2);
  xpb[1] = P::make(c3, r0);
  if constexpr (R >= 2) {
    xma[2] = L.b;
    xpa[2] = ub;
    xmb[2] = ua;
    xpb[2] = Rt.a;
  }
  if constexpr (R >= 4) {
    xma[3] = P::make(l1, l2);
    xpa[3] = P::make(c3, r0);
    xmb[3] = P::make(l3, c0);
    xpb[3] = P::make(r1, r2);
    xma[4] = L.a;
    xpa[4] = Rt.a;
    xmb[4] = L.b;
    xpb[4] = Rt.b;
  }
  P lza = P::make(T(0), T(0)), lxa = lza, lzb = lza, lxb = lza;
#pragma unroll
  for (int kk = 1; kk <= R; ++kk) {
    const P czp = P::make(cz[kk], cz[kk]);
    const P cxp = P::make(cx[kk], cx[kk]);
    lza = P::fma(czp, (w[c - kk].a - ua) + (w[c + kk].a - ua), lza);
    lxa = P::fma(cxp, (xma[kk] - ua) + (xpa[kk] - ua), lxa);
    lzb = P::fma(czp, (w[c - kk].b - ub) + (w[c + kk].b - ub), lzb);
    lxb = P::fma(cxp, (xmb[kk] - ub) + (xpb[kk] - ub), lxb);
  }
  la = lza + lxa;
  lb = lzb + lxb;
}

// One launch = a whole sweep for `gridDim.x / CL` shots, one cluster per shot.
//   FWD  (seisopt/wavesim.py:286-303): a_n = inv_m L u_n [+ amp_n w inv_m at
//        the source taps]; inc' = d (inc + dt^2 a_n); u' = d u_n + inc';
//        gathers R u_n; history a_n (HIST).
//   ADJ  (seisopt/wavesim.py:330-345, V-form, see sg_kernels.cuh):
//        w_n = d w_{n+1} + L V_n + R^T y_n; V_{n-1} = d V_n + (dt^2 inv_m d) w_n;
//        image -= a_n V_n (a_n from the history, TMA-staged one step ahead).
// Halo exchange: step k reads the neighbours' edge quads from halo slot k % 3
// and sends its own edge quads into the neighbours' slot (k + 1) % 3 with
// st.async, which completes bytes on the receiver's slot mbarrier.  Three
// slots make it race-free without a cluster barrier per step: a CTA can only
// be one step ahead of its neighbours, and a slot is rewritten two steps after
// it was read.  The own planes are ping-pong with one __syncthreads per step.
template <typename T, int R, bool ADJ, bool HIST, bool GATHER>
__global__ void __launch_bounds__(kResMaxThreads, 1)
    k_resident(const __grid_constant__ ResArgs<T> a) {
  static_assert(sizeof(T) == 4, "resident sweeps are fp32");
  using P = V2<T>;
  constexpr int NR = kResNR;
  constexpr int HW = kResHW;
  constexpr int NW = NR + 2 * R;  // window rows of a run
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t hbar[2];  // ADJ history staging
  __shared__ __align__(8) uint64_t xbar[3];  // halo slots
  __shared__ int s_src[8];
  __shared__ T s_sw[4];
  // this CTA's receivers (first kResRec staged in shared memory)
  __shared__ int s_rid[GATHER ? kResRec : 1];
  __shared__ int s_roff[GATHER ? 4 * kResRec : 1];
  __shared__ T s_rw[GATHER ? 4 * kResRec : 1];

  const int W = a.W;
  const ResSmem<T> lay(ADJ, a.SR, W, a.hrows, a.hboxes);
  T* const pl0 = reinterpret_cast<T*>(smem_raw);
  T* const hal0 = pl0 + 2 * lay.plane;       // slot s: hal0 + s * lay.halo; [L | R]
  T* const hbase = hal0 + 3 * lay.halo;      // ADJ history planes
  const int HR = a.SR * 4;                   // right half of a halo slot

  const int rank = (int)cluster_rank();
  const int b = a.s0 + (int)blockIdx.x / a.CL;  // batch shot of this cluster
  const int c0 = rank * W;                      // first padded column of this CTA
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;

  for (int e = tid; e < 2 * lay.plane + 3 * lay.halo; e += nthr) pl0[e] = T(0);
  if (!ADJ && a.src_rc != nullptr) {
    if (tid < 8) s_src[tid] = a.src_rc[b * 8 + tid];
    if (tid < 4) s_sw[tid] = a.src_w[b * 4 + tid];
  }
  int rs = 0, nrl = 0;
  if constexpr (GATHER) {
    rs = a.rec_start[rank];
    nrl = a.rec_start[rank + 1] - rs;
    for (int e = tid; e < min(nrl, kResRec); e += nthr) {
      const int r = a.rec_list[rs + e];
      s_rid[e] = r;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        s_roff[kk * kResRec + e] = a.rec_off[kk * a.nrec + r];
        s_rw[kk * kResRec + e] = a.rec_w[kk * a.nrec + r];
      }
    }
  }
  if (tid == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(&xbar[s], 1);
    if (ADJ) {
      mbar_init(&hbar[0], 1);
      mbar_init(&hbar[1], 1);
    }
    fence_barrier_init();
  }

  // this thread: quad q (columns j .. j+3), rows i0 .. i0 + NR - 1
  const int q = tid % a.Q;
  const int run = tid / a.Q;
  const bool active = run < a.runs;
  const int i0 = run * NR;
  const int j = c0 + 4 * q;
  const int nq = active ? max(0, min(NR, a.nzp - i0)) : 0;
  const bool qvalid = j < a.nxp;                // quad holds a grid column
  const bool full = nq == NR && j + 3 < a.nxp;  // no row / column masking
  const bool has_l = rank > 0, has_r = rank < a.CL - 1;
  const int to_left = (q == 0 && has_l) ? rank - 1 : -1;           // my quad is its right halo
  const int to_right = (q == a.Q - 1 && has_r) ? rank + 1 : -1;    // my quad is its left halo
  const uint32_t xbytes = (uint32_t)((has_l ? 1 : 0) + (has_r ? 1 : 0)) * a.nzp * 16u;

  T pxl[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) pxl[l] = (j + l < a.nxp) ? a.px[j + l] : T(0);
  const P pxa = P::make(pxl[0], pxl[1]), pxb = P::make(pxl[2], pxl[3]);
  T pzr[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) pzr[r] = r < nq ? a.pz[i0 + r] : T(0);
  // pointwise state in registers: inc (forward) / w (adjoint); image (adjoint)
  P sa[NR], sb[NR];
  T img[ADJ ? 4 * NR : 1];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    sa[r] = P::make(T(0), T(0));
    sb[r] = sa[r];
  }
#pragma unroll
  for (int e = 0; e < (ADJ ? 4 * NR : 1); ++e) img[e] = T(0);
  const P dt2p = P::make(a.dt2, a.dt2);

  // history TMA (adjoint): plane of step n into staging buffer k & 1
  auto issue_hist = [&](int n, int k) {
    T* dst = hbase + (k & 1) * lay.hist;
    const int pl = b * a.hist_steps + (n - a.hist_n0);
    mbar_expect_tx(&hbar[k & 1], (uint32_t)(a.hboxes * a.hrows * W * (int)sizeof(T)));
    for (int bx = 0; bx < a.hboxes; ++bx)
      tma_load_3d(dst + bx * a.hrows * W, &a.h_map, &hbar[k & 1], c0, bx * a.hrows, pl);
  };

  __syncthreads();
  int srcmask = 0;  // source taps of this shot inside this thread's cells
  if (!ADJ && a.src_rc != nullptr && nq > 0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int sr = s_src[2 * t], sc = s_src[2 * t + 1];
      if (sr >= i0 && sr < i0 + nq && sc >= j && sc < j + 4) srcmask |= 1 << t;
    }
  }
  if (ADJ && tid == 0) issue_hist(a.n1 - 1, 0);
  const int nsteps = a.n1 - a.n0;
  // halo bytes expected for step 1 (slot 1)
  if (tid == 0 && nsteps > 1 && xbytes > 0) mbar_expect_tx(&xbar[1], xbytes);
  // every CTA's barriers and zeroed planes exist before any neighbour sends
  cluster_sync_all();

  // remote addresses of the neighbours' halo slots / slot barriers (slot 0)
  uint32_t rdst = 0, rbar = 0;
  if (to_left >= 0) {
    rdst = map_rank(smem_u32(hal0 + HR), (uint32_t)to_left);
    rbar = map_rank(smem_u32(&xbar[0]), (uint32_t)to_left);
  } else if (to_right >= 0) {
    rdst = map_rank(smem_u32(hal0), (uint32_t)to_right);
    rbar = map_rank(smem_u32(&xbar[0]), (uint32_t)to_right);
  }
  const bool sender = to_left >= 0 || to_right >= 0;

  for (int k = 0; k < nsteps; ++k) {
    const int n = ADJ ? a.n1 - 1 - k : a.n0 + k;
    const int slot = k % 3, nslot = (k + 1) % 3;
    const T* cur = pl0 + (k & 1) * lay.plane;
    T* nxt = pl0 + ((k + 1) & 1) * lay.plane;
    const T* hal = hal0 + slot * lay.halo;
    if (k >= 1 && xbytes > 0) mbar_wait(&xbar[slot], ((k - (slot == 0 ? 3 : slot)) / 3) & 1);
    // bytes the neighbours will send for step k + 2 (slot (k + 2) % 3, last
    // waited at step k - 1)
    if (tid == 0 && k + 2 < nsteps && xbytes > 0) mbar_expect_tx(&xbar[(k + 2) % 3], xbytes);

    if constexpr (!ADJ && GATHER) {
      // receiver sampling before the update (seisopt/wavesim.py:225-226, :287);
      // offsets >= 0 index the own plane, < 0 the halo slot
      T* gat = a.gather + (int64_t)b * a.gather_stride + (int64_t)n * a.nrec;
      for (int e = tid; e < nrl; e += nthr) {
        if (e < kResRec) {
          auto tap = [&](int kk) {
            const int o = s_roff[kk * kResRec + e];
            return o >= 0 ? cur[o] : hal[-1 - o];
          };
          T g = s_rw[e] * tap(0);
#pragma unroll
          for (int kk = 1; kk < 4; ++kk) g += s_rw[kk * kResRec + e] * tap(kk);
          gat[s_rid[e]] = g;
        } else {
          const int r = a.rec_list[rs + e];
          auto tap = [&](int kk) {
            const int o = a.rec_off[kk * a.nrec + r];
            return o >= 0 ? cur[o] : hal[-1 - o];
          };
          T g = a.rec_w[r] * tap(0);
#pragma unroll
          for (int kk = 1; kk < 4; ++kk) g += a.rec_w[kk * a.nrec + r] * tap(kk);
          gat[r] = g;
        }
      }
    }
    const T* hcur = nullptr;
    if constexpr (ADJ) {
      if (tid == 0 && n - 1 >= a.n0) issue_hist(n - 1, k + 1);
      mbar_wait(&hbar[k & 1], (k >> 1) & 1);
      hcur = hbase + (k & 1) * lay.hist;
    }
    T amp = T(0);
    if (!ADJ && srcmask) amp = a.wav[n];
    const T* inj = nullptr;
    if (ADJ && a.inj_dense != nullptr)
      inj = a.inj_dense + (int64_t)b * a.inj_stride + (int64_t)n * a.inj_nrows * a.nxp;
    T* hout = nullptr;
    if (!ADJ && HIST) hout = a.hist + ((int64_t)b * a.hist_steps + (n - a.hist_n0)) * a.hplane;
    const bool send = sender && k + 1 < nsteps;
    const uint32_t sdst = rdst + (uint32_t)(nslot * lay.halo * (int)sizeof(T));
    const uint32_t sbar = rbar + (uint32_t)(nslot * 8);
    // horizontal neighbours: own plane, or the halo slot for the edge quads
    const T* lb_ = (q == 0) ? hal + HW * 4 : cur + HW * W + 4 * q - 4;
    const int ls = (q == 0) ? 4 : W;
    const T* rb_ = (q == a.Q - 1) ? hal + HR + HW * 4 : cur + HW * W + 4 * q + 4;
    const int rs = (q == a.Q - 1) ? 4 : W;

    if (nq > 0) {
      auto body = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        Quad<T> win[NW];
        const T* col = cur + (i0 - R + HW) * W + 4 * q;
        // sliding vertical window: rows r .. r + 2R live while row r is updated
#pragma unroll
        for (int r = 0; r < 2 * R; ++r) win[r] = lds4(col + r * W);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (!FULL && r >= nq) continue;
          win[r + 2 * R] = lds4(col + (r + 2 * R) * W);
          const int i = i0 + r;
          const Quad<T> L = lds4(lb_ + i * ls), Rt = lds4(rb_ + i * rs);
          P la, lb;
          res_lap<T, R>(win, r + R, L, Rt, a.cz, a.cx, la, lb);
          const P pzp = P::make(pzr[r], pzr[r]);
          const P dda = pzp * pxa, ddb = pzp * pxb;
          const P ua = win[r + R].a, ub = win[r + R].b;
          // 1/m of the quad (L1-resident across steps; 0 beyond nxp)
          P ma, mb;
          {
            T m4[4];
            if constexpr (FULL) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(a.inv_m + i * a.ldx + j));
              m4[0] = v.x;
              m4[1] = v.y;
              m4[2] = v.z;
              m4[3] = v.w;
            } else {
#pragma unroll
              for (int l = 0; l < 4; ++l)
                m4[l] = (j + l < a.nxp) ? __ldg(a.inv_m + i * a.ldx + j + l) : T(0);
            }
            ma = P::make(m4[0], m4[1]);
            mb = P::make(m4[2], m4[3]);
          }
          P na, nb;
          if constexpr (!ADJ) {
            P acca = la * ma, accb = lb * mb;
            if (srcmask) {
              T v[4], m[4];
              acca.split(v[0], v[1]);
              accb.split(v[2], v[3]);
              ma.split(m[0], m[1]);
              mb.split(m[2], m[3]);
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                if (!((srcmask >> t) & 1) || s_src[2 * t] != i) continue;
#pragma unroll
                for (int l = 0; l < 4; ++l)
                  if (s_src[2 * t + 1] == j + l) v[l] += amp * s_sw[t] * m[l];
              }
              acca = P::make(v[0], v[1]);
              accb = P::make(v[2], v[3]);
            }
            if (HIST && qvalid) st4(hout + i * a.ldx + j, acca, accb);
            sa[r] = P::fma(dt2p, acca, sa[r]) * dda;
            sb[r] = P::fma(dt2p, accb, sb[r]) * ddb;
            na = P::fma(dda, ua, sa[r]);
            nb = P::fma(ddb, ub, sb[r]);
          } else {
            if (inj != nullptr) {
              const int rr = i - a.inj_row0;
              if (rr >= 0 && rr < a.inj_nrows) {
                // R^T y: duplicate taps accumulate (np.add.at, seisopt/wavesim.py:229)
                T v[4];
                la.split(v[0], v[1]);
                lb.split(v[2], v[3]);
#pragma unroll
                for (int l = 0; l < 4; ++l)
                  if (j + l < a.nxp) v[l] += inj[rr * a.nxp + j + l];
                la = P::make(v[0], v[1]);
                lb = P::make(v[2], v[3]);
              }
            }
            const Quad<T> hh = lds4(hcur + i * W + 4 * q);
            sa[r] = P::fma(dda, sa[r], la);
            sb[r] = P::fma(ddb, sb[r], lb);
            na = P::fma(dda, ua, ((dt2p * ma) * dda) * sa[r]);
            nb = P::fma(ddb, ub, ((dt2p * mb) * ddb) * sb[r]);
            T v0, v1, v2, v3, h0, h1, h2, h3;
            ua.split(v0, v1);
            ub.split(v2, v3);
            hh.a.split(h0, h1);
            hh.b.split(h2, h3);
            img[4 * r + 0] -= h0 * v0;
            img[4 * r + 1] -= h1 * v1;
            img[4 * r + 2] -= h2 * v2;
            img[4 * r + 3] -= h3 * v3;
          }
          st4(nxt + (i + HW) * W + 4 * q, na, nb);
          if (send) {
            T v0, v1, v2, v3;
            na.split(v0, v1);
            nb.split(v2, v3);
            st_async4(sdst + (uint32_t)((i + HW) * 16), sbar, v0, v1, v2, v3);
          }
        }
      };
      if (full) body(std::true_type{});
      else body(std::false_type{});
    }
    // own plane (k + 1) & 1 complete; plane k & 1 free for step k + 1's writes
    __syncthreads();
  }
  if constexpr (ADJ) {
    if (nq > 0 && qvalid) {
      T* ig = a.image + (int64_t)b * a.image_stride + j;
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r < nq)
          st4(ig + (int64_t)(i0 + r) * a.ldx, P::make(img[4 * r], img[4 * r + 1]),
              P::make(img[4 * r + 2], img[4 * r + 3]));
    }
  }
  // no CTA leaves while a neighbour may still address its shared memory
  cluster_sync_all();
}

}  // namespace sg
