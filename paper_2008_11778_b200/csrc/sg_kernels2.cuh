// sg_kernels2.cuh -- two time steps per launch (temporal blocking), fp32.
//
// The one-step kernel (sg_kernels.cuh) moves ~21.6 B per shot-cell-step.  This
// kernel advances every shot of a CTA group by TWO steps per launch:
//
//   step 1 (n)    on E  = tile + a 4-cell ring (72 x 40), from the field on
//                 E + 4 = tile + 8 (80 x 48, TMA, OOB zero fill) and the state
//                 on E (TMA); the new field on E is kept in shared memory;
//   step 2 (n+1)  on the 64 x 32 tile, from that shared field.
//
// Per two steps a cell costs: field halo read 1.875 x 4 B, state read
// 1.41 x 4 B, field + state write 8 B, two history planes 8 B -> ~14.6 B per
// step instead of ~21.6 B; launches halve.  The ring recomputation costs
// +41 % stencil work in step 1, which this HBM/latency-bound kernel absorbs.
// Cells outside the padded grid have sponge factor d = 0 (zero guards of the
// profile arrays), so the ring field outside is exactly zero, reproducing the
// zero-Dirichlet exterior; results equal two launches of the one-step kernel
// bit for bit (same operation order per cell).
//
// Forward: receivers of both steps are sampled inside the tile CTAs (each
// receiver belongs to the tile holding its first tap; all four taps then lie
// in E).  Adjoint: R^T y of both steps is injected per cell (CSR), imaging
// against both history planes.
#pragma once
#include "sg_kernels.cuh"

namespace sg {

constexpr int kE = kHalo;             // ring width of step 1 (= 8th-order radius)
constexpr int kEW = kBX + 2 * kE;     // 72: step-1 region width
constexpr int kEH = kTH2 + 2 * kE;     // 40: step-1 region height
constexpr int kUW = kBX + 4 * kE;     // 80: field box width
constexpr int kUH = kTH2 + 4 * kE;     // 48: field box height
constexpr int kTY2 = 4;               // thread rows; block = kEW x kTY2 = 288 threads
constexpr int kNY1 = kEH / kTY2;      // 10 step-1 rows per thread
constexpr int kThreads2 = kEW * kTY2;

template <typename T>
struct Step2Args {
  CUtensorMap f_halo2[2];  // field buffers, box 80 x 48
  CUtensorMap s_ring[2];   // state buffers (ping-pong), box 72 x 40
  CUtensorMap m_ring[1];   // 1/m (single guarded plane), box 72 x 40
  CUtensorMap h_tile;      // history {ldx, nzp, planes}, box 64 x 32 (adjoint loads)
  T* f[2];
  int cur;                 // read f[cur], s[cur]; write f[cur ^ 1], s[cur ^ 1]
  T* state[2];
  const T* pz;
  const T* px;
  int64_t plane;
  int nzp, nxp, ldx, tiles_x, ntiles;
  int count, G;
  T dt2;
  T cz[5], cx[5];
  int n0;                  // FWD: steps n0, n0+1; ADJ: steps n0, n0-1
  // history: plane of shot b for step n = b * hist_steps + hist_slot(n)
  int hist_on, hist_steps, slot0, slot1;  // slots of the two steps
  T* hist;
  int64_t hplane;
  // forward
  const int* src_rc;
  const T* src_w;
  T amp0, amp1;
  const int* tile_rec_ptr;  // receivers anchored in each tile (CSR)
  const int* tile_rec;
  const int* rec_rc;        // (4, nrec, 2) tap rows / cols
  const T* rec_w;           // (4, nrec)
  int nrec;
  T* gather;                // gathers at step n0 (+ b*gather_stride + n*nrec + r)
  int64_t gather_stride;
  // adjoint
  int inj_row0, inj_nrows;
  const int* inj_ptr;
  const int* inj_rec;
  const T* inj_w;
  const T* ybar;            // adjoint data at step n0 (step n0-1 is ybar - nrec)
  int64_t ybar_stride;
  T* image;
  int64_t image_stride;
};

template <bool ADJ>
struct Smem2 {
  static constexpr int U = kUW * kUH;        // 3840
  static constexpr int S = kEW * kEH;        // 2880
  static constexpr int H = ADJ ? 2 * kBX * kTH2 : 0;
  static constexpr int STAGE = U + S + H;
  static constexpr int IM = kEW * kEH;
  static constexpr int MID = kEW * kEH;
  static constexpr int BYTES = (2 * STAGE + IM + MID) * 4;
};

template <bool ADJ>
__host__ __device__ constexpr int step2_smem_bytes() {
  return Smem2<ADJ>::BYTES;
}

template <int R, bool ADJ, bool HIST, bool GATHER>
__global__ void __launch_bounds__(kThreads2, 2) k_step2(const __grid_constant__ Step2Args<float> a) {
  using T = float;
  using SM = Smem2<ADJ>;
  using P = V2<T>;
  constexpr int NH = kNY1 / 2;  // pairs (q, q + NH)
  constexpr int NCOL = kNY1 + 2 * R;
  constexpr int UO = kE - R;  // U row offset of the radius-R window of E row 0
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sbase = reinterpret_cast<T*>(smem_raw);
  T* s_im = sbase + 2 * SM::STAGE;
  T* s_mid = s_im + SM::IM;
  __shared__ __align__(8) uint64_t bar[3];

  const int tid = threadIdx.y * kEW + threadIdx.x;
  const int grp = blockIdx.y;
  const int b0 = grp * a.G;
  const int nb = min(a.G, a.count - b0);
  const int tile = blockIdx.x;
  const int tzi = tile / a.tiles_x;
  const int i0 = tzi * kTH2;
  const int j0 = (tile - tzi * a.tiles_x) * kBX;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int s = k & 1;
    T* st = sbase + s * SM::STAGE;
    const int b = b0 + k;
    constexpr uint32_t bytes = (SM::U + SM::S + SM::H) * 4u;
    mbar_expect_tx(&bar[s], bytes);
    tma_load_3d(st, &a.f_halo2[a.cur], &bar[s], j0 - 2 * kE, kGuard + i0 - 2 * kE, b);
    tma_load_3d(st + SM::U, &a.s_ring[a.cur], &bar[s], j0 - kE, kGuard + i0 - kE, b);
    if (ADJ && HIST) {
      tma_load_3d(st + SM::U + SM::S, &a.h_tile, &bar[s], j0, i0, b * a.hist_steps + a.slot0);
      tma_load_3d(st + SM::U + SM::S + kBX * kTH2, &a.h_tile, &bar[s], j0, i0,
                  b * a.hist_steps + a.slot1);
    }
  };
  if (tid == 0) {
    mbar_expect_tx(&bar[2], SM::IM * 4u);
    tma_load_3d(s_im, &a.m_ring[0], &bar[2], j0 - kE, kGuard + i0 - kE, 0);
    issue(0);
  }

  // this thread: E column ex, E rows er0 .. er0 + 9
  const int ex = threadIdx.x;
  const int er0 = threadIdx.y * kNY1;
  const int gj = j0 - kE + ex;         // global column
  const int gi0 = i0 - kE + er0;       // global row of the first cell
  const bool col_in_tile = ex >= kE && ex < kE + kBX;
  const T pxj = a.px[gj];              // guarded: zero outside [0, nxp)
  T im[kNY1], dd[kNY1];
  mbar_wait(&bar[2], 0);
#pragma unroll
  for (int q = 0; q < kNY1; ++q) {
    im[q] = s_im[(er0 + q) * kEW + ex];
    dd[q] = a.pz[gi0 + q] * pxj;       // guarded: zero outside [0, nzp)
  }
  T img[kNY1];
#pragma unroll
  for (int q = 0; q < kNY1; ++q) img[q] = T(0);

  for (int k = 0; k < nb; ++k) {
    const int b = b0 + k;
    if (tid == 0 && k + 1 < nb) issue(k + 1);
    bool src_here = false;
    if (!ADJ && a.src_rc != nullptr) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r = a.src_rc[(b * 4 + t) * 2], c = a.src_rc[(b * 4 + t) * 2 + 1];
        src_here |= (r >= i0 - kE && r < i0 + kTH2 + kE && c >= j0 - kE && c < j0 + kBX + kE);
      }
    }
    const bool inj_tile = ADJ && a.ybar != nullptr && a.inj_row0 < i0 + kTH2 + kE &&
                          a.inj_row0 + a.inj_nrows > i0 - kE;
    mbar_wait(&bar[k & 1], (k >> 1) & 1);
    const T* su = sbase + (k & 1) * SM::STAGE;
    const T* ss = su + SM::U;

    // ------------------------------ step 1 on E ------------------------------
    T v1[kNY1], s1[kNY1];  // new field and state of this thread's E cells
    {
      // E cell (er, ex) is U cell (er + kE, ex + kE); window top = row er0 - R
      const T* sc = su + (er0 + UO) * kUW + ex + kE;
      T col[NCOL];
#pragma unroll
      for (int r = 0; r < NCOL; ++r) col[r] = sc[r * kUW];
#pragma unroll
      for (int q = 0; q < NH; ++q) {
        const P uc = P::make(col[q + R], col[q + NH + R]);
        const T* ra = sc + (q + R) * kUW;
        const T* rb = sc + (q + NH + R) * kUW;
        P lz = P::make(T(0), T(0)), lx = P::make(T(0), T(0));
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const P cz = P::make(a.cz[kk], a.cz[kk]);
          const P cx = P::make(a.cx[kk], a.cx[kk]);
          const P zm = P::make(col[q + R - kk], col[q + NH + R - kk]);
          const P zp = P::make(col[q + R + kk], col[q + NH + R + kk]);
          const P xm = P::make(ra[-kk], rb[-kk]);
          const P xp = P::make(ra[kk], rb[kk]);
          lz = P::fma(cz, (zm - uc) + (zp - uc), lz);
          lx = P::fma(cx, (xm - uc) + (xp - uc), lx);
        }
        T lap[2], ucs[2];
        (lz + lx).split(lap[0], lap[1]);
        uc.split(ucs[0], ucs[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int q2 = q + h * NH;
          const int gi = gi0 + q2;
          const T sv = ss[(er0 + q2) * kEW + ex];
          T lp = lap[h];
          if (!ADJ) {
            T acc = lp * im[q2];
            if (src_here) {
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int r = a.src_rc[(b * 4 + t) * 2], c = a.src_rc[(b * 4 + t) * 2 + 1];
                if (r == gi && c == gj) acc += a.amp0 * a.src_w[b * 4 + t] * im[q2];
              }
            }
            const bool in_tile = col_in_tile && (er0 + q2) >= kE && (er0 + q2) < kE + kTH2;
            if (HIST && in_tile && gi < a.nzp && gj < a.nxp)
              a.hist[((int64_t)b * a.hist_steps + a.slot0) * a.hplane + gi * a.ldx + gj] = acc;
            s1[q2] = dd[q2] * (sv + a.dt2 * acc);
            v1[q2] = dd[q2] * ucs[h] + s1[q2];
          } else {
            if (inj_tile) {
              const int rr = gi - a.inj_row0;
              if (rr >= 0 && rr < a.inj_nrows && gj >= 0 && gj < a.nxp) {
                const int cell = rr * a.nxp + gj;
                const int p1 = a.inj_ptr[cell + 1];
                for (int p = a.inj_ptr[cell]; p < p1; ++p)
                  lp += a.inj_w[p] * a.ybar[(int64_t)b * a.ybar_stride + a.inj_rec[p]];
              }
            }
            s1[q2] = dd[q2] * sv + lp;
            v1[q2] = dd[q2] * ucs[h] + (a.dt2 * im[q2] * dd[q2]) * s1[q2];
            const bool in_tile = col_in_tile && (er0 + q2) >= kE && (er0 + q2) < kE + kTH2;
            if (HIST && in_tile) {
              const int ti = er0 + q2 - kE, tj = ex - kE;
              img[q2] -= su[SM::U + SM::S + ti * kBX + tj] * ucs[h];
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kNY1; ++q) s_mid[(er0 + q) * kEW + ex] = v1[q];
    }
    __syncthreads();  // s_mid complete

    // forward receivers of both steps, sampled from the staged fields
    if (!ADJ && GATHER) {
      const int p0 = a.tile_rec_ptr[tile], p1 = a.tile_rec_ptr[tile + 1];
      for (int p = p0 + tid; p < p1; p += kThreads2) {
        const int r = a.tile_rec[p];
        T g0 = T(0), g1 = T(0);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int rr = a.rec_rc[(t * a.nrec + r) * 2] - i0;
          const int cc = a.rec_rc[(t * a.nrec + r) * 2 + 1] - j0;
          const T w = a.rec_w[t * a.nrec + r];
          if (t == 0) {
            g0 = w * su[(rr + 2 * kE) * kUW + cc + 2 * kE];
            g1 = w * s_mid[(rr + kE) * kEW + cc + kE];
          } else {
            g0 += w * su[(rr + 2 * kE) * kUW + cc + 2 * kE];
            g1 += w * s_mid[(rr + kE) * kEW + cc + kE];
          }
        }
        T* gout = a.gather + (int64_t)b * a.gather_stride + (int64_t)a.n0 * a.nrec + r;
        gout[0] = g0;
        gout[a.nrec] = g1;
      }
    }

    // ------------------------------ step 2 on the tile -----------------------
    if (col_in_tile) {
      const T* sc = s_mid + (er0 - R) * kEW + ex;  // rows er0 - R .. (inside E for tile rows)
      const int64_t sb = (int64_t)b * a.plane;
      T* __restrict__ fout = a.f[a.cur ^ 1] + sb;
      T* __restrict__ sout = a.state[a.cur ^ 1] + sb;
#pragma unroll
      for (int q = 0; q < kNY1; ++q) {
        const int er = er0 + q;
        if (er < kE || er >= kE + kTH2) continue;  // ring rows: step 1 only
        const int gi = gi0 + q;
        if (gi >= a.nzp || gj >= a.nxp) continue;
        const T uc = v1[q];
        T lz = T(0), lx = T(0);
        const T* rw = sc + (q + R) * kEW;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          lz += a.cz[kk] * ((rw[-kk * kEW] - uc) + (rw[kk * kEW] - uc));
          lx += a.cx[kk] * ((rw[-kk] - uc) + (rw[kk] - uc));
        }
        T lp = lz + lx;
        const int o = gi * a.ldx + gj;
        if (!ADJ) {
          T acc = lp * im[q];
          if (src_here) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int r = a.src_rc[(b * 4 + t) * 2], c = a.src_rc[(b * 4 + t) * 2 + 1];
              if (r == gi && c == gj) acc += a.amp1 * a.src_w[b * 4 + t] * im[q];
            }
          }
          if (HIST) a.hist[((int64_t)b * a.hist_steps + a.slot1) * a.hplane + o] = acc;
          const T so = dd[q] * (s1[q] + a.dt2 * acc);
          sout[o] = so;
          fout[o] = dd[q] * uc + so;
        } else {
          if (inj_tile) {
            const int rr = gi - a.inj_row0;
            if (rr >= 0 && rr < a.inj_nrows) {
              const int cell = rr * a.nxp + gj;
              const int p1 = a.inj_ptr[cell + 1];
              for (int p = a.inj_ptr[cell]; p < p1; ++p)
                lp += a.inj_w[p] * a.ybar[(int64_t)b * a.ybar_stride - a.nrec + a.inj_rec[p]];
            }
          }
          const T so = dd[q] * s1[q] + lp;
          sout[o] = so;
          fout[o] = dd[q] * uc + (a.dt2 * im[q] * dd[q]) * so;
          if (HIST) {
            const int ti = er - kE, tj = ex - kE;
            img[q] -= su[SM::U + SM::S + kBX * kTH2 + ti * kBX + tj] * uc;
          }
        }
      }
    }
    __syncthreads();  // stage (k & 1) and s_mid are free
  }
  if (ADJ && HIST && col_in_tile) {
    T* ig = a.image + (int64_t)grp * a.image_stride;
#pragma unroll
    for (int q = 0; q < kNY1; ++q) {
      const int er = er0 + q, gi = gi0 + q;
      if (er >= kE && er < kE + kTH2 && gi < a.nzp && gj < a.nxp) ig[gi * a.ldx + gj] += img[q];
    }
  }
}

}  // namespace sg
