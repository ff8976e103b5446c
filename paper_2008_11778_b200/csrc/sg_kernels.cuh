// sg_kernels.cuh -- sm_100a time-step kernels for the damped-leapfrog acoustic
// propagator of seisopt (seisopt/wavesim.py:259-346), re-designed for B200.
//
// Memory layout ("guarded plane", one per shot):
//   rows  -4 .. nzp+3 (4 zero guard rows top and bottom), row pitch ldx >= nxp+4
//   (multiple of 32 elements), so every stencil read of a valid cell lands on
//   either a real cell or a zero cell: the reference's zero-Dirichlet exterior
//   (seisopt/wavesim.py:216-223) costs no branches.  Columns nxp..ldx-1 are
//   zero; the left halo of column 0 wraps into the previous row's zero tail.
//   Field pointers passed to kernels point at row 0, column 0 of shot 0;
//   shot b lives at +b*plane.
//
// Recursion (algebraically identical to the reference; SURVEY s7 hard part 4):
//   forward  a_n  = inv_m (L u_n [+ g_n s]) [+ amp_n w_k inv_m at source taps]
//            inc_{n+1} = d (inc_n + dt^2 a_n),  u_{n+1} = d u_n + inc_{n+1}
//     (reference: u_{n+1} = d (2 u_n - p_n + dt^2 a_n), p_{n+1} = d u_n, with
//      inc_n = u_n - p_n).
//   adjoint  v_n  = dt^2 inv_m d lam_{n+1}
//            w_n  = d w_{n+1} + L v_n + R^T y_n,  lam_n = d lam_{n+1} + w_n
//     (reference seisopt/wavesim.py:331-341 with w_n = lam_n - d lam_{n+1}),
//            image -= a_n v_n  (seisopt/wavesim.py:342-343).
//   L is applied in difference form sum_k c_k ((u_{+k}-u) + (u_{-k}-u)), which
//   equals the reference stencil because c_0 = -2 sum_{k>0} c_k.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sg {

constexpr int kGuard = 4;       // zero guard rows above/below each plane
constexpr int kTileRowsMax = 64;  // tail padding covers tiles up to this height

template <typename T>
struct FwdArgs {
  const T* u;        // u_n     (field base, shot 0 row 0 col 0)
  T* u_next;         // u_{n+1}
  T* inc;            // increment state, updated in place
  const T* inv_m;    // 1/m on the padded grid (single plane)
  const T* pz;       // sponge profile rows (index i)
  const T* px;       // sponge profile cols (index j)
  int64_t plane;     // per-shot stride of field buffers (elements)
  int nzp, nxp, ldx, tiles_x, ntiles;
  T dt2;
  T cz[5], cx[5];    // stencil weights, index k = 1..R used
  // point source: 4 taps per shot (flat offsets i*ldx+j), weights * src_scale
  const int* src_ij; // nullptr -> no point source
  const T* src_w;
  T amp;             // wavelet[n]
  // Born grid source: a0_n (per shot stride gsrc_stride) times gscale (plane)
  const T* gsrc;
  int64_t gsrc_stride;
  const T* gscale;
  // acceleration history store for this step (per shot stride hist_stride)
  T* hist;
  int64_t hist_stride;
  // receiver sampling (gathers for this step: gather + b*gather_stride + r)
  const int* rec_ij;  // (4, nrec)
  const T* rec_w;     // (4, nrec)
  int nrec;
  T* gather;
  int64_t gather_stride;
};

template <typename T>
struct AdjArgs {
  const T* lam;       // lam_{n+1} (adjoint field)
  T* lam_next;        // lam_n
  T* w;               // increment state, in place
  const T* inv_m;
  const T* pz;
  const T* px;
  int64_t plane;
  int nzp, nxp, ldx, tiles_x, ntiles;
  T dt2;
  T cz[5], cx[5];
  // receiver injection (CSR over cells of rows [inj_row0, inj_row0+inj_nrows))
  int inj_row0, inj_nrows;
  const int* inj_ptr;  // (inj_nrows*nxp + 1)
  const int* inj_rec;  // receiver index per entry
  const T* inj_w;      // weight per entry
  const T* ybar;       // adjoint data at this step: ybar + b*ybar_stride + r
  int64_t ybar_stride;
  // imaging: image[b] -= hist[b] * v   (hist per shot stride hist_stride)
  const T* hist;
  int64_t hist_stride;
  T* image;
  int64_t image_stride;
  // optional v-history store (adjoint_solve keep_v)
  T* vhist;
  int64_t vhist_stride;
};

// ----------------------------------------------------------------------------
// forward step
// ----------------------------------------------------------------------------
template <typename T, int R, int BX, int BY, int NY>
__global__ void __launch_bounds__(BX* BY)
    k_forward_step(const FwdArgs<T> a) {
  constexpr int TH = BY * NY;
  constexpr int SW = BX + 2 * R;
  constexpr int SH = TH + 2 * R;
  __shared__ T s[SH][SW];

  const int b = blockIdx.y;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const T* __restrict__ u = a.u + (int64_t)b * a.plane;

  if ((int)blockIdx.x >= a.ntiles) {
    // receiver sampling blocks: gather[n, r] = sum_k w_k u_n[tap_k]
    // (seisopt/wavesim.py:225-226, sampled before the update, :287)
    const int r = ((int)blockIdx.x - a.ntiles) * (BX * BY) + tid;
    if (a.gather != nullptr && r < a.nrec) {
      T g = a.rec_w[r] * u[a.rec_ij[r]];
#pragma unroll
      for (int k = 1; k < 4; ++k) g += a.rec_w[k * a.nrec + r] * u[a.rec_ij[k * a.nrec + r]];
      a.gather[(int64_t)b * a.gather_stride + r] = g;
    }
    return;
  }

  const int tzi = blockIdx.x / a.tiles_x;
  const int txi = blockIdx.x - tzi * a.tiles_x;
  const int i0 = tzi * TH;
  const int j0 = txi * BX;

  // stage u_n tile + halo (guard layout: no bounds checks)
  const T* __restrict__ src = u + (int64_t)(i0 - R) * a.ldx + (j0 - R);
#pragma unroll 4
  for (int idx = tid; idx < SH * SW; idx += BX * BY) {
    const int r = idx / SW;
    const int c = idx - r * SW;
    s[r][c] = __ldg(src + (int64_t)r * a.ldx + c);
  }
  __syncthreads();

  const int j = j0 + threadIdx.x;
  if (j >= a.nxp) return;
  const int jj = threadIdx.x + R;
  const T pxj = a.px[j];
  int sij[4];
  T sw[4];
  const bool has_src = a.src_ij != nullptr;
  if (has_src) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sij[k] = a.src_ij[b * 4 + k];
      sw[k] = a.src_w[b * 4 + k];
    }
  }
#pragma unroll
  for (int q = 0; q < NY; ++q) {
    const int ii = threadIdx.y + q * BY + R;
    const int i = i0 + ii - R;
    if (i >= a.nzp) break;
    const T uc = s[ii][jj];
    T lz = T(0), lx = T(0);
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      lz += a.cz[k] * ((s[ii - k][jj] - uc) + (s[ii + k][jj] - uc));
      lx += a.cx[k] * ((s[ii][jj - k] - uc) + (s[ii][jj + k] - uc));
    }
    T lap = lz + lx;
    const int o = i * a.ldx + j;
    const T im = a.inv_m[o];
    if (a.gsrc != nullptr) lap += a.gsrc[(int64_t)b * a.gsrc_stride + o] * a.gscale[o];
    T acc = lap * im;
    if (has_src) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (o == sij[k]) acc += a.amp * sw[k] * im;
    }
    if (a.hist != nullptr) a.hist[(int64_t)b * a.hist_stride + o] = acc;
    const T d = a.pz[i] * pxj;
    const int64_t fo = (int64_t)b * a.plane + o;
    const T inc = d * (a.inc[fo] + a.dt2 * acc);
    a.inc[fo] = inc;
    a.u_next[fo] = d * uc + inc;
  }
}

// ----------------------------------------------------------------------------
// adjoint step with fused receiver injection and imaging condition
// ----------------------------------------------------------------------------
template <typename T, int R, int BX, int BY, int NY>
__global__ void __launch_bounds__(BX* BY)
    k_adjoint_step(const AdjArgs<T> a) {
  constexpr int TH = BY * NY;
  constexpr int SW = BX + 2 * R;
  constexpr int SH = TH + 2 * R;
  __shared__ T s[SH][SW];  // v_n = dt^2 inv_m d lam_{n+1} on tile + halo

  const int b = blockIdx.y;
  const int tid = threadIdx.y * BX + threadIdx.x;
  const int tzi = blockIdx.x / a.tiles_x;
  const int txi = blockIdx.x - tzi * a.tiles_x;
  const int i0 = tzi * TH;
  const int j0 = txi * BX;
  const T* __restrict__ lam = a.lam + (int64_t)b * a.plane;

#pragma unroll 4
  for (int idx = tid; idx < SH * SW; idx += BX * BY) {
    const int r = idx / SW;
    const int c = idx - r * SW;
    const int i = i0 - R + r;
    const int j = j0 - R + c;
    const int o = i * a.ldx + j;
    const T d = a.pz[i] * a.px[j];
    s[r][c] = ((d * __ldg(lam + o)) * __ldg(a.inv_m + o)) * a.dt2;
  }
  __syncthreads();

  const int j = j0 + threadIdx.x;
  if (j >= a.nxp) return;
  const int jj = threadIdx.x + R;
  const T pxj = a.px[j];
#pragma unroll
  for (int q = 0; q < NY; ++q) {
    const int ii = threadIdx.y + q * BY + R;
    const int i = i0 + ii - R;
    if (i >= a.nzp) break;
    const T vc = s[ii][jj];
    T lz = T(0), lx = T(0);
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      lz += a.cz[k] * ((s[ii - k][jj] - vc) + (s[ii + k][jj] - vc));
      lx += a.cx[k] * ((s[ii][jj - k] - vc) + (s[ii][jj + k] - vc));
    }
    T lv = lz + lx;
    const int o = i * a.ldx + j;
    const int rr = i - a.inj_row0;
    if (a.ybar != nullptr && rr >= 0 && rr < a.inj_nrows) {
      // R^T y: duplicate taps accumulate (np.add.at, seisopt/wavesim.py:229)
      const int cell = rr * a.nxp + j;
      const int p1 = a.inj_ptr[cell + 1];
      for (int p = a.inj_ptr[cell]; p < p1; ++p)
        lv += a.inj_w[p] * a.ybar[(int64_t)b * a.ybar_stride + a.inj_rec[p]];
    }
    const T d = a.pz[i] * pxj;
    const int64_t fo = (int64_t)b * a.plane + o;
    const T wn = d * a.w[fo] + lv;
    a.w[fo] = wn;
    a.lam_next[fo] = d * lam[o] + wn;
    if (a.image != nullptr)
      a.image[(int64_t)b * a.image_stride + o] -= a.hist[(int64_t)b * a.hist_stride + o] * vc;
    if (a.vhist != nullptr) a.vhist[(int64_t)b * a.vhist_stride + o] = vc;
  }
}

}  // namespace sg
