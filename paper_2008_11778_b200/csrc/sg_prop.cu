// sg_prop.cu -- propagator context, sweep orchestration and the C ABI for
// forward modelling, FWI gradients and Born/LSRTM (include/seisgpu.h).
//
// Reference behaviour reproduced here:
//   Workspace                 seisopt/wavesim.py:183-214   -> sg_handle + sg_set_*
//   _forward_sweep            seisopt/wavesim.py:259-304   -> k_forward_step x nt
//   _adjoint_sweep            seisopt/wavesim.py:307-346   -> k_adjoint_step x nt
//   fwi_synthetic / misfit    seisopt/gradients.py:98-115, :70-79
//   fwi_gradient              seisopt/gradients.py:118-155
//   BornKernel / lsrtm        seisopt/gradients.py:158-277
//   fold_pad                  seisopt/wavesim.py:135-147   -> k_fold
// Shots of one call are processed in batches (grid.y = shot), each batch's
// nt-step loops captured once into CUDA graphs and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "seisgpu.h"
#include "sg_common.cuh"
#include "sg_kernels.cuh"
// The two-step (k_step2) and cluster-resident (k_resident) kernels were
// measured slower than k_step on B200.  Their types stay
// visible, but the kernels are only instantiated with -DSG_EXPERIMENTAL=1
// (tools/ builds); the product library ships the kernels that won their A/B.
#ifndef SG_EXPERIMENTAL
#define SG_EXPERIMENTAL 0
#endif
#include "sg_kernels2.cuh"
#include "sg_resident.cuh"

namespace sg {
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

// ---- red-zone allocator (SG_REDZONE=1; see sg_common.cuh) -------------------
constexpr size_t kRedZone = 64 << 10;
struct RzRec {
  void* base;
  size_t bytes;
};
static std::mutex g_rz_mu;
static std::map<void*, RzRec> g_rz_live;       // user pointer -> allocation
static std::atomic<int64_t> g_rz_bad{0};       // corrupted guard bytes found at free time
static std::atomic<int64_t> g_rz_allocs{0};    // guarded allocations made so far

static bool rz_on() {
  static const bool on = [] {
    const char* e = getenv("SG_REDZONE");
    return e && atoi(e) != 0;
  }();
  return on;
}

// guard bytes of one allocation that no longer hold 0xFF
static int64_t rz_scan(const RzRec& r) {
  std::vector<unsigned char> hbuf(2 * kRedZone);
  cudaDeviceSynchronize();
  if (cudaMemcpy(hbuf.data(), r.base, kRedZone, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(hbuf.data() + kRedZone, (char*)r.base + kRedZone + r.bytes, kRedZone,
                 cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  int64_t bad = 0;
  for (unsigned char c : hbuf) bad += c != 0xFF;
  return bad;
}

cudaError_t rz_malloc(void** p, size_t bytes) {
  if (!rz_on()) return cudaMalloc(p, bytes);
  const size_t padded = (bytes + 255) / 256 * 256;  // keeps the tail zone aligned
  void* base = nullptr;
  cudaError_t e = cudaMalloc(&base, padded + 2 * kRedZone);
  if (e != cudaSuccess) return e;
  e = cudaMemset(base, 0xFF, padded + 2 * kRedZone);
  if (e != cudaSuccess) {
    cudaFree(base);
    return e;
  }
  *p = (char*)base + kRedZone;
  std::lock_guard<std::mutex> lk(g_rz_mu);
  g_rz_live[*p] = RzRec{base, padded};
  g_rz_allocs.fetch_add(1);
  return cudaSuccess;
}

void rz_free(void* p) {
  if (!p) return;
  if (rz_on()) {
    std::lock_guard<std::mutex> lk(g_rz_mu);
    auto it = g_rz_live.find(p);
    if (it != g_rz_live.end()) {
      g_rz_bad.fetch_add(rz_scan(it->second));
      cudaFree(it->second.base);
      g_rz_live.erase(it);
      return;
    }
  }
  cudaFree(p);
}
}  // namespace sg

using namespace sg;

namespace {

constexpr int BX = kBX, TH = kTH;  // one-step kernel tiles (64 x kTH), 256 threads
constexpr int TH2 = kTH2;          // two-step kernel tile height
constexpr int RB = kThreads;        // threads per block
constexpr int kSlack = 256;         // column slack for profile arrays

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------

// scale/m on the padded grid with edge replication (seisopt/wavesim.py:126-128,200-201;
// scale = 1, or the stencil's z scale K for the fp32 SG_GC forward)
template <typename T, typename M>
__global__ void k_set_inv_m(const M* __restrict__ m, T* __restrict__ inv_m, int nz, int nx,
                            int nzp, int nxp, int ldx, int top, int left, double scale) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= nxp || i >= nzp) return;
  const int si = min(max(i - top, 0), nz - 1);
  const int sj = min(max(j - left, 0), nx - 1);
  inv_m[i * ldx + j] = (T)(scale / (double)m[(int64_t)si * nx + sj]);
}

// edge-replicated, scaled copy onto the padded grid (Born scale -m_r_pad,
// seisopt/gradients.py:193-194)
template <typename T, typename M>
__global__ void k_extend(const M* __restrict__ m, T* __restrict__ out, int nz, int nx, int nzp,
                         int nxp, int ldx, int top, int left, double scale) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= nxp || i >= nzp) return;
  const int si = min(max(i - top, 0), nz - 1);
  const int sj = min(max(j - left, 0), nx - 1);
  out[i * ldx + j] = (T)(scale * (double)m[(int64_t)si * nx + sj]);
}

// min(m) and count of (non-finite or <= 0) entries, partials per block
template <typename M>
__global__ void k_model_stats(const M* __restrict__ m, int64_t n, double* __restrict__ part) {
  double mn = INFINITY, bad = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)m[k];
    if (!isfinite(v) || v <= 0.0) bad += 1.0;
    mn = fmin(mn, v);
  }
  __shared__ double smin[1024];
  smin[threadIdx.x] = mn;
  const double b = block_sum(bad);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = smin[0];
    part[2 * blockIdx.x + 1] = b;
  }
}

// residual, weighted adjoint source and misfit partials
//   mode 0 (FWI):  ybar = (w_t dt)(f - g), acc w_t (f-g)^2   (seisopt/gradients.py:137-147)
//   mode 1 (LSRTM): ybar = f - g,          acc (f-g)^2       (seisopt/gradients.py:269-273)
//   mode 2 (value): no ybar,               acc w_t (f-g)^2   (seisopt/gradients.py:70-79)
//   mode 3 (LSRTM value): no ybar,         acc (f-g)^2       (seisopt/gradients.py:363-369)
template <typename T>
__global__ void k_residual(const T* __restrict__ f, const T* __restrict__ g, T* ybar,
                           int64_t rows, int nt, int nrec, double dt, int mode,
                           double* __restrict__ part) {
  // rows = shots * nt time samples; each block walks a contiguous run of rows
  double acc = 0.0;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per;
  const int64_t r1 = min(rows, r0 + per);
  for (int64_t row = r0; row < r1; ++row) {
    const int n = (int)(row % nt);
    const double w = (mode == 1 || mode == 3) ? 1.0 : ((n == 0 || n == nt - 1) ? 0.5 : 1.0);
    const T wdt = (T)(w * dt);
    const int64_t base = row * nrec;
    double racc = 0.0;
    for (int r = threadIdx.x; r < nrec; r += blockDim.x) {
      const T res = f[base + r] - g[base + r];
      racc += (double)res * (double)res;
      if (mode == 0) ybar[base + r] = wdt * res;
      else if (mode == 1) ybar[base + r] = res;
    }
    acc += w * racc;
  }
  const double s = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// R^T y for every step on the receiver row band:
//   dense[b][n][rr][j] = sum_{p in CSR(rr, j)} w_p ybar[b][n][rec_p]
// in np.add.at order (seisopt/wavesim.py:228-229).  Turns the adjoint step's
// dependent CSR walk into one coalesced load per band cell.
template <typename T>
__global__ void k_inj_dense(const T* __restrict__ ybar, T* __restrict__ dense, int64_t rows,
                            int nrec, int ncell, const int* __restrict__ ptr,
                            const int* __restrict__ rec, const T* __restrict__ w) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  const int p0 = ptr[c], p1 = ptr[c + 1];
  for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
    T acc = T(0);
    const T* y = ybar + row * nrec;
    for (int p = p0; p < p1; ++p) acc += w[p] * y[rec[p]];
    dense[row * ncell + c] = acc;
  }
}

// out[0] += scale * sum(part[0..n))  -- fixed order, one block
__global__ void k_finish_sum(const double* __restrict__ part, int n, double scale,
                             double* out) {
  double acc = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) acc += part[k];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) out[0] += scale * s;
}

// acc[o] += sum_b img[b][o] over valid padded cells (shot-order sum)
template <typename T>
__global__ void k_reduce_images(const T* __restrict__ img, T* __restrict__ acc, int count,
                                int64_t stride, int nzp, int nxp, int ldx) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= nxp) return;
  const int o = i * ldx + j;
  T s = acc[o];
  for (int b = 0; b < count; ++b) s += img[(int64_t)b * stride + o];
  acc[o] = s;
}

// fold_pad: transpose of edge replication (seisopt/wavesim.py:135-147)
template <typename T>
__global__ void k_fold(const T* __restrict__ pad, T* __restrict__ out, int nz, int nx,
                       int nzp, int nxp, int ldx, int top, int left, int accumulate,
                       double* __restrict__ nonfinite) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iz = blockIdx.y;
  if (ix >= nx) return;
  const int r0 = (iz == 0) ? 0 : top + iz;
  const int r1 = (iz == nz - 1) ? nzp - 1 : top + iz;
  const int c0 = (ix == 0) ? 0 : left + ix;
  const int c1 = (ix == nx - 1) ? nxp - 1 : left + ix;
  T s = T(0);
  for (int c = c0; c <= c1; ++c) {
    T col = T(0);
    for (int r = r0; r <= r1; ++r) col += pad[r * ldx + c];
    s += col;
  }
  const int64_t o = (int64_t)iz * nx + ix;
  out[o] = accumulate ? out[o] + s : s;
  // NaN/Inf guard of the result (a diverged sweep): counted, reported by
  // sg_last_nonfinite
  if (!isfinite((double)s)) atomicAdd(nonfinite, 1.0);
}

// compact (rows x nxp) <- pitched (rows x ldx)
template <typename T>
__global__ void k_unpitch(const T* __restrict__ src, T* __restrict__ dst, int64_t rows,
                          int nxp, int ldx) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nxp) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) dst[r * nxp + j] = src[r * ldx + j];
}

// pitched <- compact with dtype conversion (gathers/data in and out)
template <typename T>
__global__ void k_copy(const T* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[k];
}

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------

struct GraphEntry {
  cudaGraphExec_t exec;
  int64_t kernels;
};

struct sg_handle {
  sg_desc d{};
  int esz = 8;
  int nzp = 0, nxp = 0, ldx = 0;
  int64_t plane = 0;   // guarded plane (elements)
  int64_t origin = 0;  // offset of row 0 inside a guarded plane
  int64_t hplane = 0;  // compact-row history plane nzp*ldx
  int64_t tail = 0;    // slack after the last plane of a batch buffer
  int tiles_x = 0, ntiles = 0, rec_blocks = 0;
  int ntiles2 = 0;  // tiles of the two-step kernel (64 x kTH2)
  double cz[5] = {0}, cx[5] = {0};
  // SG_GC (fp32): the z scale K = c_1/dz^2 folded into the model plane
  // (K/m), the source weights and the Born scale (/K); 1 otherwise
  double kfold = 1.0;
  // NaN/Inf entries of the last folded gradient / image (sg_last_nonfinite)
  double nonfinite = 0.0;
  bool nonfinite_pending = false;
  cudaStream_t stream = 0;
  cudaStream_t cap = nullptr;
  static constexpr int kMaxChains = 4;
  cudaStream_t chain[kMaxChains] = {};  // extra streams of concurrent shot chains (1..)
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxChains] = {};

  // static device data
  void* inv_m_buf = nullptr;  // plane + tail
  void* pz_buf = nullptr;
  void* px_buf = nullptr;
  void* ez_buf = nullptr;  // 1 - pz, 1 - px rounded from fp64 (SG_GC forward)
  void* ex_buf = nullptr;
  void* gscale_buf = nullptr;  // -m_r on the padded grid (Born)
  int* src_rc = nullptr;  // (n_shots, 4, 2) tap rows/cols
  void* src_w = nullptr;
  int* rec_ij = nullptr;
  void* rec_w = nullptr;
  int inj_row0 = 0, inj_nrows = 0;
  int* inj_ptr = nullptr;
  int* inj_rec = nullptr;
  void* inj_w = nullptr;
  std::vector<double> wavelet;
  bool have_model = false, have_geom = false, have_wavelet = false, have_sponge = false;
  double src_scale = 1.0;

  // batch buffers
  int B = 0;              // capacity (shots)
  int recon = SG_RECON_FULL;
  int K = 0, ncp = 0;     // checkpoint interval / count
  int64_t hist_steps = 0; // steps of history held per shot
  int G = 0;              // set once batch buffers exist; see group_for()
  int nsm = 148;          // SMs of the device
  bool pdl = true;        // programmatic dependent launch between step kernels
  int* bsrc_rc = nullptr;
  void* bsrc_w = nullptr;
  std::map<std::string, CUtensorMap> tmaps;  // TMA descriptors by buffer/kind
  void *u0 = nullptr, *u1 = nullptr, *inc = nullptr, *inc2 = nullptr;  // fields, states
  void *l0 = nullptr, *l1 = nullptr, *w = nullptr, *w2 = nullptr;
  // receivers grouped by the tile holding their first tap (two-step kernel)
  int* tile_rec_ptr = nullptr;
  int* tile_rec = nullptr;
  int* rec_rc = nullptr;
  void* gath = nullptr;
  void* inj_dense = nullptr;  // (B, nt, inj_nrows, nxp) when the band is narrow
  void* hist = nullptr;
  void* ckpt = nullptr;
  void* band = nullptr;   // BOUNDARY: (B, nt, nb) u on the sponge frame
  BandGeo bgeo{};         // frame of the band store (set with the sponge)
  void* img = nullptr;
  void* acc_img = nullptr;
  double* part = nullptr;   // reduction partials
  double* scal = nullptr;   // [0] misfit accumulator, [1..] scratch
  int npart = 0;
  double held_bytes = 0.0;

  // Born cache of background histories
  void* born_hist = nullptr;
  int born_b0 = -1, born_count = 0;

  std::map<std::string, GraphEntry> graphs;

  // phase events of the last sg_fwi_gradient call: 5 per batch (forward sweep
  // | residual + injection | adjoint sweep | image reduction), read lazily
  std::vector<cudaEvent_t> ph_ev;
  int ph_batches = 0;

  // cluster-resident whole-sweep kernels (sg_resident.cuh)
  std::vector<int> rec_rows_h, rec_cols_h;  // receiver taps (4, n_rec), host copy
  void* wav_dev = nullptr;                  // wavelet amplitudes in the device dtype
  int res_state = 0;                        // 0 = not planned, 1 = usable, -1 = unavailable
  int res_CL = 0, res_W = 0, res_Q = 0, res_runs = 0, res_SW = 0, res_SR = 0;
  int res_hrows = 0, res_hboxes = 0, res_threads = 0, res_clusters = 0;
  int* res_rec = nullptr;  // rec_off (4 n_rec) | rec_list (n_rec) | rec_start (CL + 1)
};

namespace {

// Guarded buffers are [lead row][shot 0 plane][shot 1 plane]...[tail]; the lead
// row keeps the (-R, -R) halo read of shot 0 inside the allocation.
template <typename T>
T* field(void* base, const sg_handle* h) {  // pointer to row 0 col 0 of shot 0
  return reinterpret_cast<T*>(base) + h->ldx + h->origin;
}

size_t span_bytes(const sg_handle* h, int cnt) {  // lead + cnt planes
  return ((size_t)h->ldx + (size_t)cnt * h->plane) * h->esz;
}

int dalloc(sg_handle* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = rz_malloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return fail(SG_ERR_OOM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " +
                                cudaGetErrorString(e));
  }
  SG_CK(cudaMemset(*p, 0, bytes));
  h->held_bytes += (double)bytes;
  return SG_OK;
}

void dfree(void** p) {
  if (*p) rz_free(*p);
  *p = nullptr;
}

void drop_graphs(sg_handle* h) {
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
  h->graphs.clear();
}

void free_batch(sg_handle* h) {
  drop_graphs(h);
  h->tmaps.clear();
  void** bufs[] = {(void**)&h->bsrc_rc, &h->bsrc_w, &h->u0, &h->u1, &h->inc, &h->inc2, &h->l0,
                   &h->l1, &h->w, &h->w2, &h->gath, &h->inj_dense, &h->hist, &h->ckpt, &h->band, &h->img, &h->acc_img,
                   (void**)&h->part, (void**)&h->scal};
  for (auto p : bufs) dfree(p);
  dfree((void**)&h->res_rec);
  h->res_state = 0;  // the resident plan is sized for the batch
  h->B = 0;
}

// receivers on at most this many padded rows get a dense per-step injection array
constexpr int kDenseInjRows = 16;
bool dense_injection(const sg_handle* h) { return h->inj_nrows <= kDenseInjRows; }

// bytes per shot for the batch buffers in a given reconstruction mode
double per_shot_bytes(const sg_handle* h, int recon, int K, int ncp) {
  const double e = h->esz;
  double b = 8.0 * h->plane + (double)h->d.nt * h->d.n_rec + 2.0 * h->hplane;
  if (dense_injection(h)) b += (double)h->d.nt * h->inj_nrows * h->nxp;
  if (recon == SG_RECON_FULL) b += (double)h->d.nt * h->hplane;
  else if (recon == SG_RECON_BOUNDARY) b += (double)h->hplane + (double)h->d.nt * h->bgeo.nb;
  else b += (double)K * h->hplane + 2.0 * ncp * h->plane;
  return b * e + 64.0;
}

int ensure_batch(sg_handle* h) {
  if (h->B > 0) return SG_OK;
  const int nt = h->d.nt;
  size_t free_b = 0, total_b = 0;
  SG_CK(cudaMemGetInfo(&free_b, &total_b));
  // default: half of the free memory, leaving room for the caller's tensors
  double budget = h->d.mem_budget_bytes > 0 ? h->d.mem_budget_bytes : 0.5 * (double)free_b;
  budget -= 4.0 * (h->plane + h->ldx + h->tail) * h->esz + (64 << 20);  // statics + slack
  int K = h->d.checkpoint_every > 0 ? h->d.checkpoint_every
                                    : std::max(1, (int)std::ceil(std::sqrt((double)nt)));
  if (h->d.checkpoint_every <= 0) K += K & 1;  // even: same launch pairing as FULL
  K = std::min(K, nt);
  const int ncp = (nt + K - 1) / K;
  const int want = h->d.batch > 0 ? std::min(h->d.batch, h->d.n_shots) : h->d.n_shots;
  int recon = h->d.recon;
  const double full_b = per_shot_bytes(h, SG_RECON_FULL, K, ncp);
  const double ck_b = per_shot_bytes(h, SG_RECON_CHECKPOINT, K, ncp);
  // AUTO: the whole history when the batch fits; else (fp32, large grids whose
  // steps are HBM-bound) boundary saving when it still batches >= 8 shots per
  // launch (C5: 90.0 s vs 94.6 s checkpointed); else checkpointing (least
  // memory; C4-sized grids: 583 ms vs 686 ms with boundary saving)
  if (recon == SG_RECON_AUTO) {
    const double bd_b = per_shot_bytes(h, SG_RECON_BOUNDARY, K, ncp);
    const bool big = (int64_t)h->nzp * h->nxp >= (1 << 20);
    if (full_b * want <= budget) recon = SG_RECON_FULL;
    else if (h->esz == 4 && big && bd_b * std::min(want, 8) <= budget) recon = SG_RECON_BOUNDARY;
    else recon = SG_RECON_CHECKPOINT;
  }
  const double per = recon == SG_RECON_FULL       ? full_b
                     : recon == SG_RECON_BOUNDARY ? per_shot_bytes(h, recon, K, ncp)
                                                  : ck_b;
  int B = (int)std::min<double>(want, std::floor(budget / per));
  if (B < 1)
    return fail(SG_ERR_OOM, "one shot needs " + std::to_string(per / 1e9) +
                                " GB of device memory; budget " + std::to_string(budget / 1e9));
  h->B = B;
  h->G = 1;  // group size is chosen per launch (group_for)
  h->recon = recon;
  h->K = K;
  h->ncp = ncp;
  // BOUNDARY keeps one history slot (the lock-step Born background hand-off)
  h->hist_steps = recon == SG_RECON_FULL ? nt : (recon == SG_RECON_BOUNDARY ? 1 : K);
  const size_t e = h->esz;
  const size_t fb = ((size_t)h->ldx + (size_t)B * h->plane + h->tail) * e;
  SG_TRY(dalloc(h, (void**)&h->bsrc_rc, (size_t)B * 8 * sizeof(int)));
  SG_TRY(dalloc(h, &h->bsrc_w, (size_t)B * 4 * e));
  SG_TRY(dalloc(h, &h->u0, fb));
  SG_TRY(dalloc(h, &h->u1, fb));
  SG_TRY(dalloc(h, &h->inc, fb));
  SG_TRY(dalloc(h, &h->inc2, fb));
  SG_TRY(dalloc(h, &h->l0, fb));
  SG_TRY(dalloc(h, &h->l1, fb));
  SG_TRY(dalloc(h, &h->w, fb));
  SG_TRY(dalloc(h, &h->w2, fb));
  SG_TRY(dalloc(h, &h->gath, (size_t)B * nt * h->d.n_rec * e));
  if (dense_injection(h))
    SG_TRY(dalloc(h, &h->inj_dense, (size_t)B * nt * h->inj_nrows * h->nxp * e));
  SG_TRY(dalloc(h, &h->hist, (size_t)B * h->hist_steps * h->hplane * e));
  if (recon == SG_RECON_CHECKPOINT)
    SG_TRY(dalloc(h, &h->ckpt, (size_t)ncp * 2 * span_bytes(h, B)));
  if (recon == SG_RECON_BOUNDARY)
    SG_TRY(dalloc(h, &h->band, (size_t)B * nt * h->bgeo.nb * e));
  SG_TRY(dalloc(h, &h->img, (size_t)2 * B * h->hplane * e));  // two launch-parity sets
  SG_TRY(dalloc(h, &h->acc_img, (size_t)h->hplane * e));
  h->npart = 1184;
  SG_TRY(dalloc(h, (void**)&h->part, (size_t)h->npart * 2 * sizeof(double)));
  SG_TRY(dalloc(h, (void**)&h->scal, 16 * sizeof(double)));
  return SG_OK;
}

// ---------------------------------------------------------------------------
// kernel argument builders + launchers
// ---------------------------------------------------------------------------

// Shots per CTA group for a launch over `count` shots.  Larger G amortises
// the per-cell model reads and the image read-modify-write (~12 B/G of the
// ~20 B per shot-cell); the persistent grid holds `slots` CTAs, so the
// busiest CTA processes ceil(items / slots) * G shots.  Minimise that
// critical path times the amortisation overhead.
// `amort`: per-CTA overhead in shot-equivalents (prologue, model loads, image
// read-modify-write).  0.6 for the one-field kernels; 1.5 for the fused
// reverse + adjoint kernel, whose step time per shot keeps falling with G on
// the HBM-bound C5 grid (14.5 / 13.9 / 13.5 / 13.3 / 13.1 us for G = 4..8,
// profiles/r02ag_c5_batch_group.log); its ties go to the larger group.
int group_for(const sg_handle* h, int count, int per_sm = 0, double amort = 0.6) {
  if (h->d.group > 0) return std::max(1, std::min({h->d.group, count, 8}));
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SG_GROUP");
    env = e ? std::max(0, std::min(8, atoi(e))) : 0;
  }
  if (env > 0) return std::max(1, std::min(env, count));
  const int slots = h->nsm * (per_sm > 0 ? per_sm : (h->esz == 4 ? 3 : 2));
  int best = 1;
  double best_cost = 1e300;
  for (int G = 1; G <= std::min(8, count); ++G) {
    const int64_t items = (int64_t)h->ntiles * ((count + G - 1) / G);
    const double rounds = (double)((items + slots - 1) / slots);
    const double cost = rounds * G * (1.0 + amort / G);
    if (amort > 1.0 ? cost <= best_cost + 1e-9 : cost < best_cost - 1e-9) {
      best_cost = cost;
      best = G;
    }
  }
  return best;
}


// TMA descriptors.  Guarded buffers (fields, state) are viewed as 3-D
// {ldx, nzp + 2 kGuard, B} starting after the lead row; histories as
// {ldx, nzp, planes}.  Out-of-bounds boxes read as zero and are clipped on store.
enum MapKind { MAP_HALO = 0, MAP_TILE = 1, MAP_HIST = 2, MAP_HALO2 = 3, MAP_RING = 4,
               MAP_HIST2 = 5 };

template <typename T, int R>
int get_map(sg_handle* h, void* base, int kind, int64_t planes, CUtensorMap* out) {
  char keyb[96];
  snprintf(keyb, sizeof keyb, "%p/%d/%lld/%d", base, kind, (long long)planes, R);
  const std::string key(keyb);
  auto it = h->tmaps.find(key);
  if (it != h->tmaps.end()) {
    *out = it->second;
    return SG_OK;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(SG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const bool hk = kind == MAP_HIST || kind == MAP_HIST2;
  const int rows = hk ? h->nzp : h->nzp + 2 * kGuard;
  const int64_t pl = hk ? h->hplane : h->plane;
  void* g = hk ? base : (void*)((char*)base + (size_t)h->ldx * sizeof(T));
  cuuint64_t dims[3] = {(cuuint64_t)h->ldx, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)h->ldx * sizeof(T), (cuuint64_t)pl * sizeof(T)};
  cuuint32_t bw = BX, bh = TH;
  if (kind == MAP_HALO) {
    bw = BX + 2 * kHalo;
    bh = TH + 2 * kHalo;
  } else if (kind == MAP_RING) {
    bw = kEW;
    bh = kEH;
  } else if (kind == MAP_HIST2) {
    bh = TH2;
  } else if (kind == MAP_HALO2) {
    bw = kUW;
    bh = kUH;
  }
  cuuint32_t box[3] = {bw, bh, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  CUresult r = enc(&m, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                   3, g, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SG_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  h->tmaps[key] = m;
  *out = m;
  return SG_OK;
}

template <typename T, int R>
int step_maps(sg_handle* h, StepArgs<T>& a, void* F0, void* F1, void* S0, void* S1, void* hist,
              int64_t hist_planes) {
  SG_TRY((get_map<T, R>(h, F0, MAP_HALO, h->B, &a.f_halo[0])));
  SG_TRY((get_map<T, R>(h, F1, MAP_HALO, h->B, &a.f_halo[1])));
  SG_TRY((get_map<T, R>(h, F0, MAP_TILE, h->B, &a.f_tile[0])));
  SG_TRY((get_map<T, R>(h, F1, MAP_TILE, h->B, &a.f_tile[1])));
  (void)S1;  // the one-step kernel updates its state in place
  SG_TRY((get_map<T, R>(h, S0, MAP_TILE, h->B, &a.s_tile)));
  if (hist) SG_TRY((get_map<T, R>(h, hist, MAP_HIST, hist_planes, &a.h_tile)));
  return SG_OK;
}

template <typename T>
int step_args(sg_handle* h, StepArgs<T>& a, void* F0, void* F1, void* S0, void* S1, void* hist,
              int64_t hist_planes) {
  std::memset(&a, 0, sizeof(a));
  if (h->d.order == 8) SG_TRY((step_maps<T, 4>(h, a, F0, F1, S0, S1, hist, hist_planes)));
  else SG_TRY((step_maps<T, 1>(h, a, F0, F1, S0, S1, hist, hist_planes)));
  a.f[0] = field<T>(F0, h);
  a.f[1] = field<T>(F1, h);
  a.state = field<T>(S0, h);
  a.inv_m = field<T>(h->inv_m_buf, h);
  a.pz = reinterpret_cast<const T*>(h->pz_buf) + kGuard;
  a.px = reinterpret_cast<const T*>(h->px_buf) + kGuard;
  a.plane = h->plane;
  a.nzp = h->nzp;
  a.nxp = h->nxp;
  a.ldx = h->ldx;
  a.tiles_x = h->tiles_x;
  a.ntiles = h->ntiles;
  a.G = h->G;
  a.dt2 = (T)(h->d.dt * h->d.dt);
  a.dt2l = (T)(h->d.dt * h->d.dt - (double)a.dt2);
  for (int k = 0; k < 5; ++k) {
    a.cz[k] = (T)h->cz[k];
    a.cx[k] = (T)h->cx[k];
  }
  // exact-constant forward (SG_GC): ratios to c_1 and the axis scales, hi + lo
  auto split = [](double v, T& hi, T& lo) {
    hi = (T)v;
    lo = (T)(v - (double)hi);
  };
  for (int k = 1; k < 5; ++k) split(h->cz[1] != 0.0 ? h->cz[k] / h->cz[1] : 0.0, a.rh[k], a.rl[k]);
  split(h->cx[1] / h->cz[1], a.rhoh, a.rhol);
  a.iso = (a.rhoh == (T)1 && a.rhol == (T)0 && h->cz[1] == h->cx[1]) ? 1 : 0;
  a.cdt2 = (T)(h->d.dt * h->d.dt / h->kfold);
  a.ez = reinterpret_cast<const T*>(h->ez_buf) + kGuard;
  a.ex = reinterpret_cast<const T*>(h->ex_buf) + kGuard;
  a.rec_ij = h->rec_ij;
  a.rec_w = reinterpret_cast<const T*>(h->rec_w);
  a.nrec = h->d.n_rec;
  a.rec_blocks = (h->G * h->d.n_rec + RB - 1) / RB;
  a.inj_row0 = h->inj_row0;
  a.inj_nrows = h->inj_nrows;
  a.inj_ptr = h->inj_ptr;
  a.inj_rec = h->inj_rec;
  a.inj_w = reinterpret_cast<const T*>(h->inj_w);
  a.bT = h->bgeo.bT;
  a.bB = h->bgeo.bB;
  a.bL = h->bgeo.bL;
  a.bR = h->bgeo.bR;
  a.nb = h->bgeo.nb;
  a.band_slot = -1;
  return SG_OK;
}

template <typename T, int R, bool ADJ, int FL>
int launch_step_f(const sg_handle* h, cudaStream_t s, const StepArgs<T>& a0) {
  // the shared-memory attribute is per device: one bit per ordinal
  static std::atomic<uint64_t> attr_devs{0};
  constexpr int smem = step_smem_bytes<T, R, ADJ, step_dual<ADJ, FL>()>();
  constexpr int per_sm = step_min_blocks<T, ADJ, FL>();
  const uint64_t bit = 1ull << (h->d.device & 63);
  if (!(attr_devs.load() & bit)) {
    SG_CK(cudaFuncSetAttribute(k_step<T, R, ADJ, FL>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_devs.fetch_or(bit);
  }
  StepArgs<T> a = a0;
  a.G = group_for(h, a.count, per_sm, (ADJ && step_dual<ADJ, FL>()) ? 1.5 : 0.6);
  // one-step fp32 adjoint: at most SG_ADJ_GMAX shots per CTA group (C3: 4
  // instead of the cost model's 5 -- adjoint step 14.1 -> 13.3 us,
  // profiles/r01e_ab_group2.log)
  if (sizeof(T) == 4 && ADJ && !step_dual<ADJ, FL>() && h->d.group <= 0)
    a.G = std::min(a.G, SG_ADJ_GMAX);
  a.rec_blocks = (a.G * h->d.n_rec + RB - 1) / RB;
  const int extra = (!ADJ && (FL & FL_GATHER)) ? a.rec_blocks : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(h->ntiles + extra, (a.count + a.G - 1) / a.G);
  cfg.blockDim = dim3(kTX, kTY);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  if (h->pdl) {
    cfg.attrs = attr_pdl;
    cfg.numAttrs = 1;
  }
  SG_CK(cudaLaunchKernelEx(&cfg, k_step<T, R, ADJ, FL>, a));
  count_launch();
  return SG_OK;
}

template <typename T, int R, bool ADJ>
int launch_step_r(const sg_handle* h, cudaStream_t s, const StepArgs<T>& a) {
  const int fl = (a.hist_on ? FL_HIST : 0) | (a.gsrc ? FL_GSRC : 0) |
                 (a.vhist ? FL_VHIST : 0) | (a.gather ? FL_GATHER : 0) | (a.band ? FL_BAND : 0);
  if constexpr (ADJ) {
    if (fl & FL_BAND) {
      if (a.adj3 && a.rev3) return launch_step_f<T, R, ADJ, FL_BAND | FL_ADJ3 | FL_REV3>(h, s, a);
      else if (a.adj3) return launch_step_f<T, R, ADJ, FL_BAND | FL_ADJ3>(h, s, a);
      else return launch_step_f<T, R, ADJ, FL_BAND>(h, s, a);
    } else if (a.adj3) {
      if (fl & FL_VHIST) return launch_step_f<T, R, ADJ, FL_VHIST | FL_ADJ3>(h, s, a);
      else if (fl & FL_HIST) return launch_step_f<T, R, ADJ, FL_HIST | FL_ADJ3>(h, s, a);
      else return launch_step_f<T, R, ADJ, FL_ADJ3>(h, s, a);
    }
    else if (fl & FL_VHIST) return launch_step_f<T, R, ADJ, FL_VHIST>(h, s, a);
    else if (fl & FL_HIST) return launch_step_f<T, R, ADJ, FL_HIST>(h, s, a);
    else return launch_step_f<T, R, ADJ, 0>(h, s, a);
  } else if (a.rstate != nullptr) {
    // fused lock-step Born pair (scattered gathers; background history optional)
    if (fl & FL_HIST) return launch_step_f<T, R, ADJ, FL_LOCK | FL_GATHER | FL_HIST>(h, s, a);
    else return launch_step_f<T, R, ADJ, FL_LOCK | FL_GATHER>(h, s, a);
  } else if (fl & FL_BAND) {
    // band-saving forwards: FWI gradient (gathers) and Born background (one-slot history)
    if (fl & FL_HIST) return launch_step_f<T, R, ADJ, FL_BAND | FL_HIST>(h, s, a);
    else if (fl & FL_GATHER) return launch_step_f<T, R, ADJ, FL_BAND | FL_GATHER>(h, s, a);
    else return launch_step_f<T, R, ADJ, FL_BAND>(h, s, a);
  } else {
  switch (fl & (FL_HIST | FL_GSRC | FL_GATHER)) {
    case 0: return launch_step_f<T, R, ADJ, 0>(h, s, a);
    case FL_HIST: return launch_step_f<T, R, ADJ, FL_HIST>(h, s, a);
    case FL_GATHER: return launch_step_f<T, R, ADJ, FL_GATHER>(h, s, a);
    case FL_HIST | FL_GATHER: return launch_step_f<T, R, ADJ, FL_HIST | FL_GATHER>(h, s, a);
    case FL_GSRC: return launch_step_f<T, R, ADJ, FL_GSRC>(h, s, a);
    case FL_GSRC | FL_GATHER: return launch_step_f<T, R, ADJ, FL_GSRC | FL_GATHER>(h, s, a);
    case FL_GSRC | FL_HIST: return launch_step_f<T, R, ADJ, FL_GSRC | FL_HIST>(h, s, a);
    default: return launch_step_f<T, R, ADJ, FL_GSRC | FL_HIST | FL_GATHER>(h, s, a);
  }
  }
}

template <typename T, bool ADJ>
int launch_step(const sg_handle* h, cudaStream_t s, const StepArgs<T>& a) {
  if (h->d.order == 8) return launch_step_r<T, 4, ADJ>(h, s, a);
  return launch_step_r<T, 1, ADJ>(h, s, a);
}

// ---- sweep pieces (enqueue only) --------------------------------------------

// A history buffer holds `steps` planes per shot for `shots` shots:
// plane index = b * steps + slot.
struct HistRef {
  void* base = nullptr;
  int steps = 0;
  int64_t shots = 0;
  int n0 = 0;           // step stored at slot 0
  bool rotate = false;  // slot = (n - n0) % steps
  int slot(int n) const { return rotate ? (n - n0) % steps : n - n0; }
};

HistRef main_hist(const sg_handle* h, int n0) {
  HistRef r;
  r.base = h->hist;
  r.steps = (int)h->hist_steps;
  r.shots = h->B;
  r.n0 = n0;
  return r;
}

struct FwdPlan {
  bool point = true;        // wavelet point source
  bool gathers = true;      // sample receivers into h->gath
  HistRef hist;             // acceleration store
  const void* gsrc = nullptr;  // Born source history (per shot gsrc_shot elements)
  int64_t gsrc_shot = 0;
  int gsrc_n0 = 0;
  bool ckpt_save = false;   // save (u_n, inc_n) at n % K == 0
  bool band_save = false;   // BOUNDARY: store u_n on the sponge frame every step
  void* fu0 = nullptr;      // field / state buffers (default u0/u1, inc/inc2)
  void* fu1 = nullptr;
  void* fs0 = nullptr;
  void* fs1 = nullptr;
};

// two-step (temporally blocked) kernels: fp32 only, no Born grid source, no
// v-history.  Opt-in (desc.step_mode == 2): measured slower than the one-step
// kernel on B200 at C3 and C5 (profiles/r01_step_kernels_by_config.txt).
bool two_step_ok(const sg_handle* h) {
  return SG_EXPERIMENTAL && h->esz == 4 && h->d.step_mode == 2;
}

template <typename T>
int step2_args(sg_handle* h, Step2Args<T>& a, void* F0, void* F1, void* S0, void* S1,
               void* hist, int64_t hist_planes) {
  std::memset(&a, 0, sizeof(a));
  SG_TRY((get_map<T, 4>(h, F0, MAP_HALO2, h->B, &a.f_halo2[0])));
  SG_TRY((get_map<T, 4>(h, F1, MAP_HALO2, h->B, &a.f_halo2[1])));
  SG_TRY((get_map<T, 4>(h, S0, MAP_RING, h->B, &a.s_ring[0])));
  SG_TRY((get_map<T, 4>(h, S1, MAP_RING, h->B, &a.s_ring[1])));
  SG_TRY((get_map<T, 4>(h, h->inv_m_buf, MAP_RING, 1, &a.m_ring[0])));
  if (hist) SG_TRY((get_map<T, 4>(h, hist, MAP_HIST2, hist_planes, &a.h_tile)));
  a.f[0] = field<T>(F0, h);
  a.f[1] = field<T>(F1, h);
  a.state[0] = field<T>(S0, h);
  a.state[1] = field<T>(S1, h);
  a.pz = reinterpret_cast<const T*>(h->pz_buf) + kGuard;
  a.px = reinterpret_cast<const T*>(h->px_buf) + kGuard;
  a.plane = h->plane;
  a.nzp = h->nzp;
  a.nxp = h->nxp;
  a.ldx = h->ldx;
  a.tiles_x = h->tiles_x;
  a.ntiles = h->ntiles2;
  a.dt2 = (T)(h->d.dt * h->d.dt);
  for (int k = 0; k < 5; ++k) {
    a.cz[k] = (T)h->cz[k];
    a.cx[k] = (T)h->cx[k];
  }
  a.hplane = h->hplane;
  a.tile_rec_ptr = h->tile_rec_ptr;
  a.tile_rec = h->tile_rec;
  a.rec_rc = h->rec_rc;
  a.rec_w = reinterpret_cast<const T*>(h->rec_w);
  a.nrec = h->d.n_rec;
  a.inj_row0 = h->inj_row0;
  a.inj_nrows = h->inj_nrows;
  a.inj_ptr = h->inj_ptr;
  a.inj_rec = h->inj_rec;
  a.inj_w = reinterpret_cast<const T*>(h->inj_w);
  return SG_OK;
}

// shots per group for the two-step kernel (2 CTAs/SM)
int group2_for(const sg_handle* h, int count) {
  if (h->d.group > 0) return std::max(1, std::min({h->d.group, count, 8}));
  const int slots = h->nsm * 2;
  int best = 1;
  double best_cost = 1e300;
  for (int G = 1; G <= std::min(8, count); ++G) {
    const int64_t items = (int64_t)h->ntiles2 * ((count + G - 1) / G);
    const double rounds = (double)((items + slots - 1) / slots);
    const double cost = rounds * G * (1.0 + 0.6 / G);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = G;
    }
  }
  return best;
}

template <int R, bool ADJ, bool HIST, bool GATHER>
void launch_step2_f(const sg_handle* h, cudaStream_t s, const Step2Args<float>& a) {
  static bool attr = false;
  constexpr int smem = step2_smem_bytes<ADJ>();
  if (!attr) {
    cudaFuncSetAttribute(k_step2<R, ADJ, HIST, GATHER>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(h->ntiles2, (a.count + a.G - 1) / a.G), block(kEW, kTY2);
  k_step2<R, ADJ, HIST, GATHER><<<grid, block, smem, s>>>(a);
  count_launch();
}

template <bool ADJ>
void launch_step2(const sg_handle* h, cudaStream_t s, const Step2Args<float>& a) {
  const bool hs = a.hist_on != 0;
  const bool ga = !ADJ && a.gather != nullptr;
#define L2(R)                                                           \
  do {                                                                  \
    if (hs && ga) launch_step2_f<R, ADJ, true, true>(h, s, a);          \
    else if (hs) launch_step2_f<R, ADJ, true, false>(h, s, a);          \
    else if (ga) launch_step2_f<R, ADJ, false, true>(h, s, a);          \
    else launch_step2_f<R, ADJ, false, false>(h, s, a);                 \
  } while (0)
  if (h->d.order == 8) L2(4);
  else L2(1);
#undef L2
}

template <typename T>
void launch_step2_t(const sg_handle* h, cudaStream_t s, const Step2Args<T>& a, bool adj) {
  if constexpr (sizeof(T) == 4 && SG_EXPERIMENTAL) {
    if (adj) launch_step2<true>(h, s, a);
    else launch_step2<false>(h, s, a);
  }
}

// Forward steps n0 .. n1-1.  `cur` selects the input buffers (F[cur], S[cur])
// and flips after every launch (one or two steps).
template <typename T>
int enq_forward(sg_handle* h, cudaStream_t s, int count, int n0, int n1, const FwdPlan& p,
                int* curp = nullptr, int s0 = 0) {
  void* U0 = p.fu0 ? p.fu0 : h->u0;
  void* U1 = p.fu1 ? p.fu1 : h->u1;
  const bool use2 = two_step_ok(h) && p.gsrc == nullptr && !p.band_save;
  void* S0 = p.fs0 ? p.fs0 : h->inc;
  // the one-step kernel reads and writes its own cells only: state in place
  void* S1 = use2 ? (p.fs1 ? p.fs1 : h->inc2) : S0;
  int cur_local = 0;
  int& cur = curp ? *curp : cur_local;
  StepArgs<T> a;
  SG_TRY(step_args<T>(h, a, U0, U1, S0, S1, p.hist.base, p.hist.shots * p.hist.steps));
  a.count = count;
  a.s0 = s0;
  if (p.point) {
    a.src_rc = h->bsrc_rc;
    a.src_w = reinterpret_cast<const T*>(h->bsrc_w);
  }
  if (p.gsrc) {
    a.gscale = field<T>(h->gscale_buf, h);
    a.gsrc_stride = p.gsrc_shot;
  }
  a.hist_on = p.hist.base != nullptr;
  a.hist_steps = p.hist.steps;
  a.hist = reinterpret_cast<T*>(p.hist.base);
  a.hplane = h->hplane;
  a.gather_stride = (int64_t)h->d.nt * h->d.n_rec;
  if (p.band_save) {
    a.band = reinterpret_cast<T*>(h->band);
    a.band_stride = (int64_t)h->d.nt * h->bgeo.nb;
  }
  Step2Args<T> a2;
  if (use2) {
    SG_TRY(step2_args<T>(h, a2, U0, U1, S0, S1, p.hist.base, p.hist.shots * p.hist.steps));
    a2.count = count;
    a2.G = group2_for(h, count);
    if (p.point) {
      a2.src_rc = h->bsrc_rc;
      a2.src_w = reinterpret_cast<const T*>(h->bsrc_w);
    }
    a2.hist_on = a.hist_on;
    a2.hist_steps = p.hist.steps;
    a2.hist = a.hist;
    a2.gather = p.gathers ? reinterpret_cast<T*>(h->gath) : nullptr;
    a2.gather_stride = a.gather_stride;
  }
  const size_t pb = span_bytes(h, count);
  const size_t sb = span_bytes(h, h->B);
  void* F[2] = {U0, U1};
  void* S[2] = {S0, S1};
  int n = n0;
  while (n < n1) {
    if (p.ckpt_save && n % h->K == 0) {
      // this launch's shots only (a chain owns planes s0 .. s0 + count - 1)
      const size_t off = s0 ? ((size_t)h->ldx + (size_t)s0 * h->plane) * h->esz : 0;
      const size_t len = s0 ? (size_t)count * h->plane * h->esz : pb;
      char* slot = (char*)h->ckpt + (size_t)(n / h->K) * 2 * sb;
      cudaMemcpyAsync(slot + off, (char*)F[cur] + off, len, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(slot + sb + off, (char*)S[cur] + off, len, cudaMemcpyDeviceToDevice, s);
    }
    const bool two = use2 && n + 1 < n1 && !(p.ckpt_save && (n + 1) % h->K == 0);
    if (two) {
      a2.cur = cur;
      a2.n0 = n;
      a2.amp0 = (T)h->wavelet[n];
      a2.amp1 = (T)h->wavelet[n + 1];
      if (a2.hist_on) {
        a2.slot0 = p.hist.slot(n);
        a2.slot1 = p.hist.slot(n + 1);
      }
      launch_step2_t<T>(h, s, a2, false);
      n += 2;
    } else {
      a.cur = cur;
      a.amp = (T)h->wavelet[n];
      if (a.hist_on) a.hist_slot = p.hist.slot(n);
      if (p.gsrc)
        a.gsrc = reinterpret_cast<const T*>(p.gsrc) + (int64_t)(n - p.gsrc_n0) * h->hplane;
      a.gather = p.gathers ? reinterpret_cast<T*>(h->gath) + (int64_t)n * h->d.n_rec : nullptr;
      a.band_slot = n;
      SG_TRY((launch_step<T, false>(h, s, a)));
      n += 1;
    }
    cur ^= 1;
  }
  return SG_OK;
}

struct AdjPlan {
  HistRef hist;                // imaging history (base nullptr: no imaging)
  bool inject = true;          // y from h->gath (scaled residual / data)
  void* vhist = nullptr;       // optional v store (nt planes, compact rows)
  bool band_recon = false;     // BOUNDARY: reverse-reconstruct u (u0/u1, inc) and image
  int rcur0 = 0;               // u_{n_hi-1} lives in {u0, u1}[rcur0]
};

// Adjoint steps n = n_hi-1 .. n_lo (descending); fields V in l0/l1, states w/w2;
// `cur` flips after every launch and continues across calls of one sweep.
template <typename T>
int enq_adjoint(sg_handle* h, cudaStream_t s, int count, int n_hi, int n_lo, const AdjPlan& p,
                int* curp = nullptr, int s0 = 0) {
  int cur_local = 0;
  int& cur = curp ? *curp : cur_local;
  const bool use2 = two_step_ok(h) && p.vhist == nullptr && !p.band_recon;
  void* W1 = use2 ? h->w2 : h->w;  // one-step kernel: state in place
  StepArgs<T> a;
  SG_TRY(step_args<T>(h, a, h->l0, h->l1, h->w, W1, p.hist.base, p.hist.shots * p.hist.steps));
  // one-step sweeps (also the boundary-saving fused reverse + adjoint step)
  // run the three-level adjoint: 12 instead of 16 B per cell-update, no w
  // buffer traffic; the opt-in two-step kernel keeps the V/w form
  a.adj3 = (SG_ADJ3 && !use2) ? 1 : 0;
  a.count = count;
  a.s0 = s0;
  a.g0 = s0;  // groups of the first s0 shots use at most s0 image planes
  a.ybar_stride = (int64_t)h->d.nt * h->d.n_rec;
  a.hist_on = p.hist.base != nullptr && !p.band_recon;
  a.hist_steps = p.hist.steps;
  const bool img_on = a.hist_on || p.band_recon;
  a.image = img_on ? reinterpret_cast<T*>(h->img) : nullptr;
  int rcur = p.rcur0;
  CUtensorMap utile[2];  // REV3: u_{n+1} tiles of u0 / u1
  if (p.band_recon) {
    constexpr int R8 = 4, R2 = 1;
    if (h->d.order == 8) {
      SG_TRY((get_map<T, R8>(h, h->u0, MAP_HALO, h->B, &a.r_halo[0])));
      SG_TRY((get_map<T, R8>(h, h->u1, MAP_HALO, h->B, &a.r_halo[1])));
      SG_TRY((get_map<T, R8>(h, h->inc, MAP_TILE, h->B, &a.r_stile)));
      SG_TRY((get_map<T, R8>(h, h->u0, MAP_TILE, h->B, &utile[0])));
      SG_TRY((get_map<T, R8>(h, h->u1, MAP_TILE, h->B, &utile[1])));
    } else {
      SG_TRY((get_map<T, R2>(h, h->u0, MAP_HALO, h->B, &a.r_halo[0])));
      SG_TRY((get_map<T, R2>(h, h->u1, MAP_HALO, h->B, &a.r_halo[1])));
      SG_TRY((get_map<T, R2>(h, h->inc, MAP_TILE, h->B, &a.r_stile)));
      SG_TRY((get_map<T, R2>(h, h->u0, MAP_TILE, h->B, &utile[0])));
      SG_TRY((get_map<T, R2>(h, h->u1, MAP_TILE, h->B, &utile[1])));
    }
    // three-level reversal (the sweep starts from u_{nt-1} in rf[rcur0] and
    // u_nt in rf[rcur0 ^ 1], k_band_init)
    a.rev3 = (a.adj3 && SG_REV3) ? 1 : 0;
    a.rf[0] = field<T>(h->u0, h);
    a.rf[1] = field<T>(h->u1, h);
    a.rstate = field<T>(h->inc, h);
    a.band = reinterpret_cast<T*>(h->band);
    a.band_stride = (int64_t)h->d.nt * h->bgeo.nb;
    a.src_rc = h->bsrc_rc;
    a.src_w = reinterpret_cast<const T*>(h->bsrc_w);
  }
  a.image_stride = h->hplane;
  a.vhist_stride = (int64_t)h->d.nt * h->hplane;
  Step2Args<T> a2;
  if (use2) {
    SG_TRY(step2_args<T>(h, a2, h->l0, h->l1, h->w, h->w2, p.hist.base,
                         p.hist.shots * p.hist.steps));
    a2.count = count;
    a2.G = group2_for(h, count);
    a2.ybar_stride = a.ybar_stride;
    a2.hist_on = a.hist_on;
    a2.hist_steps = p.hist.steps;
    a2.image = a.image;
    a2.image_stride = a.image_stride;
  }
  int n = n_hi - 1;
  while (n >= n_lo) {
    const T* yb = p.inject ? reinterpret_cast<const T*>(h->gath) + (int64_t)n * h->d.n_rec : nullptr;
    if (p.inject && h->inj_dense) {
      a.inj_dense = reinterpret_cast<const T*>(h->inj_dense) +
                    (int64_t)n * h->inj_nrows * h->nxp;
      a.inj_dense_stride = (int64_t)h->d.nt * h->inj_nrows * h->nxp;
    }
    if (use2 && n - 1 >= n_lo) {
      a2.cur = cur;
      a2.n0 = n;
      a2.ybar = yb;
      if (a2.hist_on) {
        a2.slot0 = p.hist.slot(n);
        a2.slot1 = p.hist.slot(n - 1);
      }
      launch_step2_t<T>(h, s, a2, true);
      n -= 2;
    } else {
      a.cur = cur;
      a.ybar = yb;
      // image accumulator set of this launch's parity (PDL-safe, see k_step)
      if (img_on) a.image = reinterpret_cast<T*>(h->img) + (int64_t)(SG_IMG_PARITY ? cur : 0) * h->B * h->hplane;
      if (p.band_recon) {
        a.rcur = rcur;
        if (a.rev3) a.r_stile = utile[rcur ^ 1];
        a.amp = (T)h->wavelet[n];
        a.band_slot = n - 1;  // u_{n-1} on the frame (none below step 0)
        rcur ^= 1;
      }
      if (a.hist_on) a.hist_slot = p.hist.slot(n);
      a.vhist = p.vhist ? reinterpret_cast<T*>(p.vhist) + (int64_t)n * h->hplane : nullptr;
      if (a.adj3) a.s_tile = a.f_tile[cur ^ 1];  // V_{n+1}, overwritten with V_{n-1}
      SG_TRY((launch_step<T, true>(h, s, a)));
      n -= 1;
    }
    cur ^= 1;
  }
  return SG_OK;
}

// Lock-step Born forward over steps n0 .. n1-1 in fused launches: the
// background (u0/u1, inc; point source; history `hist` if given; checkpoints
// in CHECKPOINT mode) and the scattered field (l0/l1, w; source a0_n *
// gscale; gathers) of shots [s0, s0 + count) advance together.
template <typename T>
int enq_lockstep(sg_handle* h, cudaStream_t s, int count, int n0, int n1, const HistRef& hist,
                 bool ckpt_save, int s0 = 0) {
  StepArgs<T> a;
  SG_TRY(step_args<T>(h, a, h->l0, h->l1, h->w, h->w, hist.base, hist.shots * hist.steps));
  if (h->d.order == 8) {
    SG_TRY((get_map<T, 4>(h, h->u0, MAP_HALO, h->B, &a.r_halo[0])));
    SG_TRY((get_map<T, 4>(h, h->u1, MAP_HALO, h->B, &a.r_halo[1])));
    SG_TRY((get_map<T, 4>(h, h->inc, MAP_TILE, h->B, &a.r_stile)));
  } else {
    SG_TRY((get_map<T, 1>(h, h->u0, MAP_HALO, h->B, &a.r_halo[0])));
    SG_TRY((get_map<T, 1>(h, h->u1, MAP_HALO, h->B, &a.r_halo[1])));
    SG_TRY((get_map<T, 1>(h, h->inc, MAP_TILE, h->B, &a.r_stile)));
  }
  a.count = count;
  a.s0 = s0;
  a.rf[0] = field<T>(h->u0, h);
  a.rf[1] = field<T>(h->u1, h);
  a.rstate = field<T>(h->inc, h);
  a.src_rc = h->bsrc_rc;
  a.src_w = reinterpret_cast<const T*>(h->bsrc_w);
  a.gscale = field<T>(h->gscale_buf, h);
  a.hist_on = hist.base != nullptr;
  a.hist_steps = hist.steps;
  a.hist = reinterpret_cast<T*>(hist.base);
  a.hplane = h->hplane;
  a.gather_stride = (int64_t)h->d.nt * h->d.n_rec;
  const size_t pb = span_bytes(h, count);
  const size_t sb = span_bytes(h, h->B);
  void* F[2] = {h->u0, h->u1};
  int cur = 0;
  for (int n = n0; n < n1; ++n) {
    if (ckpt_save && n % h->K == 0) {
      const size_t off = s0 ? ((size_t)h->ldx + (size_t)s0 * h->plane) * h->esz : 0;
      const size_t len = s0 ? (size_t)count * h->plane * h->esz : pb;
      char* slot = (char*)h->ckpt + (size_t)(n / h->K) * 2 * sb;
      cudaMemcpyAsync(slot + off, (char*)F[cur] + off, len, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(slot + sb + off, (char*)h->inc + off, len, cudaMemcpyDeviceToDevice, s);
    }
    a.cur = cur;   // scattered and background fields flip together
    a.rcur = cur;
    a.amp = (T)h->wavelet[n];
    if (a.hist_on) a.hist_slot = hist.slot(n);
    a.gather = reinterpret_cast<T*>(h->gath) + (int64_t)n * h->d.n_rec;
    SG_TRY((launch_step<T, false>(h, s, a)));
    cur ^= 1;
  }
  return SG_OK;
}

// ---- concurrent chains -------------------------------------------------------
// A batch's time loop runs as independent chains over disjoint shot ranges
// on separate streams (forked and joined inside the captured graph): every
// step of a chain waits only for its own previous step, so one chain's launch
// latency, pipeline fill and tail overlap the other chains' steady state.
int nchains(const sg_handle* h, int count) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SG_CHAINS");
    env = e ? std::max(1, std::min(sg_handle::kMaxChains, atoi(e))) : 0;
  }
  // auto: two chains (measured best on B200: C3 gradient 163 -> 123 ms; three
  // or four chains lose to the smaller per-launch batches)
  const int want = env > 0 ? env : (h->d.chains > 0 ? h->d.chains : 2);
  if (two_step_ok(h)) return 1;
  return std::max(1, std::min({want, count, sg_handle::kMaxChains}));
}

template <typename F>
int fork_chains(sg_handle* h, cudaStream_t s, int count, F&& body) {
  const int nc = nchains(h, count);
  if (nc == 1) return body(s, 0, count);
  if (!h->ev_fork) {
    SG_CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    for (int c = 1; c < sg_handle::kMaxChains; ++c) {
      SG_CK(cudaStreamCreateWithFlags(&h->chain[c], cudaStreamNonBlocking));
      SG_CK(cudaEventCreateWithFlags(&h->ev_join[c], cudaEventDisableTiming));
    }
  }
  SG_CK(cudaEventRecord(h->ev_fork, s));
  int s0 = 0;
  for (int c = 0; c < nc; ++c) {
    const int cnt = count / nc + (c < count % nc ? 1 : 0);
    cudaStream_t cs = c == 0 ? s : h->chain[c];
    if (c > 0) SG_CK(cudaStreamWaitEvent(cs, h->ev_fork, 0));
    SG_TRY(body(cs, s0, cnt));
    s0 += cnt;
  }
  for (int c = 1; c < nc; ++c) {
    SG_CK(cudaEventRecord(h->ev_join[c], h->chain[c]));
    SG_CK(cudaStreamWaitEvent(s, h->ev_join[c], 0));
  }
  return SG_OK;
}

// ---- graph capture / replay ---------------------------------------------------

template <typename F>
int run_graph(sg_handle* h, const std::string& key, F&& body) {
  if (!h->d.use_graphs) {
    SG_TRY(body(h->stream));
    SG_CK(cudaGetLastError());
    return SG_OK;
  }
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    if (!h->cap) SG_CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    const int64_t before = g_launches.load();
    SG_CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    const int brc = body(h->cap);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    if (brc != SG_OK) {
      if (g) cudaGraphDestroy(g);
      return brc;
    }
    if (e != cudaSuccess)
      return fail(SG_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    const int64_t nk = g_launches.load() - before;  // kernels per replay
    g_launches.fetch_sub(nk);
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess)
      return fail(SG_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    it = h->graphs.emplace(key, GraphEntry{ex, nk}).first;
  }
  SG_CK(cudaGraphLaunch(it->second.exec, h->stream));
  count_launch(it->second.kernels);
  return SG_OK;
}

// ---- model / geometry upload helpers --------------------------------------------

template <typename T>
int upload_cast(sg_handle* h, void** dst, const double* src, size_t n) {
  std::vector<T> tmp(n);
  for (size_t k = 0; k < n; ++k) tmp[k] = (T)src[k];
  SG_TRY(dalloc(h, dst, n * sizeof(T)));
  SG_CK(cudaMemcpy(*dst, tmp.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  return SG_OK;
}

int check_handle(sg_handle* h, bool need_model = true) {
  if (!h) return fail(SG_ERR_ARG, "null handle");
  if (!h->have_sponge || !h->have_geom || !h->have_wavelet)
    return fail(SG_ERR_STATE, "sponge, geometry and wavelet must be set first");
  if (need_model && !h->have_model) return fail(SG_ERR_STATE, "model not set");
  SG_CK(cudaSetDevice(h->d.device));
  return SG_OK;
}

int check_range(sg_handle* h, int shot0, int count) {
  if (shot0 < 0 || count < 1 || shot0 + count > h->d.n_shots)
    return fail(SG_ERR_ARG, "shot range [" + std::to_string(shot0) + ", " +
                                std::to_string(shot0 + count) + ") outside [0, " +
                                std::to_string(h->d.n_shots) + ")");
  return SG_OK;
}

// load batch-local source taps for shots [b0, b0+cnt)
int load_batch_sources(sg_handle* h, int b0, int cnt) {
  SG_CK(cudaMemcpyAsync(h->bsrc_rc, h->src_rc + (size_t)b0 * 8, (size_t)cnt * 8 * sizeof(int),
                        cudaMemcpyDeviceToDevice, h->stream));
  SG_CK(cudaMemcpyAsync(h->bsrc_w, (char*)h->src_w + (size_t)b0 * 4 * h->esz,
                        (size_t)cnt * 4 * h->esz, cudaMemcpyDeviceToDevice, h->stream));
  return SG_OK;
}

int zero_fields(sg_handle* h, bool fwd, bool adj, int cnt) {
  const size_t b = span_bytes(h, cnt);
  if (fwd) {
    SG_CK(cudaMemsetAsync(h->u0, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->u1, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->inc, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->inc2, 0, b, h->stream));
  }
  if (adj) {
    SG_CK(cudaMemsetAsync(h->l0, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->l1, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->w, 0, b, h->stream));
    SG_CK(cudaMemsetAsync(h->w2, 0, b, h->stream));
  }
  return SG_OK;
}

template <typename T>
int residual(sg_handle* h, int cnt, const T* obs, int mode) {
  const int64_t rows = (int64_t)cnt * h->d.nt;
  const int blocks = (int)std::min<int64_t>(h->npart, rows);
  k_residual<T><<<blocks, 256, 0, h->stream>>>(reinterpret_cast<const T*>(h->gath), obs,
                                               reinterpret_cast<T*>(h->gath), rows, h->d.nt,
                                               h->d.n_rec, h->d.dt, mode, h->part);
  const double scale = (mode == 1 || mode == 3) ? 0.5 : 0.5 * h->d.dt;
  k_finish_sum<<<1, 1024, 0, h->stream>>>(h->part, blocks, scale, h->scal);
  count_launch(2);
  SG_CK(cudaGetLastError());
  return SG_OK;
}

// expand the adjoint data now in h->gath into the dense band array
template <typename T>
int fill_injection(sg_handle* h, int cnt) {
  if (!h->inj_dense) return SG_OK;
  const int ncell = h->inj_nrows * h->nxp;
  const int64_t rows = (int64_t)cnt * h->d.nt;
  dim3 grid(cdiv(ncell, 128), (unsigned)std::min<int64_t>(rows, 8192));
  k_inj_dense<T><<<grid, 128, 0, h->stream>>>(
      reinterpret_cast<const T*>(h->gath), reinterpret_cast<T*>(h->inj_dense), rows,
      h->d.n_rec, ncell, h->inj_ptr, h->inj_rec, reinterpret_cast<const T*>(h->inj_w));
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

template <typename T>
int reduce_images(sg_handle* h, int cnt) {
  dim3 grid(cdiv(h->nxp, 128), h->nzp);
  k_reduce_images<T><<<grid, 128, 0, h->stream>>>(
      reinterpret_cast<const T*>(h->img), reinterpret_cast<T*>(h->acc_img), 2 * h->B, h->hplane,
      h->nzp, h->nxp, h->ldx);
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

template <typename T>
int fold_out(sg_handle* h, void* out, int accumulate) {
  dim3 grid(cdiv(h->d.nx, 128), h->d.nz);
  double* nf = h->scal + 8;  // non-finite entries of this output
  SG_CK(cudaMemsetAsync(nf, 0, sizeof(double), h->stream));
  k_fold<T><<<grid, 128, 0, h->stream>>>(reinterpret_cast<const T*>(h->acc_img),
                                         reinterpret_cast<T*>(out), h->d.nz, h->d.nx, h->nzp,
                                         h->nxp, h->ldx, h->d.pad_top, h->d.pad_left,
                                         accumulate, nf);
  count_launch();
  SG_CK(cudaGetLastError());
  SG_CK(cudaMemcpyAsync(&h->nonfinite, nf, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  h->nonfinite_pending = true;
  return SG_OK;
}

// ---- cluster-resident whole-sweep kernels (sg_resident.cuh) -------------------

bool res_enabled(const sg_handle* h) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SG_RESIDENT");
    env = e ? atoi(e) : 0;
  }
  // opt-in: measured slower than the one-step kernels on B200 at C1/C3
  // (cluster waves leave a third of the SMs idle, 1 CTA/SM)
  const int want = env != 0 ? env : h->d.resident;
  return SG_EXPERIMENTAL && h->esz == 4 && want > 0 && h->d.step_mode != 2;
}

template <typename T, int R>
int res_plan_r(sg_handle* h) {
  using K = decltype(&k_resident<T, R, true, true, false>);
  const K probe = k_resident<T, R, true, true, false>;
  int optin = 0;
  SG_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->d.device));
  const int nzp = h->nzp, nxp = h->nxp;
  const int runs = (nzp + kResNR - 1) / kResNR;
  const int hrows = std::min(nzp, 256), hboxes = (nzp + 255) / 256;
  double best = 1e300;
  int bCL = 0, bW = 0, bthreads = 0, bclusters = 0;
  for (int CL = 2; CL <= 16; ++CL) {
    const int W = (((nxp + CL - 1) / CL) + 3) / 4 * 4;
    if ((nxp + W - 1) / W != CL || W > 256 || W < 8) continue;
    const int Q = W / 4;
    const int threads = (Q * runs + 31) / 32 * 32;
    if (threads > kResMaxThreads) continue;
    const int SR = runs * kResNR + 2 * kResHW;
    const int smem = ResSmem<T>(true, SR, W, hrows, hboxes).bytes;
    if (smem > optin - 8192) continue;  // static shared memory (receiver staging) on top
    if (cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, probe, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nc < 1) continue;
    // waves of clusters x per-step work of one CTA (cells + a barrier's worth)
    const int shots = std::max(1, h->B);
    const double cost = (double)((shots + nc - 1) / nc) * ((double)W * nzp + 3000.0);
    if (cost < best) {
      best = cost;
      bCL = CL;
      bW = W;
      bthreads = threads;
      bclusters = nc;
    }
  }
  if (bCL == 0) {
    h->res_state = -1;
    return SG_OK;
  }
  h->res_CL = bCL;
  h->res_W = bW;
  h->res_Q = bW / 4;
  h->res_runs = runs;
  h->res_SW = bW;
  h->res_SR = runs * kResNR + 2 * kResHW;
  h->res_hrows = hrows;
  h->res_hboxes = hboxes;
  h->res_threads = bthreads;
  h->res_clusters = bclusters;
  // receivers by owner CTA (the column quad run holding the leftmost tap);
  // tap offsets into the owner's shared plane
  const int NRc = h->d.n_rec;
  std::vector<int> off(4 * NRc), owner(NRc), list, start(bCL + 1, 0);
  for (int r = 0; r < NRc; ++r) {
    int cmin = 1 << 30;
    for (int k = 0; k < 4; ++k) cmin = std::min(cmin, h->rec_cols_h[k * NRc + r]);
    owner[r] = cmin / bW;
    const int c0 = owner[r] * bW;
    for (int k = 0; k < 4; ++k) {
      const int rr = h->rec_rows_h[k * NRc + r], cc = h->rec_cols_h[k * NRc + r];
      if (cc - c0 < -kResHW || cc - c0 >= bW + kResHW) {
        h->res_state = -1;  // taps wider than the halo (not bilinear): one-step kernels
        return SG_OK;
      }
      // own plane offset, or -1 - (offset into the halo slot [left | right])
      const int hr4 = (rr + kResHW) * 4;
      if (cc < c0) off[k * NRc + r] = -1 - (hr4 + cc - (c0 - 4));
      else if (cc >= c0 + bW) off[k * NRc + r] = -1 - (h->res_SR * 4 + hr4 + cc - (c0 + bW));
      else off[k * NRc + r] = (rr + kResHW) * bW + (cc - c0);
    }
    start[owner[r] + 1]++;
  }
  for (int c = 0; c < bCL; ++c) start[c + 1] += start[c];
  list.resize(NRc);
  {
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int r = 0; r < NRc; ++r) list[fill[owner[r]]++] = r;
  }
  std::vector<int> all(off);
  all.insert(all.end(), list.begin(), list.end());
  all.insert(all.end(), start.begin(), start.end());
  dfree((void**)&h->res_rec);
  SG_TRY(dalloc(h, (void**)&h->res_rec, all.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->res_rec, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (!h->wav_dev) SG_TRY(upload_cast<T>(h, &h->wav_dev, h->wavelet.data(), h->wavelet.size()));
  h->res_state = 1;
  return SG_OK;
}

// whether this handle's sweeps run as resident launches (plans on first use)
template <typename T>
bool res_ready(sg_handle* h) {
  if constexpr (sizeof(T) != 4 || !SG_EXPERIMENTAL) {
    return false;
  } else {
    if (!res_enabled(h)) return false;
    if (h->res_state == 0) {
      const int rc = h->d.order == 8 ? res_plan_r<T, 4>(h) : res_plan_r<T, 1>(h);
      if (rc != SG_OK) {
        cudaGetLastError();
        h->res_state = -1;
      }
    }
    if (h->res_state > 0 && !h->wav_dev &&
        upload_cast<T>(h, &h->wav_dev, h->wavelet.data(), h->wavelet.size()) != SG_OK)
      h->res_state = -1;
    return h->res_state > 0;
  }
}

template <typename T>
void res_common(const sg_handle* h, ResArgs<T>& a, int cnt) {
  std::memset(&a, 0, sizeof(a));
  (void)cnt;
  a.inv_m = field<T>(h->inv_m_buf, h);
  a.pz = reinterpret_cast<const T*>(h->pz_buf) + kGuard;
  a.px = reinterpret_cast<const T*>(h->px_buf) + kGuard;
  a.nzp = h->nzp;
  a.nxp = h->nxp;
  a.ldx = h->ldx;
  a.W = h->res_W;
  a.CL = h->res_CL;
  a.Q = h->res_Q;
  a.runs = h->res_runs;
  a.SR = h->res_SR;
  a.hrows = h->res_hrows;
  a.hboxes = h->res_hboxes;
  a.n0 = 0;
  a.n1 = h->d.nt;
  a.dt2 = (T)(h->d.dt * h->d.dt);
  for (int k = 0; k < 5; ++k) {
    a.cz[k] = (T)h->cz[k];
    a.cx[k] = (T)h->cx[k];
  }
}

template <typename T, int R, bool ADJ, bool HIST, bool GATHER>
int launch_res_f(const sg_handle* h, cudaStream_t s, const ResArgs<T>& a, int cnt) {
  const auto kern = k_resident<T, R, ADJ, HIST, GATHER>;
  static int attr_smem = 0;
  const int smem = ResSmem<T>(ADJ, a.SR, a.W, a.hrows, a.hboxes).bytes;
  if (smem > attr_smem) {
    SG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cnt * a.CL);
  cfg.blockDim = dim3(h->res_threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SG_CK(cudaLaunchKernelEx(&cfg, kern, a));
  count_launch();
  return SG_OK;
}

// resident forward sweep over all nt steps for batch shots [s0, s0 + cnt):
// history `hr` (base nullptr: none), gathers into h->gath if `gathers`
template <typename T>
int enq_res_forward(sg_handle* h, cudaStream_t s, int cnt, const HistRef& hr, bool gathers,
                    int s0 = 0) {
  if constexpr (sizeof(T) != 4 || !SG_EXPERIMENTAL) {
    return fail(SG_ERR_STATE, "resident sweeps: fp32 and -DSG_EXPERIMENTAL=1 only");
  } else {
  ResArgs<T> a;
  res_common<T>(h, a, cnt);
  a.s0 = s0;
  a.src_rc = h->bsrc_rc;
  a.src_w = reinterpret_cast<const T*>(h->bsrc_w);
  a.wav = reinterpret_cast<const T*>(h->wav_dev);
  a.hist = reinterpret_cast<T*>(hr.base);
  a.hplane = h->hplane;
  a.hist_steps = hr.steps;
  a.hist_n0 = hr.n0;
  const int NRc = h->d.n_rec;
  a.rec_w = reinterpret_cast<const T*>(h->rec_w);
  a.rec_off = h->res_rec;
  a.rec_list = h->res_rec + 4 * NRc;
  a.rec_start = h->res_rec + 5 * NRc;
  a.nrec = NRc;
  a.gather = gathers ? reinterpret_cast<T*>(h->gath) : nullptr;
  a.gather_stride = (int64_t)h->d.nt * NRc;
  const bool hi = hr.base != nullptr;
#define RES_F(RR)                                                                         \
  do {                                                                                    \
    if (hi && gathers) return launch_res_f<T, RR, false, true, true>(h, s, a, cnt);       \
    if (hi) return launch_res_f<T, RR, false, true, false>(h, s, a, cnt);                 \
    if (gathers) return launch_res_f<T, RR, false, false, true>(h, s, a, cnt);            \
    return launch_res_f<T, RR, false, false, false>(h, s, a, cnt);                        \
  } while (0)
  if (h->d.order == 8) RES_F(4);
  RES_F(1);
#undef RES_F
  }
}

// resident adjoint sweep (steps nt-1 .. 0) imaging against history `hr`,
// R^T y from the dense band array; per-shot images into h->img planes [0, B)
template <typename T>
int enq_res_adjoint(sg_handle* h, cudaStream_t s, int cnt, const HistRef& hr, int s0 = 0) {
  if constexpr (sizeof(T) != 4 || !SG_EXPERIMENTAL) {
    return fail(SG_ERR_STATE, "resident sweeps: fp32 and -DSG_EXPERIMENTAL=1 only");
  } else {
  ResArgs<T> a;
  res_common<T>(h, a, cnt);
  a.s0 = s0;
  a.hist_steps = hr.steps;
  a.hist_n0 = hr.n0;
  {
    char keyb[96];
    snprintf(keyb, sizeof keyb, "res/%p/%lld/%d", hr.base, (long long)(hr.shots * hr.steps),
             h->res_W);
    auto it = h->tmaps.find(keyb);
    if (it == h->tmaps.end()) {
      EncodeTiledFn enc = encode_fn();
      if (!enc) return fail(SG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
      cuuint64_t dims[3] = {(cuuint64_t)h->ldx, (cuuint64_t)h->nzp,
                            (cuuint64_t)(hr.shots * hr.steps)};
      cuuint64_t strides[2] = {(cuuint64_t)h->ldx * sizeof(T), (cuuint64_t)h->hplane * sizeof(T)};
      cuuint32_t box[3] = {(cuuint32_t)h->res_W, (cuuint32_t)h->res_hrows, 1};
      cuuint32_t estr[3] = {1, 1, 1};
      CUtensorMap m;
      CUresult r = enc(&m, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                       3, hr.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(SG_ERR_CUDA, "cuTensorMapEncodeTiled (resident history) failed: " +
                                     std::to_string((int)r));
      it = h->tmaps.emplace(keyb, m).first;
    }
    a.h_map = it->second;
  }
  a.inj_dense = reinterpret_cast<const T*>(h->inj_dense);
  a.inj_stride = (int64_t)h->d.nt * h->inj_nrows * h->nxp;
  a.inj_row0 = h->inj_row0;
  a.inj_nrows = h->inj_nrows;
  a.image = reinterpret_cast<T*>(h->img);
  a.image_stride = h->hplane;
  if (h->d.order == 8) return launch_res_f<T, 4, true, true, false>(h, s, a, cnt);
  return launch_res_f<T, 1, true, true, false>(h, s, a, cnt);
  }
}

// ---------------------------------------------------------------------------
// sweep drivers (typed)
// ---------------------------------------------------------------------------

template <typename T>
int do_forward_batch(sg_handle* h, int b0, int cnt, bool store_full_hist_ckpt_mode) {
  // forward over all steps, gathers into h->gath; in gradient context also
  // stores the full history (FULL) or checkpoints (CHECKPOINT)
  SG_TRY(load_batch_sources(h, b0, cnt));
  SG_TRY(zero_fields(h, true, false, cnt));
  const int nt = h->d.nt;
  // cluster-resident sweep: one launch for the whole forward (gathers, and
  // the acceleration history in FULL gradient mode)
  if ((!store_full_hist_ckpt_mode || h->recon == SG_RECON_FULL) && res_ready<T>(h)) {
    const bool hist = store_full_hist_ckpt_mode;
    SG_TRY(run_graph(h, std::string(hist ? "res_fwd_full/" : "res_fwd_plain/") + std::to_string(cnt),
                     [&](cudaStream_t s) -> int {
                       HistRef hr;
                       if (hist) hr = main_hist(h, 0);
                       return enq_res_forward<T>(h, s, cnt, hr, true);
                     }));
    return SG_OK;
  }
  if (!store_full_hist_ckpt_mode) {
    SG_TRY(run_graph(h, "fwd_plain/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        FwdPlan p;
        return enq_forward<T>(h, cs, c, 0, nt, p, nullptr, s0);
      });
    }));
    return SG_OK;
  }
  if (h->recon == SG_RECON_BOUNDARY) {
    SG_TRY(run_graph(h, "fwd_band/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        FwdPlan p;
        p.band_save = true;
        return enq_forward<T>(h, cs, c, 0, nt, p, nullptr, s0);
      });
    }));
  } else if (h->recon == SG_RECON_FULL) {
    SG_TRY(run_graph(h, "fwd_full/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        FwdPlan p;
        p.hist = main_hist(h, 0);
        return enq_forward<T>(h, cs, c, 0, nt, p, nullptr, s0);
      });
    }));
  } else {
    SG_TRY(run_graph(h, "fwd_ckpt/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        FwdPlan p;
        p.ckpt_save = true;
        return enq_forward<T>(h, cs, c, 0, nt, p, nullptr, s0);
      });
    }));
  }
  return SG_OK;
}

// adjoint over all steps with imaging against the forward history of the
// current batch (FULL: stored; CHECKPOINT: segment recompute from checkpoints)
template <typename T>
int do_adjoint_batch(sg_handle* h, int cnt, const void* cached_hist, int64_t cached_shots) {
  SG_TRY(zero_fields(h, false, true, cnt));
  SG_CK(cudaMemsetAsync(h->img, 0, (size_t)2 * h->B * h->hplane * h->esz, h->stream));
  const int nt = h->d.nt;
  if (cached_hist != nullptr || h->recon == SG_RECON_FULL) {
    HistRef hr = main_hist(h, 0);
    if (cached_hist) {
      hr.base = const_cast<void*>(cached_hist);
      hr.steps = nt;
      hr.shots = cached_shots;
    }
    const void* hb = hr.base;
    if (h->inj_dense && res_ready<T>(h)) {
      // cluster-resident adjoint: one launch for the whole sweep
      const std::string key = std::string(cached_hist ? "res_adj_cached/" : "res_adj_full/") +
                              std::to_string(cnt) + "/" + std::to_string((uintptr_t)hb);
      SG_TRY(run_graph(h, key, [&](cudaStream_t s) -> int {
        return enq_res_adjoint<T>(h, s, cnt, hr);
      }));
      return SG_OK;
    }
    std::string key = std::string(cached_hist ? "adj_cached/" : "adj_full/") +
                      std::to_string(cnt) + "/" + std::to_string((uintptr_t)hb);
    SG_TRY(run_graph(h, key, [&](cudaStream_t s) -> int {
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        AdjPlan p;
        p.hist = hr;
        return enq_adjoint<T>(h, cs, c, nt, 0, p, nullptr, s0);
      });
    }));
    return SG_OK;
  }
  if (h->recon == SG_RECON_BOUNDARY) {
    // the forward left (u_nt, inc_nt) in ({u0,u1}[nt & 1], inc): step back to
    // u_{nt-1}, then the fused reverse-forward + adjoint sweep
    SG_TRY(run_graph(h, "adj_band/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
      const int fin = nt & 1;
      void* F[2] = {h->u0, h->u1};
      dim3 grid(cdiv(h->nxp, 128), h->nzp, cnt);
      k_band_init<T><<<grid, 128, 0, s>>>(field<T>(F[fin], h), field<T>(h->inc, h),
                                          field<T>(F[fin ^ 1], h),
                                          reinterpret_cast<const T*>(h->band),
                                          (int64_t)nt * h->bgeo.nb, nt - 1, h->bgeo, h->plane);
      count_launch();
      return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        AdjPlan ap;
        ap.band_recon = true;
        ap.rcur0 = fin ^ 1;
        return enq_adjoint<T>(h, cs, c, nt, 0, ap, nullptr, s0);
      });
    }));
    return SG_OK;
  }
  // CHECKPOINT: per segment restore -> forward with segment history -> adjoint
  SG_TRY(run_graph(h, "adj_ckpt/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
    const size_t pb = span_bytes(h, cnt);
    const size_t sb = span_bytes(h, h->B);
    int acur = 0;  // adjoint ping-pong position, continues across segments
    int acur_next = 0;
    for (int seg = h->ncp - 1; seg >= 0; --seg) {
      const int n0 = seg * h->K;
      const int n1 = std::min(nt, n0 + h->K);
      char* slot = (char*)h->ckpt + (size_t)seg * 2 * sb;
      cudaMemcpyAsync(h->u0, slot, pb, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(h->inc, slot + sb, pb, cudaMemcpyDeviceToDevice, s);
      SG_TRY(fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) -> int {
        FwdPlan fp;
        fp.gathers = false;
        fp.hist = main_hist(h, n0);
        SG_TRY(enq_forward<T>(h, cs, c, n0, n1, fp, nullptr, s0));
        AdjPlan ap;
        ap.hist = main_hist(h, n0);
        int ac = acur;  // every chain starts the segment at the same parity
        SG_TRY(enq_adjoint<T>(h, cs, c, n1, n0, ap, &ac, s0));
        if (s0 == 0) acur_next = ac;  // and ends it at the same one
        return SG_OK;
      }));
      acur = acur_next;
    }
    return SG_OK;
  }));
  return SG_OK;
}

template <typename T>
int copy_gathers_out(sg_handle* h, void* dst, int cnt) {
  if (dst == h->gath) return SG_OK;
  const size_t b = (size_t)cnt * h->d.nt * h->d.n_rec * h->esz;
  SG_CK(cudaMemcpyAsync(dst, h->gath, b, cudaMemcpyDeviceToDevice, h->stream));
  return SG_OK;
}

template <typename T>
int copy_gathers_in(sg_handle* h, const void* src, int cnt) {
  const size_t b = (size_t)cnt * h->d.nt * h->d.n_rec * h->esz;
  SG_CK(cudaMemcpyAsync(h->gath, src, b, cudaMemcpyDeviceToDevice, h->stream));
  return SG_OK;
}

// Shots of the next batch when `remaining` are left: the fewest batches the
// buffers allow, balanced (sizes differ by at most one), so a survey that is
// not a multiple of the batch never ends in a sliver batch at the per-step
// latency floor (C5: 240 shots at B = 14 ran 17 x 14 + 2; now 6 x 14 + 12 x 13)
int next_batch(const sg_handle* h, int remaining) {
  static const bool balance = [] {
    const char* e = getenv("SG_BALANCE");
    return !(e && atoi(e) == 0);
  }();
  if (!balance) return std::min(h->B, remaining);
  const int nb = (remaining + h->B - 1) / h->B;
  return (remaining + nb - 1) / nb;
}

template <typename T>
int fwi_synthetic_t(sg_handle* h, int shot0, int count, void* out) {
  SG_TRY(ensure_batch(h));
  const size_t per = (size_t)h->d.nt * h->d.n_rec * h->esz;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = next_batch(h, shot0 + count - b0);
    SG_TRY(do_forward_batch<T>(h, b0, cnt, false));
    SG_TRY(copy_gathers_out<T>(h, (char*)out + (size_t)(b0 - shot0) * per, cnt));
  }
  SG_CK(cudaGetLastError());
  return SG_OK;
}

template <typename T>
int fwi_misfit_t(sg_handle* h, int shot0, int count, const void* obs, double* misfit) {
  SG_TRY(ensure_batch(h));
  SG_CK(cudaMemsetAsync(h->scal, 0, sizeof(double), h->stream));
  const size_t per = (size_t)h->d.nt * h->d.n_rec * h->esz;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = next_batch(h, shot0 + count - b0);
    SG_TRY(do_forward_batch<T>(h, b0, cnt, false));
    SG_TRY(residual<T>(h, cnt, reinterpret_cast<const T*>((const char*)obs + (b0 - shot0) * per),
                       2));
  }
  SG_CK(cudaMemcpyAsync(misfit, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  SG_CK(cudaStreamSynchronize(h->stream));
  return SG_OK;
}

template <typename T>
int fwi_gradient_t(sg_handle* h, int shot0, int count, const void* obs, double* misfit,
                   void* grad, int accumulate) {
  SG_TRY(ensure_batch(h));
  SG_CK(cudaMemsetAsync(h->scal, 0, sizeof(double), h->stream));
  SG_CK(cudaMemsetAsync(h->acc_img, 0, (size_t)h->hplane * h->esz, h->stream));
  const size_t per = (size_t)h->d.nt * h->d.n_rec * h->esz;
  // phase events per batch (sg_phase_times; printed with SG_PHASE_TIMING=1)
  static const bool timing = getenv("SG_PHASE_TIMING") != nullptr;
  h->ph_batches = 0;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = next_batch(h, shot0 + count - b0);
    while ((int)h->ph_ev.size() < 5 * (h->ph_batches + 1)) {
      cudaEvent_t e;
      SG_CK(cudaEventCreate(&e));
      h->ph_ev.push_back(e);
    }
    cudaEvent_t* ev = h->ph_ev.data() + 5 * h->ph_batches;
    h->ph_batches++;
    SG_CK(cudaEventRecord(ev[0], h->stream));
    {
      Trace t_("forward sweep");
      SG_TRY(do_forward_batch<T>(h, b0, cnt, true));
    }
    SG_CK(cudaEventRecord(ev[1], h->stream));
    SG_TRY(residual<T>(h, cnt, reinterpret_cast<const T*>((const char*)obs + (b0 - shot0) * per),
                       0));
    SG_TRY(fill_injection<T>(h, cnt));
    SG_CK(cudaEventRecord(ev[2], h->stream));
    {
      Trace t_("adjoint sweep + imaging");
      SG_TRY(do_adjoint_batch<T>(h, cnt, nullptr, 0));
    }
    SG_CK(cudaEventRecord(ev[3], h->stream));
    SG_TRY(reduce_images<T>(h, cnt));
    SG_CK(cudaEventRecord(ev[4], h->stream));
    if (timing) {
      cudaEventSynchronize(ev[4]);
      float t[4];
      for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
      fprintf(stderr, "[sg] batch %d+%d: forward %.3f ms, residual+injection %.3f ms, "
              "adjoint %.3f ms, image reduce %.3f ms\n", b0, cnt, t[0], t[1], t[2], t[3]);
    }
  }
  SG_TRY(fold_out<T>(h, grad, accumulate));
  if (misfit) {
    SG_CK(cudaMemcpyAsync(misfit, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    SG_CK(cudaStreamSynchronize(h->stream));
  }
  SG_CK(cudaGetLastError());
  return SG_OK;
}

// ---- Born -------------------------------------------------------------------------

template <typename T>
int set_born_scale(sg_handle* h, const void* m_r) {
  if (!h->gscale_buf)
    SG_TRY(dalloc(h, &h->gscale_buf, (size_t)(h->ldx + h->plane + h->tail) * h->esz));
  dim3 grid(cdiv(h->nxp, 128), h->nzp);
  k_extend<T, T><<<grid, 128, 0, h->stream>>>(reinterpret_cast<const T*>(m_r),
                                              field<T>(h->gscale_buf, h), h->d.nz, h->d.nx,
                                              h->nzp, h->nxp, h->ldx, h->d.pad_top,
                                              h->d.pad_left, -1.0 / h->kfold);
  count_launch();
  SG_CK(cudaGetLastError());
  return SG_OK;
}

bool born_cached_covers(const sg_handle* h, int b0, int cnt) {
  return h->born_hist && b0 >= h->born_b0 && b0 + cnt <= h->born_b0 + h->born_count;
}

// Next batch [b0, b0 + cnt) of [b0, end) that lies entirely inside or entirely
// outside the cached background range.
int born_next_batch(const sg_handle* h, int b0, int end) {
  int lim = end;
  if (h->born_hist) {
    const int c0 = h->born_b0, c1 = h->born_b0 + h->born_count;
    if (b0 >= c0 && b0 < c1) lim = std::min(end, c1);
    else if (b0 < c0) lim = std::min(end, c0);
  }
  return std::min(h->B, lim - b0);
}

template <typename T>
int born_cache_t(sg_handle* h, int shot0, int count) {
  SG_TRY(ensure_batch(h));
  dfree(&h->born_hist);
  drop_graphs(h);
  h->born_b0 = -1;
  h->born_count = 0;
  const size_t per = (size_t)h->d.nt * h->hplane * h->esz;
  // cache as many shots as fit (the rest are recomputed per apply)
  size_t free_b = 0, total_b = 0;
  SG_CK(cudaMemGetInfo(&free_b, &total_b));
  const double room = 0.8 * (double)free_b - (double)(2ull << 30);  // leave room for callers
  count = (int)std::max(0.0, std::min((double)count, std::floor(room / (double)per)));
  if (const char* e = getenv("SG_BORN_CACHE_MAX")) count = std::min(count, std::max(0, atoi(e)));
  if (count == 0) return SG_OK;
  SG_TRY(dalloc(h, &h->born_hist, per * count));
  h->born_b0 = shot0;
  h->born_count = count;
  const int nt = h->d.nt;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = next_batch(h, shot0 + count - b0);
    SG_TRY(load_batch_sources(h, b0, cnt));
    SG_TRY(zero_fields(h, true, false, cnt));
    void* base = (char*)h->born_hist + (size_t)(b0 - shot0) * per;
    SG_TRY(run_graph(h, "born_fill/" + std::to_string(cnt) + "/" + std::to_string((uintptr_t)base),
                     [&](cudaStream_t s) -> int {
                       FwdPlan p;
                       p.gathers = false;
                       p.hist.base = base;
                       p.hist.steps = nt;
                       p.hist.shots = count - (b0 - shot0);
                       SG_TRY(enq_forward<T>(h, s, cnt, 0, nt, p));
                       return SG_OK;
                     }));
  }
  SG_CK(cudaStreamSynchronize(h->stream));
  return SG_OK;
}

template <typename T>
int born_forward_t(sg_handle* h, int shot0, int count, const void* m_r, void* out) {
  SG_TRY(ensure_batch(h));
  SG_TRY(set_born_scale<T>(h, m_r));
  const int nt = h->d.nt;
  const size_t gper = (size_t)nt * h->d.n_rec * h->esz;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = born_next_batch(h, b0, shot0 + count);
    if (born_cached_covers(h, b0, cnt)) {
      // scattered field driven by the cached a0 history (seisopt/wavesim.py:289-290)
      SG_TRY(zero_fields(h, true, false, cnt));
      const void* base = (char*)h->born_hist + (size_t)(b0 - h->born_b0) * nt * h->hplane * h->esz;
      SG_TRY(run_graph(h, "born_fwd_cached/" + std::to_string(cnt) + "/" +
                              std::to_string((uintptr_t)base),
                       [&](cudaStream_t s) -> int {
                         return fork_chains(h, s, cnt, [&](cudaStream_t cs, int s0, int c) {
                           FwdPlan p;
                           p.point = false;
                           p.gsrc = base;
                           p.gsrc_shot = (int64_t)nt * h->hplane;
                           return enq_forward<T>(h, cs, c, 0, nt, p, nullptr, s0);
                         });
                       }));
    } else {
      // lock-step: background step writes a0_n into a one-slot buffer, the
      // scattered step (fields l0/l1/w) consumes it in the same stream order
      SG_TRY(load_batch_sources(h, b0, cnt));
      SG_TRY(zero_fields(h, true, true, cnt));
      SG_TRY(run_graph(h, "born_fwd_lock/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
        // The background keeps its whole history (FULL) or its checkpoints
        // (CHECKPOINT) for a following LSRTM adjoint, which then needs no
        // background re-run (4 stencil sweeps per LSRTM gradient).
        // BOUNDARY: the background stores its sponge frame, handing a0_n to
        // the scattered step through the one-slot history.
        const bool full = h->recon == SG_RECON_FULL;
        if (h->recon != SG_RECON_BOUNDARY && h->d.step_mode != 2) {
          // one fused launch per step (a0_n stays in registers)
          return fork_chains(h, s, cnt, [&](cudaStream_t st, int s0, int c) -> int {
            HistRef hr;
            if (full) hr = main_hist(h, 0);
            return enq_lockstep<T>(h, st, c, 0, nt, hr, !full, s0);
          });
        }
        return fork_chains(h, s, cnt, [&](cudaStream_t st, int s0, int c) -> int {
        int cb = 0, cs = 0;  // ping-pong positions of the background / scattered fields
        for (int n = 0; n < nt; ++n) {
          FwdPlan bg;
          bg.gathers = false;
          bg.hist = main_hist(h, full ? 0 : n);
          bg.ckpt_save = h->recon == SG_RECON_CHECKPOINT;
          bg.band_save = h->recon == SG_RECON_BOUNDARY;
          SG_TRY(enq_forward<T>(h, st, c, n, n + 1, bg, &cb, s0));
          FwdPlan sc;
          sc.point = false;
          sc.gsrc = h->hist;
          sc.gsrc_shot = (int64_t)h->hist_steps * h->hplane;
          sc.gsrc_n0 = full ? 0 : n;
          sc.fu0 = h->l0;
          sc.fu1 = h->l1;
          sc.fs0 = h->w;
          sc.fs1 = h->w2;
          SG_TRY(enq_forward<T>(h, st, c, n, n + 1, sc, &cs, s0));
        }
        return SG_OK;
        });
      }));
    }
    SG_TRY(copy_gathers_out<T>(h, (char*)out + (size_t)(b0 - shot0) * gper, cnt));
  }
  SG_CK(cudaGetLastError());
  return SG_OK;
}

template <typename T>
int born_adjoint_core(sg_handle* h, int shot0, int count, const void* data, int mode_resid,
                      const void* d_r, double* value, void* image, int accumulate,
                      const void* m_r) {
  // mode_resid: 0 -> data given directly; 1 -> LSRTM: data = L m_r - d_r
  SG_TRY(ensure_batch(h));
  SG_CK(cudaMemsetAsync(h->acc_img, 0, (size_t)h->hplane * h->esz, h->stream));
  SG_CK(cudaMemsetAsync(h->scal, 0, sizeof(double), h->stream));
  const int nt = h->d.nt;
  const size_t gper = (size_t)nt * h->d.n_rec * h->esz;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = born_next_batch(h, b0, shot0 + count);
    if (mode_resid == 1) {
      SG_TRY(born_forward_t<T>(h, b0, cnt, m_r, h->gath));
      // born_forward_t copied gathers onto themselves; form the residual in place
      SG_TRY(residual<T>(h, cnt, reinterpret_cast<const T*>((const char*)d_r + (b0 - shot0) * gper), 1));
      SG_TRY(fill_injection<T>(h, cnt));
    } else {
      SG_TRY(copy_gathers_in<T>(h, (const char*)data + (size_t)(b0 - shot0) * gper, cnt));
      SG_TRY(fill_injection<T>(h, cnt));
    }
    if (born_cached_covers(h, b0, cnt)) {
      const void* base = (char*)h->born_hist + (size_t)(b0 - h->born_b0) * nt * h->hplane * h->esz;
      SG_TRY(do_adjoint_batch<T>(h, cnt, base, h->born_count - (b0 - h->born_b0)));
    } else if (mode_resid == 1) {
      // the lock-step Born forward of this batch left the background history
      // (FULL) or its checkpoints (CHECKPOINT) in place
      SG_TRY(do_adjoint_batch<T>(h, cnt, nullptr, 0));
    } else if (h->recon == SG_RECON_FULL) {
      // recompute and store the background history, then image against it
      SG_TRY(load_batch_sources(h, b0, cnt));
      SG_TRY(zero_fields(h, true, false, cnt));
      SG_TRY(run_graph(h, "born_bg_full/" + std::to_string(cnt), [&](cudaStream_t s) -> int {
        FwdPlan p;
        p.gathers = false;
        p.hist = main_hist(h, 0);
        SG_TRY(enq_forward<T>(h, s, cnt, 0, nt, p));
        return SG_OK;
      }));
      SG_TRY(do_adjoint_batch<T>(h, cnt, nullptr, 0));
    } else {
      SG_TRY(load_batch_sources(h, b0, cnt));
      SG_TRY(zero_fields(h, true, false, cnt));
      const bool bnd = h->recon == SG_RECON_BOUNDARY;
      SG_TRY(run_graph(h, (bnd ? "born_bg_band/" : "born_bg_ckpt/") + std::to_string(cnt),
                       [&](cudaStream_t s) -> int {
        FwdPlan p;
        p.gathers = false;
        p.ckpt_save = !bnd;
        p.band_save = bnd;
        SG_TRY(enq_forward<T>(h, s, cnt, 0, nt, p));
        return SG_OK;
      }));
      SG_TRY(do_adjoint_batch<T>(h, cnt, nullptr, 0));
    }
    SG_TRY(reduce_images<T>(h, cnt));
  }
  SG_TRY(fold_out<T>(h, image, accumulate));
  if (value) {
    SG_CK(cudaMemcpyAsync(value, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    SG_CK(cudaStreamSynchronize(h->stream));
  }
  SG_CK(cudaGetLastError());
  return SG_OK;
}

// LSRTM objective value J = 1/2 ||L m_r - d_r||^2 (LsrtmObjective.value,
// seisopt/gradients.py:363-369): Born forward per batch and the fused fp64
// residual reduction; the Born data never leave the device
template <typename T>
int lsrtm_misfit_t(sg_handle* h, int shot0, int count, const void* m_r, const void* d_r,
                   double* value) {
  SG_TRY(ensure_batch(h));
  SG_CK(cudaMemsetAsync(h->scal, 0, sizeof(double), h->stream));
  const size_t gper = (size_t)h->d.nt * h->d.n_rec * h->esz;
  for (int b0 = shot0, cnt = 0; b0 < shot0 + count; b0 += cnt) {
    cnt = born_next_batch(h, b0, shot0 + count);
    SG_TRY(born_forward_t<T>(h, b0, cnt, m_r, h->gath));
    SG_TRY(residual<T>(h, cnt, reinterpret_cast<const T*>((const char*)d_r + (b0 - shot0) * gper),
                       3));
  }
  SG_CK(cudaMemcpyAsync(value, h->scal, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  SG_CK(cudaStreamSynchronize(h->stream));
  return SG_OK;
}

// ---- single-shot history export (forward_solve / adjoint_solve) ----------------

template <typename T>
int forward_history_t(sg_handle* h, int shot, void* gather, void* accel) {
  SG_TRY(ensure_batch(h));
  const int nt = h->d.nt;
  void* tmp = nullptr;
  SG_TRY(dalloc(h, &tmp, (size_t)nt * h->hplane * h->esz));
  SG_TRY(load_batch_sources(h, shot, 1));
  SG_TRY(zero_fields(h, true, false, 1));
  FwdPlan p;
  p.hist.base = tmp;
  p.hist.steps = nt;
  p.hist.shots = 1;
  SG_TRY(enq_forward<T>(h, h->stream, 1, 0, nt, p));
  SG_CK(cudaGetLastError());
  SG_TRY(copy_gathers_out<T>(h, gather, 1));
  dim3 grid(cdiv(h->nxp, 128), 4096);
  k_unpitch<T><<<grid, 128, 0, h->stream>>>(reinterpret_cast<T*>(tmp), reinterpret_cast<T*>(accel),
                                            (int64_t)nt * h->nzp, h->nxp, h->ldx);
  count_launch();
  SG_CK(cudaStreamSynchronize(h->stream));
  rz_free(tmp);
  h->held_bytes -= (double)nt * h->hplane * h->esz;
  return SG_OK;
}

template <typename T>
int adjoint_history_t(sg_handle* h, const void* ybar, void* vout) {
  SG_TRY(ensure_batch(h));
  const int nt = h->d.nt;
  void* tmp = nullptr;
  SG_TRY(dalloc(h, &tmp, (size_t)nt * h->hplane * h->esz));
  SG_TRY(copy_gathers_in<T>(h, ybar, 1));
  SG_TRY(fill_injection<T>(h, 1));
  SG_TRY(zero_fields(h, false, true, 1));
  AdjPlan p;
  p.vhist = tmp;
  SG_TRY(enq_adjoint<T>(h, h->stream, 1, nt, 0, p));
  SG_CK(cudaGetLastError());
  dim3 grid(cdiv(h->nxp, 128), 4096);
  k_unpitch<T><<<grid, 128, 0, h->stream>>>(reinterpret_cast<T*>(tmp), reinterpret_cast<T*>(vout),
                                            (int64_t)nt * h->nzp, h->nxp, h->ldx);
  count_launch();
  SG_CK(cudaStreamSynchronize(h->stream));
  rz_free(tmp);
  h->held_bytes -= (double)nt * h->hplane * h->esz;
  return SG_OK;
}

template <typename T>
int time_kernel_t(sg_handle* h, int which, int count, int reps, float* ms) {
  SG_TRY(ensure_batch(h));
  count = std::min(count, h->B);
  if (which == 0 && h->recon != SG_RECON_FULL && h->hist_steps < 1)
    return fail(SG_ERR_STATE, "no history buffer");
  if ((which == 5 || which == 6) && h->recon != SG_RECON_BOUNDARY)
    return fail(SG_ERR_STATE, "band kernels need recon = BOUNDARY");
  SG_TRY(load_batch_sources(h, 0, count));
  cudaEvent_t e0, e1;
  SG_CK(cudaEventCreate(&e0));
  SG_CK(cudaEventCreate(&e1));
  const int n = h->d.nt / 2;
  // the launches run as the sweeps run them: concurrent shot chains
  // (fork_chains), so the time per repetition is the step time of the batch
  auto chain_body = [&](cudaStream_t s, int s0, int count) -> int {
    if (which == 5 || which == 6) {
      // band kernels walk the band store like a sweep (a different slot per launch)
      for (int r = 0; r < reps; ++r) {
        const int m = h->d.nt - 1 - r % (h->d.nt - 1);
        if (which == 6) {
          FwdPlan p;
          p.band_save = true;
          SG_TRY(enq_forward<T>(h, s, count, m, m + 1, p, nullptr, s0));
        } else {
          AdjPlan p;
          p.band_recon = true;
          p.rcur0 = r & 1;
          SG_TRY(enq_adjoint<T>(h, s, count, m + 1, m, p, nullptr, s0));
        }
      }
    } else if (which == 3 || which == 4) {
      // two-step launches (two time steps each); history rotates through the buffer
      HistRef hr = main_hist(h, n);
      hr.rotate = true;
      for (int r = 0; r < reps; ++r) {
        if (which == 3) {
          FwdPlan p;
          p.hist = hr;
          SG_TRY(enq_forward<T>(h, s, count, n + 2 * (r & 1), n + 2 * (r & 1) + 2, p));
        } else {
          AdjPlan p;
          p.hist = hr;
          SG_TRY(enq_adjoint<T>(h, s, count, n + 2, n, p));
        }
      }
    } else if (which == 0 || which == 2) {
      FwdPlan p;
      if (which == 0) {
        p.hist = main_hist(h, n);
        p.hist.rotate = true;
      }
      for (int r = 0; r < reps; ++r)
        SG_TRY(enq_forward<T>(h, s, count, n + (r & 1), n + (r & 1) + 1, p, nullptr, s0));
    } else {
      // walk the history like a sweep does (a different, L2-cold plane per
      // launch) so the timing includes the streaming history read
      AdjPlan p;
      p.hist = main_hist(h, 0);
      p.hist.rotate = true;
      for (int r = 0; r < reps; ++r) {
        const int m = (int)((h->d.nt - 1 - r % h->d.nt) % std::max<int64_t>(1, h->hist_steps));
        SG_TRY(enq_adjoint<T>(h, s, count, m + 1, m, p, nullptr, s0));
      }
    }
    return SG_OK;
  };
  auto body = [&](cudaStream_t s) -> int {
    if (which == 3 || which == 4) return chain_body(s, 0, count);  // two-step: one chain
    return fork_chains(h, s, count, chain_body);
  };

  SG_TRY(body(h->stream));  // warm-up
  SG_CK(cudaEventRecord(e0, h->stream));
  SG_TRY(body(h->stream));
  SG_CK(cudaEventRecord(e1, h->stream));
  SG_CK(cudaEventSynchronize(e1));
  float t = 0.f;
  SG_CK(cudaEventElapsedTime(&t, e0, e1));
  *ms = t / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  SG_CK(cudaGetLastError());
  return SG_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

#define SG_DISPATCH(h, fn, ...) \
  ((h)->esz == 4 ? fn<float>(__VA_ARGS__) : fn<double>(__VA_ARGS__))

extern "C" {

const char* sg_last_error(void) { return sg::g_err.c_str(); }
int sg_version(void) { return 2; }
int sg_build_flags(void) { return SG_EXPERIMENTAL ? SG_BUILD_EXPERIMENTAL : 0; }
int64_t sg_launch_count(void) { return sg::g_launches.load(); }

int sg_last_nonfinite(sg_handle* h, int64_t* count) {
  SG_TRY(check_handle(h));
  if (!count) return fail(SG_ERR_ARG, "null argument");
  if (h->nonfinite_pending) {
    SG_CK(cudaStreamSynchronize(h->stream));
    h->nonfinite_pending = false;
  }
  *count = (int64_t)h->nonfinite;
  return SG_OK;
}

int sg_redzone_check(int64_t* bad_bytes, int64_t* allocations, int32_t poke) {
  if (!bad_bytes || !allocations) return fail(SG_ERR_ARG, "null argument");
  *bad_bytes = 0;
  *allocations = 0;
  if (!sg::rz_on()) return SG_OK;
  std::lock_guard<std::mutex> lk(sg::g_rz_mu);
  if (poke && !sg::g_rz_live.empty()) {
    // self-test: one byte written just past the first live allocation
    const auto& r = sg::g_rz_live.begin()->second;
    SG_CK(cudaMemset((char*)r.base + sg::kRedZone + r.bytes, 0, 1));
  }
  int64_t bad = sg::g_rz_bad.load();
  for (const auto& kv : sg::g_rz_live) bad += sg::rz_scan(kv.second);
  *bad_bytes = bad;
  *allocations = sg::g_rz_allocs.load();
  return SG_OK;
}

int sg_create(const sg_desc* d, sg_handle** out) {
  if (!d || !out) return fail(SG_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->nz < 3 || d->nx < 3) return fail(SG_ERR_ARG, "grid must be at least 3x3");
  if (d->pad_top < 0 || d->pad_bottom < 0 || d->pad_left < 0 || d->pad_right < 0)
    return fail(SG_ERR_ARG, "negative pad");
  if (d->nt < 2) return fail(SG_ERR_ARG, "nt must be at least 2");
  if (d->n_shots < 1 || d->n_rec < 1) return fail(SG_ERR_ARG, "need sources and receivers");
  if (d->dtype != SG_F32 && d->dtype != SG_F64) return fail(SG_ERR_ARG, "dtype must be 4 or 8");
  if (d->order != 2 && d->order != 8) return fail(SG_ERR_ARG, "order must be 2 or 8");
  if (!(d->dx > 0 && d->dz > 0 && d->dt > 0)) return fail(SG_ERR_ARG, "spacings must be positive");
  if (d->recon < 0 || d->recon > 3) return fail(SG_ERR_ARG, "bad recon mode");
  SG_CK(cudaSetDevice(d->device));
  sg_handle* h = new sg_handle();
  h->d = *d;
  h->esz = d->dtype;
  h->nzp = d->nz + d->pad_top + d->pad_bottom;
  h->nxp = d->nx + d->pad_left + d->pad_right;
  h->ldx = ((h->nxp + 4 + 31) / 32) * 32;
  h->plane = (int64_t)(h->nzp + 2 * kGuard) * h->ldx;
  h->origin = (int64_t)kGuard * h->ldx;
  h->hplane = (int64_t)h->nzp * h->ldx;
  h->tail = (int64_t)(kTileRowsMax + 2 * kGuard + 4) * h->ldx;
  h->tiles_x = (h->nxp + BX - 1) / BX;
  h->ntiles = h->tiles_x * ((h->nzp + TH - 1) / TH);
  h->ntiles2 = h->tiles_x * ((h->nzp + TH2 - 1) / TH2);
  h->rec_blocks = (d->n_rec + RB - 1) / RB;
  cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, d->device);
  {
    const char* e = getenv("SG_PDL");
    h->pdl = !(e && atoi(e) == 0);
  }
  const double rz = 1.0 / (d->dz * d->dz), rx = 1.0 / (d->dx * d->dx);
  if (d->order == 2) {
    h->cz[1] = rz;
    h->cx[1] = rx;
  } else {
    const double c8[5] = {-205.0 / 72.0, 8.0 / 5.0, -1.0 / 5.0, 8.0 / 315.0, -1.0 / 560.0};
    for (int k = 1; k < 5; ++k) {
      h->cz[k] = c8[k] * rz;
      h->cx[k] = c8[k] * rx;
    }
  }
  if (SG_GC && h->esz == 4) h->kfold = h->cz[1];
  int rc = dalloc(h, &h->inv_m_buf, (size_t)(h->ldx + h->plane + h->tail) * h->esz);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return SG_OK;
}

int sg_destroy(sg_handle* h) {
  if (!h) return SG_OK;
  cudaSetDevice(h->d.device);
  free_batch(h);
  void** bufs[] = {(void**)&h->rec_rc, (void**)&h->tile_rec_ptr, (void**)&h->tile_rec,
                   &h->inv_m_buf, &h->pz_buf, &h->px_buf, &h->ez_buf, &h->ex_buf, &h->gscale_buf, (void**)&h->src_rc,
                   &h->src_w, (void**)&h->rec_ij, &h->rec_w, (void**)&h->inj_ptr,
                   (void**)&h->inj_rec, &h->inj_w, &h->born_hist, &h->wav_dev,
                   (void**)&h->res_rec};
  for (auto p : bufs) dfree(p);
  if (h->cap) cudaStreamDestroy(h->cap);
  for (int c = 1; c < sg_handle::kMaxChains; ++c) {
    if (h->chain[c]) cudaStreamDestroy(h->chain[c]);
    if (h->ev_join[c]) cudaEventDestroy(h->ev_join[c]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  for (auto e : h->ph_ev) cudaEventDestroy(e);
  delete h;
  return SG_OK;
}

int sg_set_stream(sg_handle* h, void* s) {
  if (!h) return fail(SG_ERR_ARG, "null handle");
  h->stream = reinterpret_cast<cudaStream_t>(s);
  return SG_OK;
}

int sg_set_sponge(sg_handle* h, const double* pz, const double* px) {
  if (!h || !pz || !px) return fail(SG_ERR_ARG, "null argument");
  SG_CK(cudaSetDevice(h->d.device));
  // guarded profile arrays: kGuard zeros before, generous zero tail after
  std::vector<double> z(h->nzp + 2 * kGuard + kTileRowsMax + 16, 0.0);
  std::vector<double> x(h->ldx + 2 * kGuard + kSlack, 0.0);
  for (int i = 0; i < h->nzp; ++i) z[kGuard + i] = pz[i];
  for (int j = 0; j < h->nxp; ++j) x[kGuard + j] = px[j];
  // frame of the band store: every row/column whose profile (in the device
  // dtype) is below 1 at either end, i.e. every cell with damp < 1
  // (fp32 with SG_GC damps by e = (float)(1 - p): the same rows/columns
  // unless p is within 2^-25 of 1, so both tests are applied)
  auto below1 = [&](double v) {
    return h->esz == 4 ? ((float)v < 1.0f || (float)(1.0 - v) > 0.0f) : v < 1.0;
  };
  auto frame = [&](const double* p, int n, int& lo, int& hi) {
    lo = 0;
    hi = 0;
    for (int i = 0; i < (n + 1) / 2; ++i)
      if (below1(p[i])) lo = i + 1;
    for (int i = n - 1; i >= (n + 1) / 2; --i)
      if (below1(p[i])) hi = n - i;
    hi = std::min(hi, n - lo);
  };
  BandGeo& g = h->bgeo;
  frame(pz, h->nzp, g.bT, g.bB);
  frame(px, h->nxp, g.bL, g.bR);
  g.nzp = h->nzp;
  g.nxp = h->nxp;
  g.ldx = h->ldx;
  g.nb = (g.bT + g.bB) * h->nxp + (h->nzp - g.bT - g.bB) * (g.bL + g.bR);
  free_batch(h);  // batch buffers are sized with the frame
  dfree(&h->pz_buf);
  dfree(&h->px_buf);
  dfree(&h->ez_buf);
  dfree(&h->ex_buf);
  // e = 1 - p in fp64, rounded once (zero guards and tails stay zero)
  std::vector<double> ezv(z.size(), 0.0), exv(x.size(), 0.0);
  for (int i = 0; i < h->nzp; ++i) ezv[kGuard + i] = 1.0 - pz[i];
  for (int j = 0; j < h->nxp; ++j) exv[kGuard + j] = 1.0 - px[j];
  if (h->esz == 4) {
    SG_TRY(upload_cast<float>(h, &h->pz_buf, z.data(), z.size()));
    SG_TRY(upload_cast<float>(h, &h->px_buf, x.data(), x.size()));
    SG_TRY(upload_cast<float>(h, &h->ez_buf, ezv.data(), ezv.size()));
    SG_TRY(upload_cast<float>(h, &h->ex_buf, exv.data(), exv.size()));
  } else {
    SG_TRY(upload_cast<double>(h, &h->pz_buf, z.data(), z.size()));
    SG_TRY(upload_cast<double>(h, &h->px_buf, x.data(), x.size()));
    SG_TRY(upload_cast<double>(h, &h->ez_buf, ezv.data(), ezv.size()));
    SG_TRY(upload_cast<double>(h, &h->ex_buf, exv.data(), exv.size()));
  }
  h->have_sponge = true;
  return SG_OK;
}

int sg_set_geometry(sg_handle* h, const int32_t* src_rows, const int32_t* src_cols,
                    const double* src_w, const int32_t* rec_rows, const int32_t* rec_cols,
                    const double* rec_w, double src_scale) {
  if (!h || !src_rows || !src_cols || !src_w || !rec_rows || !rec_cols || !rec_w)
    return fail(SG_ERR_ARG, "null argument");
  SG_CK(cudaSetDevice(h->d.device));
  const int S = h->d.n_shots, R = h->d.n_rec;
  auto in_grid = [&](int r, int c) { return r >= 0 && r < h->nzp && c >= 0 && c < h->nxp; };
  // sources: (4, S) -> per shot 4 flat offsets, weights * src_scale
  // (seisopt/wavesim.py:284: sw = src_w * src_scale)
  std::vector<int> src(8 * S);
  std::vector<double> sw(4 * S);
  for (int s = 0; s < S; ++s)
    for (int k = 0; k < 4; ++k) {
      const int r = src_rows[k * S + s], c = src_cols[k * S + s];
      if (!in_grid(r, c)) return fail(SG_ERR_ARG, "source tap outside padded grid");
      src[(s * 4 + k) * 2] = r;
      src[(s * 4 + k) * 2 + 1] = c;
      sw[s * 4 + k] = src_w[k * S + s] * src_scale / h->kfold;
    }
  std::vector<int> rij(4 * R);
  int rmin = 1 << 30, rmax = -1;
  for (int e = 0; e < 4 * R; ++e) {
    const int r = rec_rows[e], c = rec_cols[e];
    if (!in_grid(r, c)) return fail(SG_ERR_ARG, "receiver tap outside padded grid");
    rij[e] = r * h->ldx + c;
    rmin = std::min(rmin, r);
    rmax = std::max(rmax, r);
  }
  // injection CSR over the receiver row band, entries in np.add.at order
  // (flattened (4, R) index: k-major) -- seisopt/wavesim.py:228-229
  const int nrows = rmax - rmin + 1;
  const int ncell = nrows * h->nxp;
  std::vector<int> cnt(ncell + 1, 0);
  for (int e = 0; e < 4 * R; ++e) cnt[(rec_rows[e] - rmin) * h->nxp + rec_cols[e] + 1]++;
  for (int c = 0; c < ncell; ++c) cnt[c + 1] += cnt[c];
  std::vector<int> fillp(cnt.begin(), cnt.end() - 1), irec(4 * R);
  std::vector<double> iw(4 * R);
  for (int e = 0; e < 4 * R; ++e) {
    const int cell = (rec_rows[e] - rmin) * h->nxp + rec_cols[e];
    const int at = fillp[cell]++;
    irec[at] = e % R;
    iw[at] = rec_w[e];
  }
  // receivers grouped by the tile of their first tap (two-step forward)
  std::vector<int> rrc(8 * R), tcount(h->ntiles2 + 1, 0), trec(R);
  for (int e = 0; e < 4 * R; ++e) {
    rrc[2 * e] = rec_rows[e];
    rrc[2 * e + 1] = rec_cols[e];
  }
  auto tile_of = [&](int r) { return (rec_rows[r] / TH2) * h->tiles_x + rec_cols[r] / BX; };
  for (int r = 0; r < R; ++r) tcount[tile_of(r) + 1]++;
  for (int t = 0; t < h->ntiles2; ++t) tcount[t + 1] += tcount[t];
  {
    std::vector<int> fill(tcount.begin(), tcount.end() - 1);
    for (int r = 0; r < R; ++r) trec[fill[tile_of(r)]++] = r;
  }
  void** bufs[] = {(void**)&h->src_rc, &h->src_w, (void**)&h->rec_ij, &h->rec_w,
                   (void**)&h->inj_ptr, (void**)&h->inj_rec, &h->inj_w,
                   (void**)&h->rec_rc, (void**)&h->tile_rec_ptr, (void**)&h->tile_rec};
  for (auto p : bufs) dfree(p);
  SG_TRY(dalloc(h, (void**)&h->rec_rc, rrc.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->rec_rc, rrc.data(), rrc.size() * sizeof(int), cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->tile_rec_ptr, tcount.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->tile_rec_ptr, tcount.data(), tcount.size() * sizeof(int),
                   cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->tile_rec, trec.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->tile_rec, trec.data(), trec.size() * sizeof(int), cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->src_rc, src.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->src_rc, src.data(), src.size() * sizeof(int), cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->rec_ij, rij.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->rec_ij, rij.data(), rij.size() * sizeof(int), cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->inj_ptr, cnt.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->inj_ptr, cnt.data(), cnt.size() * sizeof(int), cudaMemcpyHostToDevice));
  SG_TRY(dalloc(h, (void**)&h->inj_rec, irec.size() * sizeof(int)));
  SG_CK(cudaMemcpy(h->inj_rec, irec.data(), irec.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (h->esz == 4) {
    SG_TRY(upload_cast<float>(h, &h->src_w, sw.data(), sw.size()));
    SG_TRY(upload_cast<float>(h, &h->rec_w, rec_w, 4 * (size_t)R));
    SG_TRY(upload_cast<float>(h, &h->inj_w, iw.data(), iw.size()));
  } else {
    SG_TRY(upload_cast<double>(h, &h->src_w, sw.data(), sw.size()));
    SG_TRY(upload_cast<double>(h, &h->rec_w, rec_w, 4 * (size_t)R));
    SG_TRY(upload_cast<double>(h, &h->inj_w, iw.data(), iw.size()));
  }
  h->rec_rows_h.assign(rec_rows, rec_rows + 4 * R);
  h->rec_cols_h.assign(rec_cols, rec_cols + 4 * R);
  dfree((void**)&h->res_rec);
  h->res_state = 0;
  h->inj_row0 = rmin;
  h->inj_nrows = nrows;
  h->src_scale = src_scale;
  h->have_geom = true;
  drop_graphs(h);
  return SG_OK;
}

int sg_set_wavelet(sg_handle* h, const double* amp) {
  if (!h || !amp) return fail(SG_ERR_ARG, "null argument");
  for (int n = 0; n < h->d.nt; ++n)
    if (!std::isfinite(amp[n])) return fail(SG_ERR_ARG, "wavelet contains non-finite values");
  h->wavelet.assign(amp, amp + h->d.nt);
  dfree(&h->wav_dev);
  h->have_wavelet = true;
  drop_graphs(h);  // amplitudes are baked into captured launches
  return SG_OK;
}

int sg_set_model(sg_handle* h, const void* m, int32_t mdt) {
  sg::Trace trace_("sg_set_model");
  if (!h || !m) return fail(SG_ERR_ARG, "null argument");
  if (mdt != SG_F32 && mdt != SG_F64) return fail(SG_ERR_ARG, "m dtype must be 4 or 8");
  SG_CK(cudaSetDevice(h->d.device));
  if (!h->part) {
    // model stats need a partials buffer before the batch buffers exist
    SG_TRY(ensure_batch(h));
  }
  const int64_t n = (int64_t)h->d.nz * h->d.nx;
  const int blocks = std::min<int64_t>(h->npart, cdiv(n, 256));
  if (mdt == SG_F32)
    k_model_stats<float><<<blocks, 256, 0, h->stream>>>((const float*)m, n, h->part);
  else
    k_model_stats<double><<<blocks, 256, 0, h->stream>>>((const double*)m, n, h->part);
  count_launch();
  std::vector<double> part(2 * blocks);
  SG_CK(cudaMemcpyAsync(part.data(), h->part, part.size() * sizeof(double),
                        cudaMemcpyDeviceToHost, h->stream));
  SG_CK(cudaStreamSynchronize(h->stream));
  double mn = INFINITY, bad = 0.0;
  for (int b = 0; b < blocks; ++b) {
    mn = std::min(mn, part[2 * b]);
    bad += part[2 * b + 1];
  }
  if (bad > 0 || !(mn > 0)) {
    h->have_model = false;
    return fail(SG_ERR_MODEL, "model is not positive and finite");
  }
  // CFL (seisopt/wavesim.py:92-100, 187-193); 8th order: x sqrt(4/6.5016)
  const double c_max = 1.0 / std::sqrt(mn);
  double bound = h->d.cfl_safety * std::min(h->d.dx, h->d.dz) / (c_max * std::sqrt(2.0));
  if (h->d.order == 8) {
    const double sym = 205.0 / 72.0 + 2.0 * (8.0 / 5.0 + 1.0 / 5.0 + 8.0 / 315.0 + 1.0 / 560.0);
    bound *= std::sqrt(4.0 / sym);
  }
  if (h->d.dt > bound) {
    h->have_model = false;
    char buf[256];
    snprintf(buf, sizeof buf, "dt=%g exceeds stable bound %.6g (c_max=%.6g, safety=%g)", h->d.dt,
             bound, c_max, h->d.cfl_safety);
    return fail(SG_ERR_STABILITY, buf);
  }
  dim3 grid(cdiv(h->nxp, 128), h->nzp);
  if (h->esz == 4) {
    if (mdt == SG_F32)
      k_set_inv_m<float, float><<<grid, 128, 0, h->stream>>>((const float*)m, field<float>(h->inv_m_buf, h), h->d.nz, h->d.nx, h->nzp, h->nxp, h->ldx, h->d.pad_top, h->d.pad_left, h->kfold);
    else
      k_set_inv_m<float, double><<<grid, 128, 0, h->stream>>>((const double*)m, field<float>(h->inv_m_buf, h), h->d.nz, h->d.nx, h->nzp, h->nxp, h->ldx, h->d.pad_top, h->d.pad_left, h->kfold);
  } else {
    if (mdt == SG_F32)
      k_set_inv_m<double, float><<<grid, 128, 0, h->stream>>>((const float*)m, field<double>(h->inv_m_buf, h), h->d.nz, h->d.nx, h->nzp, h->nxp, h->ldx, h->d.pad_top, h->d.pad_left, h->kfold);
    else
      k_set_inv_m<double, double><<<grid, 128, 0, h->stream>>>((const double*)m, field<double>(h->inv_m_buf, h), h->d.nz, h->d.nx, h->nzp, h->nxp, h->ldx, h->d.pad_top, h->d.pad_left, h->kfold);
  }
  count_launch();
  SG_CK(cudaGetLastError());
  h->have_model = true;
  if (h->born_hist) {  // background histories of the previous model are stale
    dfree(&h->born_hist);
    drop_graphs(h);
    h->born_b0 = -1;
    h->born_count = 0;
  }
  return SG_OK;
}

int sg_fwi_synthetic(sg_handle* h, int32_t shot0, int32_t count, void* out) {
  sg::Trace trace_("sg_fwi_synthetic");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!out) return fail(SG_ERR_ARG, "null output");
  return SG_DISPATCH(h, fwi_synthetic_t, h, shot0, count, out);
}

int sg_fwi_misfit(sg_handle* h, int32_t shot0, int32_t count, const void* obs, double* misfit) {
  sg::Trace trace_("sg_fwi_misfit");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!obs || !misfit) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, fwi_misfit_t, h, shot0, count, obs, misfit);
}

int sg_fwi_gradient(sg_handle* h, int32_t shot0, int32_t count, const void* obs, double* misfit,
                    void* grad, int32_t accumulate) {
  sg::Trace trace_("sg_fwi_gradient");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!obs || !grad) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, fwi_gradient_t, h, shot0, count, obs, misfit, grad, accumulate);
}

int sg_born_cache(sg_handle* h, int32_t shot0, int32_t count, int32_t enable) {
  sg::Trace trace_("sg_born_cache");
  SG_TRY(check_handle(h));
  if (!enable) {
    dfree(&h->born_hist);
    drop_graphs(h);
    h->born_b0 = -1;
    h->born_count = 0;
    return SG_OK;
  }
  SG_TRY(check_range(h, shot0, count));
  return SG_DISPATCH(h, born_cache_t, h, shot0, count);
}

int sg_born_forward(sg_handle* h, int32_t shot0, int32_t count, const void* m_r, void* out) {
  sg::Trace trace_("sg_born_forward");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!m_r || !out) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, born_forward_t, h, shot0, count, m_r, out);
}

int sg_born_adjoint(sg_handle* h, int32_t shot0, int32_t count, const void* data, void* image,
                    int32_t accumulate) {
  sg::Trace trace_("sg_born_adjoint");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!data || !image) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, born_adjoint_core, h, shot0, count, data, 0, nullptr, nullptr, image,
                     accumulate, nullptr);
}

int sg_lsrtm_gradient(sg_handle* h, int32_t shot0, int32_t count, const void* m_r,
                      const void* d_r, double* value, void* grad, int32_t accumulate) {
  sg::Trace trace_("sg_lsrtm_gradient");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!m_r || !d_r || !grad) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, born_adjoint_core, h, shot0, count, nullptr, 1, d_r, value, grad,
                     accumulate, m_r);
}

int sg_lsrtm_misfit(sg_handle* h, int32_t shot0, int32_t count, const void* m_r,
                    const void* d_r, double* value) {
  sg::Trace trace_("sg_lsrtm_misfit");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot0, count));
  if (!m_r || !d_r || !value) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, lsrtm_misfit_t, h, shot0, count, m_r, d_r, value);
}

int sg_forward_history(sg_handle* h, int32_t shot, void* gather, void* accel) {
  sg::Trace trace_("sg_forward_history");
  SG_TRY(check_handle(h));
  SG_TRY(check_range(h, shot, 1));
  if (!gather || !accel) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, forward_history_t, h, shot, gather, accel);
}

int sg_adjoint_history(sg_handle* h, const void* ybar, void* v) {
  sg::Trace trace_("sg_adjoint_history");
  SG_TRY(check_handle(h));
  if (!ybar || !v) return fail(SG_ERR_ARG, "null argument");
  return SG_DISPATCH(h, adjoint_history_t, h, ybar, v);
}

int sg_born_cached(sg_handle* h, int32_t* shot0, int32_t* count) {
  if (!h) return fail(SG_ERR_ARG, "null handle");
  if (shot0) *shot0 = h->born_hist ? h->born_b0 : 0;
  if (count) *count = h->born_hist ? h->born_count : 0;
  return SG_OK;
}

int sg_query(sg_handle* h, int32_t* batch, int32_t* recon, double* bytes) {
  if (!h) return fail(SG_ERR_ARG, "null handle");
  if (batch) *batch = h->B;
  if (recon) *recon = h->recon;
  if (bytes) *bytes = h->held_bytes;
  return SG_OK;
}

int sg_chains(sg_handle* h, int32_t count) { return h ? nchains(h, count) : 1; }

int sg_resident_plan(sg_handle* h, int32_t* out) {
  SG_TRY(check_handle(h, false));
  if (!out) return fail(SG_ERR_ARG, "null output");
  SG_TRY(ensure_batch(h));
  const bool on = h->esz == 4 ? res_ready<float>(h) : res_ready<double>(h);
  out[0] = on ? 1 : 0;
  out[1] = on ? h->res_CL : 0;
  out[2] = on ? h->res_W : 0;
  out[3] = on ? h->res_threads : 0;
  out[4] = on ? h->res_clusters : 0;
  out[5] = on ? ResSmem<float>(true, h->res_SR, h->res_W, h->res_hrows, h->res_hboxes).bytes : 0;
  return SG_OK;
}

int sg_phase_times(sg_handle* h, float* ms) {
  if (!h || !ms) return fail(SG_ERR_ARG, "null argument");
  if (h->ph_batches == 0) return fail(SG_ERR_STATE, "no gradient has run on this handle");
  SG_CK(cudaSetDevice(h->d.device));
  for (int k = 0; k < 4; ++k) ms[k] = 0.f;
  for (int b = 0; b < h->ph_batches; ++b) {
    cudaEvent_t* ev = h->ph_ev.data() + 5 * b;
    SG_CK(cudaEventSynchronize(ev[4]));
    for (int k = 0; k < 4; ++k) {
      float t = 0.f;
      SG_CK(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
      ms[k] += t;
    }
  }
  return SG_OK;
}

int sg_time_step_kernel(sg_handle* h, int32_t which, int32_t count, int32_t reps, float* ms) {
  SG_TRY(check_handle(h));
  if (!ms || reps < 1 || count < 1) return fail(SG_ERR_ARG, "bad arguments");
  return SG_DISPATCH(h, time_kernel_t, h, which, count, reps, ms);
}

}  // extern "C"
