// sg_kernels.cuh -- sm_100a time-step kernel for the damped-leapfrog acoustic
// propagator of seisopt (seisopt/wavesim.py:259-346), re-designed for B200.
//
// Memory layout ("guarded plane", one per shot): rows -4 .. nzp+3 (4 zero
// guard rows top and bottom) with row pitch ldx >= nxp+4 (multiple of 32
// elements); buffers are [lead row][shot 0 plane][shot 1 plane]...[tail].
// Columns nxp..ldx-1 stay zero.  Field pointers point at row 0 col 0 of shot 0.
//
// One CTA owns a 64 x 32 tile for a GROUP of G shots.  The halo'd field tile
// (72 x 40) of each shot is brought into shared memory by TMA
// (cp.async.bulk.tensor.2d, out-of-bounds zero fill == the reference's
// zero-Dirichlet exterior, seisopt/wavesim.py:216-223), double-buffered so
// shot k+1 streams in while shot k computes.  Per-cell model data (1/m,
// sponge factor) stay in registers across the group; each thread owns 8
// consecutive rows of one column and keeps the vertical stencil window in
// registers (z-marching inside the tile), so a cell costs ~10 shared loads.
//
// Forward (FWD) and adjoint (ADJ) share the kernel shape:
//   FWD  a_n = inv_m (L u_n [+ g_n s]) [+ amp_n w_k inv_m at the source taps]
//        inc_{n+1} = d (inc_n + dt^2 a_n),   u_{n+1} = d u_n + inc_{n+1}
//        (reference: u_{n+1} = d (2 u_n - p_n + dt^2 a_n), p_{n+1} = d u_n,
//         with inc_n = u_n - p_n -- the increment form keeps fp32 accurate)
//   ADJ  state V_n = v_n = dt^2 inv_m d lam_{n+1} (seisopt/wavesim.py:331-333)
//        w_n = d w_{n+1} + L V_n + R^T y_n,   V_{n-1} = d V_n + (dt^2 inv_m d) w_n
//        image -= a_n V_n                       (seisopt/wavesim.py:342-343)
//        (reference lam_n = L v_n + 2 d lam_{n+1} + d pbar + R^T y with
//         w_n = lam_n - d lam_{n+1}; algebraically identical, exact transpose)
//   L is applied in difference form sum_k c_k ((u_{+k}-u) + (u_{-k}-u)),
//   identical to the reference stencil because c_0 = -2 sum_{k>0} c_k.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sg {

constexpr int kGuard = 4;         // zero guard rows above/below each plane
constexpr int kTileRowsMax = 64;  // tail padding covers tiles up to this height
constexpr int kBX = 64, kBY = 4, kNY = 8, kTH = kBY * kNY;  // 64 x 32 tile, 256 threads
// TMA halo boxes are always kHalo wide (the 8th-order radius); the 2nd-order
// stencil reads the inner ring only.  72 x 40 boxes keep every TMA row a
// multiple of 16 B for fp32 and fp64.
constexpr int kHalo = 4;
#ifndef SG_HINT_FIELD
#define SG_HINT_FIELD 0
#endif
#ifndef SG_HINT_HIST
#define SG_HINT_HIST 0
#endif
#ifndef SG_STCS
#define SG_STCS 0
#endif
#ifndef SG_STAGES
#define SG_STAGES 2
#endif
#ifndef SG_FP32_MINB
#define SG_FP32_MINB 3
#endif

template <typename T>
struct StepArgs {
  // TMA descriptors (3-D views {ldx, rows, planes}; see sg_prop.cu tmap_*)
  CUtensorMap f_halo[2];  // field buffers, box = halo'd tile (load)
  CUtensorMap f_tile[2];  // field buffers, box = tile (store)
  CUtensorMap s_tile;     // state buffer (inc / w, updated in place), box = tile
  CUtensorMap h_tile;     // history buffer {ldx, nzp, shots*steps}, box = tile
  T* f[2];                // field buffers (row 0, col 0, shot 0)
  T* state;               // inc (forward) / w (adjoint), updated in place
  int cur;                // read f[cur], write f[cur ^ 1]
  const T* inv_m;         // 1/m on the padded grid (single plane)
  const T* pz;            // sponge profile, rows
  const T* px;            // sponge profile, cols
  int64_t plane;          // per-shot stride of field/state buffers
  int nzp, nxp, ldx, tiles_x, ntiles;
  int count, G;           // shots in this launch, shots per CTA group
  T dt2;
  T cz[5], cx[5];         // stencil weights k = 1..R
  int hist_on;            // FWD: store history; ADJ: image against history
  int hist_steps, hist_slot;  // history plane of shot b at this step: b*hist_steps + slot
  T* hist;                // history base (plain stores of the forward)
  int64_t hplane;         // history plane stride nzp*ldx
  // ---- forward --------------------------------------------------------------
  const int* src_rc;      // (count, 4, 2) tap rows/cols; nullptr: no point source
  const T* src_w;         // (count, 4) weights * src_scale
  T amp;                  // wavelet[n]
  const T* gsrc;          // Born source a0_n (per-shot stride gsrc_stride)
  int64_t gsrc_stride;
  const T* gscale;        // -m_r on the padded grid
  const int* rec_ij;      // (4, nrec) flat offsets
  const T* rec_w;         // (4, nrec)
  int nrec, rec_blocks;   // receiver blocks per group
  T* gather;              // gathers at this step (+ b*gather_stride + r)
  int64_t gather_stride;
  // ---- adjoint --------------------------------------------------------------
  int inj_row0, inj_nrows;
  const int* inj_ptr;     // CSR over cells of the receiver row band
  const int* inj_rec;
  const T* inj_w;
  const T* ybar;          // adjoint data at this step (+ b*ybar_stride + r)
  int64_t ybar_stride;
  const T* inj_dense;     // R^T y of this step on the receiver row band
  int64_t inj_dense_stride;  // (+ b*stride + rr*nxp + j); nullptr: CSR walk
  T* image;               // per-group image planes (stride image_stride)
  int64_t image_stride;
  T* vhist;               // optional v history (adjoint_solve keep_v)
  int64_t vhist_stride;
};

// ---- PTX helpers -----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Programmatic dependent launch: let the next kernel in the stream start its
// prologue once every CTA of this grid is resident, and wait for the previous
// grid's completion (and memory) before touching data it produced or reads.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE_%=;\n"
      "bra.uni WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// L2 eviction-priority policies (the encodings CUTLASS uses for
// CacheHintSm90::EVICT_FIRST / EVICT_LAST)
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map,
                                                 uint64_t* bar, int x, int y, int z,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x,
                                             int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          map),
      "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- paired arithmetic: two cells per instruction -------------------------
// fp32 uses Blackwell's packed FADD2/FMUL2/FFMA2 (add/sub/mul/fma.rn.f32x2);
// fp64 falls back to two scalar ops.  Results are bitwise those of the scalar
// code (fma stays fused, rounding per op unchanged).
template <typename T>
struct V2;

template <>
struct V2<float> {
  unsigned long long v;
  __device__ __forceinline__ static V2 make(float a, float b) {
    V2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
  }
  __device__ __forceinline__ void split(float& a, float& b) const {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  }
  __device__ __forceinline__ friend V2 operator+(V2 a, V2 b) {
    V2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
  }
  __device__ __forceinline__ friend V2 operator-(V2 a, V2 b) {
    V2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
  }
  __device__ __forceinline__ friend V2 operator*(V2 a, V2 b) {
    V2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
  }
  __device__ __forceinline__ static V2 fma(V2 a, V2 b, V2 c) {
    V2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
  }
};

template <>
struct V2<double> {
  double x, y;
  __device__ __forceinline__ static V2 make(double a, double b) { return V2{a, b}; }
  __device__ __forceinline__ void split(double& a, double& b) const {
    a = x;
    b = y;
  }
  __device__ __forceinline__ friend V2 operator+(V2 a, V2 b) { return V2{a.x + b.x, a.y + b.y}; }
  __device__ __forceinline__ friend V2 operator-(V2 a, V2 b) { return V2{a.x - b.x, a.y - b.y}; }
  __device__ __forceinline__ friend V2 operator*(V2 a, V2 b) { return V2{a.x * b.x, a.y * b.y}; }
  __device__ __forceinline__ static V2 fma(V2 a, V2 b, V2 c) {
    return V2{__fma_rn(a.x, b.x, c.x), __fma_rn(a.y, b.y, c.y)};
  }
};

// shared-memory plan of one CTA (element counts; every region 128-B aligned):
// two stages of {halo'd field tile, state tile[, history tile (adjoint)]}
template <typename T, int R, bool ADJ>
struct Smem {
  static constexpr int SW = kBX + 2 * kHalo;
  static constexpr int SH = kTH + 2 * kHalo;
  static constexpr int A = 128 / (int)sizeof(T);  // elements per 128 B
  static constexpr int HALO = ((SW * SH + A - 1) / A) * A;
  static constexpr int TILE = kBX * kTH;           // multiple of 128 B
  static constexpr int STAGE = HALO + (ADJ ? 2 : 1) * TILE;
  static constexpr int BYTES = SG_STAGES * STAGE * (int)sizeof(T);
};

template <typename T, int R, bool ADJ>
__host__ __device__ constexpr int step_smem_bytes() {
  return Smem<T, R, ADJ>::BYTES;
}

// ----------------------------------------------------------------------------
// the step kernel
// ----------------------------------------------------------------------------
// FL_* feature flags (compile-time; dead paths vanish from the SASS)
constexpr int FL_HIST = 1;    // FWD: store a_n; ADJ: image against a_n
constexpr int FL_GSRC = 2;    // FWD: Born grid source a0_n * gscale
constexpr int FL_VHIST = 4;   // ADJ: store v_n (adjoint_solve keep_v)
constexpr int FL_GATHER = 8;  // FWD: receiver sampling blocks present

template <typename T, int R, bool ADJ, int FL>
__global__ void __launch_bounds__(kBX* kBY, sizeof(T) == 4 ? SG_FP32_MINB : 2)
    k_step(const __grid_constant__ StepArgs<T> a) {
  using SM = Smem<T, R, ADJ>;
  constexpr int SW = SM::SW;
  constexpr int NCOL = kNY + 2 * R;
  constexpr int HO = kHalo - R;  // offset of the radius-R window inside the halo box
  constexpr bool HIST = (FL & FL_HIST) != 0;
  constexpr bool GSRC = !ADJ && (FL & FL_GSRC) != 0;
  constexpr bool VHIST = ADJ && (FL & FL_VHIST) != 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sbase = reinterpret_cast<T*>(smem_raw);
  __shared__ __align__(8) uint64_t bar[SG_STAGES];
  constexpr int NS = SG_STAGES;

  const int tid = threadIdx.y * kBX + threadIdx.x;
  const int grp = blockIdx.y;
  const int b0 = grp * a.G;
  const int nb = min(a.G, a.count - b0);

  if constexpr (!ADJ && (FL & FL_GATHER) != 0) {
    if ((int)blockIdx.x >= a.ntiles) {
      pdl_wait();
      pdl_launch_dependents();
      // receiver sampling for this group's shots: gather[n, r] = sum_k w_k u_n[tap_k]
      // (seisopt/wavesim.py:225-226, sampled before the update, :287)
      const T* __restrict__ u = a.f[a.cur];
      const int total = nb * a.nrec;
      for (int e = ((int)blockIdx.x - a.ntiles) * (kBX * kBY) + tid; e < total;
           e += a.rec_blocks * (kBX * kBY)) {
        const int bb = b0 + e / a.nrec;
        const int r = e - (e / a.nrec) * a.nrec;
        const T* ub = u + (int64_t)bb * a.plane;
        T g = a.rec_w[r] * ub[a.rec_ij[r]];
#pragma unroll
        for (int k = 1; k < 4; ++k) g += a.rec_w[k * a.nrec + r] * ub[a.rec_ij[k * a.nrec + r]];
        a.gather[(int64_t)bb * a.gather_stride + r] = g;
      }
      return;
    }
  }

  const int tzi = blockIdx.x / a.tiles_x;
  const int txi = blockIdx.x - tzi * a.tiles_x;
  const int i0 = tzi * kTH;
  const int j0 = txi * kBX;
  constexpr bool LOAD_HIST = ADJ && HIST;

  // source taps of the group's shots, staged once (static data, PDL-safe)
  __shared__ int s_src[8 * 8];
  __shared__ T s_sw[8 * 4];
  if (!ADJ && a.src_rc != nullptr) {
    if (tid < nb * 8) s_src[tid] = a.src_rc[b0 * 8 + tid];
    if (tid < nb * 4) s_sw[tid] = a.src_w[b0 * 4 + tid];
  }

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int k) {
    const int s = k % NS;
    T* st = sbase + s * SM::STAGE;
    const int b = b0 + k;
    constexpr uint32_t bytes =
        (SM::SW * SM::SH + (LOAD_HIST ? 2 : 1) * SM::TILE) * (uint32_t)sizeof(T);
    mbar_expect_tx(&bar[s], bytes);
    // rows of a guarded plane: data row i lives at plane row kGuard + i
    // the working set (fields, state) is kept in L2; the history stream,
    // read once, is evicted first so it does not push the working set out
#if SG_HINT_FIELD
    tma_load_3d_hint(st, &a.f_halo[a.cur], &bar[s], j0 - kHalo, kGuard + i0 - kHalo, b,
                     kEvictLast);
    tma_load_3d_hint(st + SM::HALO, &a.s_tile, &bar[s], j0, kGuard + i0, b, kEvictLast);
#else
    tma_load_3d(st, &a.f_halo[a.cur], &bar[s], j0 - kHalo, kGuard + i0 - kHalo, b);
    tma_load_3d(st + SM::HALO, &a.s_tile, &bar[s], j0, kGuard + i0, b);
#endif
    if (LOAD_HIST) {
#if SG_HINT_HIST
      tma_load_3d_hint(st + SM::HALO + SM::TILE, &a.h_tile, &bar[s], j0, i0,
                       b * a.hist_steps + a.hist_slot, kEvictFirst);
#else
      tma_load_3d(st + SM::HALO + SM::TILE, &a.h_tile, &bar[s], j0, i0,
                  b * a.hist_steps + a.hist_slot);
#endif
    }
  };
  const int j = j0 + threadIdx.x;
  const bool vj = j < a.nxp;
  const int rb = threadIdx.y * kNY;  // first tile row owned by this thread
  const int ib = i0 + rb;
  const int nq = vj ? max(0, min(kNY, a.nzp - ib)) : 0;
  const int o0 = ib * a.ldx + j;     // offset of this thread's first cell
  const int ldx = a.ldx;

  // per-cell model data, reused for every shot of the group; the image
  // accumulator starts from the stored image (prefetched, lands during shot 0)
  T im[kNY], dd[kNY], img[kNY];
  const T pxj = vj ? a.px[j] : T(0);
  // Prologue (may overlap the previous step under PDL): model data and the
  // image accumulator of this launch's parity, last written two launches ago
  // (complete: the previous grid signalled its dependents only after its own
  // griddepcontrol.wait).
  T* ig = nullptr;
  if (LOAD_HIST) ig = a.image + (int64_t)grp * a.image_stride + o0;
#pragma unroll
  for (int q = 0; q < kNY; ++q) {
    if (q < nq) {
      im[q] = a.inv_m[o0 + q * ldx];
      dd[q] = a.pz[ib + q] * pxj;
      img[q] = LOAD_HIST ? ig[q * ldx] : T(0);
    } else {
      im[q] = T(0);
      dd[q] = T(0);
      img[q] = T(0);
    }
  }
  // everything below reads or writes fields/states of the previous step
  pdl_wait();
  pdl_launch_dependents();
  if (tid == 0)
    for (int k = 0; k < NS - 1 && k < nb; ++k) issue(k);

  for (int k = 0; k < nb; ++k) {
    const int b = b0 + k;
    if (tid == 0 && k + NS - 1 < nb) issue(k + NS - 1);

    // does this tile hold a source tap of shot b?  (CTA-uniform)
    bool src_here = false;
    if (!ADJ && a.src_rc != nullptr) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int r = s_src[(k * 4 + t) * 2], c = s_src[(k * 4 + t) * 2 + 1];
        src_here |= (r >= i0 && r < i0 + kTH && c >= j0 && c < j0 + kBX);
      }
    }
    // receiver injection rows inside this tile?  (CTA-uniform)
    const bool inj_here = ADJ && a.ybar != nullptr && a.inj_row0 < i0 + kTH &&
                          a.inj_row0 + a.inj_nrows > i0;
    const int64_t sb = (int64_t)b * a.plane;
    T* __restrict__ fout = a.f[a.cur ^ 1] + sb + o0;
    T* __restrict__ sout = a.state + sb + o0;
    T* __restrict__ hout = nullptr;
    if (!ADJ && HIST) hout = a.hist + ((int64_t)b * a.hist_steps + a.hist_slot) * a.hplane + o0;
    const T* __restrict__ gin = nullptr;
    if (GSRC) gin = a.gsrc + (int64_t)b * a.gsrc_stride + o0;

    mbar_wait(&bar[k % NS], (k / NS) & 1);
    const T* st = sbase + (k % NS) * SM::STAGE;
    // this thread's column, from tile row rb - R
    const T* sc = st + (rb + HO) * SW + threadIdx.x + kHalo;
    const T* sst = st + SM::HALO + rb * kBX + threadIdx.x;

    if (nq > 0) {
      using P = V2<T>;
      constexpr int NH = kNY / 2;  // cells q and q + NH form one pair
      T col[NCOL];
#pragma unroll
      for (int r = 0; r < NCOL; ++r) col[r] = sc[r * SW];
#pragma unroll
      for (int q = 0; q < NH; ++q) {
        // Laplacian of cells (q, q + NH) in difference form, two per instruction
        const P uc = P::make(col[q + R], col[q + NH + R]);
        const T* ra = sc + (q + R) * SW;
        const T* rbw = sc + (q + NH + R) * SW;
        P lz = P::make(T(0), T(0)), lx = P::make(T(0), T(0));
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const P cz = P::make(a.cz[kk], a.cz[kk]);
          const P cx = P::make(a.cx[kk], a.cx[kk]);
          const P zm = P::make(col[q + R - kk], col[q + NH + R - kk]);
          const P zp = P::make(col[q + R + kk], col[q + NH + R + kk]);
          const P xm = P::make(ra[-kk], rbw[-kk]);
          const P xp = P::make(ra[kk], rbw[kk]);
          lz = P::fma(cz, (zm - uc) + (zp - uc), lz);
          lx = P::fma(cx, (xm - uc) + (xp - uc), lx);
        }
        T lap[2], ucs[2];
        (lz + lx).split(lap[0], lap[1]);
        uc.split(ucs[0], ucs[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int qq = q + h * NH;
          if (qq >= nq) continue;
          const T sv = sst[qq * kBX];
          T lp = lap[h];
          if (!ADJ) {
            if (GSRC) lp += gin[qq * ldx] * a.gscale[o0 + qq * ldx];
            T acc = lp * im[qq];
            if (src_here) {
              const int i = ib + qq;
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int r = s_src[(k * 4 + t) * 2], c = s_src[(k * 4 + t) * 2 + 1];
                if (r == i && c == j) acc += a.amp * s_sw[k * 4 + t] * im[qq];
              }
            }
  #if SG_STCS
          if (HIST) __stcs(hout + qq * ldx, acc);  // streaming store: evict first
#else
          if (HIST) hout[qq * ldx] = acc;
#endif
            const T so = dd[qq] * (sv + a.dt2 * acc);
            sout[qq * ldx] = so;
            fout[qq * ldx] = dd[qq] * ucs[h] + so;
          } else {
            if (inj_here) {
              const int rr = ib + qq - a.inj_row0;
              if (rr >= 0 && rr < a.inj_nrows) {
                // R^T y: duplicate taps accumulate (np.add.at, seisopt/wavesim.py:229)
                const int cell = rr * a.nxp + j;
                if (a.inj_dense != nullptr) {
                  lp += a.inj_dense[(int64_t)b * a.inj_dense_stride + cell];
                } else {
                  const int p1 = a.inj_ptr[cell + 1];
                  for (int p = a.inj_ptr[cell]; p < p1; ++p)
                    lp += a.inj_w[p] * a.ybar[(int64_t)b * a.ybar_stride + a.inj_rec[p]];
                }
              }
            }
            const T so = dd[qq] * sv + lp;
            sout[qq * ldx] = so;
            fout[qq * ldx] = dd[qq] * ucs[h] + (a.dt2 * im[qq] * dd[qq]) * so;
            if (LOAD_HIST) img[qq] -= sst[qq * kBX + SM::TILE] * ucs[h];
            if (VHIST) a.vhist[(int64_t)b * a.vhist_stride + o0 + qq * ldx] = ucs[h];
          }
        }
      }
    }
    __syncthreads();  // stage (k % NS) is free for shot k + NS
  }
  if (LOAD_HIST) {
#pragma unroll
    for (int q = 0; q < kNY; ++q)
      if (q < nq) ig[q * ldx] = img[q];
  }
}

}  // namespace sg
