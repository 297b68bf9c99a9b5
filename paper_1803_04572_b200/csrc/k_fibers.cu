// k_fibers.cu — the two streaming passes over the projected fibers X'_k (smooth path), FP64 on
// the tensor cores (mma.sync m8n8k4 f64 = SASS DMMA; 36.9 TFLOP/s measured).
//
// Fiber (k, j): the l-vector x'_kj = X'_k(:, j) = C_k^T X_k(:, j). Fibers of a patient are
// contiguous and sorted by the RELABELED feature id j' = perm[j]: features are dealt round-robin
// by fiber mass into G x W equal-size label ranges, so every range carries about the same work.
//
// Pass A  P'_k = X'_k V(cols_k, :)  (m_k x R) — warp per patient, dynamic scheduling over patients
//         sorted by fiber count, V staged (relabeled) in shared memory, fiber loads software-
//         pipelined one 8-fiber tile ahead across patient boundaries.
//         MMA per 4 fibers: M = basis index a (8/tile), N = r (8/tile), K = fibers.
// Pass B  F_V(j, :) += x'_kj^T N_k  (J x R) — CTA (range p, group g) owns the F_V rows of label group
//         g in shared memory for patient range p; warp w owns label sub-range (g, w) so no two warps
//         ever update the same row (no atomics). N_k of 32-patient chunks is staged into shared
//         memory with cp.async (double buffer), the chunk metadata one chunk further ahead, so
//         each warp prefetches its next fiber tile across patient and chunk boundaries.
//         MMA per 8 fibers: M = fibers, N = r (8/tile), K = a (4/step). Per-CTA F_V partials are
//         summed in a fixed order (deterministic) and un-relabeled.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>

#include "copa_internal.cuh"

namespace copa {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// ------------------------------------------------------------------ pass A
template <int MT>
struct TileA {  // one k-step pair (8 fibers) of pass A: lane's fiber f = fb + 4 s + t
  double a[2][MT];
  int32_t col[2];
};

template <int MT>
__device__ __forceinline__ void load_tile_a(TileA<MT>& T, int64_t fb, int64_t f1, int l, const int32_t* fiber_col,
                                            const double* fiber_val) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int64_t f = fb + 4 * s + t;
    const bool ok = f < f1;
    T.col[s] = ok ? fiber_col[f] : -1;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = mt * 8 + g;
      T.a[s][mt] = (ok && a < l) ? fiber_val[f * l + a] : 0.0;
    }
  }
}

template <int MT, int NT, bool VSMEM>
__global__ void __launch_bounds__(512) k_spmm_mma(const int64_t* __restrict__ fiber_ptr,
                                                  const int32_t* __restrict__ fiber_col,
                                                  const double* __restrict__ fiber_val, const int32_t* __restrict__ m,
                                                  const int32_t* __restrict__ order, const int32_t* __restrict__ inv,
                                                  int64_t K, int l, int R, int64_t Jl, const double* __restrict__ Vg,
                                                  double* __restrict__ Pp, int* counter) {
  extern __shared__ double smem_v[];
  if (VSMEM) {
    for (int64_t x = threadIdx.x; x < Jl * R; x += blockDim.x) {
      const int64_t nj = x / R, r = x - nj * R;
      const int32_t j = inv[nj];
      smem_v[x] = j >= 0 ? Vg[(int64_t)j * R + r] : 0.0;
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  // current patient and the one grabbed ahead
  int idx = 0;
  if (lane == 0) idx = atomicAdd(counter, 1);
  idx = __shfl_sync(0xffffffffu, idx, 0);
  int64_t k = idx < K ? order[idx] : -1;
  int64_t f0 = k >= 0 ? fiber_ptr[k] : 0, f1 = k >= 0 ? fiber_ptr[k + 1] : 0;
  TileA<MT> cur;
  if (k >= 0) load_tile_a<MT>(cur, f0, f1, l, fiber_col, fiber_val);
  while (k >= 0) {
    int nidx = 0;
    if (lane == 0) nidx = atomicAdd(counter, 1);
    nidx = __shfl_sync(0xffffffffu, nidx, 0);
    const int64_t kn = nidx < K ? order[nidx] : -1;
    const int64_t g0 = kn >= 0 ? fiber_ptr[kn] : 0, g1 = kn >= 0 ? fiber_ptr[kn + 1] : 0;
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    if (f0 >= f1 && kn >= 0) load_tile_a<MT>(cur, g0, g1, l, fiber_col, fiber_val);
    for (int64_t fb = f0; fb < f1; fb += 8) {
      // prefetch the next tile (this patient's or the next patient's first)
      TileA<MT> nxt;
      if (fb + 8 < f1) load_tile_a<MT>(nxt, fb + 8, f1, l, fiber_col, fiber_val);
      else if (kn >= 0) load_tile_a<MT>(nxt, g0, g1, l, fiber_col, fiber_val);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double bfr[NT];
        const int64_t j = cur.col[s];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int r = nt * 8 + g;
          bfr[nt] = (j >= 0 && r < R) ? (VSMEM ? smem_v[j * R + r] : Vg[(int64_t)inv[j] * R + r]) : 0.0;
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], cur.a[s][mt], bfr[nt]);
      }
      cur = nxt;
    }
    const int mk = m[k];
    double* out = Pp + k * l * R;  // smooth state rows: srow[k] = k * l
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = mt * 8 + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = nt * 8 + 2 * t + i;
          if (a < mk && r < R) out[a * R + r] = acc[mt][nt][i];
        }
    }
    k = kn;
    f0 = g0;
    f1 = g1;
  }
}

template <int MT, int NT, bool VS>
static void spmm_inst(Handle& h, int smem_bytes) {
  auto fn = k_spmm_mma<MT, NT, VS>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, smem_bytes);
  if (per_sm < 1) per_sm = 1;
  cudaMemsetAsync(h.counter, 0, sizeof(int), h.stream);
  fn<<<148 * per_sm, 512, smem_bytes, h.stream>>>(h.fiber_ptr, h.fiber_col, h.fiber_val, h.m, h.order, h.inv, h.K,
                                                   h.l, h.R, h.Jl, h.V, h.Pp, h.counter);
}

template <int MT, int NT>
static void spmm_dispatch_v(Handle& h) {
  size_t vbytes = sizeof(double) * (size_t)(h.Jl * h.R);
  if (vbytes <= 200 * 1024) spmm_inst<MT, NT, true>(h, (int)vbytes);
  else spmm_inst<MT, NT, false>(h, 0);
}

template <int MT>
static void spmm_dispatch_n(Handle& h) {
  switch ((h.R + 7) / 8) {
    case 1: spmm_dispatch_v<MT, 1>(h); break;
    case 2: spmm_dispatch_v<MT, 2>(h); break;
    case 3: spmm_dispatch_v<MT, 3>(h); break;
    case 4: spmm_dispatch_v<MT, 4>(h); break;
    case 5: spmm_dispatch_v<MT, 5>(h); break;
    case 6: spmm_dispatch_v<MT, 6>(h); break;
    case 7: spmm_dispatch_v<MT, 7>(h); break;
    default: spmm_dispatch_v<MT, 8>(h); break;
  }
}

void launch_spmm_fibers(Handle& h) {
  if (h.l <= 8) spmm_dispatch_n<1>(h);
  else spmm_dispatch_n<2>(h);
}

// ------------------------------------------------------------------ pass B
constexpr int kScW = 8;        // warps per scatter CTA = label sub-ranges per group
constexpr int kWoffStride = 16;  // uint16 entries per (group, patient) row of woff (>= kScW + 1)

struct MetaB {  // per chunk, in shared memory
  int64_t f0[64];
  int32_t m[64];
  uint16_t wo[64][kWoffStride];
};

template <int KS>
struct TileB {
  double a[KS];
  int32_t col;   // label of the lane's fiber (-1: none)
  int p;         // visit (patient index within its chunk), -1 = end
  int chunk;     // chunk index (relative) of the visit: 0 = current, 1 = next
  int64_t fb, fz;
};

template <int KS, int NT>
__global__ void __launch_bounds__(32 * kScW) k_scatter_grp(
    const int64_t* __restrict__ fiber_ptr, const int32_t* __restrict__ fiber_col,
    const double* __restrict__ fiber_val, const int32_t* __restrict__ m, const uint16_t* __restrict__ woff,
    const int64_t* __restrict__ range_k, int G, int64_t Jg, int l, int R, int RS, int CH,
    const double* __restrict__ Nst, double* __restrict__ FVpart) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int grp = blockIdx.x % G;
  const int64_t rng = blockIdx.x / G;
  const int64_t k0 = range_k[rng], k1 = range_k[rng + 1];
  const int64_t jbase = grp * Jg;
  double* Fs = sm;                                       // Jg x RS
  double* Nb = sm + Jg * RS;                             // [2][CH * l * R]
  MetaB* mb = (MetaB*)(Nb + 2 * (int64_t)CH * l * R);    // [3]
  const int64_t per = (int64_t)l * R;
  for (int64_t x = threadIdx.x; x < Jg * RS; x += blockDim.x) Fs[x] = 0.0;
  const int64_t nch = (k1 - k0 + CH - 1) / CH;
  auto stage_meta = [&](int64_t c) {
    MetaB& M = mb[c % 3];
    const int64_t kc = k0 + c * CH;
    for (int i = threadIdx.x; i < CH; i += blockDim.x) {
      const int64_t k = kc + i;
      if (k < k1) {
        cp_async8(&M.f0[i], fiber_ptr + k);
        cp_async16(&M.wo[i][0], woff + (k * G + grp) * kWoffStride);
        cp_async16(&M.wo[i][8], woff + (k * G + grp) * kWoffStride + 8);
      }
    }
    for (int i = threadIdx.x; i < CH; i += blockDim.x) {
      const int64_t k = kc + i;
      if (k < k1) {
        // m as 4-byte copies (8-byte aligned pairs are not guaranteed)
        unsigned s = (unsigned)__cvta_generic_to_shared(&M.m[i]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(m + k));
      }
    }
  };
  auto stage_n = [&](int64_t c) {
    double* dst = Nb + (c & 1) * (int64_t)CH * per;
    const int64_t kc = k0 + c * CH;
    const int64_t np = (kc + CH < k1 ? CH : k1 - kc) * per;
    const double* src = Nst + kc * per;
    for (int64_t x = threadIdx.x; x < np; x += blockDim.x) cp_async8(dst + x, src + x);
  };
  // prologue: group 0 = meta(0), group 1 = [N(0), meta(1)]
  if (nch > 0) stage_meta(0);
  cp_async_commit();
  if (nch > 0) stage_n(0);
  if (nch > 1) stage_meta(1);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // the warp's tile iterator over (chunk, visit, tile)
  auto first_visit = [&](int64_t c, int p_start, TileB<KS>& T) {
    // find the first visit p >= p_start of chunk c with a non-empty range; T.p = -1 if none
    const MetaB& M = mb[c % 3];
    const int64_t kc = k0 + c * CH;
    const int np = (int)(kc + CH < k1 ? CH : k1 - kc);
    for (int p = p_start; p < np; ++p) {
      const int64_t fa = M.f0[p] + M.wo[p][w], fz = M.f0[p] + M.wo[p][w + 1];
      if (fa < fz) { T.p = p; T.fb = fa; T.fz = fz; return; }
    }
    T.p = -1;
  };
  auto load_b = [&](TileB<KS>& T) {
    const int64_t f = T.fb + g;
    const bool ok = f < T.fz;
    T.col = ok ? fiber_col[f] : -1;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int a = 4 * ks + t;
      T.a[ks] = (ok && a < l) ? fiber_val[f * l + a] : 0.0;
    }
  };
  // next tile after T (same visit, later visit of the same chunk, or first visit of chunk c+1)
  auto advance = [&](const TileB<KS>& T, int64_t c, TileB<KS>& N) {
    if (T.fb + 8 < T.fz) { N = T; N.fb = T.fb + 8; load_b(N); return; }
    int64_t cc = c + T.chunk;
    first_visit(cc, T.p + 1, N);
    N.chunk = T.chunk;
    if (N.p < 0 && T.chunk == 0 && cc + 1 < nch) {
      first_visit(cc + 1, 0, N);
      N.chunk = 1;
    }
    if (N.p >= 0) load_b(N);
  };

  TileB<KS> cur;
  cur.p = -1;
  cur.chunk = 0;
  for (int64_t c = 0; c < nch; ++c) {
    // stage N(c+1) and meta(c+2); wait for N(c)/meta(c+1) (committed one group earlier)
    if (c + 1 < nch) stage_n(c + 1);
    if (c + 2 < nch) stage_meta(c + 2);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (cur.p < 0) {  // iterator ran dry (no prefetched tile): restart in this chunk
      first_visit(c, 0, cur);
      cur.chunk = 0;
      if (cur.p >= 0) load_b(cur);
    }
    const double* Nc = Nb + (c & 1) * (int64_t)CH * per;
    int curp = -1;
    double bfr[KS][NT];
    // process tiles belonging to chunk c (cur.chunk == 0)
    while (cur.p >= 0 && cur.chunk == 0) {
      if (cur.p != curp) {  // B fragments of the visit: B[t][g] = N(a = 4 ks + t, r = 8 nt + g)
        curp = cur.p;
        const MetaB& M = mb[c % 3];
        const int mp = M.m[cur.p];
        const double* Np = Nc + (int64_t)cur.p * per;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int a = 4 * ks + t, r = 8 * nt + g;
            bfr[ks][nt] = (a < mp && r < R) ? Np[a * R + r] : 0.0;
          }
      }
      TileB<KS> nxt;
      advance(cur, c, nxt);
      double cc[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        cc[nt][0] = cc[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma(cc[nt][0], cc[nt][1], cur.a[ks], bfr[ks][nt]);
      }
      if (cur.col >= 0) {
        double* row = Fs + (cur.col - jbase) * RS;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int r = 8 * nt + 2 * t;
          if (r < RS) {
            double2 v = *reinterpret_cast<double2*>(row + r);
            v.x += cc[nt][0];
            v.y += cc[nt][1];
            *reinterpret_cast<double2*>(row + r) = v;
          }
        }
      }
      cur = nxt;
    }
    // tiles of chunk c+1 already prefetched keep chunk = 1 -> becomes the current chunk
    if (cur.p >= 0) cur.chunk = 0;
    __syncthreads();  // everyone done with N(c) and meta(c) before they are overwritten
  }
  cp_async_wait<0>();
  __syncthreads();
  double* out = FVpart + rng * (G * Jg) * (int64_t)R + jbase * R;
  for (int64_t x = threadIdx.x; x < Jg * R; x += blockDim.x) {
    const int64_t jj = x / R, r = x - jj * R;
    out[x] = Fs[jj * RS + r];
  }
}

// FV[inv[j']] = sum over ranges of part[range][j'] (fixed order), for every used label j'
__global__ void k_sum_ranges(const double* __restrict__ part, int nr, int64_t Jl, int R,
                             const int32_t* __restrict__ inv, double* __restrict__ FV) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= Jl * R) return;
  const int64_t nj = x / R, r = x - nj * R;
  const int32_t j = inv[nj];
  if (j < 0) return;
  double s = 0.0;
  for (int b = 0; b < nr; ++b) s += part[(int64_t)b * Jl * R + x];
  FV[(int64_t)j * R + r] = s;
}

size_t scatter_smem_bytes(const Handle& h) {
  return sizeof(double) * (size_t)(h.sc_Jg * h.sc_RS + 2 * (int64_t)h.sc_CH * h.l * h.R) + 3 * sizeof(MetaB);
}

template <int KS, int NT>
static void scatter_inst(Handle& h) {
  auto fn = k_scatter_grp<KS, NT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const size_t smem = scatter_smem_bytes(h);
  const int nr = h.sc_ranges;
  fn<<<nr * h.sc_G, 32 * kScW, smem, h.stream>>>(h.fiber_ptr, h.fiber_col, h.fiber_val, h.m, h.woff, h.block_k,
                                                   h.sc_G, h.sc_Jg, h.l, h.R, h.sc_RS, h.sc_CH, h.Nst, h.fv_part);
  int64_t n = h.Jl * h.R;
  k_sum_ranges<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.fv_part, nr, h.Jl, h.R, h.inv, h.FV);
}

template <int KS>
static void scatter_dispatch_n(Handle& h) {
  switch ((h.R + 7) / 8) {
    case 1: scatter_inst<KS, 1>(h); break;
    case 2: scatter_inst<KS, 2>(h); break;
    case 3: scatter_inst<KS, 3>(h); break;
    case 4: scatter_inst<KS, 4>(h); break;
    case 5: scatter_inst<KS, 5>(h); break;
    case 6: scatter_inst<KS, 6>(h); break;
    case 7: scatter_inst<KS, 7>(h); break;
    default: scatter_inst<KS, 8>(h); break;
  }
}

int launch_scatter_fibers(Handle& h) {
  switch ((h.l + 3) / 4) {
    case 1: scatter_dispatch_n<1>(h); break;
    case 2: scatter_dispatch_n<2>(h); break;
    case 3: scatter_dispatch_n<3>(h); break;
    default: scatter_dispatch_n<4>(h); break;
  }
  return 2;
}

// Chooses G (label groups), chunk size and label ranges so that a scatter CTA fits in shared memory.
void plan_scatter(Handle& h) {
  const size_t budget = 220 * 1024;
  h.sc_RS = (h.R + 1) & ~1;
  h.sc_ok = 0;
  for (int G = 1; G <= 8 && !h.sc_ok; ++G) {
    const int64_t Js = (h.J + (int64_t)G * kScW - 1) / ((int64_t)G * kScW);
    const int64_t Jg = Js * kScW;
    for (int CH = 64; CH >= 8; CH /= 2) {
      size_t bytes = sizeof(double) * (size_t)(Jg * h.sc_RS + 2 * (int64_t)CH * h.l * h.R) + 3 * sizeof(MetaB);
      if (bytes <= budget) {
        h.sc_G = G;
        h.sc_Js = Js;
        h.sc_Jg = Jg;
        h.sc_CH = CH;
        h.sc_ok = 1;
        break;
      }
    }
  }
  if (!h.sc_ok) {  // fall back: one label range per group of 1 (atomic scatter path handles it)
    h.sc_G = 1;
    h.sc_Js = (h.J + kScW - 1) / kScW;
    h.sc_Jg = h.sc_Js * kScW;
    h.sc_CH = 8;
  }
  h.Jl = (int64_t)h.sc_G * h.sc_Jg;
  int64_t ranges = (148 + h.sc_G - 1) / h.sc_G;
  if (ranges > h.K) ranges = h.K > 0 ? h.K : 1;
  h.sc_ranges = (int)ranges;
}

bool scatter_smem_ok(const Handle& h) { return h.sc_ok != 0; }

// ------------------------------------------------------------------ init-time layout for the passes
__global__ void k_fiber_counts(const int64_t* fiber_ptr, int64_t K, int32_t* cnt, int32_t* idx) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  cnt[k] = (int32_t)(fiber_ptr[k + 1] - fiber_ptr[k]);
  idx[k] = (int32_t)k;
}

// woff[(k G + grp) 16 + w] = lower_bound(label (grp W + w) * Js) within the patient's sorted labels
__global__ void k_warp_offsets(const int64_t* fiber_ptr, const int32_t* fiber_col, int64_t K, int G, int64_t Js,
                               uint16_t* woff) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int per = G * (kScW + 1);
  if (x >= K * per) return;
  int64_t k = x / per;
  int rem = (int)(x - k * per);
  int grp = rem / (kScW + 1), w = rem - grp * (kScW + 1);
  int64_t f0 = fiber_ptr[k], f1 = fiber_ptr[k + 1];
  int64_t key = ((int64_t)grp * kScW + w) * Js;
  int64_t lo = f0, hi = f1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (fiber_col[mid] < key) lo = mid + 1; else hi = mid;
  }
  woff[(k * G + grp) * kWoffStride + w] = (uint16_t)(lo - f0);
}

// range_k[b] = first patient whose fiber start >= b F / nb (balanced patient ranges)
__global__ void k_block_ranges(const int64_t* fiber_ptr, int64_t K, int nb, int64_t* block_k) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) { block_k[nb] = K; return; }
  int64_t F = fiber_ptr[K];
  int64_t target = (F * b) / nb;
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (fiber_ptr[mid] < target) lo = mid + 1; else hi = mid;
  }
  block_k[b] = lo;
}

size_t fiber_layout_temp_bytes(int64_t K) {
  size_t a = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                            (int32_t*)nullptr, (int)K);
  return a + 256;
}

// Feature relabeling from the per-feature fiber counts: features sorted by count (descending,
// ties by id) are dealt round-robin over the G*W label ranges of Js labels each; perm[j] = new label,
// inv[new] = j. Host-side (J <= 65535).
void compute_relabel(int64_t J, int ranges, const unsigned long long* hist, int32_t* perm, int32_t* inv, int64_t* Js) {
  std::vector<int32_t> idx((size_t)J);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return hist[a] > hist[b]; });
  const int64_t js = (J + ranges - 1) / ranges;
  std::vector<int64_t> fill((size_t)ranges, 0);
  int64_t total = (int64_t)ranges * js;
  for (int64_t x = 0; x < total; ++x) inv[x] = -1;
  for (int64_t i = 0; i < J; ++i) {
    // serpentine deal keeps the range masses close
    int64_t round = i / ranges, pos = i % ranges;
    int64_t rr = (round & 1) ? ranges - 1 - pos : pos;
    int64_t label = rr * js + fill[(size_t)rr]++;
    perm[idx[(size_t)i]] = (int32_t)label;
    inv[label] = idx[(size_t)i];
  }
  *Js = js;
}

// Builds order (pass A), woff / range_k (pass B). tmp: >= fiber_layout_temp_bytes(K) + 12 K bytes.
void build_fiber_layout(Handle& h, void* tmp, size_t tmp_bytes) {
  cudaStream_t s = h.stream;
  char* p = (char*)tmp;
  auto take = [&](size_t n) { char* r = p; p += (n + 255) & ~(size_t)255; return (void*)r; };
  int32_t* cnt = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  int32_t* cnt_sorted = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  int32_t* idx = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  size_t sort_bytes = fiber_layout_temp_bytes(h.K);
  void* sort_tmp = take(sort_bytes);
  if (h.K > 0) {
    k_fiber_counts<<<(unsigned)((h.K + 255) / 256), 256, 0, s>>>(h.fiber_ptr, h.K, cnt, idx);
    cub::DeviceRadixSort::SortPairsDescending(sort_tmp, sort_bytes, cnt, cnt_sorted, idx, h.order, (int)h.K, 0, 32, s);
    int64_t n = h.K * h.sc_G * (kScW + 1);
    k_warp_offsets<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.fiber_ptr, h.fiber_col, h.K, h.sc_G, h.sc_Js,
                                                               h.woff);
  }
  k_block_ranges<<<(h.sc_ranges + 1 + 255) / 256, 256, 0, s>>>(h.fiber_ptr, h.K, h.sc_ranges, h.block_k);
}

}  // namespace copa
