// k_fibers.cu — the two streaming passes over the projected fibers X'_k (smooth path), FP64 on
// the tensor cores (mma.sync m8n8k4 f64 = SASS DMMA; 36.9 TFLOP/s measured).
//
// Fiber (k, j): the l-vector x'_kj = X'_k(:, j) = C_k^T X_k(:, j).
//
// g-stream layout. Features are relabeled by fiber mass and dealt into G x W equal-mass label
// sub-ranges of Js labels each; label group g = sub-ranges [g W, (g+1) W) = labels [g Jg, (g+1) Jg).
// Stream g holds, patient after patient, the fibers of that patient whose label is in group g,
// sorted by label: patient k's run in stream g is [gptr[g][k], gptr[g][k+1]). Within a run, the
// fibers of sub-range (g, w) are a contiguous sub-run.
//
// Pass A  P'_k = X'_k V(cols_k, :)  (m_k x R) — warp per patient (dynamic scheduling over patients
//         sorted by fiber count), the patient's G runs one after the other, fiber tiles loaded one
//         tile ahead, the next patient's runs bulk-prefetched into L2 (cp.async.bulk.prefetch.L2).
//         MMA per 4 fibers: M = basis index a (8/tile), N = r (8/tile), K = fibers.
// Pass B  F_V(j, :) += x'_kj^T N_k  (J x R) — CTA = (patient range, label group g) owns the F_V rows
//         of group g in shared memory. One producer warp streams the range's run of stream g in
//         stages (<= FB fibers, <= PB patients) into an NS-deep shared-memory ring with 1-D TMA bulk
//         copies (cp.async.bulk + mbarrier complete_tx): fiber labels, fiber values and the N_k rows
//         of the stage's patients. W consumer warps: warp w owns label sub-range (g, w), so no two
//         warps ever update the same F_V row (no atomics); it finds its sub-run of every patient of
//         the stage with two warp ballots and runs MMA tiles of 8 fibers: M = fibers, N = r (8/tile),
//         K = a (4/step). Per-CTA F_V partials are summed in a fixed order (deterministic) and
//         un-relabeled.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <numeric>
#include <type_traits>

#include "copa_internal.cuh"

namespace copa {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Bulk-prefetch [p, p + bytes) into L2 (16-byte aligned outward).
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
  const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15;
  const uintptr_t e = ((uintptr_t)p + bytes + 15) & ~(uintptr_t)15;
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// ------------------------------------------------------------------ mbarrier / bulk-copy helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
      "DONE%=:\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// try_wait with a suspend-time hint: the thread is parked until the phase completes (or the hint
// expires), without issuing instructions in between.
__device__ __forceinline__ void mbar_wait_park(uint64_t* b, uint32_t parity, uint32_t hint_ns) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
      "DONE%=:\n}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(hint_ns)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// Copy [src, src + bytes) with a 16-byte aligned bulk copy that starts at or before src; returns
// the byte offset of src inside dst. dst must have 16 bytes of slack.
__device__ __forceinline__ uint32_t bulk_g2s_span(void* dst, const void* src, size_t bytes, uint64_t* bar,
                                                  uint32_t* tx) {
  const uintptr_t a = (uintptr_t)src & ~(uintptr_t)15;
  const uint32_t shift = (uint32_t)((uintptr_t)src - a);
  const uint32_t nb = (uint32_t)((shift + bytes + 15) & ~(size_t)15);
  if (nb) bulk_g2s(dst, (const void*)a, nb, bar);
  *tx += nb;
  return shift;
}

// ------------------------------------------------------------------ V̄ in label order
// (pass A, k_passA.cu, gathers V̄ rows by fiber label)
__global__ void k_relabel_V(const double* V, const int32_t* inv, int64_t Jl, int R, double* Vl) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= Jl * R) return;
  const int64_t nj = x / R, r = x - nj * R;
  const int32_t j = inv[nj];
  Vl[x] = j >= 0 ? V[(int64_t)j * R + r] : 0.0;
}

void launch_relabel_V(Handle& h) {
  const int64_t n = h.Jl * h.R;
  k_relabel_V<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.V, h.inv, h.Jl, h.R, h.Vl);
}

// ------------------------------------------------------------------ pass B (TMA-staged scatter)
// Stage slot layout (bytes, each part 16-byte aligned):
//   meta  : int32 npat, shift_lh, shift_col, shift_val, shift_n (32)
//   lh    : uint32 [PB][W] + 16  sub-run bounds lo | hi << 16 of every (patient, sub-range), relative
//           to the stage's first fiber (st_tab, built at init; bulk copy, shifted)
//   col   : int32 [FB] + 16  F_V row byte offsets (bulk copy, shifted)
//   val   : f64 [FB l] + 16   fiber values     (bulk copy, shifted)
//   nrows : f64 [PB l R] + 16 N_k rows         (bulk copy, shifted)
struct SlotGeom {
  uint32_t lh, col, val, nrows, bytes;
};
__host__ __device__ inline uint32_t al16(uint64_t x) { return (uint32_t)((x + 15) & ~(uint64_t)15); }
__host__ __device__ inline SlotGeom slot_geom(int FB, int PB, int W, int l, int R) {
  SlotGeom s;
  s.lh = 32;
  s.col = s.lh + al16(4ull * W * PB + 16);
  s.val = s.col + al16(4ull * FB + 16);
  s.nrows = s.val + al16(8ull * FB * l + 16);
  s.bytes = (s.nrows + al16(8ull * PB * l * R + 16) + 127) & ~127u;
  return s;
}

constexpr int kScW = 4;          // pass-B consumer warps per CTA (label sub-ranges per group)
constexpr int kScrD = 128;       // per-sub-range scratch doubles behind the F_V slice (redirected row updates)

// Shared-memory accesses by 32-bit shared addresses: the consumers hold their base addresses in
// registers (with generic pointers the compiler re-derived the shared window, S2UR + ULEA, per tile).
// All are volatile: they keep program order among themselves (F_V read-modify-writes of one lane).
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_s32_if(uint32_t a, bool p, int dflt) {
  int v = dflt;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.b32 %0, [%1];\n}" : "+r"(v) : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ double lds_f64_if(uint32_t a, bool p) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}" : "+d"(v) : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ double2 lds_v2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_v2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
      "DONE%=:\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// W label sub-ranges per group, CS consumer warps per sub-range: warp (w, c) owns the F_V rows of
// sub-range w, columns [8 NT/CS c, 8 NT/CS (c + 1)) — disjoint words, no atomics. Per stage it reads
// its sub-run bounds of every patient from the staged lh table, then runs 8-fiber MMA tiles
// (M = fibers, N = r, K = a) with one tile in flight: the next tile's loads and MMAs are issued
// before the F_V read-modify-write of the pending one (updates stay in tile order). Lanes outside
// the sub-run or past column R are redirected to scratch words (branch-free updates).
template <int KS, int NT, int W, int LT, int RT, int CS>
__global__ void __launch_bounds__(32 * (W * CS + 1)) k_scatter_tma(
    const int32_t* __restrict__ fiber_col, const double* __restrict__ fiber_val, int G, int64_t Jg,
    const int64_t* __restrict__ st_f, const int32_t* __restrict__ st_k, const int32_t* __restrict__ st_t,
    const uint32_t* __restrict__ st_tab, const int32_t* __restrict__ cta_st, int l_, int R_, int RS_, int FB, int PB,
    int NSt, const double* __restrict__ Nst, double* __restrict__ FVpart) {
  const int R = RT ? RT : R_;  // compile-time for the configured (R, l) shapes
  const int l = LT ? LT : l_;
  const int RS = RT ? ((RT + 1) & ~1) : RS_;
  static_assert(NT % CS == 0, "column splits divide the n-tiles");
  constexpr int NTW = NT / CS;  // n-tiles per consumer warp
  extern __shared__ __align__(128) unsigned char smraw[];
  int tid;  // in a register the compiler cannot rebuild from SR_TID
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const int lane = tid & 31, wc = tid >> 5;
  const int w = wc % W, cpart = wc / W;
  const int grp = blockIdx.x % G;
  const int64_t rng = blockIdx.x / G;
  const SlotGeom sg = slot_geom(FB, PB, W, l, R);
  double* Fs = (double*)smraw;  // Jg x RS, then W x kScrD doubles of scratch
  const uint32_t fs_bytes = (uint32_t)(((uint64_t)Jg * RS * 8 + (uint64_t)W * kScrD * 8 + 127) & ~127ull);
  uint64_t* full = (uint64_t*)(smraw + fs_bytes);
  uint64_t* empty = full + NSt;
  const uint32_t slots_off = fs_bytes + ((2 * NSt * 8 + 127) & ~127);
  unsigned char* slots = smraw + slots_off;
  for (int64_t x = threadIdx.x; x < Jg * RS; x += blockDim.x) Fs[x] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSt; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, W * CS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int s0 = cta_st[blockIdx.x], ns = cta_st[blockIdx.x + 1] - s0;
  if (wc == W * CS) {
    // ---------------- producer (one lane); stage metadata loaded one stage ahead
    if (lane == 0) {
      int64_t nf0 = 0, nf1 = 0;
      int32_t nk0 = 0, nk1 = 0, nt0 = 0;
      if (ns > 0) {
        nf0 = st_f[2 * (int64_t)s0]; nf1 = st_f[2 * (int64_t)s0 + 1];
        nk0 = st_k[2 * (int64_t)s0]; nk1 = st_k[2 * (int64_t)s0 + 1];
        nt0 = st_t[s0];
      }
      int slot = 0, phase = 1;  // the producer's first pass over the ring does not wait
      for (int i = 0; i < ns; ++i) {
        const int64_t f0 = nf0, f1 = nf1;
        const int32_t k0 = nk0, k1 = nk1, t0 = nt0;
        if (i + 1 < ns) {
          const int64_t st = s0 + i + 1;
          nf0 = st_f[2 * st]; nf1 = st_f[2 * st + 1];
          nk0 = st_k[2 * st]; nk1 = st_k[2 * st + 1];
          nt0 = st_t[st];
        }
        mbar_wait_park(empty + slot, phase, 1000000u);  // parked, no issue slots taken from consumers
        unsigned char* base = slots + (size_t)slot * sg.bytes;
        int32_t* mi = (int32_t*)base;
        const uintptr_t sl = (uintptr_t)(st_tab + t0), sc = (uintptr_t)(fiber_col + f0),
                        sv = (uintptr_t)(fiber_val + f0 * l), sn = (uintptr_t)(Nst + (int64_t)k0 * l * R);
        const size_t bl = 4ull * W * (k1 - k0), bc = 4ull * (f1 - f0), bv = 8ull * (f1 - f0) * l,
                     bn = 8ull * (k1 - k0) * l * R;
        mi[0] = k1 - k0;
        mi[1] = (int32_t)(sl & 15);
        mi[2] = (int32_t)(sc & 15);
        mi[3] = (int32_t)(sv & 15);
        mi[4] = (int32_t)(sn & 15);
        // expected bytes first (same rounding as bulk_g2s_span), then the copies
        const uint32_t tx = al16((sl & 15) + bl) + al16((sc & 15) + bc) + al16((sv & 15) + bv) + al16((sn & 15) + bn);
        mbar_arrive_tx(full + slot, tx);
        uint32_t t2 = 0;
        bulk_g2s_span(base + sg.lh, (const void*)sl, bl, full + slot, &t2);
        bulk_g2s_span(base + sg.col, (const void*)sc, bc, full + slot, &t2);
        bulk_g2s_span(base + sg.val, (const void*)sv, bv, full + slot, &t2);
        bulk_g2s_span(base + sg.nrows, (const void*)sn, bn, full + slot, &t2);
        if (++slot == NSt) { slot = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- consumers
    const int g = lane >> 2, t = lane & 3;
    const int per = l * R;
    const int c0 = 8 * NTW * cpart;  // first F_V column of this warp's n-tiles
    const uint32_t sbase = smem_u32(smraw);
    const uint32_t fwA = sbase + 8u * (uint32_t)(c0 + 2 * t);  // + row byte offset + 64 nt: the lane's pair
    // scratch words of this lane (the CS warps of a sub-range share them: redirected updates are
    // never read back, so their interleaving is immaterial); + 64 nt stays inside kScrD doubles
    const uint32_t scrA = sbase + 8u * (uint32_t)(Jg * RS + w * kScrD + 2 * lane);
    // B fragment B[t][g] = N(a = 4 ks + t, r = c0 + 8 nt + g); lanes outside (a < l, r < R) load nothing
    const int nb0 = t * R + g + c0;
    unsigned nok = 0;  // bit (ks NTW + nt): the lane's fragment is inside N
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
        if (4 * ks + t < l && c0 + 8 * nt + g < R) nok |= 1u << (ks * NTW + nt);
    bool colok[NTW];  // the lane's two columns of n-tile nt are inside R (else: scratch)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) colok[nt] = c0 + 8 * nt + 2 * t < R;
    bool aok[KS];  // the lane's A fragment (a = 4 ks + t) is inside l
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) aok[ks] = 4 * ks + t < l;
    uint32_t pA = scrA;  // pending tile: the lane's F_V row address (or scratch) and its products
    double pcc[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) pcc[nt][0] = pcc[nt][1] = 0.0;
    auto commit = [&]() {
      uint32_t a[NTW];
      double2 v[NTW];
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        a[nt] = (colok[nt] ? pA : scrA) + 64u * nt;
        v[nt] = lds_v2(a[nt]);
      }
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        v[nt].x += pcc[nt][0];
        v[nt].y += pcc[nt][1];
        sts_v2(a[nt], v[nt]);
      }
    };
    const uint32_t fullA = smem_u32(full), emptyA = smem_u32(empty);
    int slot = 0, phase = 0;
    for (int i = 0; i < ns; ++i) {
      mbar_wait_a(fullA + 8u * slot, phase);
      const uint32_t sb = sbase + slots_off + (uint32_t)slot * sg.bytes;
      const int npat = lds_s32(sb);
      const uint32_t lhA = sb + sg.lh + lds_s32(sb + 4) + 4u * w;
      const uint32_t colA = sb + sg.col + lds_s32(sb + 8) + 4u * g;
      const uint32_t valA = sb + sg.val + lds_s32(sb + 12) + 8u * (uint32_t)(t + l * g);
      const uint32_t nA = sb + sg.nrows + lds_s32(sb + 16) + 8u * nb0;
      // per-patient setup (sub-run bounds, B fragments) one patient ahead of its tiles
      auto setup = [&](int p, int& lo_, int& hi_, double (&b)[KS][NTW]) {
        const uint32_t lh = (uint32_t)lds_s32(lhA + 4u * W * p);
        lo_ = (int)(lh & 0xffffu);
        hi_ = (int)(lh >> 16);
        const uint32_t np = nA + 8u * (uint32_t)(p * per);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt)
            b[ks][nt] = lds_f64_if(np + 8u * (4 * ks * R + 8 * nt), (nok >> (ks * NTW + nt)) & 1u);
      };
      int nlo = 0, nhi = 0;
      double nbfr[KS][NTW];
      if (npat > 0) setup(0, nlo, nhi, nbfr);
      for (int p = 0; p < npat; ++p) {
        const int lo = nlo, hi = nhi;
        double bfr[KS][NTW];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) bfr[ks][nt] = nbfr[ks][nt];
        if (p + 1 < npat) setup(p + 1, nlo, nhi, nbfr);
#pragma unroll 2
        for (int tb = lo; tb < hi; tb += 8) {
          const bool ok = tb + g < hi;
          const int rb = lds_s32_if(colA + 4u * tb, ok, 0);  // the fiber's F_V row byte offset
          double av[KS];
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) av[ks] = lds_f64_if(valA + 8u * (uint32_t)(l * tb + 4 * ks), ok && aok[ks]);
          double cc[NTW][2];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) cc[nt][0] = cc[nt][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) dmma(cc[nt][0], cc[nt][1], av[ks], bfr[ks][nt]);
          commit();  // the previous tile (or a zero update of the scratch words)
          pA = ok ? fwA + (uint32_t)rb : scrA;
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) { pcc[nt][0] = cc[nt][0]; pcc[nt][1] = cc[nt][1]; }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(emptyA + 8u * slot) : "memory");
      if (++slot == NSt) { slot = 0; phase ^= 1; }
    }
    commit();  // the last tile
  }
  __syncthreads();
  double* out = FVpart + rng * (G * Jg) * (int64_t)R + (int64_t)grp * Jg * R;
  for (int64_t x = threadIdx.x; x < Jg * R; x += blockDim.x) {
    const int64_t jj = x / R, r = x - jj * R;
    out[x] = Fs[jj * RS + r];
  }
}

// Init: the pass-B stage table of sub-run bounds. CTA c = (range, group c % G) walks its stages;
// entry (stage s, patient k in [k0, k1), sub-range w) = lo | hi << 16 with [lo, hi) the fibers of
// sub-range (g, w) of patient k inside the stage's fiber window [f0, f1), relative to f0.
__global__ void k_stage_tab(const int64_t* __restrict__ gptr, const uint16_t* __restrict__ woff, int64_t K, int G,
                            int W, const int64_t* __restrict__ st_f, const int32_t* __restrict__ st_k,
                            const int32_t* __restrict__ st_t, const int32_t* __restrict__ cta_st,
                            uint32_t* __restrict__ st_tab) {
  const int c = blockIdx.x, grp = c % G;
  const int64_t* gp = gptr + (int64_t)grp * (K + 1);
  for (int s = cta_st[c] + threadIdx.x; s < cta_st[c + 1]; s += blockDim.x) {
    const int64_t f0 = st_f[2 * (int64_t)s], f1 = st_f[2 * (int64_t)s + 1];
    const int32_t k0 = st_k[2 * (int64_t)s], k1 = st_k[2 * (int64_t)s + 1];
    uint32_t* out = st_tab + st_t[s];
    for (int32_t k = k0; k < k1; ++k) {
      const uint16_t* wo = woff + ((int64_t)grp * K + k) * kWoS;
      for (int w = 0; w < W; ++w) {
        const int64_t lo = min(max(gp[k] + wo[w], f0), f1) - f0;
        const int64_t hi = min(max(gp[k] + wo[w + 1], f0), f1) - f0;
        out[(int64_t)(k - k0) * W + w] = (uint32_t)lo | ((uint32_t)hi << 16);
      }
    }
  }
}

void launch_stage_tab(Handle& h) {
  if (!h.sc_ok || h.nst == 0) return;
  k_stage_tab<<<(unsigned)(h.sc_ranges * h.sc_G), 128, 0, h.stream>>>(h.gptr, h.woff, h.K, h.sc_G, h.sc_W, h.st_f,
                                                                      h.st_k, h.st_t, h.cta_st, h.st_tab);
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

template <int KS, int NT, int W, int LT = 0, int RT = 0, int CS = 1>
static void scatter_inst_w(Handle& h) {
  constexpr auto fn = k_scatter_tma<KS, NT, W, LT, RT, CS>;
  max_smem_attr<fn>(h);
  const int ctas = h.sc_ranges * h.sc_G;
  fn<<<ctas, 32 * (W * CS + 1), h.sc_smem, h.stream>>>(h.fiber_col, h.fiber_val, h.sc_G, h.sc_Jg, h.st_f, h.st_k,
                                                        h.st_t, h.st_tab, h.cta_st, h.l, h.R, h.sc_RS, h.sc_FB,
                                                        h.sc_PB, h.sc_NS, h.Nst, h.fv_part);
  int64_t n = h.Jl * h.R;
  k_sum_ranges<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.fv_part, h.sc_ranges, h.Jl, h.R, h.inv, h.FV);
}

template <int KS, int NT>
static void scatter_inst(Handle& h) {
  if (h.sc_W == 2) scatter_inst_w<KS, NT, 2>(h);
  else scatter_inst_w<KS, NT, 4>(h);
}

// Column splits for the configured shapes (measured at Scale: CS = 3 23.3 ms vs CS = 1 24.7 ms;
// Medium CS = 2 1.26 vs 1.40 ms; Large CS = 5 8.1 vs 9.0 ms; 2 or 8 sub-ranges per group slower).
template <int KS>
static void scatter_dispatch_n(Handle& h) {
  if (h.sc_W == 4) {
    if (KS == 2 && h.l == 7 && h.R == 20) { scatter_inst_w<2, 3, 4, 7, 20, 3>(h); return; }
    if (KS == 2 && h.l == 7 && h.R == 15) { scatter_inst_w<2, 2, 4, 7, 15, 2>(h); return; }
    if (KS == 3 && h.l == 9 && h.R == 40) { scatter_inst_w<3, 5, 4, 9, 40, 5>(h); return; }
  }
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

// Chooses the label groups G (F_V slice of a CTA), stage geometry and the number of pass-B patient
// ranges so that one CTA's F_V slice plus its NS-stage ring fits in shared memory.
void plan_scatter(Handle& h) {
  const size_t budget = 225 * 1024;
  h.sc_W = kScW;  // label sub-ranges per group (2 or 4)
  h.sc_RS = (h.R + 1) & ~1;
  h.sc_FB = 256;
  h.sc_ok = 0;
  const int pbs[3] = {16, 8, 4};
  const int gmin = 1;
  for (int pass = 0; pass < 2 && !h.sc_ok; ++pass)  // pass 0: >= 3 stages of >= 8 patients
    for (int G = gmin; G <= kMaxGroups && !h.sc_ok; ++G) {
      const int64_t Js = (h.J + (int64_t)G * h.sc_W - 1) / ((int64_t)G * h.sc_W);
      const int64_t Jg = Js * h.sc_W;
      const size_t fs = ((size_t)Jg * h.sc_RS * 8 + (size_t)h.sc_W * kScrD * 8 + 127) & ~(size_t)127;
      for (int NSt = 4; NSt >= (pass ? 2 : 3) && !h.sc_ok; --NSt)
        for (int pi = 0; pi < (pass ? 3 : 2) && !h.sc_ok; ++pi) {
          const SlotGeom sg = slot_geom(h.sc_FB, pbs[pi], h.sc_W, h.l, h.R);
          const size_t bytes = fs + ((2 * NSt * 8 + 127) & ~127) + (size_t)NSt * sg.bytes;
          if (bytes <= budget) {
            h.sc_G = G;
            h.sc_Js = Js;
            h.sc_Jg = Jg;
            h.sc_PB = pbs[pi];
            h.sc_NS = NSt;
            h.sc_slot = sg.bytes;
            h.sc_smem = bytes;
            h.sc_ok = 1;
          }
        }
    }
  // Larger stages (FB = 512: fewer per-stage overheads; measured 43 -> 40 ms at Scale, 2.26 -> 2.10 ms
  // at Medium) when they still fit at the same G with >= 3 slots of >= 8 patients.
  if (h.sc_ok) {
    const size_t fs = ((size_t)h.sc_Jg * h.sc_RS * 8 + (size_t)h.sc_W * kScrD * 8 + 127) & ~(size_t)127;
    bool done = false;
    for (int NSt = 4; NSt >= 3 && !done; --NSt)
      for (int pi = 0; pi < 2 && !done; ++pi) {
        const SlotGeom sg = slot_geom(512, pbs[pi], h.sc_W, h.l, h.R);
        const size_t bytes = fs + ((2 * NSt * 8 + 127) & ~127) + (size_t)NSt * sg.bytes;
        if (bytes <= budget) {
          h.sc_FB = 512;
          h.sc_PB = pbs[pi];
          h.sc_NS = NSt;
          h.sc_slot = sg.bytes;
          h.sc_smem = bytes;
          done = true;
        }
      }
  }
  if (!h.sc_ok) {  // F_V does not fit even split 8 ways: global-atomic fallback (k_iter.cu)
    h.sc_G = kMaxGroups;
    h.sc_Js = (h.J + (int64_t)h.sc_G * h.sc_W - 1) / ((int64_t)h.sc_G * h.sc_W);
    h.sc_Jg = h.sc_Js * h.sc_W;
  }
  h.Jl = (int64_t)h.sc_G * h.sc_Jg;
  int bps = h.sc_ok ? (int)((228 * 1024) / (h.sc_smem + 1024)) : 1;
  if (bps < 1) bps = 1;
  int64_t ranges = (h.sms * (int64_t)bps + h.sc_G - 1) / h.sc_G;
  if (ranges > h.K) ranges = h.K > 0 ? h.K : 1;
  h.sc_ranges = (int)ranges;
}

bool scatter_smem_ok(const Handle& h) { return h.sc_ok != 0; }

// Init (after layoutA has copied the labels): the g-stream labels become F_V slice offsets
// (label - g Jg) RS, so pass B addresses a fiber's F_V row without index arithmetic.
__global__ void k_fiber_rowoff(const int64_t* __restrict__ gptr, int64_t K, int G, int64_t Jg, int RS,
                               int32_t* __restrict__ fiber_col) {
  for (int g = 0; g < G; ++g) {
    const int64_t f0 = gptr[(int64_t)g * (K + 1)], f1 = gptr[(int64_t)g * (K + 1) + K];
    for (int64_t f = f0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < f1; f += (int64_t)gridDim.x * blockDim.x)
      fiber_col[f] = (int32_t)((fiber_col[f] - g * Jg) * RS * 8);  // bytes
  }
}

void launch_fiber_rowoff(Handle& h) {
  if (!h.sc_ok || h.K == 0) return;
  k_fiber_rowoff<<<(unsigned)(h.sms * 8), 256, 0, h.stream>>>(h.gptr, h.K, h.sc_G, h.sc_Jg, h.sc_RS, h.fiber_col);
}

// stage-table entries: every stage holds its patients' sub-range bounds; a patient's run is split
// over at most (run / FB + 2) stages, so sum over stages of (k1 - k0) <= G K + nst
int64_t stage_tab_cap(const Handle& h) { return ((int64_t)h.sc_G * h.K + stage_cap(h)) * h.sc_W + 16; }

int64_t stage_cap(const Handle& h) {
  return h.F / h.sc_FB + (int64_t)h.sc_G * (h.K / h.sc_PB + 1) + (int64_t)h.sc_ranges * h.sc_G + 16;
}

// Host planning from the per-group run lengths gcnt[g][k]: stream offsets gptr (absolute), pass-B
// patient ranges (balanced by fibers) and the stage table of every (range, group) CTA.
void plan_streams(Handle& h, const int32_t* gcnt, int64_t* gptr, std::vector<int64_t>& st_f, std::vector<int32_t>& st_k,
                  std::vector<int32_t>& st_t, std::vector<int32_t>& cta_st, std::vector<int64_t>& block_k) {
  const int G = h.sc_G;
  const int64_t K = h.K, K1 = K + 1;
  int64_t base = 0;
  for (int g = 0; g < G; ++g) {
    int64_t* gp = gptr + g * K1;
    gp[0] = base;
    for (int64_t k = 0; k < K; ++k) gp[k + 1] = gp[k] + gcnt[g * K + k];
    base = gp[K];
  }
  // balanced patient ranges by total fibers
  const int nr = h.sc_ranges;
  block_k.assign((size_t)nr + 1, 0);
  std::vector<int64_t> tot((size_t)K1, 0);
  for (int64_t k = 0; k < K; ++k) {
    int64_t c = 0;
    for (int g = 0; g < G; ++g) c += gcnt[g * K + k];
    tot[(size_t)k + 1] = tot[(size_t)k] + c;
  }
  for (int b = 0; b <= nr; ++b) {
    if (b == nr) { block_k[(size_t)b] = K; break; }
    const int64_t target = (tot[(size_t)K] * b) / nr;
    block_k[(size_t)b] = std::lower_bound(tot.begin(), tot.end(), target) - tot.begin();
    if (block_k[(size_t)b] > K) block_k[(size_t)b] = K;
  }
  st_f.clear();
  st_k.clear();
  cta_st.assign((size_t)nr * G + 1, 0);
  const int64_t FB = h.sc_FB, PB = h.sc_PB;
  for (int r = 0; r < nr; ++r)
    for (int g = 0; g < G; ++g) {
      cta_st[(size_t)r * G + g] = (int32_t)(st_k.size() / 2);
      const int64_t* gp = gptr + g * K1;
      const int64_t kr0 = block_k[(size_t)r], kr1 = block_k[(size_t)r + 1];
      if (kr0 >= kr1) continue;
      int64_t f = gp[kr0];
      const int64_t fend = gp[kr1];
      int64_t k = kr0;
      while (f < fend) {
        while (gp[k + 1] <= f) ++k;  // first patient whose run ends after f
        int64_t f1 = std::min(f + FB, fend);
        int64_t kk = k + 1;
        while (kk < kr1 && gp[kk] < f1) ++kk;
        if (kk - k > PB) {
          kk = k + PB;
          f1 = gp[kk];
        }
        st_f.push_back(f);
        st_f.push_back(f1);
        st_k.push_back((int32_t)k);
        st_k.push_back((int32_t)kk);
        f = f1;
        k = kk - 1;
      }
    }
  cta_st[(size_t)nr * G] = (int32_t)(st_k.size() / 2);
  // offsets of every stage's (patient, sub-range) entries in the stage table st_tab
  const size_t nst = st_k.size() / 2;
  st_t.assign(nst + 1, 0);
  int64_t acc = 0;  // (the caller rejects tables beyond int32)
  for (size_t x = 0; x < nst; ++x) {
    acc += (int64_t)(st_k[2 * x + 1] - st_k[2 * x]) * h.sc_W;
    st_t[x + 1] = (int32_t)std::min<int64_t>(acc, INT32_MAX);
  }
}

// ------------------------------------------------------------------ init-time relabeling
// Feature relabeling from the per-feature fiber counts: features sorted by count (descending,
// ties by id) are dealt serpentine over the G*W label sub-ranges of Js labels each; perm[j] = new
// label, inv[new] = j. Host-side (J <= 65535).
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

}  // namespace copa
