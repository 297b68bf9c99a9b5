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
#include <thread>
#include <type_traits>
#include <vector>

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

// ------------------------------------------------------------------ pass B (tiled stream, TMA-staged)
// Tiled stream (built once at init from the g-streams, k_build_tiles): per label group g, patient
// after patient, sub-range after sub-range, the sub-run of (patient k, sub-range (g, w)) is cut into
// ceil(n / 8) tiles of 8 fiber slots, each tile
//   int32 rowoff[8]   F_V row byte offset (label - g Jg) RS 8 inside the CTA's shared-memory slice
//   f64   val         x'(a, slot) in blocks of nb = min(4, l - 4 b) a's (b = a / 4): byte 256 b +
//                     32 nb (slot / 4) + 32 (a % 4) + 8 (slot % 4), so the MMA A fragment of a
//                     k-step (a = 4 ks + t, slot g) is one block whose two half-warps each read 32 nb
//                     contiguous bytes (two conflict-free wavefronts; a-major rows of 64 bytes
//                     measured 4, a zero-padded last block made the tiles larger and pass B slower)
// Padding slots hold zeros and address one of the scratch rows behind the slice. The slots of a tile
// are paired (2i, 2i + 1) so that the two rows one quarter-warp touches in an F_V read-modify-write
// lie in opposite halves of the 32 banks (row labels differ by D mod M, see pair_rule); pads are
// wildcards that take the partner class. tptr[g][k]: first tile of (g, k); twoff[g][k][w]: tile
// offset of sub-range w inside it.
__host__ __device__ inline uint32_t tile_bytes(int l) { return 32u + 64u * (uint32_t)l; }
__host__ __device__ inline uint32_t tile_val_off(int l, int a, int slot) {  // byte offset of x'(a, slot)
  const int b = a >> 2, nb = min(4, l - 4 * b);
  return 32u + 256u * b + 32u * nb * (slot >> 2) + 32u * (a & 3) + 8u * (slot & 3);
}
constexpr int kScrRows = 8;  // scratch rows behind the F_V slice (pads; any label class mod M <= 8)

// Rows j0, j1 with byte offsets 8 RS j: their 64-byte segments (same columns) are bank-disjoint iff
// 8 RS (j0 - j1) = 64 mod 128, i.e. RS (j0 - j1) = 8 mod 16. With RS = 2^a b (b odd, 1 <= a <= 3):
// j0 - j1 = D mod M with M = 2^(4 - a), D = M / 2. RS is chosen with a <= 3 (plan_scatter).
__host__ __device__ inline void pair_rule(int RS, int* M, int* D) {
  int a = 0;
  while (((RS >> a) & 1) == 0 && a < 4) ++a;
  *M = 1 << (4 - a);
  *D = *M / 2;
}

// Stage slot layout (bytes, each part 16-byte aligned):
//   meta  : int32 npat, shift_list, shift_tiles, shift_n (32)
//   list  : uint32 [8 + FT] + 16   the stage's tile list (st_list, built at init; bulk copy, shifted):
//           8 offsets e[w] (w = 0..W), then the tiles grouped by sub-range, entry = tile | patient << 16
//           (relative to the stage), sub-range w's tiles at [e[w], e[w + 1])
//   tiles : [FT] x tile_bytes + 16  (bulk copy, shifted)
//   nrows : f64 [PB l R] + 16      N_k rows (bulk copy, shifted)
struct SlotGeom {
  uint32_t lh, tiles, nrows, bytes;
};
__host__ __device__ inline uint32_t al16(uint64_t x) { return (uint32_t)((x + 15) & ~(uint64_t)15); }
__host__ __device__ inline SlotGeom slot_geom(int FT, int PB, int W, int l, int R) {
  SlotGeom s;
  s.lh = 32;
  s.tiles = s.lh + al16(4ull * (8 + FT) + 16);
  s.nrows = s.tiles + al16((uint64_t)tile_bytes(l) * FT + 16);
  s.bytes = (s.nrows + al16(8ull * PB * l * R + 16) + 127) & ~127u;
  return s;
}
__host__ __device__ inline uint32_t slice_bytes(int64_t Jg, int RS) {
  return (uint32_t)(((uint64_t)(Jg + kScrRows) * RS * 8 + 127) & ~127ull);
}

constexpr int kScW = 4;  // pass-B label sub-ranges per group

// Shared-memory accesses by 32-bit shared addresses: the consumers hold their base addresses in
// registers (with generic pointers the compiler re-derived the shared window, S2UR + ULEA, per tile).
// All are volatile: they keep program order among themselves (F_V read-modify-writes of one lane).
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64_if(uint32_t a, bool p) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}" : "+d"(v) : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ double2 lds_v2_if(uint32_t a, bool p) {
  double2 v = make_double2(0.0, 0.0);
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q ld.shared.v2.f64 {%0, %1}, [%2];\n}"
               : "+d"(v.x), "+d"(v.y)
               : "r"(a), "r"((int)p));
  return v;
}
__device__ __forceinline__ void lds_f64_keep(double& v, uint32_t a, bool p) {  // v unchanged when !p
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}" : "+d"(v) : "r"(a), "r"((int)p));
}
__device__ __forceinline__ void sts_v2_if(uint32_t a, double2 v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a),
               "d"(v.x), "d"(v.y), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
      "DONE%=:\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// CTA = (patient range, label group g) owns the F_V rows of group g in shared memory. One producer
// warp streams the range's stages (<= FT tiles, <= PB patients) of the group's tiled stream into an
// NS-deep ring with 1-D TMA bulk copies. W x CS consumer warps: warp (w, c) owns the rows of
// sub-range (g, w), columns [8 NT/CS c, 8 NT/CS (c + 1)) — disjoint words, no atomics. Per stage
// it reads its tile bounds of every patient from the staged lh table and runs one MMA per tile and
// k-step (M = 8 slots, N = r, K = a) with one tile in flight: the next tile's loads and MMAs are
// issued before the F_V read-modify-write of the pending one (updates stay in tile order). Lanes
// whose columns are past R are predicated off.
template <int KS, int NT, int W, int LT, int RT, int CS>
__global__ void __launch_bounds__(32 * (W * CS + 1)) k_scatter_tma(
    const unsigned char* __restrict__ tiles, int G, int64_t Jg, const int64_t* __restrict__ st_f,
    const int32_t* __restrict__ st_k, const int32_t* __restrict__ st_t, const uint32_t* __restrict__ st_list,
    const int32_t* __restrict__ cta_st, int l_, int R_, int RS_, int FT, int PB, int NSt,
    const double* __restrict__ Nst, double* __restrict__ FVpart) {
  const int R = RT ? RT : R_;  // compile-time for the configured (R, l) shapes
  const int l = LT ? LT : l_;
  const int RS = RS_;
  static_assert(NT % CS == 0, "column splits divide the n-tiles");
  constexpr int NTW = NT / CS;  // n-tiles per consumer warp
  extern __shared__ __align__(128) unsigned char smraw[];
  int tid;  // in a register the compiler cannot rebuild from SR_TID
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
  const int lane = tid & 31, wc = tid >> 5;
  const int w = wc % W, cpart = wc / W;
  const int grp = blockIdx.x % G;
  const int64_t rng = blockIdx.x / G;
  const SlotGeom sg = slot_geom(FT, PB, W, l, R);
  const uint32_t TB = tile_bytes(l);
  double* Fs = (double*)smraw;  // (Jg + kScrRows) x RS
  const uint32_t fs_bytes = slice_bytes(Jg, RS);
  uint64_t* full = (uint64_t*)(smraw + fs_bytes);
  uint64_t* empty = full + NSt;
  const uint32_t slots_off = fs_bytes + ((2 * NSt * 8 + 127) & ~127);
  unsigned char* slots = smraw + slots_off;
  for (int64_t x = threadIdx.x; x < (Jg + kScrRows) * RS; x += blockDim.x) Fs[x] = 0.0;
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
        const uintptr_t sl = (uintptr_t)(st_list + t0), sc = (uintptr_t)(tiles + (size_t)f0 * TB),
                        sn = (uintptr_t)(Nst + (int64_t)k0 * l * R);
        const size_t bl = 4ull * (8 + (f1 - f0)), bc = (size_t)TB * (f1 - f0), bn = 8ull * (k1 - k0) * l * R;
        mi[0] = k1 - k0;
        mi[1] = (int32_t)(sl & 15);
        mi[2] = (int32_t)(sc & 15);
        mi[3] = (int32_t)(sn & 15);
        // expected bytes first (same rounding as bulk_g2s_span), then the copies
        const uint32_t tx = al16((sl & 15) + bl) + al16((sc & 15) + bc) + al16((sn & 15) + bn);
        mbar_arrive_tx(full + slot, tx);
        uint32_t t2 = 0;
        bulk_g2s_span(base + sg.lh, (const void*)sl, bl, full + slot, &t2);
        bulk_g2s_span(base + sg.tiles, (const void*)sc, bc, full + slot, &t2);
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
    // B fragment B[t][g] = N(a = 4 ks + t, r = c0 + 8 nt + g); lanes outside (a < l, r < R) load nothing
    const int nb0 = t * R + g + c0;
    unsigned nok = 0;  // bit (ks NTW + nt): the lane's fragment is inside N
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
        if (4 * ks + t < l && c0 + 8 * nt + g < R) nok |= 1u << (ks * NTW + nt);
    bool colok[NTW];  // the lane's two columns of n-tile nt are inside R (else: no access)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) colok[nt] = c0 + 8 * nt + 2 * t < R;
    bool aok[KS];      // the lane's A fragment (a = 4 ks + t) is inside l
    uint32_t aoff[KS];  // ... and its byte offset inside a tile
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      aok[ks] = 4 * ks + t < l;
      aoff[ks] = aok[ks] ? tile_val_off(l, 4 * ks + t, g) : 0u;
    }
    // pending tile: the lane's F_V row address and its products (initially a zero update of a
    // scratch row)
    uint32_t pA = fwA + 8u * (uint32_t)(Jg * RS);
    double pcc[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) pcc[nt][0] = pcc[nt][1] = 0.0;
    auto commit = [&]() {
      double2 v[NTW];
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) v[nt] = lds_v2_if(pA + 64u * nt, colok[nt]);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        v[nt].x += pcc[nt][0];
        v[nt].y += pcc[nt][1];
        sts_v2_if(pA + 64u * nt, v[nt], colok[nt]);
      }
    };
    const uint32_t fullA = smem_u32(full), emptyA = smem_u32(empty);
    int slot = 0, phase = 0;
    for (int i = 0; i < ns; ++i) {
      mbar_wait_a(fullA + 8u * slot, phase);
      const uint32_t sb = sbase + slots_off + (uint32_t)slot * sg.bytes;
      const uint32_t lA = sb + sg.lh + lds_s32(sb + 4);
      const uint32_t tA = sb + sg.tiles + lds_s32(sb + 8);
      const uint32_t nA = sb + sg.nrows + lds_s32(sb + 12) + 8u * nb0;
      const int e0 = lds_s32(lA + 4u * w), e1 = lds_s32(lA + 4u * (w + 1));
      // Software pipeline over this warp's tiles of the stage (flat list): iteration e issues the
      // F_V load of the pending tile e - 1, the loads of tile e + 1 (entry of e + 2), the MMAs of
      // tile e, then the F_V update of e - 1. B fragments are reloaded only when the patient changes.
      if (e0 < e1) {
        const uint32_t eA = lA + 32u;
        uint32_t ent = (uint32_t)lds_s32(eA + 4u * e0);
        uint32_t ent2 = (uint32_t)lds_s32(eA + 4u * min(e0 + 1, e1 - 1));
        int pc = (int)(ent >> 16);
        double bc[KS][NTW], ac[KS];
        int rc;
        {
          const uint32_t ta = tA + TB * (ent & 0xffffu);
          rc = lds_s32(ta + 4u * g);
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) ac[ks] = lds_f64_if(ta + aoff[ks], aok[ks]);
          const uint32_t np = nA + 8u * (uint32_t)(pc * per);
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt)
              bc[ks][nt] = lds_f64_if(np + 8u * (4 * ks * R + 8 * nt), (nok >> (ks * NTW + nt)) & 1u);
        }
        for (int e = e0; e < e1; ++e) {
          // F_V rows of the pending tile
          double2 v[NTW];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) v[nt] = lds_v2_if(pA + 64u * nt, colok[nt]);
          // next tile's operands (entry e + 1 = ent2) and the entry after it
          double an[KS], bn[KS][NTW];
          int rn = 0, pn = pc;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) bn[ks][nt] = bc[ks][nt];
          const bool more = e + 1 < e1;
          {
            const uint32_t ta = tA + TB * (ent2 & 0xffffu);
            pn = more ? (int)(ent2 >> 16) : pc;
            rn = lds_s32(ta + 4u * g);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) an[ks] = lds_f64_if(ta + aoff[ks], aok[ks] && more);
            const uint32_t np = nA + 8u * (uint32_t)(pn * per);
            const bool newp = pn != pc;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt)
                lds_f64_keep(bn[ks][nt], np + 8u * (4 * ks * R + 8 * nt), newp && ((nok >> (ks * NTW + nt)) & 1u));
            ent2 = (uint32_t)lds_s32(eA + 4u * min(e + 2, e1 - 1));
          }
          double cc[NTW][2];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) cc[nt][0] = cc[nt][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) dmma(cc[nt][0], cc[nt][1], ac[ks], bc[ks][nt]);
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) {
            v[nt].x += pcc[nt][0];
            v[nt].y += pcc[nt][1];
            sts_v2_if(pA + 64u * nt, v[nt], colok[nt]);
          }
          pA = fwA + (uint32_t)rc;
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) { pcc[nt][0] = cc[nt][0]; pcc[nt][1] = cc[nt][1]; }
          rc = rn;
          pc = pn;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            ac[ks] = an[ks];
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) bc[ks][nt] = bn[ks][nt];
          }
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

// ------------------------------------------------------------------ init: the tiled stream
// Warp per (group, patient) run, its W sub-runs one after the other: a sub-run's n fibers (g-stream,
// sorted by label) go to 8 ceil(n / 8) slots paired as described above. Pairs, in order: (class c
// rank i, class c + D rank i) for every c < D; each class's surplus with a pad; the remaining surplus
// fibers with each other (consecutive, possibly a same-half pair); pads with pads. Slot = 2 pair +
// side. Class ranks come from per-class warp ballots, 32 fibers at a time; the lanes then write
// their fibers (and the pads) in parallel.
__global__ void k_build_tiles(const int64_t* __restrict__ gptr, const uint16_t* __restrict__ woff,
                              const int64_t* __restrict__ tptr, const uint16_t* __restrict__ twoff, int64_t K, int G,
                              int W, int64_t Jg, int RS, int l, const int64_t* __restrict__ fp,
                              const int32_t* __restrict__ fiber_col, const double* __restrict__ fiber_val,
                              unsigned char* __restrict__ tiles) {
  const int lane = threadIdx.x & 31;
  const int64_t gk = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gk >= (int64_t)G * K) return;
  const int g = (int)(gk / K);
  const int64_t k = gk - (int64_t)g * K;
  const uint16_t* wo = woff + gk * kWoS;
  const uint32_t TB = tile_bytes(l);
  int M, D;
  pair_rule(RS, &M, &D);
  const int64_t lab0 = (int64_t)g * Jg;
  const unsigned lt = (1u << lane) - 1u;
  auto scr = [&](int cls) -> int64_t { return Jg + (((int64_t)cls - Jg) & (M - 1)); };
  // the run (g, k) inside layout A (patient k's G runs concatenated at fp[k]); the tiles overwrite
  // the g-streams, so they are read from layout A
  int64_t run0 = fp[k];
  for (int gg = 0; gg < g; ++gg) run0 += gptr[(int64_t)gg * (K + 1) + k + 1] - gptr[(int64_t)gg * (K + 1) + k];
  for (int w = 0; w < W; ++w) {
    const int64_t f0 = run0 + wo[w];
    const int n = wo[w + 1] - wo[w];
    if (n == 0) continue;
    const int T = (n + 7) >> 3, P = 8 * T - n;
    unsigned char* tb = tiles + (size_t)TB * (size_t)(tptr[(int64_t)g * (K + 1) + k] + twoff[gk * kWoS + w]);
    auto put = [&](int slot, int64_t rowlab, const double* v) {
      unsigned char* tp = tb + (size_t)TB * (slot >> 3);
      const int pos = slot & 7;
      reinterpret_cast<int32_t*>(tp)[pos] = (int32_t)(rowlab * RS * 8);
      for (int a = 0; a < l; ++a) *reinterpret_cast<double*>(tp + tile_val_off(l, a, pos)) = v ? v[a] : 0.0;
    };
    int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i0 = 0; i0 < n; i0 += 32) {
      const bool ok = i0 + lane < n;
      const int c = ok ? (int)((fiber_col[f0 + i0 + lane] - lab0) & (M - 1)) : -1;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) cnt[cc] += __popc(__ballot_sync(0xffffffffu, c == cc));
    }
    // pair bookkeeping per class pair c < D (warp-uniform)
    int m[4], q[4], base1[4], base2[4], off3[4], X[4];
    int pair = 0, padsLeft = P, tot3 = 0, nq = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < D) {
        m[c] = min(cnt[c], cnt[c + D]);
        base1[c] = pair;
        pair += m[c];
        X[c] = cnt[c] >= cnt[c + D] ? c : c + D;
      }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < D) {
        const int sur = abs(cnt[c] - cnt[c + D]);
        q[c] = min(sur, padsLeft);
        padsLeft -= q[c];
        base2[c] = pair;
        pair += q[c];
        off3[c] = tot3;
        tot3 += sur - q[c];
        nq += q[c];
      }
    const int base3 = pair;  // phase-3 pairs: base3 .. base3 + ceil(tot3 / 2)
    int seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i0 = 0; i0 < n; i0 += 32) {
      const bool ok = i0 + lane < n;
      const int64_t lab = ok ? fiber_col[f0 + i0 + lane] - lab0 : 0;
      const int c = ok ? (int)(lab & (M - 1)) : -1;
      int r = 0;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const unsigned b = __ballot_sync(0xffffffffu, c == cc);
        if (c == cc) r = seen[cc] + __popc(b & lt);
        seen[cc] += __popc(b);
      }
      if (ok) {
        const int cp = c % D;
        int mm = 0, qq = 0, b1 = 0, b2 = 0, o3 = 0;
#pragma unroll
        for (int x = 0; x < 4; ++x)
          if (x == cp) { mm = m[x]; qq = q[x]; b1 = base1[x]; b2 = base2[x]; o3 = off3[x]; }
        int slot;
        if (r < mm) {
          slot = 2 * (b1 + r) + (c >= D ? 1 : 0);
        } else {
          const int j = r - mm;  // surplus rank (c == X[cp])
          slot = j < qq ? 2 * (b2 + j) : 2 * base3 + o3 + (j - qq);  // phase 3: consecutive slots
        }
        put(slot, lab, fiber_val + (f0 + i0 + lane) * l);
      }
    }
    // pads: partners of the phase-2 surplus (nq), then the odd phase-3 tail and pad pairs
    const int npads = nq + (8 * T - 2 * base3 - tot3);
    for (int j = lane; j < npads; j += 32) {
      if (j < nq) {
        int jj = j, slot = 0, cls = 0;
#pragma unroll
        for (int x = 0; x < 4; ++x)
          if (x < D) {
            if (jj >= 0 && jj < q[x]) { slot = 2 * (base2[x] + jj) + 1; cls = (X[x] + D) & (M - 1); }
            jj -= q[x];
          }
        put(slot, scr(cls), nullptr);
      } else {
        const int s = 2 * base3 + tot3 + (j - nq);
        put(s, scr((s & 1) ? D : 0), nullptr);
      }
    }
  }
}

void launch_build_tiles(Handle& h) {
  if (!h.sc_ok || h.K == 0) return;
  const int64_t n = (int64_t)h.sc_G * h.K;  // warps
  k_build_tiles<<<(unsigned)((n + 7) / 8), 256, 0, h.stream>>>(h.gptr, h.woff, h.tptr, h.twoff, h.K, h.sc_G,
                                                                   h.sc_W, h.sc_Jg, h.sc_RS, h.l, h.fiber_ptr,
                                                                   h.fa_col, h.fa_val, h.tiles);
}

// Init: the pass-B stage lists. CTA c = (range, group c % G) walks its stages; stage s (tile window
// [t0, t1), patients [k0, k1)) gets at st_list + st_t[s]: 8 offsets, then for w = 0..W-1 the tiles
// of sub-range (g, w) of every patient inside the window, entry = (tile - t0) | (k - k0) << 16.
__global__ void k_stage_tab(const int64_t* __restrict__ tptr, const uint16_t* __restrict__ twoff, int64_t K, int G,
                            int W, const int64_t* __restrict__ st_f, const int32_t* __restrict__ st_k,
                            const int32_t* __restrict__ st_t, const int32_t* __restrict__ cta_st,
                            uint32_t* __restrict__ st_list) {
  const int c = blockIdx.x, grp = c % G;
  const int64_t* tp = tptr + (int64_t)grp * (K + 1);
  for (int s = cta_st[c] + threadIdx.x; s < cta_st[c + 1]; s += blockDim.x) {
    const int64_t t0 = st_f[2 * (int64_t)s], t1 = st_f[2 * (int64_t)s + 1];
    const int32_t k0 = st_k[2 * (int64_t)s], k1 = st_k[2 * (int64_t)s + 1];
    uint32_t* hdr = st_list + st_t[s];
    uint32_t* ent = hdr + 8;
    uint32_t n = 0;
    for (int w = 0; w < W; ++w) {
      hdr[w] = n;
      for (int32_t k = k0; k < k1; ++k) {
        const uint16_t* tw = twoff + ((int64_t)grp * K + k) * kWoS;
        const int64_t lo = min(max(tp[k] + tw[w], t0), t1), hi = min(max(tp[k] + tw[w + 1], t0), t1);
        for (int64_t x = lo; x < hi; ++x) ent[n++] = (uint32_t)(x - t0) | ((uint32_t)(k - k0) << 16);
      }
    }
    for (int w = W; w < 8; ++w) hdr[w] = n;
  }
}

void launch_stage_tab(Handle& h) {
  if (!h.sc_ok || h.nst == 0) return;
  k_stage_tab<<<(unsigned)(h.sc_ranges * h.sc_G), 128, 0, h.stream>>>(h.tptr, h.twoff, h.K, h.sc_G, h.sc_W, h.st_f,
                                                                      h.st_k, h.st_t, h.cta_st, h.st_list);
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
  fn<<<ctas, 32 * (W * CS + 1), h.sc_smem, h.stream>>>(h.tiles, h.sc_G, h.sc_Jg, h.st_f, h.st_k, h.st_t, h.st_list,
                                                        h.cta_st, h.l, h.R, h.sc_RS, h.sc_FB, h.sc_PB, h.sc_NS, h.Nst,
                                                        h.fv_part);
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

// Chooses the label groups G (F_V slice of a CTA), stage geometry (sc_FB = tiles per stage) and the
// number of pass-B patient ranges so that one CTA's F_V slice plus its NS-stage ring fits in shared
// memory. RS (F_V row stride) = R rounded up to even, with 2-adic order <= 3 (pair_rule).
void plan_scatter(Handle& h) {
  const size_t budget = 225 * 1024;
  h.sc_W = kScW;
  h.sc_RS = (h.R + 1) & ~1;
  if (h.sc_RS % 16 == 0) h.sc_RS += 2;
  h.sc_FB = 32;
  h.sc_ok = 0;
  const int pbs[3] = {16, 8, 4};
  for (int pass = 0; pass < 2 && !h.sc_ok; ++pass)  // pass 0: >= 3 stages of >= 8 patients
    for (int G = 1; G <= kMaxGroups && !h.sc_ok; ++G) {
      const int64_t Js = (h.J + (int64_t)G * h.sc_W - 1) / ((int64_t)G * h.sc_W);
      const int64_t Jg = Js * h.sc_W;
      const size_t fs = slice_bytes(Jg, h.sc_RS);
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
  // Larger stages (64 tiles: fewer per-stage overheads) when they still fit at the same G with >= 3
  // slots of >= 8 patients.
  if (h.sc_ok) {
    const size_t fs = slice_bytes(h.sc_Jg, h.sc_RS);
    bool done = false;
    for (int NSt = 4; NSt >= 3 && !done; --NSt)
      for (int pi = 0; pi < 2 && !done; ++pi) {
        const SlotGeom sg = slot_geom(64, pbs[pi], h.sc_W, h.l, h.R);
        const size_t bytes = fs + ((2 * NSt * 8 + 127) & ~127) + (size_t)NSt * sg.bytes;
        if (bytes <= budget) {
          h.sc_FB = 64;
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

// Tiles of the tiled stream: sum over sub-runs of ceil(n / 8) <= F / 8 + (non-empty sub-runs).
int64_t tiles_cap(const Handle& h) {
  const int64_t runs = std::min<int64_t>(h.F, (int64_t)h.sc_G * h.K * h.sc_W);
  return h.F / 8 + runs + 8;
}

// stage-list words: 8 per stage plus one per tile
int64_t stage_tab_cap(const Handle& h) { return 8 * stage_cap(h) + tiles_cap(h) + 16; }

int64_t stage_cap(const Handle& h) {
  return tiles_cap(h) / h.sc_FB + (int64_t)h.sc_G * (h.K / h.sc_PB + 1) + (int64_t)h.sc_ranges * h.sc_G + 16;
}

// ------------------------------------------------------------------ init: pass-B planning on the device
// (the host only reads back three totals: host arrays of K-proportional size cost more in page faults
// than the planning itself; measured 180 ms of host planning at Scale)
namespace {
struct ToI64 {
  __host__ __device__ int64_t operator()(int32_t x) const { return (int64_t)x; }
};

// tmp = exclusive scan of the flat [G][K] counts (GK + 1 entries) -> ptr[g][k], k = 0..K (the groups
// back to back: ptr[g][K] = ptr[g + 1][0])
__global__ void k_runs_layout(const int64_t* __restrict__ tmp, int64_t K, int G, int64_t* __restrict__ ptr) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= (int64_t)G * (K + 1)) return;
  const int64_t g = x / (K + 1), k = x - g * (K + 1);
  ptr[x] = tmp[g * K + k];
}

__device__ __forceinline__ int64_t tiles_before(const int64_t* tptr, int G, int64_t K, int64_t k) {
  int64_t c = 0;
  for (int g = 0; g < G; ++g) c += tptr[g * (K + 1) + k] - tptr[g * (K + 1)];
  return c;
}

// pass-B patient ranges balanced by tiles: block_k[b] = first k with tiles_before(k) >= total b / nr
__global__ void k_block_ranges(const int64_t* __restrict__ tptr, int G, int64_t K, int nr, int64_t* __restrict__ block_k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nr) return;
  if (b == nr) { block_k[b] = K; return; }
  const int64_t target = tiles_before(tptr, G, K, K) * b / nr;
  int64_t lo = 0, hi = K + 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (tiles_before(tptr, G, K, mid) < target) lo = mid + 1; else hi = mid;
  }
  block_k[b] = lo < K ? lo : K;
}

// Stages of CTA c = (range c / G, group c % G): from the range's first tile, a stage ends at FT tiles
// or at the PB-th patient boundary, whichever comes first (greedy walk). Warp per CTA: the walk is
// sequential, its two patient searches are warp ballots over 32 run starts. Counting pass (st_f
// null): cnt[c] = stages; writing pass: stages at cta_st[c].
__global__ void k_stage_walk(const int64_t* __restrict__ tptr, const int64_t* __restrict__ block_k, int G, int64_t K,
                             int nc, int64_t FT, int64_t PB, int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ cta_st, int64_t* __restrict__ st_f, int32_t* __restrict__ st_k) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= nc) return;
  const int r = c / G, g = c % G;
  const int64_t* gp = tptr + (int64_t)g * (K + 1);
  const int64_t kr0 = block_k[r], kr1 = block_k[r + 1];
  int64_t n = 0;
  const int64_t o = st_f ? cta_st[c] : 0;
  if (kr0 < kr1) {
    int64_t f = gp[kr0];
    const int64_t fend = gp[kr1];
    int64_t k = kr0;
    while (f < fend) {
      // first patient whose run ends after f: first k' >= k with gp[k' + 1] > f (exists: f < fend)
      for (;;) {
        const int64_t q = k + 1 + lane;
        const unsigned b = __ballot_sync(0xffffffffu, q > kr1 || gp[q] > f);
        if (b) { k += __ffs(b) - 1; break; }
        k += 32;
      }
      int64_t f1 = f + FT < fend ? f + FT : fend;
      // first kk >= k + 1 with kk >= kr1 or gp[kk] >= f1
      int64_t kk = k + 1;
      for (;;) {
        const int64_t q = kk + lane;
        const unsigned b = __ballot_sync(0xffffffffu, q >= kr1 || gp[q] >= f1);
        if (b) { kk += __ffs(b) - 1; break; }
        kk += 32;
      }
      if (kk - k > PB) {
        kk = k + PB;
        f1 = gp[kk];
      }
      if (st_f && lane == 0) {
        st_f[2 * (o + n)] = f;
        st_f[2 * (o + n) + 1] = f1;
        st_k[2 * (o + n)] = (int32_t)k;
        st_k[2 * (o + n) + 1] = (int32_t)kk;
      }
      ++n;
      f = f1;
      k = kk - 1;
    }
  }
  if (!st_f && lane == 0) cnt[c] = (int32_t)n;
}

__global__ void k_cta_scan(const int32_t* __restrict__ cnt, int nc, int32_t* __restrict__ cta_st) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int64_t a = 0;
    for (int c = 0; c < nc; ++c) {
      cta_st[c] = (int32_t)(a < INT32_MAX ? a : INT32_MAX);
      a += cnt[c];
    }
    cta_st[nc] = (int32_t)(a < INT32_MAX ? a : INT32_MAX);
  }
}

// words of every stage's list: 8 header words + one per tile (last entry 0: the exclusive scan's total)
__global__ void k_stage_len(const int64_t* __restrict__ st_f, int64_t nst, int32_t* __restrict__ len) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s > nst) return;
  len[s] = s < nst ? (int32_t)(8 + st_f[2 * s + 1] - st_f[2 * s]) : 0;
}
}  // namespace

// cub temporary bytes of the planning scans (carve): flat run counts (G K + 1) and stage lists
size_t plan_cub_bytes(const Handle& h) {
  size_t a = 0, b = 0;
  const int64_t gk = (int64_t)h.sc_G * h.K;
  cub::TransformInputIterator<int64_t, ToI64, const int32_t*> it(nullptr, ToI64());
  cub::DeviceScan::ExclusiveSum(nullptr, a, it, (int64_t*)nullptr, (int)(gk + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int32_t*)nullptr, (int32_t*)nullptr, (int)(stage_cap(h) + 1));
  return std::max(a, b);
}
int64_t plan_tmp_words(const Handle& h) {  // int64 words of the planning scratch (after the counts)
  return std::max<int64_t>((int64_t)h.sc_G * h.K + 1, stage_cap(h) + 1) + 8;
}

// gcnt / tcnt: [G][K] fiber and tile counts per run (device, k_count_groups). Writes gptr, tptr,
// block_k, cta_st, st_f, st_k, st_t and h.nst, h.ntiles; returns false if a table exceeds its bound.
bool plan_streams_device(Handle& h, const int32_t* gcnt, const int32_t* tcnt, int64_t* tmp, int64_t* gtotal) {
  cudaStream_t s = h.stream;
  const int G = h.sc_G;
  const int64_t K = h.K, GK = (int64_t)G * K, n1 = (int64_t)G * (K + 1);
  size_t tb = h.cub_temp_bytes;
  cub::TransformInputIterator<int64_t, ToI64, const int32_t*> ig(gcnt, ToI64()), it(tcnt, ToI64());
  // GK + 1 items: the last reads the zero the caller keeps one past each count array
  cub::DeviceScan::ExclusiveSum(h.cub_temp, tb, ig, tmp, (int)(GK + 1), s);
  k_runs_layout<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>(tmp, K, G, h.gptr);
  tb = h.cub_temp_bytes;
  cub::DeviceScan::ExclusiveSum(h.cub_temp, tb, it, tmp, (int)(GK + 1), s);
  k_runs_layout<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>(tmp, K, G, h.tptr);
  const int nr = h.sc_ranges, nc = nr * G;
  k_block_ranges<<<(unsigned)((nr + 1 + 127) / 128), 128, 0, s>>>(h.tptr, G, K, nr, h.block_k);
  int32_t* cnt = reinterpret_cast<int32_t*>(tmp);
  k_stage_walk<<<(unsigned)((nc + 1) / 2), 64, 0, s>>>(h.tptr, h.block_k, G, K, nc, h.sc_FB, h.sc_PB, cnt, nullptr,
                                                       nullptr, nullptr);
  k_cta_scan<<<1, 32, 0, s>>>(cnt, nc, h.cta_st);
  int64_t tot[3] = {0, 0, 0};  // stages, tiles, fibers
  int32_t nst32 = 0;
  cudaMemcpyAsync(&nst32, h.cta_st + nc, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&tot[1], h.tptr + n1 - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&tot[2], h.gptr + n1 - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return false;
  h.nst = nst32;
  h.ntiles = tot[1];
  *gtotal = tot[2];
  if (h.nst >= INT32_MAX || h.nst > h.nst_cap || h.ntiles > tiles_cap(h) || tot[2] > h.F ||
      8 * h.nst + h.ntiles > stage_tab_cap(h) || stage_tab_cap(h) > INT32_MAX)
    return false;
  k_stage_walk<<<(unsigned)((nc + 1) / 2), 64, 0, s>>>(h.tptr, h.block_k, G, K, nc, h.sc_FB, h.sc_PB, nullptr,
                                                       h.cta_st, h.st_f, h.st_k);
  int32_t* len = reinterpret_cast<int32_t*>(tmp);
  k_stage_len<<<(unsigned)((h.nst + 1 + 255) / 256), 256, 0, s>>>(h.st_f, h.nst, len);
  tb = h.cub_temp_bytes;
  cub::DeviceScan::ExclusiveSum(h.cub_temp, tb, len, h.st_t, (int)(h.nst + 1), s);
  return true;
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
