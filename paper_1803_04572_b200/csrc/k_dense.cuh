// k_dense.cuh — per-patient dense work of the smooth ("wide": m_k <= l < R) path, organised in
// warp rounds of 32 patients: the R-dimension contractions run on the FP64 tensor cores
// (mma.sync m8n8k4 f64, warp-cooperative, one patient per MMA tile) and the small sequential
// m_k x m_k algebra (Givens QR, one-sided Jacobi, row ADMM solves) runs one patient per thread.
//
//   polar_wide : A_k = P'_k S_k H̄^T (MMA, 8-column slabs) -> Givens QR of A_k^T (thread)
//                -> Jacobi (thread) -> Q~_k = K_k A_k (thread, K_k = V Σ^-1 V^T on the range)
//                -> F_H += Q~_k^T P'_k S_k (MMA, per-warp accumulators)        (Alg.1 l.4-6, l.12)
//   passB_wide : T_k = Q~_k H̄ (MMA) -> F_W(k,:) = colsum(T_k ∘ P'_k) -> W-row ADMM (thread)
//                -> N_k = T_k S_k (MMA recompute) -> M += N_k^T N_k, W̄^T W̄ (MMA)  (l.12-19, FIT)
// Templates of the wide per-patient kernels; instantiated by k_polar_l*.cu and k_passB_m*.cu
// (split so that the heavily unrolled instantiations compile in parallel).
#pragma once
#include <algorithm>
#include <cstdlib>

#include "copa_internal.cuh"

namespace copa {

__device__ __forceinline__ void dmma2(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void pf_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// Prefetch the byte range [p, p + bytes) with the 32 lanes of a warp (128-byte lines).
__device__ __forceinline__ void warp_prefetch(const void* p, size_t bytes, bool to_l1) {
  const int lane = threadIdx.x & 31;
  const char* c = (const char*)((uintptr_t)p & ~(uintptr_t)127);
  const char* e = (const char*)p + bytes;
  for (const char* x = c + 128 * lane; x < e; x += 128 * 32) {
    if (to_l1) pf_l1(x); else pf_l2(x);
  }
}

// Prefetch the state rows of patients [base, base + 32) (srow-contiguous) and their W rows.
__device__ __forceinline__ void round_prefetch(int64_t base, int64_t K, int R, const int64_t* srow, const double* A,
                                               const double* B, const double* Wrows, bool to_l1) {
  if (base >= K) return;
  int64_t last = base + 32 < K ? base + 32 : K;
  int64_t s0 = srow[base], s1 = srow[last];
  warp_prefetch(A + s0 * R, sizeof(double) * (size_t)((s1 - s0) * R), to_l1);
  if (B) warp_prefetch(B + s0 * R, sizeof(double) * (size_t)((s1 - s0) * R), to_l1);
  if (Wrows) warp_prefetch(Wrows + base * R, sizeof(double) * (size_t)((last - base) * R), to_l1);
}

// Givens insert of column vector c[0..L) into the upper-triangular Rf (L x L, registers).
template <int L>
__device__ __forceinline__ void givens_insert_reg(double (&Rf)[L][L], double (&c)[L]) {
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const double aj = c[j];
    if (aj != 0.0) {
      const double r = Rf[j][j];
      const double n2 = fma(r, r, aj * aj);
      const double inv = rsqrt(n2);
      const double cs = r * inv, sn = aj * inv;
      Rf[j][j] = n2 * inv;
#pragma unroll
      for (int t = j + 1; t < L; ++t) {
        const double x = Rf[j][t], y = c[t];
        Rf[j][t] = fma(cs, x, sn * y);
        c[t] = fma(cs, y, -sn * x);
      }
    }
  }
}

// One-sided Jacobi on the rows of Wm (L x L, registers) until mutually orthogonal. Round-robin
// (tournament) ordering: every round rotates floor(L/2) disjoint row pairs, whose dot products and
// rotation parameters are independent (instruction-level parallelism in the thread-per-patient
// layout); a sweep (L-1 or L rounds) meets every pair once. Each rotation is jacobi_rot()
// (copa_internal.cuh: Hestenes' angle from two reciprocal square roots).
constexpr double kJacobiDoneCos2 = 1e-24;  // (1e-12)^2, see jacobi_rows_reg

template <int L>
__device__ __forceinline__ void jacobi_rows_reg(double (&Wm)[L][L]) {
  constexpr int N = (L % 2) ? L + 1 : L;  // players, with a dummy (index L) when L is odd
  constexpr double eps = 2.220446049250313e-16 * (double)L;
  constexpr double tol2 = eps * eps;
  double tr = 0.0;  // trace of the Gram (invariant under the rotations): residue-row threshold
#pragma unroll
  for (int p = 0; p < L; ++p)
#pragma unroll
    for (int x = 0; x < L; ++x) tr = fma(Wm[p][x], Wm[p][x], tr);
  const double negl = kJacobiNegl2 * tr;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0, big = 0;  // big: some rotation of this sweep had (x.y)^2 > 1e-24 |x|^2 |y|^2
#pragma unroll
    for (int rd = 0; rd < N - 1; ++rd) {
      double cs[N / 2], sn[N / 2];
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const int p = i == 0 ? 0 : 1 + (i - 1 + rd) % (N - 1);
        const int q = 1 + (N - 2 - i + rd) % (N - 1);
        cs[i] = 1.0;
        sn[i] = 0.0;
        if (p < L && q < L) {
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
          for (int x = 0; x < L; ++x) {
            a = fma(Wm[p][x], Wm[p][x], a);
            b = fma(Wm[q][x], Wm[q][x], b);
            c = fma(Wm[p][x], Wm[q][x], c);
          }
          if (a > negl && b > negl && c * c > tol2 * (a * b)) {
            rotated = 1;
            big |= c * c > kJacobiDoneCos2 * (a * b);
            jacobi_rot(a, b, c, cs[i], sn[i]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const int p = i == 0 ? 0 : 1 + (i - 1 + rd) % (N - 1);
        const int q = 1 + (N - 2 - i + rd) % (N - 1);
        if (p < L && q < L) {
#pragma unroll
          for (int x = 0; x < L; ++x) {
            const double u = Wm[p][x], v = Wm[q][x];
            Wm[p][x] = fma(cs[i], u, -sn[i] * v);
            Wm[q][x] = fma(sn[i], u, cs[i] * v);
          }
        }
      }
    }
    // converged when no pair needed a rotation, or when every rotation of this sweep was below
    // 1e-12 in cosine (the sweep has left the rows orthogonal to ~1e-24 (quadratic convergence); a
    // further sweep would only confirm it)
    if (__all_sync(0xffffffffu, rotated == 0 || !big)) break;
  }
}

__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kRing = 4;  // patients staged ahead (per warp) by the cp.async rings of the wide kernels
constexpr int kRingA = 3; // ... by the polar A-slab ring (smaller, for 3 polar CTAs per SM)
// F_H ring depth of the wide polar: 3 for l > 8, so that the ring fits in the A slab it reuses
__host__ __device__ constexpr int polar_fh_ring(int L) { return L > 8 ? 3 : kRing; }
constexpr bool kSplitK = false;  // even/odd k-step accumulators in the A slabs (changes rounding order)

__device__ __forceinline__ uint32_t su32d(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Per-warp ring of kRing patient records in shared memory: record p holds NSEG segments (segment j:
// len[j] doubles from src[j] + p stride[j]). BULK: one lane issues 1-D TMA bulk copies completing on
// the slot's mbarrier (all segments 16-byte aligned: R even); otherwise every lane issues 8-byte
// cp.async granules (any alignment) as one commit group per record. issue(p) fills slot p % kRing;
// wait(p) makes record p visible to the whole warp. init() (re)arms the barriers for a new pass.
template <int NSEG, bool BULK, int NR = kRing>
struct WarpRing {
  double* buf;
  uint64_t* bar;           // NR mbarriers (BULK), armed once per kernel (ring_bars_init)
  int q0;                  // records issued by earlier passes of this warp (slot / phase continuity)
  int per;                 // doubles per record
  const double* src[NSEG];
  int64_t stride[NSEG];
  int len[NSEG];
  __device__ __forceinline__ double* slot(int p) const { return buf + ((q0 + p) % NR) * per; }
  __device__ __forceinline__ void issue(int p, int np) {
    if (BULK) {
      if (p < np && (threadIdx.x & 31) == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior reads of the slot first
        uint64_t* b = bar + ((q0 + p) % NR);
        uint32_t tx = 0;
#pragma unroll
        for (int j = 0; j < NSEG; ++j) tx += 8u * (uint32_t)len[j];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32d(b)), "r"(tx) : "memory");
        double* dst = slot(p);
#pragma unroll
        for (int j = 0; j < NSEG; ++j) {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32d(dst)),
              "l"(src[j] + (int64_t)p * stride[j]), "r"(8u * (uint32_t)len[j]), "r"(su32d(b))
              : "memory");
          dst += len[j];
        }
      }
    } else {
      if (p < np) {
        const int lane = threadIdx.x & 31;
        double* dst = slot(p);
#pragma unroll
        for (int j = 0; j < NSEG; ++j) {
          const double* sp = src[j] + (int64_t)p * stride[j];
          for (int x = lane; x < len[j]; x += 32) cpa8(dst + x, sp + x);
          dst += len[j];
        }
      }
      cpa_commit();
    }
  }
  __device__ __forceinline__ void wait(int p) {
    if (BULK) {
      const int q = q0 + p;
      const uint32_t a = su32d(bar + (q % NR)), parity = (uint32_t)((q / NR) & 1);
      asm volatile(
          "{\n .reg .pred P1;\n"
          "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
          "DONE%=:\n}" ::"r"(a),
          "r"(parity)
          : "memory");
    } else {
      cpa_wait<NR - 1>();
      __syncwarp();
    }
  }
  // records p and p + 1 (consumed in pairs; the pair loop issues two groups per step)
  __device__ __forceinline__ void wait_pair(int p, bool two) {
    if (BULK) {
      wait(p);
      if (two) wait(p + 1);
    } else {
      cpa_wait<NR - 2>();
      __syncwarp();
    }
  }
  __device__ __forceinline__ void drain() {
    if (!BULK) cpa_wait<0>();
  }
};

__device__ __forceinline__ void ring_bars_init(uint64_t* bar, int n = kRing) {
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < n; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32d(bar + i)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

// Warp-cooperative A slab: slab[p][a][cc] = A_p(a, s = 8 nt + cc) for the round's patients.
// A_p = P'_p S_p H^T. MMA: M = a (MT tiles), N = s (this slab), K = r (KS steps). Rows a >= m_p of
// P'_p are zero (never written), so only a < l is checked. P'_p and w̄_p arrive through the warp's
// cp.async ring, kRing patients ahead of the MMAs.
//
// FAST (MT == 1, l >= 7, R % 4 == 0): fragment loads without masks from a per-lane base. Every K
// index r = 4 ks + t is < R; the only out-of-range operand row is a = g >= l (g = 7 when l = 7),
// which reads in-record values (the w̄ part) and only feeds row 7 of D, never stored.
template <int MT, int KS, bool BULK, int SR, bool FAST = false>
__device__ __forceinline__ void a_slab(int nt, int64_t base, int64_t K, int l, int R, const double* Pp,
                                       const double* W, const double* Hs, double* slab, double* ringbuf,
                                       uint64_t* bars, int& q0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int s = 8 * nt + g;
  double hb[KS];
  int offp[KS][MT];  // lane's fragment offsets inside a patient's P' block (-1: outside)
  int offw[KS];
  const int lR = l * R;
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int r = 4 * ks + t;
    hb[ks] = (r < R && s < R) ? Hs[s * R + r] : 0.0;  // B[t][g] = H^T(r, s)
    offw[ks] = r < R ? lR + r : -1;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = 8 * mt + g;
      offp[ks][mt] = (a < l && r < R) ? a * R + r : -1;
    }
  }
  const int np = (int)(K - base < 32 ? K - base : 32);
  WarpRing<2, BULK, kRingA> ring;
  ring.buf = ringbuf;
  ring.bar = bars;
  ring.q0 = q0;
  ring.per = lR + R;
  ring.src[0] = Pp + base * lR;
  ring.stride[0] = lR;
  ring.len[0] = lR;
  ring.src[1] = W + base * R;
  ring.stride[1] = R;
  ring.len[1] = R;
#pragma unroll
  for (int p = 0; p < kRingA; ++p) ring.issue(p, np);
  for (int p = 0; p < np; ++p) {
    ring.wait(p);
    const double* rec = ring.slot(p);
    double c[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) c[mt][0] = c[mt][1] = 0.0;
    if (FAST) {
      const double* ra = rec + g * R + t;
      const double* rw = rec + lR + t;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma2(c[0][0], c[0][1], ra[4 * ks] * rw[4 * ks], hb[ks]);
    } else {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double wr = offw[ks] >= 0 ? rec[offw[ks]] : 0.0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double av = offp[ks][mt] >= 0 ? rec[offp[ks][mt]] * wr : 0.0;  // A[g][t] = (P'S)(a, r)
          dmma2(c[mt][0], c[mt][1], av, hb[ks]);
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
      if (8 * mt + g < SR)
        *reinterpret_cast<double2*>(slab + (p * SR + 8 * mt + g) * 8 + 2 * t) = make_double2(c[mt][0], c[mt][1]);
    __syncwarp();  // slot p fully read before it is refilled
    ring.issue(p + kRingA, np);
  }
  ring.drain();
  q0 += np;
  for (int p = np; p < 32; ++p)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
      if (8 * mt + g < SR)
        *reinterpret_cast<double2*>(slab + (p * SR + 8 * mt + g) * 8 + 2 * t) = make_double2(0.0, 0.0);
}

template <int L, int MT, int NT, int RT, int LT>
__global__ void __launch_bounds__(128, (L > 8 ? 1 : 3)) k_polar_wide(const int32_t* __restrict__ m, int64_t K, int R_, int l_,
                                                       const double* __restrict__ Pp, const double* __restrict__ W,
                                                       const double* __restrict__ Hg, double tau,
                                                       double* __restrict__ Qt, int32_t* __restrict__ rank,
                                                       double* __restrict__ FHwarp, int nextpf,
                                                       unsigned long long* __restrict__ diag) {
  constexpr int KS = RT ? (RT + 3) / 4 : (NT * 8 + 3) / 4;  // r steps of 4 covering R (an all-zero step
                                                             // costs a DMMA like any other)
  // fixed-shape slab path: unmasked fragment loads (needs l >= 7, one M tile, R % 4 == 0; see a_slab)
  constexpr bool FAST = MT == 1 && LT >= 7 && RT > 0 && RT % 4 == 0;
  constexpr int RP = 8 * NT;
  const int R = RT ? RT : R_;           // compile-time for the configured (R, l) pairs
  const int l = LT ? LT : l_;
  extern __shared__ double sm[];
  const int hoff = ((R * R + 31) / 32) * 32;
  double* Hs = sm;                                      // R x R
  const int wib = threadIdx.x >> 5;
  constexpr bool BULK = RT > 0 && (RT % 2) == 0;     // 16-byte aligned records: TMA bulk copies
  constexpr int SR = LT ? LT : MT * 8;                 // A rows kept per patient in the slab
  constexpr int NRF = polar_fh_ring(L);  // F_H ring depth
  // per warp: a-slab ring + 2 barrier sets, kept a multiple of 2 doubles (16-byte bulk-copy alignment)
  const int ringd = kRingA * (l * R + R) + ((kRingA + NRF + 1) & ~1);
  // per warp: slab of 32 patients x SR x 8, reused as the F_H ring (NRF x (2 l R + R))
  const int slabd = 32 * SR * 8 > NRF * (2 * l * R + R) ? 32 * SR * 8 : NRF * (2 * l * R + R);
  double* slab = sm + hoff + wib * (slabd + ringd);
  double* ringbuf = slab + slabd;
  uint64_t* bars = (uint64_t*)(ringbuf + kRingA * (l * R + R));  // kRingA (a-slab ring)
  uint64_t* barsf = bars + kRingA;                                 // NRF (F_H ring)
  if (BULK) {
    ring_bars_init(bars, kRingA);
    ring_bars_init(barsf, NRF);
  }
  int q0 = 0, qf = 0;  // records pulled through each ring (mbarrier phase continuity)
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Hs[x] = Hg[x];
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t rounds = (K + 31) / 32;
  const int64_t pstride = (int64_t)l * R;
  // this warp's F_H partial (RP x RP, MMA fragment order), accumulated round by round
  double* fhw = FHwarp + ((int64_t)blockIdx.x * (blockDim.x >> 5) + wib) * (RP * RP) + lane;
#pragma unroll
  for (int x = 0; x < NT * NT * 2; ++x) fhw[32 * x] = 0.0;
  for (int64_t rd = blockIdx.x * (blockDim.x >> 5) + wib; rd < rounds; rd += nwarps_total) {
    const int64_t base = rd * 32;
    {  // prefetch the next round's P' and W rows into L2
      const int64_t nb = base + 32 * (int64_t)nwarps_total;
      if (nextpf && nb < K) {
        const int64_t nl = nb + 32 < K ? nb + 32 : K;
        warp_prefetch(Pp + nb * pstride, sizeof(double) * (size_t)((nl - nb) * pstride), false);
        warp_prefetch(W + nb * R, sizeof(double) * (size_t)((nl - nb) * R), false);
      }
    }
    const int64_t kme = base + lane;
    const int mme = kme < K ? m[kme] : 0;
    // ---- Givens QR of A^T (rows of A^T = columns of A), slab by slab
    double Rf[L][L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
      for (int j = 0; j < L; ++j) Rf[i][j] = 0.0;
#pragma unroll 1
    for (int nt = 0; nt < NT; ++nt) {
      a_slab<MT, KS, BULK, SR, FAST>(nt, base, K, l, R, Pp, W, Hs, slab, ringbuf, bars, q0);
      __syncwarp();
#pragma unroll 1
      for (int cc = 0; cc < 8; ++cc) {
        if (8 * nt + cc < R) {
          double col[L];
#pragma unroll
          for (int a = 0; a < L; ++a) col[a] = slab[(lane * SR + a) * 8 + cc];
          givens_insert_reg<L>(Rf, col);
        }
      }
      __syncwarp();
    }
    // ---- SVD of the m x m factor: rows of Rf -> sigma_j v_j; u_j = v_j / sqrt(sigma_j) so that
    //      K = sum_kept u_j u_j^T = V Σ^-1 V^T on the numerical range (reading R-polar-2/3)
    jacobi_rows_reg<L>(Rf);
    double smax = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) s = fma(Rf[j][i], Rf[j][i], s);
      smax = fmax(smax, s);
    }
    smax = sqrt(smax);
    int rk = 0;
    RatioDiag dg;  // rank-cut diagnostics (copa_stats)
#pragma unroll
    for (int j = 0; j < L; ++j) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) s = fma(Rf[j][i], Rf[j][i], s);
      const double sg = sqrt(s);
      const bool keep = smax > 0.0 && sg > tau * smax;
      if (smax > 0.0 && j < mme) dg.note(sg / smax, keep, tau);
      rk += keep ? 1 : 0;
      const double sc = keep ? 1.0 / (sg * sqrt(sg)) : 0.0;
#pragma unroll
      for (int i = 0; i < L; ++i) Rf[j][i] *= sc;
    }
    if (kme < K) rank[kme] = mme > 0 ? rk : 0;
    ratio_diag_warp(diag, D_POLAR_NEAR, dg);
    // ---- Q~ = K A, slab by slab (A recomputed on the tensor cores)
#pragma unroll 1
    for (int nt = 0; nt < NT; ++nt) {
      a_slab<MT, KS, BULK, SR, FAST>(nt, base, K, l, R, Pp, W, Hs, slab, ringbuf, bars, q0);
      __syncwarp();
      if (kme < K && mme > 0) {
        double* Q = Qt + kme * pstride;
#pragma unroll 1
        for (int cc = 0; cc < 8; ++cc) {
          const int s = 8 * nt + cc;
          if (s < R) {
            double y[L];
#pragma unroll
            for (int a = 0; a < L; ++a) y[a] = slab[(lane * SR + a) * 8 + cc];
            double q[L];
#pragma unroll
            for (int a = 0; a < L; ++a) q[a] = 0.0;
#pragma unroll
            for (int j = 0; j < L; ++j) {
              double d = 0.0;
#pragma unroll
              for (int a = 0; a < L; ++a) d = fma(Rf[j][a], y[a], d);
#pragma unroll
              for (int a = 0; a < L; ++a) q[a] = fma(Rf[j][a], d, q[a]);
            }
#pragma unroll
            for (int a = 0; a < L; ++a)
              if (a < mme) Q[a * R + s] = q[a];
          }
        }
      }
      __syncwarp();
    }
    // Q~ rows were just written by this warp's threads (generic proxy) and are read back below by
    // TMA bulk copies (async proxy): every writer fences its stores into the async proxy first.
    if (BULK) asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    // ---- F_H += Q~_p^T (P'_p S_p): MMA with M = r, N = s, K = a (rows a >= m_p are zero)
    {
      int offq[2 * MT][NT];
      int offw[NT];
#pragma unroll
      for (int ks = 0; ks < 2 * MT; ++ks)
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          const int a = 4 * ks + t, rr = 8 * i + g;
          offq[ks][i] = (a < l && rr < R) ? a * R + rr : -1;
        }
#pragma unroll
      for (int i = 0; i < NT; ++i) offw[i] = 8 * i + g < R ? 8 * i + g : -1;
      double fh[NT][NT][2];
#pragma unroll
      for (int a = 0; a < NT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) fh[a][b][0] = fh[a][b][1] = 0.0;
      const int np = (int)(K - base < 32 ? K - base : 32);
      const int lR = l * R;
      WarpRing<3, BULK, NRF> ring;  // record: Q~_p (l R), P'_p (l R), w̄_p (R), staged in the (free) slab
      ring.buf = slab;
      ring.bar = barsf;
      ring.q0 = qf;
      ring.per = 2 * lR + R;
      ring.src[0] = Qt + base * lR;
      ring.stride[0] = lR;
      ring.len[0] = lR;
      ring.src[1] = Pp + base * lR;
      ring.stride[1] = lR;
      ring.len[1] = lR;
      ring.src[2] = W + base * R;
      ring.stride[2] = R;
      ring.len[2] = R;
#pragma unroll
      for (int p = 0; p < NRF; ++p) ring.issue(p, np);
      for (int p = 0; p < np; ++p) {
        ring.wait(p);
        const double* rec = ring.slot(p);
        double wv[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) wv[i] = offw[i] >= 0 ? rec[2 * lR + offw[i]] : 0.0;
        double af[2 * MT][NT], bf[2 * MT][NT];
#pragma unroll
        for (int ks = 0; ks < 2 * MT; ++ks)
#pragma unroll
          for (int i = 0; i < NT; ++i) {
            af[ks][i] = offq[ks][i] >= 0 ? rec[offq[ks][i]] : 0.0;               // A[g][t] = Q~^T(r, a)
            bf[ks][i] = offq[ks][i] >= 0 ? rec[lR + offq[ks][i]] * wv[i] : 0.0;  // B[t][g] = (P'S)(a, s)
          }
#pragma unroll
        for (int ks = 0; ks < 2 * MT; ++ks)
#pragma unroll
          for (int i = 0; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma2(fh[i][j][0], fh[i][j][1], af[ks][i], bf[ks][j]);
        __syncwarp();
        ring.issue(p + NRF, np);
      }
      ring.drain();
      qf += np;
      __syncwarp();  // the slab is rewritten by the next round
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int c = 0; c < 2; ++c) fhw[32 * ((i * NT + j) * 2 + c)] += fh[i][j][c];
    }
  }
}

// F_H = sum over warps (fixed order) of the fragment-ordered partials
// F_H = sum over the per-warp fragment-ordered partials, in a fixed order (deterministic):
// stage 1 sums kFhChunks contiguous warp chunks per fragment position, stage 2 sums the chunks.
constexpr int kFhChunks = 32;
static __global__ void k_sum_fh1(const double* __restrict__ part, int nw, int P, double* __restrict__ tmp) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= P) return;
  const int c = blockIdx.y;
  const int w0 = (int)((int64_t)nw * c / kFhChunks), w1 = (int)((int64_t)nw * (c + 1) / kFhChunks);
  double v = 0.0;
  for (int w = w0; w < w1; ++w) v += part[(int64_t)w * P + pos];
  tmp[(int64_t)c * P + pos] = v;
}
static __global__ void k_sum_fh(const double* __restrict__ tmp, int R, int NT, double* __restrict__ FH) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= R * R) return;
  const int r = x / R, s = x - r * R;
  // fragment position of (r, s): tile (i = r/8, j = s/8), lane g = r%8, t = (s%8)/2, c = s%2
  const int i = r >> 3, j = s >> 3, g = r & 7, t = (s & 7) >> 1, c = s & 1;
  const int off = 32 * ((i * NT + j) * 2 + c) + g * 4 + t;
  const int P = 64 * NT * NT;
  double v = 0.0;
  for (int ch = 0; ch < kFhChunks; ++ch) v += tmp[(int64_t)ch * P + off];
  FH[x] = v;
}

static __global__ void k_sum_rr(const double* part, int nb, int n, double* out) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * n + x];
  out[x] = s;
}

constexpr int kDenseThreads = 128;

template <int L, int NT, int RT = 0, int LT = 0>
static void polar_wide_inst(Handle& h) {
  constexpr int MT = (L + 7) / 8;
  constexpr auto fn = k_polar_wide<L, MT, NT, RT, LT>;
  const size_t hoff = (size_t)((h.R * h.R + 31) / 32) * 32;
  constexpr int SR = LT ? LT : MT * 8;
  constexpr int NRF = polar_fh_ring(L);
  const size_t slabd = (size_t)std::max(32 * SR * 8, NRF * (2 * h.l * h.R + h.R));
  const size_t per_warp = slabd + (size_t)(kRingA * (h.l * h.R + h.R) + ((kRingA + NRF + 1) & ~1));
  max_smem_attr<fn>(h);
  // warps per block (4, 2 or 1): the one with the most resident warps per SM (the R x R H̄ copy is
  // per block, so large per-warp slabs can favour smaller blocks)
  int wpb = 1, per_sm = 1, best = -1;
  for (int cand = kDenseThreads / 32; cand >= 1; cand /= 2) {
    const size_t sm_c = sizeof(double) * (hoff + cand * per_warp);
    if (sm_c > 227 * 1024) continue;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * cand, sm_c);
    if (occ * cand > best) { best = occ * cand; wpb = cand; per_sm = occ; }
  }
  const int threads = 32 * wpb;
  size_t smem = sizeof(double) * (hoff + wpb * per_warp);
  int64_t rounds = (h.K + 31) / 32;
  int64_t blocks = (rounds + wpb - 1) / wpb;
  int64_t cap = h.sms * (int64_t)(per_sm > 0 ? per_sm : 1);
  if (cap > kPartBlocks * 4 / wpb) cap = kPartBlocks * 4 / wpb;  // fh_warp holds kPartBlocks x 4 warps
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  fn<<<(unsigned)blocks, threads, smem, h.stream>>>(h.m, h.K, h.R, h.l, h.Pp, h.W, h.H, h.o.rank_tol, h.Qt, h.rank,
                                                    h.fh_warp, 0, h.diag);
  const int RR = h.R * h.R;
  const int P = 64 * NT * NT;
  k_sum_fh1<<<dim3((P + 127) / 128, kFhChunks), 128, 0, h.stream>>>(h.fh_warp, (int)blocks * wpb, P, h.partial);
  k_sum_fh<<<(RR + 255) / 256, 256, 0, h.stream>>>(h.partial, h.R, NT, h.FH);
}

template <int L>
static void polar_wide_n(Handle& h) {
  // compile-time (R, l) for the BASELINE configs (Medium, Large, Scale); generic otherwise
  if (L == 7 && h.l == 7 && h.R == 20) { polar_wide_inst<7, 3, 20, 7>(h); return; }
  if (L == 7 && h.l == 7 && h.R == 15) { polar_wide_inst<7, 2, 15, 7>(h); return; }
  if (L == 9 && h.l == 9 && h.R == 40) { polar_wide_inst<9, 5, 40, 9>(h); return; }
  switch ((h.R + 7) / 8) {
    case 1: polar_wide_inst<L, 1>(h); break;
    case 2: polar_wide_inst<L, 2>(h); break;
    case 3: polar_wide_inst<L, 3>(h); break;
    case 4: polar_wide_inst<L, 4>(h); break;
    case 5: polar_wide_inst<L, 5>(h); break;
    case 6: polar_wide_inst<L, 6>(h); break;
    case 7: polar_wide_inst<L, 7>(h); break;
    default: polar_wide_inst<L, 8>(h); break;
  }
}

// ------------------------------------------------------------------ pass B (wide): F_W, W ADMM, N, M, W^T W
// Per patient p of a warp round (one MMA tile set per patient, the next patient's fragments loaded
// while the current one's MMAs run):
//   T_p = Q~_p H̄ (MMA: M = a, N = r, K = i), F_W(p, r) = sum_a T_p(a, r) P'_p(a, r)   (Alg.1 l.12, W mode)
// thread per patient: 5 ADMM row steps z = Ginv (f + rho (w̄ + d)), w̄ = prox(z - d), d += w̄ - z with
//   Ginv = (G_W + rho I)^-1 formed once from the cached Cholesky factor (k_admm_H)          (l.13-19)
//   N_p = T_p S_p (new w̄_p) -> HBM, M += N_p^T N_p (MMA via the warp's smem scratch), W̄^T W̄ += w̄ w̄^T
// W-row ADMM with the per-row stop of reading R-inner-tol (used when admm_tol > 0): the same steps
// as the fixed-count loop in k_passB_wide on the [r * 32] strided shared-memory rows of one lane.
static __device__ __noinline__ int w_row_admm_tol(const double* Gs, int R, const double* fw, double* wb, double* dd,
                                           double rho, int n_inner, int kind, double param, double tol) {
  double rhs[kMaxR];
  int it = 0;
  while (it < n_inner) {
    for (int r = 0; r < R; ++r) rhs[r] = fw[r * 32] + rho * (wb[r * 32] + dd[r * 32]);
    RowResid res;
    for (int r = 0; r < R; ++r) {
      double z = 0.0;
      for (int q = 0; q < R; ++q) z = fma(Gs[r * R + q], rhs[q], z);
      const double d0 = dd[r * 32];
      const double nb = prox(kind, param, rho, z - d0);
      res.add(nb, z, wb[r * 32]);
      dd[r * 32] = d0 + nb - z;
      wb[r * 32] = nb;
    }
    ++it;
    if (res.done(tol)) break;
  }
  return it;
}

template <int MT, int NT, int RT, int LT>
__global__ void __launch_bounds__(128) k_passB_wide(int64_t K, int R_, int l_, const double* __restrict__ Pp,
                                                    const double* __restrict__ Qt, const double* __restrict__ Hg,
                                                    const double* __restrict__ GWi, const double* __restrict__ scal,
                                                    int n_inner, int kind, double param, double tol,
                                                    double* __restrict__ W, double* __restrict__ DW,
                                                    double* __restrict__ Nst,
                                                    double* __restrict__ part /* [blocks][2][R R] */,
                                                    int l1_prefetch, int nextpf, unsigned long long* __restrict__ steps) {
  constexpr int RP = 8 * NT;
  constexpr int KS = RT ? (RT + 3) / 4 : (NT * 8 + 3) / 4;  // i steps of 4 covering R
  const int R = RT ? RT : R_;
  const int l = LT ? LT : l_;
  extern __shared__ double sm[];
  const int hoff = ((R * R + 31) / 32) * 32;
  constexpr int KA = 2 * NT;       // k-steps of the batched W-row solves (K = columns, permuted, see below)
  // Shared memory (passB_wide_smem): H̄ [R x R] | (G_W + rho I)^-1 as MMA B fragments [KA][NT][lane] |
  // with the per-row stop only: (G_W + rho I)^-1 [R x R] | per warp: F_W and w̄ as [r][lane] (+ d as
  // [r][lane] and a separate N scratch with the per-row stop; otherwise the N scratch reuses the F_W
  // rows, dead after the solves, and d stays in registers).
  const bool tolpath = tol > 0.0;
  // TBUF (fixed steps, small tiles): the round runs as four sub-rounds of 8 patients and keeps each
  // patient's T = Q~ H̄ fragments in shared memory between the F_W and N steps (no recompute, no
  // second read of Q~); per warp: F_W [RP][8], w̄ [RP][8], N scratch, T [8][MT][NT][2][lane]
  constexpr bool TBUF_OK = MT * NT <= 4;
  const bool tbuf = TBUF_OK && !tolpath;
  double* Hs = sm;
  double* gfr = sm + hoff;
  double* Gs = tolpath ? gfr + KA * NT * 32 : nullptr;
  const int fwd = RP * 32 > MT * 8 * RP ? RP * 32 : MT * 8 * RP;
  const int per_warp = tolpath ? 3 * RP * 32 + MT * 8 * RP
                       : tbuf ? 2 * RP * 8 + MT * 8 * RP + 8 * 32 * MT * NT * 2 : fwd + RP * 32;
  const int wib = threadIdx.x >> 5;
  double* wv = sm + hoff + KA * NT * 32 + (tolpath ? hoff : 0) + wib * per_warp;
  double* fwv = wv;
  double* wbv = tolpath ? wv + RP * 32 : tbuf ? wv + RP * 8 : wv + fwd;
  double* dv = tolpath ? wv + 2 * RP * 32 : nullptr;
  double* ns = tolpath ? wv + 3 * RP * 32 : tbuf ? wv + 2 * RP * 8 : wv;  // N_p (MT 8 x RP)
  double* tb = tbuf ? ns + MT * 8 * RP : nullptr;
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    Hs[x] = Hg[x];
    if (tolpath) Gs[x] = GWi[x];
  }
  // Batched W-row solve z_p = Ginv rhs_p of a warp round as MMAs (M = 8 patients, N = r, K = q) whose
  // A operand is the rhs in accumulator (C) layout: k-step ks, lane t covers column
  // q = 8 (ks / 2) + 2 t + ks % 2 — exactly the C-fragment element (n-tile ks / 2, ks % 2) a lane
  // holds, so the ADMM steps need no shuffles. B[t][g] = Ginv^T(q, r = 8 nt + g) = Ginv(r, q).
  for (int x = threadIdx.x; x < KA * NT * 32; x += blockDim.x) {
    const int ln = x & 31, nt = (x >> 5) % NT, ks = (x >> 5) / NT;
    const int q = 8 * (ks >> 1) + 2 * (ln & 3) + (ks & 1), r = 8 * nt + (ln >> 2);
    gfr[x] = (q < R && r < R) ? GWi[r * R + q] : 0.0;
  }
  __syncthreads();
  const double rho = scal[S_RHO_W];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const int64_t rounds = (K + 31) / 32;
  const int64_t pstride = (int64_t)l * R;
  // lane-constant fragment offsets (-1: padding)
  int offq[KS][MT];   // A[g][t] = Q~(a = 8 mt + g, i = 4 ks + t)
  int offp[MT][NT][2];  // C-layout (a = 8 mt + g, r = 8 nt + 2 t + c)
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = 8 * mt + g, i = 4 * ks + t;
      offq[ks][mt] = (a < l && i < R) ? a * R + i : -1;
    }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int a = 8 * mt + g, r = 8 * nt + 2 * t + c;
        offp[mt][nt][c] = (a < l && r < R) ? a * R + r : -1;
      }
  double hb[KS][NT];  // B[t][g] = H̄(i = 4 ks + t, r = 8 nt + g), kept in registers
#pragma unroll
  for (int ks = 0; ks < KS; ++ks)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int i = 4 * ks + t, r = 8 * nt + g;
      hb[ks][nt] = (i < R && r < R) ? Hs[i * R + r] : 0.0;
    }
  auto load_q = [&](const double* Q, double (&f)[KS][MT]) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) f[ks][mt] = offq[ks][mt] >= 0 ? Q[offq[ks][mt]] : 0.0;
  };
  auto t_mma = [&](const double (&f)[KS][MT], double (&c)[MT][NT][2]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) c[mt][nt][0] = c[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma2(c[mt][nt][0], c[mt][nt][1], f[ks][mt], hb[ks][nt]);
  };
  double macc[NT][NT][2], wacc[NT][NT][2];
#pragma unroll
  for (int a = 0; a < NT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) macc[a][b][0] = macc[a][b][1] = wacc[a][b][0] = wacc[a][b][1] = 0.0;
  for (int64_t rd = blockIdx.x * (blockDim.x >> 5) + wib; rd < rounds; rd += nwarps_total) {
    const int64_t base = rd * 32;
    const int np = (int)(K - base < 32 ? K - base : 32);
    {  // this round's rows into L1 (measured better than L2-only), the next round's into L2
      const bool l1 = l1_prefetch;
      if (l1) {
        warp_prefetch(Pp + base * pstride, sizeof(double) * (size_t)(np * pstride), true);
        warp_prefetch(Qt + base * pstride, sizeof(double) * (size_t)(np * pstride), true);
        warp_prefetch(W + base * R, sizeof(double) * (size_t)(np * R), true);
        warp_prefetch(DW + base * R, sizeof(double) * (size_t)(np * R), true);
      }
      const int64_t nb = base + 32 * (int64_t)nwarps_total;
      if (nextpf && nb < K) {
        const int64_t nn = K - nb < 32 ? K - nb : 32;
        warp_prefetch(Pp + nb * pstride, sizeof(double) * (size_t)(nn * pstride), false);
        warp_prefetch(Qt + nb * pstride, sizeof(double) * (size_t)(nn * pstride), false);
      }
    }
    if (TBUF_OK && tbuf) {
      const double* Q = Qt + base * pstride;
      const double* P = Pp + base * pstride;
      double* Nrow = Nst + base * pstride;
      double fq[KS][MT];
      load_q(Q, fq);
#pragma unroll 1
      for (int sr = 0; sr < 4; ++sr) {
        const int p0 = 8 * sr;
        const int n8 = np - p0 < 8 ? (np - p0 > 0 ? np - p0 : 0) : 8;
        // ---- F_W rows of the sub-round, T_p fragments kept
        for (int pp = 0; pp < n8; ++pp) {
          double pv[MT][NT][2];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int c = 0; c < 2; ++c) pv[mt][nt][c] = offp[mt][nt][c] >= 0 ? P[offp[mt][nt][c]] : 0.0;
          double c[MT][NT][2];
          t_mma(fq, c);
          Q += pstride;
          P += pstride;
          if (p0 + pp + 1 < np) load_q(Q, fq);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int i = 0; i < 2; ++i) tb[(((pp * MT + mt) * NT + nt) * 2 + i) * 32 + lane] = c[mt][nt][i];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              double sv = 0.0;
#pragma unroll
              for (int mt = 0; mt < MT; ++mt) sv = fma(c[mt][nt][i], pv[mt][nt][i], sv);
              sv += __shfl_xor_sync(0xffffffffu, sv, 4);
              sv += __shfl_xor_sync(0xffffffffu, sv, 8);
              sv += __shfl_xor_sync(0xffffffffu, sv, 16);
              if (g == 0) fwv[(8 * nt + 2 * t + i) * 8 + pp] = sv;
            }
        }
        __syncwarp();
        // ---- W-row ADMM of the sub-round's 8 rows (rows past np stay zero)
        {
          const int p = p0 + g;
          double f[NT][2], wb[NT][2], dd[NT][2];
          const int64_t rowo = (base + p) * R;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int r = 8 * nt + 2 * t + c;
              const bool in = r < R && p < np;
              f[nt][c] = in ? fwv[r * 8 + g] : 0.0;
              wb[nt][c] = in ? W[rowo + r] : 0.0;
              dd[nt][c] = in ? DW[rowo + r] : 0.0;
            }
#pragma unroll 1
          for (int it = 0; it < n_inner; ++it) {
            double a[KA], z[NT][2];
#pragma unroll
            for (int ks = 0; ks < KA; ++ks)
              a[ks] = f[ks >> 1][ks & 1] + rho * (wb[ks >> 1][ks & 1] + dd[ks >> 1][ks & 1]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              z[nt][0] = z[nt][1] = 0.0;
#pragma unroll
              for (int ks = 0; ks < KA; ++ks) dmma2(z[nt][0], z[nt][1], a[ks], gfr[(ks * NT + nt) * 32 + lane]);
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const double nb = prox(kind, param, rho, z[nt][c] - dd[nt][c]);
                dd[nt][c] = dd[nt][c] + nb - z[nt][c];
                wb[nt][c] = nb;
              }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int r = 8 * nt + 2 * t + c;
              if (r < R) wbv[r * 8 + g] = wb[nt][c];
              if (r < R && p < np) {
                W[rowo + r] = wb[nt][c];
                DW[rowo + r] = dd[nt][c];
              }
            }
        }
        __syncwarp();
        // ---- W̄^T W̄ += sum_p w̄_p w̄_p^T over the sub-round (K = patients)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int pp = 4 * ks + t;
          double af[NT];
#pragma unroll
          for (int i = 0; i < NT; ++i) {
            const int r = 8 * i + g;
            af[i] = r < R ? wbv[r * 8 + pp] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma2(wacc[i][j][0], wacc[i][j][1], af[i], af[j]);
        }
        // ---- N_p = T_p S_p (new w̄_p) -> HBM; M += N_p^T N_p
        for (int pp = 0; pp < n8; ++pp) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              double v[2];
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int r = 8 * nt + 2 * t + i;
                v[i] = r < R ? tb[(((pp * MT + mt) * NT + nt) * 2 + i) * 32 + lane] * wbv[r * 8 + pp] : 0.0;
                if (offp[mt][nt][i] >= 0) Nrow[offp[mt][nt][i]] = v[i];
              }
              *reinterpret_cast<double2*>(ns + (8 * mt + g) * RP + 8 * nt + 2 * t) = make_double2(v[0], v[1]);
            }
          __syncwarp();
#pragma unroll
          for (int ks = 0; ks < 2 * MT; ++ks) {
            const int a = 4 * ks + t;
            double af[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) af[i] = a < l ? ns[a * RP + 8 * i + g] : 0.0;
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma2(macc[i][j][0], macc[i][j][1], af[i], af[j]);
          }
          __syncwarp();
          Nrow += pstride;
        }
      }
      steps_warp(steps + 1, base + lane < K ? n_inner : 0);
      continue;
    }
    // ---- F_W rows: F_W(p, r) = sum_a T_p(a, r) P'_p(a, r)
    {
      const double* Q = Qt + base * pstride;
      const double* P = Pp + base * pstride;
      double fq[KS][MT];
      load_q(Q, fq);
      for (int p = 0; p < np; ++p) {
        double pv[MT][NT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) pv[mt][nt][c] = offp[mt][nt][c] >= 0 ? P[offp[mt][nt][c]] : 0.0;
        double c[MT][NT][2];
        t_mma(fq, c);
        Q += pstride;
        P += pstride;
        if (p + 1 < np) load_q(Q, fq);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            double sv = 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) sv = fma(c[mt][nt][i], pv[mt][nt][i], sv);
            sv += __shfl_xor_sync(0xffffffffu, sv, 4);
            sv += __shfl_xor_sync(0xffffffffu, sv, 8);
            sv += __shfl_xor_sync(0xffffffffu, sv, 16);
            if (g == 0) fwv[(8 * nt + 2 * t + i) * 32 + p] = sv;
          }
      }
    }
    __syncwarp();
    // ---- W-row ADMM: z = Ginv (f + rho (w̄ + d)), w̄ = prox(z - d), d += w̄ - z, n_inner steps
    const int64_t kme = base + lane;
    int nsteps = 0;
    if (tolpath) {
      // per-row inner stop (reading R-inner-tol): thread per patient, out of line
      if (kme < K) {
        for (int r = 0; r < R; ++r) { wbv[r * 32 + lane] = W[kme * R + r]; dv[r * 32 + lane] = DW[kme * R + r]; }
        nsteps = w_row_admm_tol(Gs, R, fwv + lane, wbv + lane, dv + lane, rho, n_inner, kind, param, tol);
        for (int r = 0; r < R; ++r) { W[kme * R + r] = wbv[r * 32 + lane]; DW[kme * R + r] = dv[r * 32 + lane]; }
      } else {
        for (int r = 0; r < R; ++r) wbv[r * 32 + lane] = 0.0;
      }
    } else {
      // fixed steps: the warp's 32 rows at once, 8 patients (one M tile) at a time; the rows of
      // patients past K stay zero (f = w̄ = d = 0 and prox(0) = 0)
      __syncwarp();
#pragma unroll 1
      for (int mt = 0; mt < 4; ++mt) {
        const int p = 8 * mt + g;
        double f[NT][2], wb[NT][2], dd[NT][2];
        const int64_t rowo = (base + p) * R;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int r = 8 * nt + 2 * t + c;
            const bool in = r < R && p < np;  // (F_W rows p >= np hold stale sums)
            f[nt][c] = in ? fwv[r * 32 + p] : 0.0;
            wb[nt][c] = in ? W[rowo + r] : 0.0;
            dd[nt][c] = in ? DW[rowo + r] : 0.0;
          }
#pragma unroll 1
        for (int it = 0; it < n_inner; ++it) {
          double a[KA], z[NT][2];
#pragma unroll
          for (int ks = 0; ks < KA; ++ks) a[ks] = f[ks >> 1][ks & 1] + rho * (wb[ks >> 1][ks & 1] + dd[ks >> 1][ks & 1]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            z[nt][0] = z[nt][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KA; ++ks) dmma2(z[nt][0], z[nt][1], a[ks], gfr[(ks * NT + nt) * 32 + lane]);
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const double nb = prox(kind, param, rho, z[nt][c] - dd[nt][c]);
              dd[nt][c] = dd[nt][c] + nb - z[nt][c];
              wb[nt][c] = nb;
            }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int r = 8 * nt + 2 * t + c;
            if (r < R) wbv[r * 32 + p] = wb[nt][c];  // zero for rows p >= np
            if (r < R && p < np) {
              W[rowo + r] = wb[nt][c];
              DW[rowo + r] = dd[nt][c];
            }
          }
      }
      __syncwarp();
      nsteps = kme < K ? n_inner : 0;
    }
    steps_warp(steps + 1, nsteps);
    __syncwarp();
    // ---- W̄^T W̄ += sum_p w̄_p w̄_p^T  (MMA with K = patients)
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int p = 4 * ks + t;
      double af[NT];
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int r = 8 * i + g;
        af[i] = r < R ? wbv[r * 32 + p] : 0.0;  // A[g][t] = w̄_p(r) ; B[t][g] = w̄_p(s) (same values)
      }
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma2(wacc[i][j][0], wacc[i][j][1], af[i], af[j]);
    }
    // ---- N_p = T_p S_p (new w̄_p) -> HBM; M += N_p^T N_p
    {
      const double* Q = Qt + base * pstride;
      double* Nrow = Nst + base * pstride;
      double fq[KS][MT];
      load_q(Q, fq);
      for (int p = 0; p < np; ++p) {
        double c[MT][NT][2];
        t_mma(fq, c);
        Q += pstride;
        if (p + 1 < np) load_q(Q, fq);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double v[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = 8 * nt + 2 * t + i;
              v[i] = r < R ? c[mt][nt][i] * wbv[r * 32 + p] : 0.0;
              if (offp[mt][nt][i] >= 0) Nrow[offp[mt][nt][i]] = v[i];
            }
            *reinterpret_cast<double2*>(ns + (8 * mt + g) * RP + 8 * nt + 2 * t) = make_double2(v[0], v[1]);
          }
        __syncwarp();
        // M += N^T N: A[g][t] = N(a = 4 ks + t, r = 8 i + g), B[t][g] = N(a, s = 8 j + g)
#pragma unroll
        for (int ks = 0; ks < 2 * MT; ++ks) {
          const int a = 4 * ks + t;
          double af[NT];
#pragma unroll
          for (int i = 0; i < NT; ++i) af[i] = a < l ? ns[a * RP + 8 * i + g] : 0.0;
#pragma unroll
          for (int i = 0; i < NT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma2(macc[i][j][0], macc[i][j][1], af[i], af[j]);
        }
        __syncwarp();
        Nrow += pstride;
      }
    }
  }
  // block partials of M and W̄^T W̄, one after the other through warps x RP^2 doubles at offset 0
  double* red = sm;
  const int nw = blockDim.x >> 5;
#pragma unroll 1
  for (int which = 0; which < 2; ++which) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c)
          red[wib * RP * RP + (8 * i + g) * RP + 8 * j + 2 * t + c] = which == 0 ? macc[i][j][c] : wacc[i][j][c];
    __syncthreads();
    for (int y = threadIdx.x; y < R * R; y += blockDim.x) {
      const int r = y / R, s2 = y - r * R;
      double v = 0.0;
      for (int ww = 0; ww < nw; ++ww) v += red[ww * RP * RP + r * RP + s2];
      part[((int64_t)blockIdx.x * 2 + which) * R * R + y] = v;
    }
  }
}

// dynamic shared memory of k_passB_wide (layout in the kernel)
inline size_t passB_wide_smem(int R, int NT, int MT, bool tolpath, int warps) {
  const size_t RP = 8 * (size_t)NT, hoff = (size_t)((R * R + 31) / 32) * 32;
  const size_t fwd = std::max(RP * 32, (size_t)MT * 8 * RP);
  const bool tbuf = MT * NT <= 4 && !tolpath;
  const size_t per_warp = tolpath ? 3 * RP * 32 + (size_t)MT * 8 * RP
                          : tbuf ? 2 * RP * 8 + (size_t)MT * 8 * RP + 8 * 32 * (size_t)MT * NT * 2 : fwd + RP * 32;
  const size_t main = hoff + 2 * NT * (size_t)NT * 32 + (tolpath ? hoff : 0) + warps * per_warp;
  return sizeof(double) * std::max(main, (size_t)warps * RP * RP);
}

static __global__ void k_sum_rr2(const double* part, int nb, int RR, double* M, double* WtW) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= 2 * RR) return;
  int which = x / RR, y = x - which * RR;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[((int64_t)b * 2 + which) * RR + y];
  (which == 0 ? M : WtW)[y] = s;
}

template <int MT, int NT, int RT = 0, int LT = 0>
static void passB_wide_inst(Handle& h) {
  constexpr auto fn = k_passB_wide<MT, NT, RT, LT>;
  const size_t smem = passB_wide_smem(h.R, NT, MT, h.o.admm_tol > 0.0, kDenseThreads / 32);
  max_smem_attr<fn>(h);
  int64_t rounds = (h.K + 31) / 32;
  int64_t blocks = (rounds + 3) / 4;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kDenseThreads, smem);
  int64_t cap = h.sms * (int64_t)(per_sm > 0 ? per_sm : 1);
  if (cap > kPartBlocks) cap = kPartBlocks;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  fn<<<(unsigned)blocks, kDenseThreads, smem, h.stream>>>(h.K, h.R, h.l, h.Pp, h.Qt, h.H, h.GWi, h.scal,
                                                         h.o.admm_inner, h.o.on_W.kind, h.o.on_W.param,
                                                         h.o.admm_tol, h.W, h.DW, h.Nst, h.partial, 1, 0, h.steps);
  const int RR = h.R * h.R;
  k_sum_rr2<<<(2 * RR + 255) / 256, 256, 0, h.stream>>>(h.partial, (int)blocks, RR, h.M, h.WtW);
}

// Generic NT instantiations of the W pass, grouped so the object files compile in parallel
// (k_passB_g*.cu); the configured (R, l) shapes are in k_passB_s.cu.
template <int MT, int NT0, int NT1>
static void passB_wide_group(Handle& h, int nt) {
  if constexpr (NT0 <= NT1) {
    if (nt == NT0) { passB_wide_inst<MT, NT0>(h); return; }
    passB_wide_group<MT, NT0 + 1, NT1>(h, nt);
  }
}

// F_W + W-ADMM + N + M + W^T W for smooth patients (m_k <= l <= 16). Returns kernels launched.
}  // namespace copa
