// k_passA.cu — pass A of the smooth path: P'_k = X'_k V(cols_k, :) (m_k x R) for every patient
// (Alg.1 l.4 input X_k V S_k H^T, projected form P:342-347), FP64 on the tensor cores.
//
// Layout A: a patient-major copy of the fibers (built once at init from the g-streams, k_layoutA):
// patient k's fibers are [fp[k], fp[k+1]) in fa_col / fa_val. Each warp owns a contiguous patient
// range balanced by fibers (plan_passA), i.e. ONE contiguous fiber stream, which it pulls through a
// private NS-slot shared-memory ring of 32-fiber chunks with 1-D TMA bulk copies (cp.async.bulk +
// an mbarrier per slot): the chunk c + NS is requested as soon as chunk c is consumed, so ~NS x 2 KB
// are in flight per warp without any register staging.
//
// MMA (mma.sync m8n8k4 f64): M = basis index a (8 / tile), N = r (8 / tile), K = 4 fibers. V̄ rows
// come from shared memory when V̄ (label order) fits, else from L1/L2 (Vl). A k-step that straddles
// a patient boundary is split with a fiber mask; P'_k is written when the patient's last fiber has
// been consumed (rows a >= m_k are exact zeros: x'_kj(a) = 0 there).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "copa_internal.cuh"

namespace copa {

namespace {

__device__ __forceinline__ void dmma_a(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE%=;\n bra WAIT%=;\n"
      "DONE%=:\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

constexpr int kAWarps = 8;   // warps per CTA
constexpr int kANS = 4;      // ring slots per warp (power of two)
constexpr int kAChunk = 32;  // fibers per chunk

__host__ __device__ inline int chunk_val_off() { return kAChunk * 4; }  // col block, then val block
__host__ __device__ inline int chunk_bytes(int l) { return kAChunk * 4 + kAChunk * l * 8; }

}  // namespace

// Layout A: patient k's G runs concatenated at fp[k] (same label order inside each run).
__global__ void k_layoutA(const int64_t* __restrict__ gptr, int G, int64_t K, const int64_t* __restrict__ fp,
                          const int32_t* __restrict__ gcol, const double* __restrict__ gval, int l,
                          int32_t* __restrict__ acol, double* __restrict__ aval) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < K; k += nw) {
    int64_t dst = fp[k];
    for (int g = 0; g < G; ++g) {
      const int64_t s0 = gptr[g * (K + 1) + k], s1 = gptr[g * (K + 1) + k + 1];
      for (int64_t x = lane; x < s1 - s0; x += 32) acol[dst + x] = gcol[s0 + x];
      for (int64_t x = lane; x < (s1 - s0) * l; x += 32) aval[dst * l + x] = gval[s0 * l + x];
      dst += s1 - s0;
    }
  }
}

template <int MT, int NT, int LT, int RT, bool VS>
__global__ void __launch_bounds__(32 * kAWarps) k_passA(const int64_t* __restrict__ fp,
                                                        const int64_t* __restrict__ warp_k,
                                                        const int32_t* __restrict__ acol,
                                                        const double* __restrict__ aval, int64_t K, int l_, int R_,
                                                        int64_t Jl, const double* __restrict__ Vl,
                                                        double* __restrict__ Pp) {
  const int R = RT ? RT : R_;
  const int l = LT ? LT : l_;
  extern __shared__ __align__(128) unsigned char sraw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int cb = (chunk_bytes(l) + 127) & ~127;
  // VS: all of V̄ (label order) in smem; otherwise gathers through L1/L2 (a hot-label smem cache
  // measured slower at Scale: 12.1 vs 11.0 ms).
  double* Vs = (double*)sraw;
  const size_t vbytes = VS ? (((size_t)Jl * R * 8 + 127) & ~(size_t)127) : 0;
  uint64_t* bars = (uint64_t*)(sraw + vbytes) + wib * kANS;
  unsigned char* ring = sraw + vbytes + kAWarps * kANS * 8 + (size_t)wib * kANS * cb;
  if (VS) {
    for (int64_t x = threadIdx.x; x < Jl * R; x += blockDim.x) Vs[x] = Vl[x];
  }
  if (lane == 0) {
    for (int i = 0; i < kANS; ++i) mb_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t wid = (int64_t)blockIdx.x * kAWarps + wib;
  const int64_t ka = warp_k[wid], kb = warp_k[wid + 1];
  if (ka >= kb) return;
  const int64_t F0 = fp[ka], F1 = fp[kb];
  const int64_t C0 = F0 & ~(int64_t)3;  // chunk grid aligned to 4 fibers (16-byte bulk copies)
  const int64_t nch = (F1 - C0 + kAChunk - 1) / kAChunk;
  const uint32_t vbytes_chunk = (uint32_t)(kAChunk * l * 8);
  const int nchi = (int)nch;  // chunks per warp stream (< 2^31)
  auto issue = [&](int c) {
    if (lane == 0 && c < nchi) {
      unsigned char* dst = ring + (c & (kANS - 1)) * cb;
      uint64_t* bar = bars + (c & (kANS - 1));
      const int64_t cs = C0 + (int64_t)c * kAChunk;
      mb_arrive_tx(bar, kAChunk * 4 + vbytes_chunk);
      bulk_copy(dst, acol + cs, kAChunk * 4, bar);
      bulk_copy(dst + chunk_val_off(), aval + cs * l, vbytes_chunk, bar);
    }
  };
#pragma unroll
  for (int c = 0; c < kANS; ++c) issue(c);
  // patient cursor: fe = end of patient k; fp window in registers (lane i holds fp[kw + i])
  int64_t k = ka;
  int64_t kw = ka + 1;
  int64_t fpw = kw + lane <= K ? fp[kw + lane] : 0;
  auto fp_at = [&](int64_t kk) -> int64_t {  // fp[kk] for kk >= kw (warp-uniform)
    if (kk >= kw + 32) {
      kw = kk;
      fpw = kw + lane <= K ? fp[kw + lane] : 0;
    }
    return __shfl_sync(0xffffffffu, fpw, (int)(kk - kw));
  };
  int64_t fe = fp_at(k + 1);
  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  auto flush = [&](int64_t kk) {
    double* out = Pp + kk * l * R;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = 8 * mt + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int r = 8 * nt + 2 * t;
        if (a < l) {
          if (r < R) out[a * R + r] = acc[mt][nt][0];
          if (r + 1 < R) out[a * R + r + 1] = acc[mt][nt][1];
        }
        acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      }
    }
  };
  // Chunk fragments: k-step j covers fibers cs + 4 j .. + 3. A[g][t] = x'_{cs+4j+t}(a = 8 mt + g),
  // B[t][g] = V̄(label_{cs+4j+t}, r = 8 nt + g). Loads are unpredicated: fibers outside the current
  // patient segment are masked to zero in the A operand at MMA time; rows a >= l and columns r >= R
  // only feed accumulator entries that are never written (labels are always valid: the slack of
  // fa_col is zeroed and V̄ rows are padded).
  // the lane's k index t kept in a register (opaque to the compiler): otherwise it is rebuilt from
  // SR_TID.X right before the masked MMAs of every patient boundary (S2R latency on the MMA path)
  int tk;
  asm volatile("mov.b32 %0, %1;" : "=r"(tk) : "r"(t));
  for (int c = 0; c < nchi; ++c) {
    mb_wait(bars + (c & (kANS - 1)), (uint32_t)((c / kANS) & 1));
    const unsigned char* buf = ring + (c & (kANS - 1)) * cb;
    const int32_t* colS = (const int32_t*)buf;
    const double* valS = (const double*)(buf + chunk_val_off());
    const int64_t cs = C0 + (int64_t)c * kAChunk;
    double x[8][MT], bv[8][NT];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int fl = 4 * j + t;
      const int32_t col = colS[fl];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) x[j][mt] = valS[fl * l + 8 * mt + g];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if (VS) {
          bv[j][nt] = Vs[col * R + 8 * nt + g];
        } else {
          bv[j][nt] = __ldg(Vl + (int64_t)col * R + 8 * nt + g);
        }
      }
    }
    // patient segments of this chunk: [lo, hi) relative to cs
    int lo = (int)(F0 > cs ? F0 - cs : 0);
    const int ce = (int)(F1 - cs < kAChunk ? F1 - cs : kAChunk);
    while (lo < ce && k < kb) {
      const int hi = (int)(fe - cs < ce ? fe - cs : ce);
      const int j0 = lo >> 2, j1 = (hi + 3) >> 2;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= j0 && j < j1) {
          const int fl = 4 * j + tk;
          const bool in = fl >= lo && fl < hi;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma_a(acc[mt][nt][0], acc[mt][nt][1], in ? x[j][mt] : 0.0, bv[j][nt]);
        }
      }
      if (cs + hi == fe) {
        flush(k);
        ++k;
        if (k < kb) fe = fp_at(k + 1);
      }
      lo = hi;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads of the slot before its refill
    issue(c + kANS);
  }
  // patients with no fibers left at the end of the range (fe == F1 already flushed above)
  while (k < kb) {
    flush(k);
    ++k;
  }
}

template <int MT, int NT, int LT, int RT>
static void passA_inst(Handle& h) {
  const int cb = (chunk_bytes(h.l) + 127) & ~127;
  const size_t ring = (size_t)kAWarps * kANS * (8 + cb);
  const bool vs = h.pa_vs;
  const size_t vbytes = vs ? (((size_t)h.Jl * h.R * 8 + 127) & ~(size_t)127) : 0;
  const size_t smem = vbytes + ring + 128;
  launch_relabel_V(h);  // V̄ in label order (read by every CTA: smem copy or L1/L2 gathers)
  if (vs) {
    constexpr auto fn = k_passA<MT, NT, LT, RT, true>;
    max_smem_attr<fn>(h);
    fn<<<h.pa_ctas, 32 * kAWarps, smem, h.stream>>>(h.fiber_ptr, h.pa_wk, h.fa_col, h.fa_val, h.K, h.l, h.R, h.Jl,
                                                    h.Vl, h.Pp);
  } else {
    constexpr auto fn = k_passA<MT, NT, LT, RT, false>;
    max_smem_attr<fn>(h);
    fn<<<h.pa_ctas, 32 * kAWarps, smem, h.stream>>>(h.fiber_ptr, h.pa_wk, h.fa_col, h.fa_val, h.K, h.l, h.R, h.Jl,
                                                    h.Vl, h.Pp);
  }
}

template <int MT>
static void passA_n(Handle& h) {
  if (MT == 1 && h.l == 7 && h.R == 20) { passA_inst<1, 3, 7, 20>(h); return; }
  if (MT == 1 && h.l == 7 && h.R == 15) { passA_inst<1, 2, 7, 15>(h); return; }
  if (MT == 2 && h.l == 9 && h.R == 40) { passA_inst<2, 5, 9, 40>(h); return; }
  switch ((h.R + 7) / 8) {
    case 1: passA_inst<MT, 1, 0, 0>(h); break;
    case 2: passA_inst<MT, 2, 0, 0>(h); break;
    case 3: passA_inst<MT, 3, 0, 0>(h); break;
    case 4: passA_inst<MT, 4, 0, 0>(h); break;
    case 5: passA_inst<MT, 5, 0, 0>(h); break;
    case 6: passA_inst<MT, 6, 0, 0>(h); break;
    case 7: passA_inst<MT, 7, 0, 0>(h); break;
    default: passA_inst<MT, 8, 0, 0>(h); break;
  }
}

void launch_spmm_fibers(Handle& h) {
  if (h.l <= 8) passA_n<1>(h);
  else passA_n<2>(h);
}

// CTAs / warps of pass A and where V̄ lives: all of it in shared memory when it fits (VS),
// otherwise gathered through L1/L2.
void plan_passA(Handle& h) {
  const int cb = (chunk_bytes(h.l) + 127) & ~127;
  const size_t ring = (size_t)kAWarps * kANS * (8 + cb);
  const size_t vbytes = ((size_t)h.Jl * h.R * 8 + 127) & ~(size_t)127;
  h.pa_vs = vbytes + ring + 128 <= 225 * 1024;
  const size_t smem = (h.pa_vs ? vbytes : 0) + ring + 128;
  int per_sm = (int)((228 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 2048 / (32 * kAWarps)) per_sm = 2048 / (32 * kAWarps);
  h.pa_ctas = h.sms * per_sm;
  h.pa_nw = (int64_t)h.pa_ctas * kAWarps;
}

// Warp ranges of pass A: contiguous patient ranges with balanced fibers, from the fiber prefix fp:
// wk[w] = first patient k with fp[k] >= F w / nw (K if none), wk[0] = 0, wk[nw] = K.
__global__ void k_passA_ranges(const int64_t* __restrict__ fp, int64_t K, int64_t nw, int64_t* __restrict__ wk) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w > nw) return;
  if (w == 0 || w == nw) { wk[w] = w == 0 ? 0 : K; return; }
  const int64_t target = (fp[K] * w) / nw;
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (fp[mid] < target) lo = mid + 1; else hi = mid;
  }
  wk[w] = lo;
}

void launch_passA_ranges(Handle& h) {
  k_passA_ranges<<<(unsigned)((h.pa_nw + 1 + 255) / 256), 256, 0, h.stream>>>(h.fiber_ptr, h.K, h.pa_nw, h.pa_wk);
}

void launch_layoutA(Handle& h) {
  if (h.K == 0) return;
  int64_t blocks = (h.K + 7) / 8;
  if (blocks > h.sms * 16) blocks = h.sms * 16;
  k_layoutA<<<(unsigned)blocks, 256, 0, h.stream>>>(h.gptr, h.sc_G, h.K, h.fiber_ptr, h.fiber_col, h.fiber_val, h.l,
                                                    h.fa_col, h.fa_val);
}

}  // namespace copa
