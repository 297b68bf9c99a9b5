// copa_api.cu — the C ABI (include/copa.h): validation, workspace layout, orchestration of one
// outer iteration on one stream, and the allreduce hand-off points C1/C2.
#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: phase ranges for nsys/ncu timelines

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "copa_internal.cuh"

using namespace copa;

namespace {

thread_local std::string g_last_error;

copa_status fail(copa_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

copa_status cuda_fail(cudaError_t e, const char* where) {
  return fail(COPA_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(call, where)                     \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(int64_t n) {
    size_t o = off;
    off = align_up(off + sizeof(T) * (size_t)(n > 0 ? n : 1));
    return base ? reinterpret_cast<T*>(base + o) : nullptr;
  }
};

// Segment layout shared by workspace_size (base = nullptr) and init.
size_t carve(Handle& h, char* base) {
  Carver c{base};
  const int64_t R = h.R, RR = R * R;
  h.err = c.take<int>(16);
  h.scal = c.take<double>(S_COUNT);
  h.H = c.take<double>(RR);
  h.DH = c.take<double>(RR);
  h.FH = c.take<double>(RR);
  h.HtH = c.take<double>(RR);
  h.VtV = c.take<double>(RR);
  h.LW = c.take<double>(RR);
  h.GWi = c.take<double>(RR);
  h.HT = c.take<double>(RR);
  h.comm2 = c.take<double>(h.J * R + 2 * RR);
  if (base) { h.FV = h.comm2; h.WtW = h.comm2 + h.J * R; h.M = h.WtW + RR; }
  h.V = c.take<double>(h.J * R);
  h.DV = c.take<double>(h.J * R);
  h.W = c.take<double>(h.K * R);
  h.DW = c.take<double>(h.K * R);
  h.m = c.take<int32_t>(h.K);
  h.rank = c.take<int32_t>(h.K);
  h.srow = c.take<int64_t>(h.K + 1);
  h.Pp = c.take<double>(h.S * R + 4);   // +4: bulk copies round up to 16 bytes
  h.Qt = c.take<double>(h.S * R + 4);
  h.Nst = c.take<double>(h.S * R + 4);
  {  // per-block partials of the R x R reductions; also the chunk sums of the F_H reduction
    const int64_t NT = (R + 7) / 8, a = 2 * (int64_t)kPartBlocks * RR, b = 32 * 64 * NT * NT;
    h.partial = c.take<double>(a > b ? a : b);
  }
  {
    const int64_t RP = 8 * ((R + 7) / 8);
    h.fh_warp = c.take<double>(h.fib ? (int64_t)kPartBlocks * 4 * RP * RP : 1);
  }
  h.fit_ring = c.take<double>(1024);  // device ring of per-iteration FIT values
  h.diag = c.take<unsigned long long>(kDiagSlots);
  h.porder = c.take<int32_t>(h.K);
  h.steps = c.take<unsigned long long>(4);
  if (h.fib) {
    const int G = h.sc_G;
    h.Fcap = h.F + 8;
    h.Bk = c.take<double>(h.K * h.l * h.l);
    h.fiber_ptr = c.take<int64_t>(h.K + 1);
    h.gptr = c.take<int64_t>((int64_t)G * (h.K + 1) + 2);  // +2: bulk copies round up to 16 bytes
    {  // the tiled stream's buffer first holds the g-streams (init only: layout A is built from
       // them, the tiles from layout A; without a shared-memory F_V slice the g-streams stay)
      const size_t gcol = align_up(sizeof(int32_t) * (size_t)h.Fcap);
      const size_t gsz = gcol + sizeof(double) * (size_t)(h.Fcap * h.l);
      const size_t tsz = (size_t)tiles_cap(h) * tile_bytes_host(h.l) + 64;
      h.tiles = c.take<unsigned char>((int64_t)(gsz > tsz ? gsz : tsz));
      h.fiber_col = reinterpret_cast<int32_t*>(h.tiles);
      h.fiber_val = h.tiles ? reinterpret_cast<double*>(h.tiles + gcol) : nullptr;
    }
    h.cub_temp_bytes = std::max(h.cub_temp_bytes, plan_cub_bytes(h));
    h.cub_temp = c.take<char>((int64_t)h.cub_temp_bytes);
    h.perm = c.take<int32_t>(h.J);
    h.inv = c.take<int32_t>(h.Jl);
    h.Vl = c.take<double>(h.Jl * R + 64);  // +64: unpredicated pass-A gathers past the last row
    h.fa_col = c.take<int32_t>(h.F + 64);
    h.fa_val = c.take<double>((h.F + 64) * h.l);
    h.pa_wk = c.take<int64_t>(h.pa_nw + 1);
    h.block_k = c.take<int64_t>(h.sc_ranges + 1);
    h.fv_part = c.take<double>((int64_t)h.sc_ranges * h.Jl * R);
    h.fhist = c.take<unsigned long long>(h.J);
    h.woff = c.take<uint16_t>((int64_t)G * h.K * kWoS + 16);
    h.twoff = c.take<uint16_t>((int64_t)G * h.K * kWoS + 16);
    h.tptr = c.take<int64_t>((int64_t)G * (h.K + 1) + 2);
    h.nst_cap = stage_cap(h);
    h.st_f = c.take<int64_t>(2 * h.nst_cap);
    h.st_k = c.take<int32_t>(2 * h.nst_cap);
    h.cta_st = c.take<int32_t>((int64_t)h.sc_ranges * G + 1);
    h.st_t = c.take<int32_t>(h.nst_cap + 1);
    h.st_list = c.take<uint32_t>(stage_tab_cap(h));
    // per-run fiber and tile counts (each followed by a zero), then the planning scans' scratch
    h.layout_tmp_bytes = 2 * sizeof(int32_t) * ((size_t)G * (size_t)h.K + 4) + sizeof(int64_t) * plan_tmp_words(h);
    h.layout_tmp = c.take<char>((int64_t)h.layout_tmp_bytes);
  } else {
    if (h.rowproj) {
      h.Bk = c.take<double>(h.K * h.l * h.l);
      h.Prow = c.take<double>(h.rows * R);
      h.Nrow = c.take<double>(h.rows * R);
    }
    h.row_patient = c.take<int32_t>(h.rows);
    h.csc_ptr = c.take<int64_t>(h.J + 1);
    h.csc_row = c.take<int32_t>(h.nnz);
    h.csc_val = c.take<double>(h.nnz);
    h.csc_chunk_cap = h.nnz / kCscChunk + h.J + 1;
    h.csc_chunk = c.take<int64_t>(2 * h.csc_chunk_cap);
    h.csc_chunk_first = c.take<int64_t>(h.J + 1);
    h.csc_part = c.take<double>(h.csc_chunk_cap * R);
    h.csc_tmp_bytes = csc_temp_bytes(h);
    h.csc_tmp = c.take<char>((int64_t)h.csc_tmp_bytes);
  }
  return c.off;
}

copa_status check_args(const copa_problem* p, const copa_options* o) {
  if (!p || !o) return fail(COPA_E_ARG, "null problem/options");
  if (p->R < 1) return fail(COPA_E_ARG, "R must be >= 1");
  if (p->R > kMaxR) return fail(COPA_E_UNSUPPORTED, "R > 64 not supported by this build");
  if (p->J < 1 || p->J > kMaxJ) return fail(COPA_E_UNSUPPORTED, "J must be in [1, 65535]");
  if (p->K_local < 0 || p->rows < 0 || p->nnz < 0) return fail(COPA_E_ARG, "negative size");
  if (p->K_local > 0 && (!p->patient_row_ptr || !p->row_ptr)) return fail(COPA_E_ARG, "null CSR pointer");
  if (p->nnz > 0 && (!p->col || !p->val)) return fail(COPA_E_ARG, "null col/val");
  if (o->admm_inner < 1) return fail(COPA_E_ARG, "admm_inner must be >= 1");
  const copa_constraint* cs[3] = {&o->on_H, &o->on_W, &o->on_V};
  for (auto c : cs) {
    if (c->kind < COPA_NONE || c->kind > COPA_L0) return fail(COPA_E_ARG, "unknown constraint kind");
    if ((c->kind == COPA_L1 || c->kind == COPA_NONNEG_L1) && !(c->param >= 0)) return fail(COPA_E_ARG, "lambda < 0");
    if (c->kind == COPA_L0 && !(c->param > 0)) return fail(COPA_E_ARG, "mu <= 0");
  }
  if (!(o->rank_tol >= 0) || !(o->basis_tol >= 0) || !(o->admm_tol >= 0))
    return fail(COPA_E_ARG, "tolerances must be >= 0");
  if (o->smooth_l < 0) return fail(COPA_E_ARG, "smooth_l < 0");
  if (o->smooth_l > 0) {
    if (o->smooth_l > kMaxL) return fail(COPA_E_UNSUPPORTED, "smooth_l > 64 not supported");
    if (o->smooth_degree < 0 || o->smooth_degree > kMaxDeg || o->smooth_degree >= o->smooth_l)
      return fail(COPA_E_ARG, "smooth_degree must be in [0, min(7, l-1)]");
    if (p->K_local > 0 && !p->visit_time) return fail(COPA_E_ARG, "smoothness requires visit times");
  }
  if (!o->H0 || !o->V0 || (p->K_local > 0 && !o->W0_local)) return fail(COPA_E_ARG, "null initial factors");
  return COPA_OK;
}

void fill_sizes(Handle& h, const copa_problem* p, const copa_options* o) {
  h.p = *p;
  h.o = *o;
  h.stream = (cudaStream_t)o->stream;
  if (cudaGetDevice(&h.dev) != cudaSuccess) { cudaGetLastError(); h.dev = 0; }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.dev) == cudaSuccess && sms > 0) h.sms = sms;
  else cudaGetLastError();
  h.smooth = o->smooth_l > 0;
  h.fib = h.smooth && o->smooth_l <= kMaxFiberL;
  h.rowproj = h.smooth && !h.fib;
  h.l = o->smooth_l;
  h.d = o->smooth_degree;
  h.K = p->K_local;
  h.J = p->J;
  h.rows = p->rows;
  h.nnz = p->nnz;
  h.R = p->R;
  h.S = h.smooth ? h.K * h.l : h.rows;
  h.Jl = h.J;
  if (h.fib) {
    plan_scatter(h);
    plan_passA(h);
  }
}

copa_status count_fibers(Handle& h, int64_t* F_out, size_t* cub_bytes) {
  *F_out = 0;
  *cub_bytes = 0;
  if (!h.fib) return COPA_OK;
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(h.K + 1));
  *cub_bytes = tb;
  if (h.K == 0) return COPA_OK;
  int64_t* counts = nullptr;
  void* tmp = nullptr;
  CUDA_TRY(cudaMallocAsync(&counts, sizeof(int64_t) * (size_t)(h.K + 2), h.stream), "cudaMallocAsync(count)");
  CUDA_TRY(cudaMallocAsync(&tmp, tb + 256, h.stream), "cudaMallocAsync(scan)");
  launch_count_fibers(h, counts, nullptr);
  cub::DeviceScan::InclusiveSum(tmp, tb, counts, counts, (int)(h.K + 1), h.stream);
  int64_t F = 0;
  CUDA_TRY(cudaMemcpyAsync(&F, counts + h.K, sizeof(int64_t), cudaMemcpyDeviceToHost, h.stream), "count copy");
  cudaFreeAsync(counts, h.stream);
  cudaFreeAsync(tmp, h.stream);
  CUDA_TRY(cudaStreamSynchronize(h.stream), "count sync");
  CUDA_TRY(cudaGetLastError(), "count kernels");
  *F_out = F;
  return COPA_OK;
}

copa_status allreduce(Handle& h, double* buf, int64_t n) {
  if (!h.o.allreduce) return COPA_OK;
  int rc = h.o.allreduce(buf, n, (void*)h.stream, h.o.allreduce_ctx);
  if (rc != 0) return fail(COPA_E_COMM, "allreduce callback returned " + std::to_string(rc));
  return COPA_OK;
}

copa_status check_err(Handle& h) {
  int err = 0;
  CUDA_TRY(cudaMemcpyAsync(&err, h.err, sizeof(int), cudaMemcpyDeviceToHost, h.stream), "err copy");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "stream sync");
  CUDA_TRY(cudaGetLastError(), "kernel launch");
  if (err & ERR_SHAPE) return fail(COPA_E_SHAPE, "invalid CSR/times (monotonicity, column range, duplicates)");
  if (err & ERR_INPUT_NONFINITE) return fail(COPA_E_NONFINITE, "non-finite input value");
  if (err & ERR_DEGEN) return fail(COPA_E_DEGENERATE, "trace(G) = 0 with automatic rho");
  if (err & ERR_CHOL) return fail(COPA_E_CHOL, "non-positive pivot in chol(G + rho I)");
  if (err & ERR_NONFINITE) return fail(COPA_E_NONFINITE, "non-finite FIT");
  return COPA_OK;
}

__global__ void k_srow_smooth(int64_t K, int l, int64_t* srow) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k <= K) srow[k] = k * l;
}

__global__ void k_rank_deficient(const int32_t* m, const int32_t* rank, int64_t K, int R, unsigned long long* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  int q = m[k] < R ? m[k] : R;
  if (rank[k] < q) atomicAdd(out, 1ull);
}

}  // namespace

struct copa_handle {
  Handle h;
};

extern "C" {

void copa_get_limits(copa_limits* out) {
  if (!out) return;
  out->max_R = kMaxR;
  out->max_q = kMaxR;
  out->max_smooth_l = kMaxL;
  out->max_J = kMaxJ;
}

const char* copa_last_error(void) { return g_last_error.c_str(); }

copa_status copa_workspace_size(const copa_problem* p, const copa_options* o, size_t* bytes) {
  copa_status st = check_args(p, o);
  if (st != COPA_OK) return st;
  if (!bytes) return fail(COPA_E_ARG, "null bytes");
  Handle h{};
  fill_sizes(h, p, o);
  st = count_fibers(h, &h.F, &h.cub_temp_bytes);
  if (st != COPA_OK) return st;
  *bytes = carve(h, nullptr);
  return COPA_OK;
}

// Init stage timing (COPA_INIT_TIMES=1): synchronises the stream at each mark and prints the
// elapsed host time per stage to stderr. Off by default (the marks are no-ops).
namespace {
struct InitTimer {
  bool on = getenv("COPA_INIT_TIMES") != nullptr;
  cudaStream_t s = nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* name) {
    nvtxMarkA(name);  // init stage boundary on the NVTX timeline
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[copa init] %-16s %9.2f ms\n", name, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
}  // namespace

// Values arriving in chunks (copa_fit): chunk i holds the values of patients [k[i-1], k[i]) (entries
// [e[i-1], e[i])) and is on the device once ev[i] has completed; until then only the other inputs
// may be read. The first init stages run meanwhile, and the fiber build follows chunk by chunk.
struct ValChunks {
  int n = 0;
  int64_t e0 = 0;               // first referenced value (row_ptr[patient_row_ptr[0]])
  int64_t k[8] = {}, e[8] = {};  // chunk i: patients [k[i-1], k[i]), values [e[i-1], e[i]) (absolute)
  cudaEvent_t ev[8] = {};
};

static copa_status init_impl(const copa_problem* p, const copa_options* o, void* ws, size_t bytes, copa_handle** out,
                             const ValChunks* vc);

copa_status copa_init(const copa_problem* p, const copa_options* o, void* ws, size_t bytes, copa_handle** out) {
  return init_impl(p, o, ws, bytes, out, nullptr);
}

static copa_status init_impl(const copa_problem* p, const copa_options* o, void* ws, size_t bytes, copa_handle** out,
                             const ValChunks* vc) {
  copa_status st = check_args(p, o);
  if (st != COPA_OK) return st;
  if (!out || !ws) return fail(COPA_E_ARG, "null workspace/out");
  if (((uintptr_t)ws & 255) != 0) return fail(COPA_E_WORKSPACE, "workspace must be 256-byte aligned");
  copa_handle* H = new (std::nothrow) copa_handle();
  if (!H) return fail(COPA_E_ARG, "out of host memory");
  Handle& h = H->h;
  fill_sizes(h, p, o);
  InitTimer tm;
  tm.s = h.stream;
  tm.mark("start");
  st = count_fibers(h, &h.F, &h.cub_temp_bytes);
  if (st != COPA_OK) { delete H; return st; }
  tm.mark("count_fibers F");
  size_t need = carve(h, nullptr);
  if (bytes < need) { delete H; return fail(COPA_E_WORKSPACE, "workspace too small: need " + std::to_string(need)); }
  carve(h, (char*)ws);
  cudaStream_t s = h.stream;
  const size_t RR = (size_t)h.R * h.R;
  cudaMemsetAsync(h.err, 0, 16 * sizeof(int), s);
  cudaMemsetAsync(h.scal, 0, S_COUNT * sizeof(double), s);
  cudaMemsetAsync(h.Pp, 0, sizeof(double) * (size_t)(h.S * h.R), s);
  cudaMemsetAsync(h.Qt, 0, sizeof(double) * (size_t)(h.S * h.R), s);
  cudaMemsetAsync(h.Nst, 0, sizeof(double) * (size_t)(h.S * h.R), s);
  cudaMemsetAsync(h.rank, 0, sizeof(int32_t) * (size_t)(h.K > 0 ? h.K : 1), s);
  cudaMemsetAsync(h.steps, 0, 4 * sizeof(unsigned long long), s);
  {  // rank-cut diagnostics: counts 0, min-kept ratios +inf, max-dropped ratios 0
    static const unsigned long long d0[kDiagSlots] = {0, 0x7ff0000000000000ull, 0, 0, 0x7ff0000000000000ull, 0, 0, 0};
    CUDA_TRY(cudaMemcpyAsync(h.diag, d0, sizeof(d0), cudaMemcpyHostToDevice, s), "diag init");
  }
  launch_validate(h, vc == nullptr);
  st = check_err(h);
  if (st != COPA_OK) { delete H; return st; }
  tm.mark("memset+validate");
  auto values_in = [&]() -> copa_status {  // every value chunk has landed (copa_fit) and is finite
    if (!vc) return COPA_OK;
    for (int i = 0; i < vc->n; ++i) {
      cudaStreamWaitEvent(s, vc->ev[i], 0);
      launch_validate_vals(h, i ? vc->e[i - 1] : vc->e0, vc->e[i]);
    }
    return check_err(h);
  };
  if (h.fib) {
    if (h.K > 0) k_srow_smooth<<<(unsigned)((h.K + 256) / 256), 256, 0, s>>>(h.K, h.l, h.srow);
    launch_count_fibers(h, h.fiber_ptr, h.fhist);
    size_t tb = h.cub_temp_bytes;
    if (h.K > 0) cub::DeviceScan::InclusiveSum(h.cub_temp, tb, h.fiber_ptr, h.fiber_ptr, (int)(h.K + 1), s);
    tm.mark("fiber_ptr");
    {  // feature relabeling by fiber mass (host, J <= 65535)
      std::vector<unsigned long long> hist((size_t)h.J);
      std::vector<int32_t> perm((size_t)h.J), inv((size_t)h.Jl);
      CUDA_TRY(cudaMemcpyAsync(hist.data(), h.fhist, sizeof(unsigned long long) * (size_t)h.J, cudaMemcpyDeviceToHost,
                               s), "hist copy");
      CUDA_TRY(cudaStreamSynchronize(s), "hist sync");
      int64_t Js = 0;
      compute_relabel(h.J, h.sc_G * h.sc_W, hist.data(), perm.data(), inv.data(), &Js);
      CUDA_TRY(cudaMemcpyAsync(h.perm, perm.data(), sizeof(int32_t) * (size_t)h.J, cudaMemcpyHostToDevice, s), "perm");
      CUDA_TRY(cudaMemcpyAsync(h.inv, inv.data(), sizeof(int32_t) * (size_t)h.Jl, cudaMemcpyHostToDevice, s), "inv");
      CUDA_TRY(cudaStreamSynchronize(s), "perm sync");
    }
    tm.mark("relabel");
    {  // g-stream layout: per-group run lengths (device) -> offsets and pass-B stage table (host)
      const int G = h.sc_G;
      // per-run fiber and tile counts (device), then the planning on the device
      const int64_t GK = (int64_t)G * h.K;
      int32_t* gcnt_dev = (int32_t*)h.layout_tmp;
      int32_t* tcnt_dev = gcnt_dev + GK + 4;
      int64_t* plan_tmp = reinterpret_cast<int64_t*>((char*)h.layout_tmp + 2 * sizeof(int32_t) * (GK + 4));
      CUDA_TRY(cudaMemsetAsync(gcnt_dev + GK, 0, 4 * sizeof(int32_t), s), "counts pad");
      CUDA_TRY(cudaMemsetAsync(tcnt_dev + GK, 0, 4 * sizeof(int32_t), s), "counts pad");
      launch_count_groups(h, gcnt_dev, tcnt_dev);
      tm.mark("count_groups");
      int64_t gtotal = 0;
      if (!plan_streams_device(h, gcnt_dev, tcnt_dev, plan_tmp, &gtotal)) {
        delete H;
        return fail(COPA_E_WORKSPACE, "internal: stage table exceeds its bound");
      }
      if (tm.on)
        fprintf(stderr,
                "[copa init] pass B: G=%d Jg=%lld W=%d RS=%d tiles/stage=%d patients/stage=%d slots=%d smem=%zu "
                "ranges=%d stages=%lld tiles=%lld (cap %lld) fibers=%lld workspace=%zu\n",
                h.sc_G, (long long)h.sc_Jg, h.sc_W, h.sc_RS, h.sc_FB, h.sc_PB, h.sc_NS, h.sc_smem, h.sc_ranges,
                (long long)h.nst, (long long)h.ntiles, (long long)tiles_cap(h), (long long)h.F, bytes);
      tm.mark("plan_streams+h2d");
      launch_passA_ranges(h);  // pass-A warp ranges (fiber-balanced) from fiber_ptr
    }
    tm.mark("passA ranges");
    launch_basis(h);
    tm.mark("basis");
    if (vc) {  // fiber build chunk by chunk as the values land
      for (int i = 0; i < vc->n; ++i) {
        cudaStreamWaitEvent(s, vc->ev[i], 0);
        launch_validate_vals(h, i ? vc->e[i - 1] : vc->e0, vc->e[i]);
        launch_build_fibers(h, i ? vc->k[i - 1] : 0, vc->k[i]);
      }
      st = check_err(h);
      if (st != COPA_OK) { delete H; return st; }
    } else {
      launch_build_fibers(h);
    }
    tm.mark("build_fibers");
    cudaMemsetAsync(h.fa_col + h.F, 0, 64 * sizeof(int32_t), s);  // slack read by the pass-A chunk grid
    cudaMemsetAsync(h.fa_val + h.F * h.l, 0, 64 * sizeof(double) * (size_t)h.l, s);
    cudaMemsetAsync(h.Vl, 0, sizeof(double) * (size_t)(h.Jl * h.R + 64), s);
    launch_layoutA(h);
    launch_build_tiles(h);  // pass B's tiled stream (k_fibers.cu) ...
    launch_stage_tab(h);    // ... and its stage table of tile bounds
    tm.mark("layoutA");
  } else {
    launch_row_patient(h);
    if (h.K == 0) cudaMemsetAsync(h.srow, 0, sizeof(int64_t), s);
    if (h.rowproj) {  // state rows k l (srow), m_k = l'_k from the per-patient basis
      if (h.K > 0) k_srow_smooth<<<(unsigned)((h.K + 256) / 256), 256, 0, s>>>(h.K, h.l, h.srow);
      launch_basis(h);
      cudaMemsetAsync(h.Prow, 0, sizeof(double) * (size_t)(h.rows * h.R), s);
      cudaMemsetAsync(h.Nrow, 0, sizeof(double) * (size_t)(h.rows * h.R), s);
    }
    st = values_in();
    if (st != COPA_OK) { delete H; return st; }
    const int rc = build_csc(h);
    if (rc != 0) {
      delete H;
      return rc == -2 ? fail(COPA_E_WORKSPACE, "internal: CSC chunk table exceeds its bound")
                      : cuda_fail(cudaGetLastError(), "CSC build");
    }
  }
  if (!polar_wide_ok(h) && plan_polar_order(h) != 0) {
    delete H;
    return cuda_fail(cudaGetLastError(), "polar order");
  }
  cudaMemcpyAsync(h.H, o->H0, sizeof(double) * RR, cudaMemcpyDefault, s);
  cudaMemcpyAsync(h.V, o->V0, sizeof(double) * (size_t)(h.J * h.R), cudaMemcpyDefault, s);
  if (h.K > 0) cudaMemcpyAsync(h.W, o->W0_local, sizeof(double) * (size_t)(h.K * h.R), cudaMemcpyDefault, s);
  cudaMemsetAsync(h.DH, 0, sizeof(double) * RR, s);
  cudaMemsetAsync(h.DV, 0, sizeof(double) * (size_t)(h.J * h.R), s);
  cudaMemsetAsync(h.DW, 0, sizeof(double) * (size_t)(h.K > 0 ? h.K * h.R : 1), s);
  // normX, W^T W and V^T V of the initial factors (C0: normX and W^T W are summed over ranks)
  launch_sumsq(h, h.scal + S_NORMX);
  launch_gram(h, h.W, h.W, h.K, 0, h.WtW);
  launch_gram(h, h.V, h.V, h.J, 0, h.VtV);
  // C0 payload: [normX] and [WtW]
  if (h.o.allreduce) {
    st = allreduce(h, h.scal + S_NORMX, 1);
    if (st == COPA_OK) st = allreduce(h, h.WtW, (int64_t)RR);
    if (st != COPA_OK) { delete H; return st; }
  }
  st = check_err(h);
  if (st != COPA_OK) { delete H; return st; }
  tm.mark("factors+grams");
  *out = H;
  return COPA_OK;
}

// Phase timing (copa_set_profiling): event pairs around each phase of the iteration, on the
// library's stream, summed at the next synchronisation point.
static const char* kPhaseNames[kPhases] = {"spmm", "polar", "fh", "allreduce_c1", "admm_H", "passB1",
                                           "grams_B", "scatter", "allreduce_c2", "admm_V", "fit"};

static void phase_begin(Handle& h, int ph) {
  if (!h.profiling) return;
  if (h.ev_used + 2 > (int)h.events.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    h.events.push_back(a);
    h.events.push_back(b);
  }
  h.ev_phase.push_back(ph);
  cudaEventRecord(h.events[h.ev_used], h.stream);
}
static void phase_end(Handle& h) {
  if (!h.profiling) return;
  cudaEventRecord(h.events[h.ev_used + 1], h.stream);
  h.ev_used += 2;
}
static void phase_collect(Handle& h) {
  for (int i = 0; i < h.ev_used; i += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, h.events[i], h.events[i + 1]) == cudaSuccess) {
      h.phase_ms[h.ev_phase[i / 2]] += ms;
      h.phase_calls[h.ev_phase[i / 2]] += 1;
    }
  }
  h.ev_used = 0;
  h.ev_phase.clear();
}

#define PHASE(ph, expr)                                                    \
  do {                                                                     \
    nvtxRangePushA(kPhaseNames[ph]);                                       \
    phase_begin(h, ph);                                                    \
    h.launches += (expr);                                                  \
    phase_end(h);                                                          \
    nvtxRangePop();                                                        \
    const cudaError_t pe_ = cudaGetLastError();                            \
    if (pe_ != cudaSuccess) return cuda_fail(pe_, kPhaseNames[ph]);         \
  } while (0)

static copa_status iterate_once(Handle& h) {
  copa_status st = COPA_OK;
  const int64_t RR = (int64_t)h.R * h.R;
  const bool wide = polar_wide_ok(h);
  PHASE(0, launch_spmm(h));
  PHASE(1, wide ? launch_polar_wide(h) : launch_polar_warp(h));  // wide: F_H fused into the polar kernel
  if (!wide) PHASE(2, launch_fh(h));
  PHASE(3, (st = allreduce(h, h.FH, RR), 0));  // C1
  if (st != COPA_OK) return st;
  PHASE(4, launch_admm_H(h));
  if (wide) {
    PHASE(5, launch_passB_wide(h));  // F_W, W rows, N, M and W^T W in one pass
  } else {
    PHASE(5, launch_passB_warp(h));
    PHASE(6, launch_gram(h, h.W, h.W, h.K, 0, h.WtW) + launch_gram(h, h.Nst, h.Nst, h.S, 0, h.M));
  }
  PHASE(7, launch_scatter(h));
  PHASE(8, (st = allreduce(h, h.comm2, h.J * h.R + 2 * RR), 0));  // C2
  if (st != COPA_OK) return st;
  PHASE(9, launch_admm_V(h));
  PHASE(10, launch_fit(h));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "iteration launch");
  return COPA_OK;
}

// One outer iteration, replayed from a CUDA graph when possible (the small workloads are
// launch-bound). The graph is captured on the second call of a single-rank, non-profiled handle
// (the first call runs eagerly, so one-off host work such as function attributes is done) and
// replayed afterwards; every kernel argument is a workspace pointer or an option, so the graph
// stays valid for the handle's lifetime. Multi-rank iterations call the allreduce callback and
// run eagerly.
static copa_status iterate_step(Handle& h) {
  if (h.o.allreduce || h.profiling || h.graph_failed || !h.use_graph) return iterate_once(h);
  if (!h.graph_exec) {
    if (h.eager_done < 1) {
      ++h.eager_done;
      return iterate_once(h);
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(h.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      h.graph_failed = true;
      return iterate_once(h);
    }
    copa_status st = iterate_once(h);
    const cudaError_t ce = cudaStreamEndCapture(h.stream, &g);
    if (st != COPA_OK || ce != cudaSuccess || !g ||
        cudaGraphInstantiate(&h.graph_exec, g, 0) != cudaSuccess) {
      cudaGetLastError();
      if (g) cudaGraphDestroy(g);
      h.graph_exec = nullptr;
      h.graph_failed = true;
      if (st != COPA_OK) return st;
      return iterate_once(h);  // nothing ran during the capture
    }
    h.graph = g;
  }
  CUDA_TRY(cudaGraphLaunch(h.graph_exec, h.stream), "graph launch");
  return COPA_OK;
}

copa_status copa_iterate(copa_handle* H, int32_t n_outer, double* fit_host) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  if (n_outer < 0) return fail(COPA_E_ARG, "n_outer < 0");
  Handle& h = H->h;
  int32_t done = 0;
  while (done < n_outer) {
    int32_t chunk = n_outer - done < 1024 ? n_outer - done : 1024;
    for (int32_t t = 0; t < chunk; ++t) {
      copa_status st = iterate_step(h);
      if (st != COPA_OK) return st;
      cudaMemcpyAsync(h.fit_ring + t, h.scal + S_FIT, sizeof(double), cudaMemcpyDeviceToDevice, h.stream);
      ++h.iterations;
    }
    if (fit_host)
      CUDA_TRY(cudaMemcpyAsync(fit_host + done, h.fit_ring, sizeof(double) * chunk, cudaMemcpyDefault, h.stream),
               "fit copy");
    copa_status st = check_err(h);
    if (st != COPA_OK) return st;
    phase_collect(h);
    done += chunk;
  }
  return COPA_OK;
}

copa_status copa_iterate_until(copa_handle* H, int32_t max_outer, double outer_tol, double* fit_host,
                               int32_t* n_done) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  if (max_outer < 0 || !(outer_tol >= 0)) return fail(COPA_E_ARG, "max_outer < 0 or outer_tol < 0");
  Handle& h = H->h;
  if (n_done) *n_done = 0;
  double prev = 0.0;
  for (int32_t t = 0; t < max_outer; ++t) {
    copa_status st = iterate_step(h);
    if (st != COPA_OK) return st;
    ++h.iterations;
    double fit = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&fit, h.scal + S_FIT, sizeof(double), cudaMemcpyDeviceToHost, h.stream), "fit copy");
    st = check_err(h);  // synchronises
    if (st != COPA_OK) return st;
    phase_collect(h);
    if (fit_host) fit_host[t] = fit;
    if (n_done) *n_done = t + 1;
    if (t >= 1 && std::fabs(fit - prev) < outer_tol * std::fmax(std::fabs(prev), 1.0)) break;
    prev = fit;
  }
  return COPA_OK;
}

copa_status copa_get_state(copa_handle* H, const copa_state* out) {
  if (!H || !out) return fail(COPA_E_ARG, "null handle/state");
  Handle& h = H->h;
  const size_t RR = sizeof(double) * (size_t)h.R * h.R, JR = sizeof(double) * (size_t)(h.J * h.R),
               KR = sizeof(double) * (size_t)(h.K * h.R);
  cudaStream_t s = h.stream;
  const double* src[8] = {h.H, h.V, h.W, h.DH, h.DV, h.DW, h.WtW, h.VtV};
  double* dst[8] = {out->H, out->V, out->W_local, out->DH, out->DV, out->DW_local, out->WtW, out->VtV};
  const size_t sz[8] = {RR, JR, KR, RR, JR, KR, RR, RR};
  for (int i = 0; i < 8; ++i) {
    if (sz[i] == 0) continue;
    if (!dst[i]) return fail(COPA_E_ARG, "null state pointer");
    CUDA_TRY(cudaMemcpyAsync(dst[i], src[i], sz[i], cudaMemcpyDefault, s), "get state");
  }
  CUDA_TRY(cudaStreamSynchronize(s), "get state sync");
  // the caller's struct is const; iterations is reported through copa_get_stats
  return COPA_OK;
}

copa_status copa_set_state(copa_handle* H, const copa_state* in) {
  if (!H || !in) return fail(COPA_E_ARG, "null handle/state");
  Handle& h = H->h;
  if (!in->H || !in->V || !in->DH || !in->DV || (h.K > 0 && (!in->W_local || !in->DW_local)))
    return fail(COPA_E_ARG, "null state pointer");
  const size_t RR = sizeof(double) * (size_t)h.R * h.R, JR = sizeof(double) * (size_t)(h.J * h.R),
               KR = sizeof(double) * (size_t)(h.K * h.R);
  cudaStream_t s = h.stream;
  CUDA_TRY(cudaMemcpyAsync(h.H, in->H, RR, cudaMemcpyDefault, s), "set H");
  CUDA_TRY(cudaMemcpyAsync(h.DH, in->DH, RR, cudaMemcpyDefault, s), "set DH");
  CUDA_TRY(cudaMemcpyAsync(h.V, in->V, JR, cudaMemcpyDefault, s), "set V");
  CUDA_TRY(cudaMemcpyAsync(h.DV, in->DV, JR, cudaMemcpyDefault, s), "set DV");
  if (h.K > 0) {
    CUDA_TRY(cudaMemcpyAsync(h.W, in->W_local, KR, cudaMemcpyDefault, s), "set W");
    CUDA_TRY(cudaMemcpyAsync(h.DW, in->DW_local, KR, cudaMemcpyDefault, s), "set DW");
  }
  // the Grams the next iteration's H-mode reads (Alg.1 l.11)
  if (in->VtV) CUDA_TRY(cudaMemcpyAsync(h.VtV, in->VtV, RR, cudaMemcpyDefault, s), "set VtV");
  else launch_gram(h, h.V, h.V, h.J, 0, h.VtV);
  if (in->WtW) {
    CUDA_TRY(cudaMemcpyAsync(h.WtW, in->WtW, RR, cudaMemcpyDefault, s), "set WtW");
  } else {
    launch_gram(h, h.W, h.W, h.K, 0, h.WtW);
    copa_status st = allreduce(h, h.WtW, (int64_t)h.R * h.R);
    if (st != COPA_OK) return st;
  }
  h.iterations = in->iterations;
  return check_err(h);
}

copa_status copa_get_factors(copa_handle* H, double* Hout, double* Vout, double* Wout) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  Handle& h = H->h;
  if (Hout) CUDA_TRY(cudaMemcpyAsync(Hout, h.H, sizeof(double) * h.R * h.R, cudaMemcpyDefault, h.stream), "get H");
  if (Vout) CUDA_TRY(cudaMemcpyAsync(Vout, h.V, sizeof(double) * h.J * h.R, cudaMemcpyDefault, h.stream), "get V");
  if (Wout && h.K > 0)
    CUDA_TRY(cudaMemcpyAsync(Wout, h.W, sizeof(double) * h.K * h.R, cudaMemcpyDefault, h.stream), "get W");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "get sync");
  return COPA_OK;
}

copa_status copa_get_duals(copa_handle* H, double* DH, double* DV, double* DW) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  Handle& h = H->h;
  if (DH) CUDA_TRY(cudaMemcpyAsync(DH, h.DH, sizeof(double) * h.R * h.R, cudaMemcpyDefault, h.stream), "get DH");
  if (DV) CUDA_TRY(cudaMemcpyAsync(DV, h.DV, sizeof(double) * h.J * h.R, cudaMemcpyDefault, h.stream), "get DV");
  if (DW && h.K > 0)
    CUDA_TRY(cudaMemcpyAsync(DW, h.DW, sizeof(double) * h.K * h.R, cudaMemcpyDefault, h.stream), "get DW");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "get sync");
  return COPA_OK;
}

copa_status copa_get_U(copa_handle* H, double* U) {
  if (!H || !U) return fail(COPA_E_ARG, "null handle/U");
  Handle& h = H->h;
  cudaPointerAttributes attr{};
  cudaError_t e = cudaPointerGetAttributes(&attr, U);
  if (e != cudaSuccess) cudaGetLastError();
  if (e == cudaSuccess && (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged)) {
    launch_U(h, U, 0, h.K);
  } else if (h.K > 0) {
    // host destination: patient chunks staged through the state buffer N (S x R doubles; overwritten,
    // rebuilt by the next iteration's pass B)
    std::vector<int64_t> prp((size_t)h.K + 1);
    CUDA_TRY(cudaMemcpyAsync(prp.data(), h.p.patient_row_ptr, sizeof(int64_t) * prp.size(), cudaMemcpyDeviceToHost,
                             h.stream), "get U prp");
    CUDA_TRY(cudaStreamSynchronize(h.stream), "get U sync");
    const int64_t cap = h.S > 0 ? h.S : 0;
    int64_t k0 = 0;
    while (k0 < h.K) {
      int64_t k1 = k0;
      while (k1 < h.K && prp[(size_t)k1 + 1] - prp[(size_t)k0] <= cap) ++k1;
      if (k1 == k0) return fail(COPA_E_UNSUPPORTED, "host U: a patient has more rows than the state buffer");
      launch_U(h, h.Nst, k0, k1);
      CUDA_TRY(cudaMemcpyAsync(U + prp[(size_t)k0] * h.R, h.Nst,
                               sizeof(double) * (size_t)(prp[(size_t)k1] - prp[(size_t)k0]) * h.R,
                               cudaMemcpyDeviceToHost, h.stream), "get U");
      CUDA_TRY(cudaStreamSynchronize(h.stream), "get U sync");  // N is reused by the next chunk
      k0 = k1;
    }
  }
  return check_err(h);
}

copa_status copa_get_stats(copa_handle* H, copa_stats* out) {
  if (!H || !out) return fail(COPA_E_ARG, "null handle/out");
  Handle& h = H->h;
  double sc[S_COUNT];
  CUDA_TRY(cudaMemcpyAsync(sc, h.scal, sizeof(sc), cudaMemcpyDeviceToHost, h.stream), "stats copy");
  unsigned long long* cnt = (unsigned long long*)(h.partial);
  cudaMemsetAsync(cnt, 0, sizeof(*cnt), h.stream);
  if (h.K > 0)
    k_rank_deficient<<<(unsigned)((h.K + 255) / 256), 256, 0, h.stream>>>(h.m, h.rank, h.K, h.R, cnt);
  unsigned long long rd = 0;
  CUDA_TRY(cudaMemcpyAsync(&rd, cnt, sizeof(rd), cudaMemcpyDeviceToHost, h.stream), "stats copy");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "stats sync");
  out->fit = sc[S_FIT];
  out->rho[0] = sc[S_RHO_H];
  out->rho[1] = sc[S_RHO_W];
  out->rho[2] = sc[S_RHO_V];
  out->normX = sc[S_NORMX];
  out->iterations = h.iterations;
  out->fibers = h.F;
  out->tiles = h.ntiles;
  out->state_rows = h.S;
  out->rank_deficient = (int64_t)rd;
  unsigned long long dg[kDiagSlots], stp[4];
  launch_count_zeros(h);
  CUDA_TRY(cudaMemcpyAsync(dg, h.diag, sizeof(dg), cudaMemcpyDeviceToHost, h.stream), "stats diag");
  CUDA_TRY(cudaMemcpyAsync(stp, h.steps, sizeof(stp), cudaMemcpyDeviceToHost, h.stream), "stats steps");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "stats sync");
  auto ratio = [](unsigned long long b, double none) {
    double v;
    memcpy(&v, &b, sizeof(v));
    return std::isinf(v) ? none : v;
  };
  out->sparsity_V = (double)stp[3] / (double)(h.J * h.R);
  for (int i = 0; i < 3; ++i) out->inner_steps[i] = (int64_t)stp[i];
  out->polar_near = (int64_t)dg[D_POLAR_NEAR];
  out->polar_min_kept = ratio(dg[D_POLAR_KEPT], 1.0);
  out->polar_max_dropped = ratio(dg[D_POLAR_DROP], 0.0);
  out->basis_near = (int64_t)dg[D_BASIS_NEAR];
  out->basis_min_kept = ratio(dg[D_BASIS_KEPT], 1.0);
  out->basis_max_dropped = ratio(dg[D_BASIS_DROP], 0.0);
  return COPA_OK;
}

copa_status copa_debug_state(copa_handle* H, double* Pp, double* Qt, int32_t* m, int64_t* srow, int32_t* rank) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  Handle& h = H->h;
  size_t SR = sizeof(double) * (size_t)(h.S * h.R);
  if (Pp) CUDA_TRY(cudaMemcpyAsync(Pp, h.Pp, SR, cudaMemcpyDefault, h.stream), "dbg Pp");
  if (Qt) CUDA_TRY(cudaMemcpyAsync(Qt, h.Qt, SR, cudaMemcpyDefault, h.stream), "dbg Qt");
  if (m && h.K) CUDA_TRY(cudaMemcpyAsync(m, h.m, sizeof(int32_t) * h.K, cudaMemcpyDefault, h.stream), "dbg m");
  if (srow) CUDA_TRY(cudaMemcpyAsync(srow, h.srow, sizeof(int64_t) * (h.K + 1), cudaMemcpyDefault, h.stream), "dbg srow");
  if (rank && h.K) CUDA_TRY(cudaMemcpyAsync(rank, h.rank, sizeof(int32_t) * h.K, cudaMemcpyDefault, h.stream), "dbg rank");
  CUDA_TRY(cudaStreamSynchronize(h.stream), "dbg sync");
  return COPA_OK;
}

void copa_destroy(copa_handle* H) {
  if (!H) return;
  for (auto e : H->h.events) cudaEventDestroy(e);
  if (H->h.graph_exec) cudaGraphExecDestroy(H->h.graph_exec);
  if (H->h.graph) cudaGraphDestroy(H->h.graph);
  delete H;
}

copa_status copa_set_profiling(copa_handle* H, int32_t on) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  Handle& h = H->h;
  h.profiling = on != 0;
  for (int i = 0; i < kPhases; ++i) { h.phase_ms[i] = 0; h.phase_calls[i] = 0; }
  h.launches = 0;
  return COPA_OK;
}

copa_status copa_get_phase_times(copa_handle* H, double* ms, int64_t* calls, int32_t n, int32_t* n_phases,
                                 int64_t* launches) {
  if (!H) return fail(COPA_E_ARG, "null handle");
  Handle& h = H->h;
  CUDA_TRY(cudaStreamSynchronize(h.stream), "phase sync");
  phase_collect(h);
  for (int i = 0; i < n && i < kPhases; ++i) {
    if (ms) ms[i] = h.phase_ms[i];
    if (calls) calls[i] = h.phase_calls[i];
  }
  if (n_phases) *n_phases = kPhases;
  if (launches) *launches = h.launches;
  return COPA_OK;
}

const char* copa_phase_name(int32_t i) { return (i >= 0 && i < kPhases) ? kPhaseNames[i] : ""; }

// ---------------------------------------------------------------- end-to-end with host inputs
static size_t input_bytes(const copa_problem* p) {
  size_t b = 0;
  b += align_up(sizeof(int64_t) * (size_t)(p->K_local + 1));
  b += align_up(sizeof(int64_t) * (size_t)(p->rows + 1));
  b += align_up(sizeof(int32_t) * (size_t)(p->nnz > 0 ? p->nnz : 1));
  b += align_up(sizeof(double) * (size_t)(p->nnz > 0 ? p->nnz : 1));
  b += align_up(sizeof(double) * (size_t)(p->rows > 0 ? p->rows : 1));
  b += 3 * align_up(sizeof(double) * 1);  // placeholders
  return b;
}

copa_status copa_fit_workspace_size(const copa_problem* p, const copa_options* o, size_t* bytes) {
  copa_status st = check_args(p, o);
  if (st != COPA_OK) return st;
  if (!bytes) return fail(COPA_E_ARG, "null bytes");
  Handle h{};
  fill_sizes(h, p, o);
  // fibers = distinct (patient, feature) pairs, counted from the host CSR (the workspace grows
  // ~150 bytes per fiber, so the sum_k min(J, nnz_k) bound overshoots a B200 at Scale); host threads
  // over patient chunks, a feature bitmap each. Out-of-range columns are left to init's validation
  // and counted as distinct.
  int64_t F = 0;
  if (h.fib) {
    const int64_t K = p->K_local;
    const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<int64_t> part(nth, 0);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nth; ++t)
      pool.emplace_back([&, t]() {
        std::vector<uint64_t> bits((size_t)((p->J + 63) / 64), 0);
        int64_t cnt = 0;
        auto rowp = [&](int64_t k) -> int64_t {  // unvalidated input: every host read stays in bounds
          const int64_t r = std::min<int64_t>(std::max<int64_t>(p->patient_row_ptr[k], 0), p->rows);
          return std::min<int64_t>(std::max<int64_t>(p->row_ptr[r], 0), p->nnz);
        };
        for (int64_t k = K * t / nth; k < K * (t + 1) / nth; ++k) {
          const int64_t a = rowp(k), b = std::max(a, rowp(k + 1));
          for (int64_t x = a; x < b; ++x) {
            const int32_t j = p->col[x];
            if (j < 0 || j >= p->J) { ++cnt; continue; }
            uint64_t& wd = bits[(size_t)j >> 6];
            const uint64_t m = 1ull << (j & 63);
            cnt += (wd & m) ? 0 : 1;
            wd |= m;
          }
          for (int64_t x = a; x < b; ++x) {
            const int32_t j = p->col[x];
            if (j >= 0 && j < p->J) bits[(size_t)j >> 6] = 0;
          }
        }
        part[t] = cnt;
      });
    for (auto& th : pool) th.join();
    for (auto v : part) F += v;
    cub::DeviceScan::InclusiveSum(nullptr, h.cub_temp_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)(h.K + 1));
  }
  h.F = F;
  size_t need = carve(h, nullptr) + input_bytes(p) + align_up(sizeof(double) * ((size_t)p->J * p->R * 2 +
                                                                               (size_t)p->R * p->R +
                                                                               (size_t)p->K_local * p->R)) + 4096;
  *bytes = need;
  return COPA_OK;
}

copa_status copa_fit(const copa_problem* hp, const copa_options* ho, void* ws, size_t bytes, int32_t n_outer,
                     double* fit_host, double* H_out, double* V_out, double* W_out) {
  copa_status st = check_args(hp, ho);
  if (st != COPA_OK) return st;
  if (!ws || ((uintptr_t)ws & 255)) return fail(COPA_E_WORKSPACE, "workspace null or misaligned");
  cudaStream_t s = (cudaStream_t)ho->stream;
  Carver c{(char*)ws};
  copa_problem dp = *hp;
  int64_t* prp = c.take<int64_t>(hp->K_local + 1);
  int64_t* rp = c.take<int64_t>(hp->rows + 1);
  int32_t* col = c.take<int32_t>(hp->nnz);
  double* val = c.take<double>(hp->nnz);
  double* tim = c.take<double>(hp->rows);
  double* H0 = c.take<double>((int64_t)hp->R * hp->R);
  double* V0 = c.take<double>(hp->J * hp->R);
  double* W0 = c.take<double>(hp->K_local * hp->R);
  if (c.off > bytes) return fail(COPA_E_WORKSPACE, "workspace too small for the inputs");
  // the structure, columns and times first (on the caller's stream, read by the first init
  // stages), then the values on a second stream, overlapped with those stages (init_impl waits for
  // them before the fiber build)
  CUDA_TRY(cudaMemcpyAsync(prp, hp->patient_row_ptr, sizeof(int64_t) * (hp->K_local + 1), cudaMemcpyDefault, s), "h2d");
  CUDA_TRY(cudaMemcpyAsync(rp, hp->row_ptr, sizeof(int64_t) * (hp->rows + 1), cudaMemcpyDefault, s), "h2d");
  if (hp->nnz > 0) CUDA_TRY(cudaMemcpyAsync(col, hp->col, sizeof(int32_t) * hp->nnz, cudaMemcpyDefault, s), "h2d");
  if (hp->visit_time && hp->rows > 0)
    CUDA_TRY(cudaMemcpyAsync(tim, hp->visit_time, sizeof(double) * hp->rows, cudaMemcpyDefault, s), "h2d");
  struct Aux {
    cudaStream_t s2 = nullptr;
    cudaEvent_t first = nullptr;
    ValChunks vc;
    ~Aux() {
      if (s2) cudaStreamSynchronize(s2);
      if (first) cudaEventDestroy(first);
      for (int i = 0; i < vc.n; ++i) cudaEventDestroy(vc.ev[i]);
      if (s2) cudaStreamDestroy(s2);
    }
  } aux;
  CUDA_TRY(cudaStreamCreateWithFlags(&aux.s2, cudaStreamNonBlocking), "fit stream");
  CUDA_TRY(cudaEventCreateWithFlags(&aux.first, cudaEventDisableTiming), "fit event");
  CUDA_TRY(cudaEventRecord(aux.first, s), "fit event");
  CUDA_TRY(cudaStreamWaitEvent(aux.s2, aux.first, 0), "fit event");
  {  // the values in 4 patient chunks (host CSR offsets), one event each
    // (validated structure is not known yet: the offsets are clamped to [0, nnz]; a malformed
    // row_ptr is rejected by init's validation before any value is read)
    const int nch = 4;
    const int64_t K = hp->K_local, nnz = hp->nnz;
    auto at = [&](int64_t k) -> int64_t {  // host reads of unvalidated input stay in bounds
      if (K <= 0) return 0;
      const int64_t r = std::min<int64_t>(std::max<int64_t>(hp->patient_row_ptr[k], 0), hp->rows);
      const int64_t e = hp->row_ptr[r];
      return e < 0 ? 0 : (e > nnz ? nnz : e);
    };
    aux.vc.e0 = at(0);
    int64_t c0 = 0;  // copy ranges cover [0, nnz) whatever the offsets
    for (int i = 0; i < nch; ++i) {
      const int64_t k1 = K * (i + 1) / nch;
      int64_t e1 = std::max(at(k1), i ? aux.vc.e[i - 1] : aux.vc.e0);
      const int64_t c1 = i == nch - 1 ? nnz : std::max(e1, c0);
      CUDA_TRY(cudaEventCreateWithFlags(&aux.vc.ev[i], cudaEventDisableTiming), "fit event");
      aux.vc.n = i + 1;
      aux.vc.k[i] = k1;
      aux.vc.e[i] = e1;
      if (c1 > c0)
        CUDA_TRY(cudaMemcpyAsync(val + c0, hp->val + c0, sizeof(double) * (c1 - c0), cudaMemcpyDefault, aux.s2), "h2d");
      c0 = c1;
      CUDA_TRY(cudaEventRecord(aux.vc.ev[i], aux.s2), "fit event");
    }
  }
  copa_options dopt = *ho;
  CUDA_TRY(cudaMemcpyAsync(H0, ho->H0, sizeof(double) * hp->R * hp->R, cudaMemcpyDefault, s), "h2d");
  CUDA_TRY(cudaMemcpyAsync(V0, ho->V0, sizeof(double) * hp->J * hp->R, cudaMemcpyDefault, s), "h2d");
  if (hp->K_local > 0)
    CUDA_TRY(cudaMemcpyAsync(W0, ho->W0_local, sizeof(double) * hp->K_local * hp->R, cudaMemcpyDefault, s), "h2d");
  dopt.H0 = H0; dopt.V0 = V0; dopt.W0_local = W0;
  dp.patient_row_ptr = prp; dp.row_ptr = rp; dp.col = col; dp.val = val;
  dp.visit_time = hp->visit_time ? tim : nullptr;
  copa_handle* h = nullptr;
  st = init_impl(&dp, &dopt, (char*)ws + c.off, bytes - c.off, &h, &aux.vc);
  if (st != COPA_OK) return st;
  st = copa_iterate(h, n_outer, fit_host);
  if (st == COPA_OK) st = copa_get_factors(h, H_out, V_out, W_out);
  copa_destroy(h);
  return st;
}

}  // extern "C"
