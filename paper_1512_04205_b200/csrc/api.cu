#include <cstdlib>
// api.cu — the C ABI of libcdmd (include/cdmd.h): host-side validation, handle
// state, workspace carving and kernel launches.  No torch types cross this
// boundary; the Python binding (paper_1512_04205_b200/cdmd.py) only marshals
// pointers and sizes.
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <math.h>
#include <string.h>

#include "handle.h"

namespace cdmd {
cudaError_t smem_optin(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, kern})) return cudaSuccess;
  cudaFuncAttributes a;
  if ((e = cudaFuncGetAttributes(&a, kern)) != cudaSuccess) return e;
  int optin = 0;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({dev, kern});
  return e;
}
}  // namespace cdmd

using namespace cdmd;

namespace cdmd {
int persistent_ctas(int sms) {
  static int reserve = -1;
  if (reserve < 0) {
    const char* e = getenv("CDMD_PERSIST_RESERVE");
    reserve = e ? atoi(e) : 0;
    if (reserve < 0) reserve = 0;
  }
  int g = sms - reserve;
  if (g_persist_limit > 0 && g > g_persist_limit) g = g_persist_limit;   // cdmd_sm_partition
  return g < 1 ? 1 : g;
}

size_t hqr_smem_bytes(int k);
cudaError_t launch_hqr_eig(int k, const double* A, double* W, double* VR, int* info, double* scratch,
                           cudaStream_t st);
}  // namespace cdmd

namespace {

size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

cdmd_status cuda_status(cudaError_t e) { return e == cudaSuccess ? CDMD_OK : CDMD_ERR_CUDA; }

cdmd_status check_video(const cdmd_video* v) {
  if (!v || !v->X) return CDMD_ERR_ARG;
  if (v->m < 2) return CDMD_ERR_RANGE;
  if (v->n_total < 1 || v->n_local < 1 || v->pix0 < 0 || v->pix0 + v->n_local > v->n_total)
    return CDMD_ERR_RANGE;
  if ((reinterpret_cast<uintptr_t>(v->X) & 15) != 0) return CDMD_ERR_ARG;
  if (v->ld < v->n_local || (v->ld & 15) != 0) return CDMD_ERR_ARG;
  if (v->pix0 % 128 != 0) return CDMD_ERR_ARG;
  if (v->n_total > (int64_t)8421504) return CDMD_ERR_RANGE;  // 255 n < 2^31 (exact int32 sums)
  return CDMD_OK;
}

cdmd_status check_sensing(int64_t n_total, const cdmd_sensing* c) {
  if (!c) return CDMD_ERR_ARG;
  if (c->kind < CDMD_SPIXEL || c->kind > CDMD_SRFT) return CDMD_ERR_ARG;
  if (c->kind == CDMD_SRFT) {   // p real rows = Re, Im of p/2 distinct frequencies
    if (c->p < 2 || (c->p & 1) || c->p > 2 * n_total) return CDMD_ERR_RANGE;
    return CDMD_OK;
  }
  if (c->p < 1 || c->p > n_total) return CDMD_ERR_RANGE;
  if (c->kind == CDMD_SPARSE && c->s > 0 && c->s <= 1.0) return CDMD_ERR_RANGE;
  if (c->kind == CDMD_SPARSE && c->s <= 0 && n_total < 3) return CDMD_ERR_RANGE;  // n/ln n > 1
  return CDMD_OK;
}

int64_t kpad_of(int k) { return round_up(k, CDMD_NBLK); }
int64_t mpad_of(int64_t m) { return round_up(m - 1, CDMD_KBLK); }

struct ModelLayout {
  size_t lambda, omega, pair, sigma, Mfold, beta, support, Mq, Mq_scale, coef, coef_col, dev_info, total;
};

ModelLayout model_layout(int k, int K, int64_t m) {
  ModelLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += al256(b); return o; };
  const int64_t kp = kpad_of(k), mp = mpad_of(m);
  L.lambda = take(sizeof(double) * 2 * k);
  L.omega = take(sizeof(double) * 2 * k);
  L.pair = take(sizeof(int32_t) * k);
  L.sigma = take(sizeof(double) * k);
  L.Mfold = take(sizeof(double) * (m - 1) * k);
  L.beta = take(sizeof(double) * 2 * K);
  L.support = take(sizeof(int32_t) * K);
  L.Mq = take((size_t)kp * CDMD_LIMBS * mp);
  L.Mq_scale = take(sizeof(double) * kp);
  L.coef = take(sizeof(float) * 2 * K * m);
  L.coef_col = take(sizeof(int32_t) * 2 * K);
  L.dev_info = take(sizeof(int32_t) * 8);
  L.total = off;
  return L;
}

cdmd_status check_model(const cdmd_model* M, int64_t m) {
  if (!M || !M->lambda || !M->Mq || !M->coef) return CDMD_ERR_ARG;
  if (M->m != m) return CDMD_ERR_ARG;
  if (M->k_eff < 1 || M->k_eff > M->k) return CDMD_ERR_ARG;  // cdmd_fit not run
  return CDMD_OK;
}

}  // namespace

extern "C" {

const char* cdmd_version(void) { return "cdmd-b200 0.1 (sm_100a)"; }


uint64_t cdmd_kernel_launches(void) { return cdmd::launch_counter().load(std::memory_order_relaxed); }

cdmd_status cdmd_eigensolver_stats(cdmd_handle h, uint64_t* runs, uint64_t* fallbacks) {
  if (!h) return CDMD_ERR_ARG;
  if (runs) *runs = h->lz_runs.load();
  if (fallbacks) *fallbacks = h->lz_fallbacks.load();
  return CDMD_OK;
}

cdmd_status cdmd_set_background_selection(cdmd_handle h, double omega_eps) {
  if (!h) return CDMD_ERR_ARG;
  if (!(omega_eps >= 0.0) || !isfinite(omega_eps)) return CDMD_ERR_RANGE;
  h->omega_eps = omega_eps;
  return CDMD_OK;
}

const char* cdmd_status_str(cdmd_status s) {
  switch (s) {
    case CDMD_OK: return "ok";
    case CDMD_ERR_ARG: return "invalid argument";
    case CDMD_ERR_RANGE: return "argument out of range";
    case CDMD_ERR_NUMERIC: return "numerical failure";
    case CDMD_ERR_CUDA: return "CUDA error";
    case CDMD_ERR_WORKSPACE: return "workspace too small";
    case CDMD_ERR_UNSUPPORTED: return "unsupported device (needs sm_100a)";
  }
  return "unknown status";
}

cdmd_status cdmd_create(int device, cdmd_handle* out) {
  if (!out) return CDMD_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return CDMD_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return CDMD_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return CDMD_ERR_UNSUPPORTED;  // built for sm_100a only
  if (cudaSetDevice(device) != cudaSuccess) return CDMD_ERR_CUDA;
  cdmd_handle h = new cdmd_handle_s();
  h->device = device;
  h->sm_count = prop.multiProcessorCount;
  cdmd_status st = CDMD_OK;
  if (cublasCreate(&h->blas) != CUBLAS_STATUS_SUCCESS) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK) cublasSetMathMode(h->blas, CUBLAS_DEFAULT_MATH);  // fp64, no emulation
  if (st == CDMD_OK && cusolverDnCreate(&h->solver) != CUSOLVER_STATUS_SUCCESS) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cusolverDnCreateParams(&h->params) != CUSOLVER_STATUS_SUCCESS) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cudaMalloc(&h->gauss_table, 65536 * sizeof(uint16_t)) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cudaMallocHost(&h->host_info, 16 * sizeof(int32_t)) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cudaMalloc(&h->sched, CDMD_SCHED_SLOTS * sizeof(int)) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && launch_gaussian_table(h->gauss_table, 0) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cudaMalloc(&h->srft_table, 16385 * sizeof(uint16_t)) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && launch_srft_table(h->srft_table, 0) != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st == CDMD_OK && cudaDeviceSynchronize() != cudaSuccess) st = CDMD_ERR_CUDA;
  if (st != CDMD_OK) {
    cdmd_destroy(h);
    return st;
  }
  *out = h;
  return CDMD_OK;
}

void cdmd_destroy(cdmd_handle h) {
  if (!h) return;
  if (h->params) cusolverDnDestroyParams(h->params);
  if (h->solver) cusolverDnDestroy(h->solver);
  if (h->blas) cublasDestroy(h->blas);
  if (h->gauss_table) cudaFree(h->gauss_table);
  if (h->srft_table) cudaFree(h->srft_table);
  if (h->host_info) cudaFreeHost(h->host_info);
  if (h->sched) cudaFree(h->sched);
  for (auto& kv : h->sparse_csc) {
    cudaFree(kv.second.pos);
    cudaFree(kv.second.rs);
  }
  delete h;
}

// ------------------------------------------------------------------- sketch
// A sparse row longer than its ELL capacity (mu + 12 sqrt(mu) + 16 entries; a
// binomial tail below 1e-20 per row) would be truncated.  The index lists depend
// only on (n, p, s, seed), so the first call with a plan reads the overflow flag back
// once (one stream sync) and reports CDMD_ERR_NUMERIC; later calls with a checked plan
// do not sync.
static bool sparse_checked(cdmd_handle h, const SensingPlan& P, uint64_t seed) {
  std::lock_guard<std::mutex> g(h->mu);
  return h->sparse_checked.count(std::make_tuple(P.n, P.p, P.s, seed)) != 0;
}

static cdmd_status check_sparse_once(cdmd_handle h, const SensingPlan& P, uint64_t seed, const int32_t* flags,
                                     cudaStream_t st) {
  int32_t f = 0;
  if (cudaMemcpyAsync(&f, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return CDMD_ERR_CUDA;
  if (f & FLAG_SPARSE_OVERFLOW) return CDMD_ERR_NUMERIC;
  std::lock_guard<std::mutex> g(h->mu);
  h->sparse_checked.insert(std::make_tuple(P.n, P.p, P.s, seed));
  return CDMD_OK;
}

static size_t sketch_ws_bytes(const cdmd_video* v, const SensingPlan& P) {
  size_t b = al256(sensing_ws_bytes(P));
  if (P.kind == CDMD_GAUSSIAN || P.kind == CDMD_SRFT) b += al256(sizeof(float) * (size_t)gaussian_part_floats(*v, P.p));
  return b;
}

size_t cdmd_sketch_workspace_bytes(const cdmd_video* v, const cdmd_sensing* c) {
  if (!v || !c || check_sensing(v->n_total, c) != CDMD_OK) return 0;
  return sketch_ws_bytes(v, make_plan(v->n_total, c));
}

cdmd_status cdmd_sketch(cdmd_handle h, const cdmd_video* v, const cdmd_sensing* c, void* Y,
                        int64_t ldy, void* ws, size_t ws_bytes, cdmd_stream st_) {
  cudaStream_t st = (cudaStream_t)st_;
  if (!h || !Y) return CDMD_ERR_ARG;
  cdmd_status s = check_video(v);
  if (s != CDMD_OK) return s;
  if ((s = check_sensing(v->n_total, c)) != CDMD_OK) return s;
  if (ldy < c->p) return CDMD_ERR_ARG;
  const SensingPlan P = make_plan(v->n_total, c);
  const size_t need = sketch_ws_bytes(v, P);
  if (ws_bytes < need || (need > 256 && !ws)) return CDMD_ERR_WORKSPACE;
  if (ws && (reinterpret_cast<uintptr_t>(ws) & 255) != 0) return CDMD_ERR_ARG;
  cudaError_t e = cudaSuccess;
  switch (P.kind) {
    case CDMD_SPIXEL: {
      int32_t* rows = (int32_t*)ws;
      e = launch_spixel_rows(P, rows, st);
      if (e == cudaSuccess) e = launch_sketch_spixel(*v, P, rows, (int32_t*)Y, ldy, st);
      break;
    }
    case CDMD_SPARSE: {
      const bool checked = sparse_checked(h, P, c->seed);
      if (!checked) {   // the first call of a plan syncs once: not inside a graph capture
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) return CDMD_ERR_CUDA;
        if (cap != cudaStreamCaptureStatusNone) return CDMD_ERR_ARG;
      }
      int32_t* ell = (int32_t*)ws;
      int32_t* counts = (int32_t*)((char*)ws + al256(sizeof(int32_t) * P.p * P.cap));
      int32_t* flags = (int32_t*)((char*)counts + al256(sizeof(int32_t) * P.p));
      const bool sorted = sketch_sparse_sorted_supported(P.p) && !getenv("CDMD_SPARSE_ELL");
      const SparseCsc* csc = nullptr;
      if (sorted && checked) {   // the cached pixel-sorted C: no per-call index generation
        csc = sparse_csc_get(h, P, c->seed, nullptr, nullptr, st, &e);
      }
      if (!csc) {
        e = cudaMemsetAsync(flags, 0, 16, st);
        if (e == cudaSuccess) e = launch_sparse_rows(P, ell, counts, flags, st);
        if (e == cudaSuccess && !checked) {
          const cdmd_status cs = check_sparse_once(h, P, c->seed, flags, st);
          if (cs != CDMD_OK) return cs;
        }
        if (e == cudaSuccess && sorted) csc = sparse_csc_get(h, P, c->seed, ell, counts, st, &e);
      }
      if (e == cudaSuccess) {
        if (csc) e = launch_sketch_sparse_sorted(*v, P, csc->pos, csc->rs, csc->nent, (int32_t*)Y, ldy, st);
        else e = launch_sketch_sparse(*v, P, ell, counts, (int32_t*)Y, ldy, st);
      }
      break;
    }
    case CDMD_RADEMACHER:
      e = launch_sketch_rademacher(*v, P, (int32_t*)Y, ldy, st);
      break;
    case CDMD_GAUSSIAN:
      e = launch_sketch_gaussian(*v, P, h->gauss_table, (float*)Y, ldy,
                                 (float*)((char*)ws + al256(sensing_ws_bytes(P))), st);
      break;
    case CDMD_SRFT: {
      if (!sketch_srft_supported(*v)) return CDMD_ERR_UNSUPPORTED;
      int32_t* freqs = (int32_t*)ws;
      e = launch_srft_freqs(P, freqs, st);
      if (e == cudaSuccess)
        e = launch_sketch_srft(*v, P, freqs, h->srft_table, (float*)Y, ldy,
                               (float*)((char*)ws + al256(sensing_ws_bytes(P))), st);
      break;
    }
  }
  return cuda_status(e);
}

// ---------------------------------------------------------------------- fit
size_t cdmd_model_bytes(int k, int K, int64_t m) {
  if (k < 1 || K < 1 || m < 2) return 0;
  return model_layout(k, K, m).total;
}

cdmd_status cdmd_model_bind(cdmd_model* M, void* buf, size_t bytes, int k, int K, int64_t m) {
  if (!M || !buf) return CDMD_ERR_ARG;
  if (k < 1 || k > 256 || K < 1 || K > 32 || K > k || m < 2) return CDMD_ERR_RANGE;
  if ((reinterpret_cast<uintptr_t>(buf) & 255) != 0) return CDMD_ERR_ARG;
  const ModelLayout L = model_layout(k, K, m);
  if (bytes < L.total) return CDMD_ERR_WORKSPACE;
  char* b = (char*)buf;
  memset(M, 0, sizeof(*M));
  M->k = k;
  M->K = K;
  M->limbs = CDMD_LIMBS;
  M->kpad = (int32_t)kpad_of(k);
  M->m = m;
  M->mpad = mpad_of(m);
  M->lambda = (double*)(b + L.lambda);
  M->omega = (double*)(b + L.omega);
  M->pair = (int32_t*)(b + L.pair);
  M->sigma = (double*)(b + L.sigma);
  M->Mfold = (double*)(b + L.Mfold);
  M->beta = (double*)(b + L.beta);
  M->support = (int32_t*)(b + L.support);
  M->Mq = (int8_t*)(b + L.Mq);
  M->Mq_scale = (double*)(b + L.Mq_scale);
  M->coef = (float*)(b + L.coef);
  M->coef_col = (int32_t*)(b + L.coef_col);
  M->dev_info = (int32_t*)(b + L.dev_info);
  M->dt = 1.0;
  return CDMD_OK;
}

size_t cdmd_fit_workspace_bytes(cdmd_handle h, int64_t p, int64_t m, int k) {
  if (!h || p < 1 || m < 2 || k < 1) return 0;
  return fit_ws_bytes(h, p, m, k);
}

cdmd_status cdmd_fit(cdmd_handle h, const void* Y, int64_t ldy, int32_t kind, int64_t p, int64_t m,
                     int k, int K, double dt, cdmd_model* model, void* ws, size_t ws_bytes,
                     cdmd_stream st) {
  if (!h || !Y || !model || !ws) return CDMD_ERR_ARG;
  if (kind < CDMD_SPIXEL || kind > CDMD_SRFT) return CDMD_ERR_ARG;
  if (m < 2 || p < 1) return CDMD_ERR_RANGE;
  const int kmax = k < 0 ? -k : k;   // k < 0: Gavish-Donoho rank, at most -k (Remark 2)
  if (kmax < 1 || kmax > p || kmax > m - 1 || kmax > model->k) return CDMD_ERR_RANGE;  // P:355 "p >= k"
  if (K < 1 || K > kmax || K > model->K) return CDMD_ERR_RANGE;
  if (ldy < p || !(dt > 0.0)) return CDMD_ERR_ARG;
  if (model->m != m) return CDMD_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return CDMD_ERR_ARG;
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing((cudaStream_t)st, &cst) != cudaSuccess) return CDMD_ERR_CUDA;
  // under capture the model keeps the sizes of its previous (eager) fit: the graph assumes them
  if (cst == cudaStreamCaptureStatusNone) model->k_eff = model->K_eff = model->n_coef = model->info = 0;
  return fit_impl(h, Y, ldy, kind, p, m, k, K, dt, model, ws, ws_bytes, (cudaStream_t)st);
}

// -------------------------------------------------------------------- modes
static cdmd_status modes_common(cdmd_handle h, const cdmd_video* v, const cdmd_model* M, float* Phi,
                                int64_t ldphi) {
  if (!h || !Phi) return CDMD_ERR_ARG;
  cdmd_status s = check_video(v);
  if (s != CDMD_OK) return s;
  if ((s = check_model(M, v->m)) != CDMD_OK) return s;
  if (ldphi < v->n_local) return CDMD_ERR_ARG;
  return CDMD_OK;
}

cdmd_status cdmd_modes(cdmd_handle h, const cdmd_video* v, const cdmd_model* M, float* Phi,
                       int64_t ldphi, cdmd_stream st) {
  cdmd_status s = modes_common(h, v, M, Phi, ldphi);
  if (s != CDMD_OK) return s;
  return cuda_status(launch_modes_tc(*v, *M, Phi, ldphi, sched_slot(h), (cudaStream_t)st));
}

cdmd_status cdmd_modes_simt(cdmd_handle h, const cdmd_video* v, const cdmd_model* M, float* Phi,
                            int64_t ldphi, cdmd_stream st) {
  cdmd_status s = modes_common(h, v, M, Phi, ldphi);
  if (s != CDMD_OK) return s;
  return cuda_status(launch_modes_simt(*v, *M, Phi, ldphi, (cudaStream_t)st));
}

// ---------------------------------------------------------- background / mask
cdmd_status cdmd_background(cdmd_handle h, const float* Phi, int64_t ldphi, int64_t n_local,
                            const cdmd_model* M, int32_t mode, int64_t t0, int64_t nt, float* L,
                            int64_t ldl, cdmd_stream st) {
  if (!h || !Phi || !L || !M) return CDMD_ERR_ARG;
  if (mode != CDMD_BG_STATIC && mode != CDMD_BG_DYNAMIC) return CDMD_ERR_ARG;
  if (n_local < 1 || ldphi < n_local || ldl < n_local) return CDMD_ERR_ARG;
  cdmd_status s = check_model(M, M->m);
  if (s != CDMD_OK) return s;
  if (t0 < 0 || nt < 1 || t0 + nt > M->m || nt > 65535) return CDMD_ERR_RANGE;
  return cuda_status(launch_background(Phi, ldphi, n_local, *M, mode, t0, nt, L, ldl, (cudaStream_t)st));
}

cdmd_status cdmd_foreground(cdmd_handle h, const cdmd_video* v, const cdmd_model* M,
                            const float* Phi, int64_t ldphi, int32_t mode, float tau,
                            uint32_t* mask, int64_t ldw, cdmd_stream st) {
  if (!h || !mask) return CDMD_ERR_ARG;
  if (mode != CDMD_BG_STATIC && mode != CDMD_BG_DYNAMIC) return CDMD_ERR_ARG;
  cdmd_status s = check_video(v);
  if (s != CDMD_OK) return s;
  if ((s = check_model(M, v->m)) != CDMD_OK) return s;
  if (!(tau > 0.0f)) return CDMD_ERR_RANGE;
  if (ldw < ceil_div(v->n_local, 32)) return CDMD_ERR_ARG;
  if (!Phi) {   // N11: the support's modes computed in-slab from X (fused_tc.cu)
    if (!fused_supported(*v, *M, mode)) return CDMD_ERR_UNSUPPORTED;
    return cuda_status(launch_fused_fg(*v, *M, mode, tau, mask, ldw, sched_slot(h), (cudaStream_t)st));
  }
  if (ldphi < v->n_local) return CDMD_ERR_ARG;
  return cuda_status(launch_foreground(*v, *M, Phi, ldphi, mode, tau, mask, ldw, sched_slot(h), (cudaStream_t)st));
}

// --------------------------------------------------------------- amplitudes
size_t cdmd_amplitudes_workspace_bytes(cdmd_handle h, int k) {
  if (!h || k < 1 || k > 128) return 0;
  return al256(amp_gram_ws_bytes(h->sm_count, k));
}

cdmd_status cdmd_amplitudes_gram(cdmd_handle h, const cdmd_video* v, const cdmd_model* M,
                                 const float* Phi, int64_t ldphi, double* G, void* ws,
                                 size_t ws_bytes, cdmd_stream st) {
  if (!h || !Phi || !G || !ws) return CDMD_ERR_ARG;
  cdmd_status s = check_video(v);
  if (s != CDMD_OK) return s;
  if ((s = check_model(M, v->m)) != CDMD_OK) return s;
  if (M->k_eff > 128) return CDMD_ERR_RANGE;
  if (ldphi < v->n_local) return CDMD_ERR_ARG;
  if (ws_bytes < amp_gram_ws_bytes(h->sm_count, M->k_eff)) return CDMD_ERR_WORKSPACE;
  return cuda_status(launch_amp_gram(h->sm_count, Phi, ldphi, v->X, v->n_local, M->k_eff,
                                     static_cast<double*>(ws), G, (cudaStream_t)st));
}

cdmd_status cdmd_amplitudes_solve(cdmd_handle h, const cdmd_model* M, const double* G, double* b,
                                  int32_t* dropped, cdmd_stream st) {
  if (!h || !G || !b || !M || !M->pair) return CDMD_ERR_ARG;
  if (M->k_eff < 1 || M->k_eff > M->k) return CDMD_ERR_ARG;
  if (M->k_eff > 128) return CDMD_ERR_RANGE;
  return cuda_status(launch_amp_solve(G, M->k_eff, M->pair, b, dropped, (cudaStream_t)st));
}

int32_t cdmd_modes_path(const cdmd_model* M) {
  if (!M || M->k < 1) return -1;
  if (!modes_tc_supported(*M)) return 0;
  return (M->kpad > 64 && !getenv("CDMD_MODES_NO_MC")) ? 2 : 1;
}

int32_t cdmd_foreground_path(const cdmd_video* v, const cdmd_model* M, int32_t mode) {
  if (!v || !M) return -1;
  if (mode == CDMD_BG_STATIC) return 0;
  if (mode != CDMD_BG_DYNAMIC) return -1;
  return foreground_tc_supported(*v, *M) ? 2 : 1;
}

size_t cdmd_foreground_median3_ws_bytes(int64_t width, int64_t height) {
  if (width < 1 || height < 1) return 0;
  return al256(sizeof(int) * ((size_t)height + 1));   // a completion counter per image row + the row queue
}

cdmd_status cdmd_foreground_median3(cdmd_handle h, const cdmd_video* v, const cdmd_model* M, int32_t mode, float tau,
                                    int64_t width, int64_t height, uint32_t* raw, uint32_t* out, int64_t ldw, void* ws,
                                    size_t ws_bytes, cdmd_stream st) {
  if (!h || !raw || !out || !ws) return CDMD_ERR_ARG;
  if (mode != CDMD_BG_STATIC && mode != CDMD_BG_DYNAMIC) return CDMD_ERR_ARG;
  cdmd_status s = check_video(v);
  if (s != CDMD_OK) return s;
  if ((s = check_model(M, v->m)) != CDMD_OK) return s;
  if (!(tau > 0.0f)) return CDMD_ERR_RANGE;
  if (width < 1 || height < 1 || width * height != v->n_total || v->pix0 != 0 || v->n_local != v->n_total)
    return CDMD_ERR_ARG;
  if (ldw < ceil_div(v->n_local, 32)) return CDMD_ERR_ARG;
  const char *a0 = (const char*)raw, *a1 = a0 + sizeof(uint32_t) * ldw * v->m;
  const char *b0 = (const char*)out, *b1 = b0 + sizeof(uint32_t) * ldw * v->m;
  if (a0 < b1 && b0 < a1) return CDMD_ERR_ARG;   // aliasing
  if (ws_bytes < cdmd_foreground_median3_ws_bytes(width, height)) return CDMD_ERR_WORKSPACE;
  if ((width % 32) != 0 || width > (int64_t)1 << 24 || !fused_supported(*v, *M, mode)) return CDMD_ERR_UNSUPPORTED;
  return cuda_status(launch_fused_fg_median(*v, *M, mode, tau, raw, ldw, sched_slot(h), (int)width, (int)height, out,
                                            (int*)ws, (cudaStream_t)st));
}

cdmd_status cdmd_mask_median3(const uint32_t* mask, int64_t ldw, int64_t width, int64_t height, int64_t m,
                              uint32_t* out, cdmd_stream st) {
  if (!mask || !out) return CDMD_ERR_ARG;
  if (width < 1 || height < 1 || m < 1 || m > 65535) return CDMD_ERR_RANGE;
  const int64_t nw = ceil_div(width * height, 32);
  if (ldw < nw) return CDMD_ERR_ARG;
  const char *a0 = (const char*)mask, *a1 = a0 + sizeof(uint32_t) * ldw * m;
  const char *b0 = (const char*)out, *b1 = b0 + sizeof(uint32_t) * ldw * m;
  if (a0 < b1 && b0 < a1) return CDMD_ERR_ARG;   // aliasing
  return cuda_status(launch_mask_median3(mask, ldw, width, height, m, out, (cudaStream_t)st));
}

// --------------------------------------------------------------- test hooks
cdmd_status cdmd_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, int64_t count,
                        cdmd_stream st) {
  if (count < 0 || (count > 0 && (!ctr || !out))) return CDMD_ERR_ARG;
  return cuda_status(launch_philox_test(ctr, k0, k1, out, count, (cudaStream_t)st));
}

cdmd_status cdmd_gaussian_table(cdmd_handle h, uint16_t* out, cdmd_stream st) {
  if (!h || !out) return CDMD_ERR_ARG;
  return cuda_status(cudaMemcpyAsync(out, h->gauss_table, 65536 * sizeof(uint16_t),
                                     cudaMemcpyDeviceToDevice, (cudaStream_t)st));
}

cdmd_status cdmd_srft_table(cdmd_handle h, uint16_t* out, cdmd_stream st) {
  if (!h || !out) return CDMD_ERR_ARG;
  return cuda_status(cudaMemcpyAsync(out, h->srft_table, 16385 * sizeof(uint16_t), cudaMemcpyDeviceToDevice,
                                     (cudaStream_t)st));
}

int64_t cdmd_sparse_cap(int64_t n_total, int64_t p, double s) {
  cdmd_sensing c{CDMD_SPARSE, p, s, 0};
  return make_plan(n_total, &c).cap;
}

cdmd_status cdmd_sensing_rows(cdmd_handle h, int64_t n_total, const cdmd_sensing* c,
                              int32_t* rows_or_ell, int32_t* counts, cdmd_stream st_) {
  cudaStream_t st = (cudaStream_t)st_;
  if (!h || !rows_or_ell) return CDMD_ERR_ARG;
  cdmd_status s = check_sensing(n_total, c);
  if (s != CDMD_OK) return s;
  const SensingPlan P = make_plan(n_total, c);
  if (P.kind == CDMD_SPIXEL) return cuda_status(launch_spixel_rows(P, rows_or_ell, st));
  if (P.kind == CDMD_SRFT) return cuda_status(launch_srft_freqs(P, rows_or_ell, st));
  if (P.kind == CDMD_SPARSE) {
    if (!counts) return CDMD_ERR_ARG;
    int32_t* flags = nullptr;
    if (cudaMallocAsync((void**)&flags, 16, st) != cudaSuccess) return CDMD_ERR_CUDA;
    cudaMemsetAsync(flags, 0, 16, st);
    cudaError_t e = launch_sparse_rows(P, rows_or_ell, counts, flags, st);
    int32_t f = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&f, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(flags, st);
    if (e == cudaSuccess && (f & FLAG_SPARSE_OVERFLOW)) return CDMD_ERR_NUMERIC;
    return cuda_status(e);
  }
  return CDMD_ERR_ARG;
}

cdmd_status cdmd_eig(const double* A, int k, double* W, double* VR, int32_t* info, cdmd_stream st) {
  if (!A || !W || !VR || !info) return CDMD_ERR_ARG;
  if (k < 1 || hqr_smem_bytes(k) > 227 * 1024) return CDMD_ERR_RANGE;
  double* scratch = nullptr;
  if (cudaMallocAsync((void**)&scratch, sizeof(double) * 2 * (size_t)k * k, (cudaStream_t)st) != cudaSuccess)
    return CDMD_ERR_CUDA;
  const cudaError_t e = launch_hqr_eig(k, A, W, VR, info, scratch, (cudaStream_t)st);
  cudaFreeAsync(scratch, (cudaStream_t)st);
  return cuda_status(e);
}

}  // extern "C"
