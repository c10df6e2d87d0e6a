// Context, memory, spec upload and small C-ABI glue for libltb.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "ltb_common.cuh"

int ltb_set_error(ltb_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->last_error = buf;
  return code;
}

int ltb_ws_alloc(ltb_ctx* ctx, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync(out, bytes, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return ltb_set_error(ctx, LTB_EOOM, "device allocation of %zu bytes failed: %s", bytes,
                         cudaGetErrorString(e));
  }
  return LTB_OK;
}

void ltb_ws_free(ltb_ctx* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
}

namespace {
std::mutex g_attr_mu;
std::unordered_map<const void*, size_t> g_smem_set;
std::map<std::tuple<const void*, int, size_t>, int> g_occ;
}  // namespace

int ltb_ensure_smem(ltb_ctx* ctx, const void* kern, size_t smem, bool carveout) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  auto it = g_smem_set.find(kern);
  if (it != g_smem_set.end() && it->second >= smem) return LTB_OK;
  if (smem > 48 * 1024) LTB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (carveout)
    LTB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           (int)cudaSharedmemCarveoutMaxShared));
  g_smem_set[kern] = smem;
  return LTB_OK;
}

int ltb_occupancy(const void* kern, int threads, size_t smem) {
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_tuple(kern, threads, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  g_occ[key] = per_sm;
  return per_sm;
}

extern "C" {

int ltb_version(void) { return 1; }

int ltb_device_count(int* count) {
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return LTB_ECUDA;
  }
  return LTB_OK;
}

int ltb_ctx_create(int device, ltb_ctx** out) {
  *out = nullptr;
  ltb_ctx* ctx = new ltb_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return LTB_ECUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return LTB_ECUDA;
  }
  ctx->stream = ctx->own_stream;
  // keep freed pool memory cached instead of returning it at every sync
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMallocHost(&ctx->h_scratch, 64 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ctx->d_scratch, 64 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ctx->d_counter, 64 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc(&ctx->d_stats, 8 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    delete ctx;
    return LTB_EOOM;
  }
  cudaMemset(ctx->d_counter, 0, 64 * sizeof(unsigned int));
  cudaMemset(ctx->d_stats, 0, 8 * sizeof(unsigned long long));
  cudaDeviceSynchronize();
  *out = ctx;
  return LTB_OK;
}

void ltb_ctx_destroy(ltb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  if (ctx->d_scratch) cudaFree(ctx->d_scratch);
  if (ctx->d_counter) cudaFree(ctx->d_counter);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  if (ctx->split_hi) cudaStreamDestroy(ctx->split_hi);
  if (ctx->split_hi2) cudaStreamDestroy(ctx->split_hi2);
  if (ctx->split_lo) cudaStreamDestroy(ctx->split_lo);
  if (ctx->h_big) cudaFreeHost(ctx->h_big);
  for (int b = 0; b < 2; ++b) {
    if (ctx->h_stage[b]) cudaFreeHost(ctx->h_stage[b]);
    if (ctx->ev_stage[b]) cudaEventDestroy(ctx->ev_stage[b]);
  }
  delete ctx;
}

const char* ltb_ctx_last_error(const ltb_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int ltb_ctx_set_stream(ltb_ctx* ctx, void* stream) {
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return LTB_OK;
}

int ltb_ctx_set_option(ltb_ctx* ctx, int option, int64_t value) {
  switch (option) {
    case LTB_OPT_FORCE_BLOCKED_SVD: ctx->opt_force_blocked = value != 0; return LTB_OK;
    case LTB_OPT_TC_TIMELINE: ctx->opt_tc_timeline = (unsigned long long*)(uintptr_t)value; return LTB_OK;
    case LTB_OPT_QR_TIMELINE: ctx->opt_qr_timeline = (unsigned long long*)(uintptr_t)value; return LTB_OK;
    case LTB_OPT_JACOBI_PAIRS: ctx->opt_jacobi_pairs = (int)value; return LTB_OK;
    case LTB_OPT_FULL_SWEEPS: ctx->opt_full_sweeps = value != 0; return LTB_OK;
  }
  return ltb_set_error(ctx, LTB_EPARAM, "unknown context option %d", option);
}

int ltb_ctx_make_current(ltb_ctx* ctx) {
  LTB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
  return LTB_OK;
}

int ltb_ctx_synchronize(ltb_ctx* ctx) {
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  LTB_CUDA_TRY(ctx, cudaGetLastError());
  return LTB_OK;
}

int64_t ltb_ctx_launch_count(const ltb_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ltb_ctx_stats(ltb_ctx* ctx, int64_t* h_out, int reset) {
  unsigned long long v[3] = {0, 0, 0};
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(v, ctx->d_stats, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  h_out[0] = (int64_t)v[0];
  h_out[1] = (int64_t)v[1];
  h_out[2] = (int64_t)v[2];
  if (reset) LTB_CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_stats, 0, sizeof(v), ctx->stream));
  return LTB_OK;
}

int ltb_malloc(ltb_ctx* ctx, int64_t bytes, void** d_out) {
  if (bytes < 0) return ltb_set_error(ctx, LTB_EPARAM, "negative allocation size");
  cudaSetDevice(ctx->device);
  return ltb_ws_alloc(ctx, (size_t)bytes, d_out);
}

int ltb_free(ltb_ctx* ctx, void* d_ptr) {
  // the buffer may belong to a context other than the calling thread's current device
  int cur = ctx->device;
  cudaGetDevice(&cur);
  if (cur != ctx->device) cudaSetDevice(ctx->device);
  ltb_ws_free(ctx, d_ptr);
  if (cur != ctx->device) cudaSetDevice(cur);
  return LTB_OK;
}

// ---------------------------------------------------------------- host <-> device copies
// A pageable numpy buffer is what the drop-in API receives and returns.  cudaMemcpy from or
// to pageable memory runs at ~4.5 GB/s here (the driver's own staging); instead the copy is
// pipelined through two pinned buffers: the DMA of chunk c overlaps the host copy of chunk
// c - 1, and each host copy is split over a few threads (page faults of a fresh output and
// a single memcpy thread each cap a copy at a few GB/s).  Pinned / registered host memory
// goes straight to the DMA engine.
namespace {
constexpr size_t kStageBytes = 16u << 20;
constexpr int kCopyThreads = 8;

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// persistent workers for the host side of staged copies
class CopyPool {
 public:
  CopyPool() {
    for (int t = 1; t < kCopyThreads; ++t) workers_.emplace_back([this, t] { run(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void copy(char* dst, const char* src, size_t n) {
    if (n < (1u << 20)) {
      std::memcpy(dst, src, n);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);  // one staged copy at a time (several contexts)
    std::unique_lock<std::mutex> l(mu_);
    dst_ = dst;
    src_ = src;
    n_ = n;
    pending_ = kCopyThreads - 1;
    ++gen_;
    l.unlock();
    cv_.notify_all();
    part(0);
    l.lock();
    done_cv_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void part(int t) {
    const size_t per = ((n_ + kCopyThreads - 1) / kCopyThreads + 63) & ~size_t(63);  // covers n_
    const size_t b = std::min(n_, per * t), e = std::min(n_, b + per);
    if (e > b) std::memcpy(dst_ + b, src_ + b, e - b);
  }
  void run(int t) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> l(mu_);
    for (;;) {
      cv_.wait(l, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      l.unlock();
      part(t);
      l.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

std::mutex g_pool_mu;
CopyPool& copy_pool() {
  std::lock_guard<std::mutex> l(g_pool_mu);
  static CopyPool* pool = new CopyPool();  // never destroyed: workers may outlive static teardown order
  return *pool;
}

}  // namespace

bool ltb_is_pinned(const void* p) { return is_pinned(p); }
void ltb_host_copy(void* dst, const void* src, size_t n) { copy_pool().copy((char*)dst, (const char*)src, n); }

int ltb_pinned_scratch(ltb_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->h_big_bytes) {
    if (ctx->h_big) {
      LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFreeHost(ctx->h_big);
      ctx->h_big = nullptr;
      ctx->h_big_bytes = 0;
    }
    LTB_CUDA_TRY(ctx, cudaHostAlloc(&ctx->h_big, bytes, cudaHostAllocDefault));
    ctx->h_big_bytes = bytes;
  }
  *out = ctx->h_big;
  return LTB_OK;
}

namespace {
int ensure_stage(ltb_ctx* ctx) {
  for (int b = 0; b < 2; ++b) {
    if (!ctx->h_stage[b]) LTB_CUDA_TRY(ctx, cudaHostAlloc(&ctx->h_stage[b], kStageBytes, cudaHostAllocDefault));
    if (!ctx->ev_stage[b]) LTB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_stage[b], cudaEventDisableTiming));
  }
  return LTB_OK;
}
}  // namespace

int ltb_memcpy_h2d(ltb_ctx* ctx, void* d_dst, const void* h_src, int64_t bytes) {
  if (bytes <= 0) return LTB_OK;
  if ((size_t)bytes <= (1u << 20) || is_pinned(h_src)) {
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(d_dst, h_src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return LTB_OK;
  }
  LTB_TRY(ensure_stage(ctx));
  const char* src = (const char*)h_src;
  char* dst = (char*)d_dst;
  int c = 0;
  for (int64_t off = 0; off < bytes; off += kStageBytes, ++c) {
    const int b = c & 1;
    const size_t len = std::min<int64_t>(kStageBytes, bytes - off);
    // the DMA that last read this buffer (chunk c - 2) must be done before it is refilled
    LTB_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_stage[b]));
    copy_pool().copy((char*)ctx->h_stage[b], src + off, len);
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(dst + off, ctx->h_stage[b], len, cudaMemcpyHostToDevice, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_stage[b], ctx->stream));
  }
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return LTB_OK;
}

int ltb_memcpy_d2h(ltb_ctx* ctx, void* h_dst, const void* d_src, int64_t bytes) {
  if (bytes <= 0) return LTB_OK;
  if ((size_t)bytes <= (1u << 20) || is_pinned(h_dst)) {
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(h_dst, d_src, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return LTB_OK;
  }
  LTB_TRY(ensure_stage(ctx));
  char* dst = (char*)h_dst;
  const char* src = (const char*)d_src;
  const int64_t nch = (bytes + (int64_t)kStageBytes - 1) / (int64_t)kStageBytes;
  auto chunk = [&](int64_t c, size_t* len) {
    const int64_t off = c * (int64_t)kStageBytes;
    *len = (size_t)std::min<int64_t>(kStageBytes, bytes - off);
    return off;
  };
  size_t len = 0;
  int64_t off = chunk(0, &len);
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stage[0], src + off, len, cudaMemcpyDeviceToHost, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_stage[0], ctx->stream));
  for (int64_t c = 0; c < nch; ++c) {
    const int b = (int)(c & 1);
    if (c + 1 < nch) {  // next chunk's DMA into the other buffer (its previous contents are copied out)
      size_t l2 = 0;
      const int64_t o2 = chunk(c + 1, &l2);
      LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stage[b ^ 1], src + o2, l2, cudaMemcpyDeviceToHost, ctx->stream));
      LTB_CUDA_TRY(ctx, cudaEventRecord(ctx->ev_stage[b ^ 1], ctx->stream));
    }
    LTB_CUDA_TRY(ctx, cudaEventSynchronize(ctx->ev_stage[b]));
    off = chunk(c, &len);
    copy_pool().copy(dst + off, (const char*)ctx->h_stage[b], len);
  }
  return LTB_OK;
}

int ltb_memcpy_d2d(ltb_ctx* ctx, void* d_dst, const void* d_src, int64_t bytes) {
  if (bytes <= 0) return LTB_OK;
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(d_dst, d_src, (size_t)bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  return LTB_OK;
}

int ltb_memset_zero(ltb_ctx* ctx, void* d_dst, int64_t bytes) {
  if (bytes <= 0) return LTB_OK;
  LTB_CUDA_TRY(ctx, cudaMemsetAsync(d_dst, 0, (size_t)bytes, ctx->stream));
  return LTB_OK;
}

int ltb_spec_create(ltb_ctx* ctx, int ntrail, const int64_t* trail_dims, int nmodes, const int* axes,
                    int is_complex, const double* h_fwd, const double* h_inv, ltb_spec** out) {
  *out = nullptr;
  if (ntrail < 0 || ntrail > 16 || nmodes < 0 || nmodes > ntrail)
    return ltb_set_error(ctx, LTB_ETRANSFORM, "spec: bad mode count (%d trailing, %d modes)", ntrail, nmodes);
  ltb_spec* s = new ltb_spec();
  s->ctx = ctx;
  s->ntrail = ntrail;
  s->P = 1;
  for (int i = 0; i < ntrail; ++i) {
    if (trail_dims[i] < 1) {
      delete s;
      return ltb_set_error(ctx, LTB_ESHAPE, "spec: trailing dim %d is %lld", i, (long long)trail_dims[i]);
    }
    s->trail_dims[i] = trail_dims[i];
    s->P *= trail_dims[i];
  }
  s->nmodes = nmodes;
  s->is_complex = is_complex ? 1 : 0;
  int64_t total = 0;
  for (int k = 0; k < nmodes; ++k) {
    if (axes[k] < 0 || axes[k] >= ntrail || (k > 0 && axes[k] <= axes[k - 1])) {
      delete s;
      return ltb_set_error(ctx, LTB_ETRANSFORM, "spec: axes must be ascending and within the trailing dims");
    }
    s->axes[k] = axes[k];
    s->sizes[k] = (int)trail_dims[axes[k]];
    s->mat_off[k] = total;
    total += (int64_t)s->sizes[k] * s->sizes[k];
  }
  s->mat_total = total;
  const int comp = is_complex ? 2 : 1;
  const size_t n_el = (size_t)(total > 0 ? total : 1) * comp;
  std::vector<float> tmpf(n_el);
  for (int dir = 0; dir < 2; ++dir) {
    const double* src = dir == 0 ? h_fwd : h_inv;
    for (size_t i = 0; i < n_el; ++i) tmpf[i] = total > 0 ? (float)src[i] : 0.f;
    void *d32 = nullptr, *d64 = nullptr;
    if (cudaMalloc(&d32, n_el * sizeof(float)) != cudaSuccess || cudaMalloc(&d64, n_el * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      delete s;
      return ltb_set_error(ctx, LTB_EOOM, "spec: matrix upload allocation failed");
    }
    cudaMemcpy(d32, tmpf.data(), n_el * sizeof(float), cudaMemcpyHostToDevice);
    if (total > 0) cudaMemcpy(d64, src, n_el * sizeof(double), cudaMemcpyHostToDevice);
    s->d_mats[0][dir] = d32;
    s->d_mats[1][dir] = d64;
  }
  // even/odd symmetric real mode matrices (the DCT and its inverse); a match within 1e-12
  // of the largest entry (the fp32 engine then uses half of the matrix)
  if (!is_complex && total > 0) {
    for (int dir = 0; dir < 2; ++dir)
      for (int k = 0; k < nmodes; ++k) {
        const int n = s->sizes[k];
        if (n % 2 || n < 8) continue;
        const double* M = (dir == 0 ? h_fwd : h_inv) + s->mat_off[k];
        double mx = 0.0;
        for (int64_t l = 0; l < (int64_t)n * n; ++l) mx = std::max(mx, std::fabs(M[l]));
        const double tol = 1e-12 * mx;
        bool c1 = mx > 0.0, c2 = mx > 0.0;
        for (int i = 0; i < n && (c1 || c2); ++i)
          for (int j = 0; j < n; ++j) {
            const double a = M[(int64_t)i * n + j];
            if (c1 && std::fabs(M[(int64_t)i * n + (n - 1 - j)] - ((i & 1) ? -a : a)) > tol) c1 = false;
            if (c2 && std::fabs(M[(int64_t)(n - 1 - i) * n + j] - ((j & 1) ? -a : a)) > tol) c2 = false;
          }
        s->sym[dir][k] = c1 ? 1 : (c2 ? 2 : 0);
      }
  }
  // conjugate-slice pairing for real input data (complex specs): every transformed
  // mode is real (partner index j) or has exactly Hermitian rows (partner (n - j) mod n)
  if (is_complex && nmodes > 0) {
    std::vector<int> herm(ntrail, 0);
    bool ok = true, any = false;
    for (int k = 0; k < nmodes && ok; ++k) {
      const int n = s->sizes[k];
      const double* M = h_fwd + 2 * s->mat_off[k];
      bool real = true, hrow = true;
      for (int i = 0; i < n && (real || hrow); ++i)
        for (int j = 0; j < n; ++j) {
          const double re = M[2 * ((int64_t)i * n + j)], im = M[2 * ((int64_t)i * n + j) + 1];
          if (im != 0.0) real = false;
          const int ip = (n - i) % n;
          const double re2 = M[2 * ((int64_t)ip * n + j)], im2 = M[2 * ((int64_t)ip * n + j) + 1];
          if (re2 != re || im2 != -im) hrow = false;
        }
      if (real) continue;
      if (hrow) {
        herm[axes[k]] = 1;
        any = true;
      } else {
        ok = false;
      }
    }
    if (ok && any && s->P < (int64_t(1) << 31)) {
      const int64_t P = s->P;
      std::vector<int> partner((size_t)P), uniq;
      std::vector<int64_t> idx(ntrail);
      for (int64_t q = 0; q < P; ++q) {
        int64_t r = q;
        for (int a = ntrail - 1; a >= 0; --a) {
          idx[a] = r % trail_dims[a];
          r /= trail_dims[a];
        }
        int64_t qp = 0;
        for (int a = 0; a < ntrail; ++a) {
          const int64_t j = herm[a] ? (trail_dims[a] - idx[a]) % trail_dims[a] : idx[a];
          qp = qp * trail_dims[a] + j;
        }
        partner[(size_t)q] = (int)qp;
        if (q <= qp) uniq.push_back((int)q);
      }
      if ((int64_t)uniq.size() < P && cudaMalloc(&s->d_partner, sizeof(int) * P) == cudaSuccess &&
          cudaMalloc(&s->d_uniq, sizeof(int) * uniq.size()) == cudaSuccess) {
        cudaMemcpy(s->d_partner, partner.data(), sizeof(int) * P, cudaMemcpyHostToDevice);
        cudaMemcpy(s->d_uniq, uniq.data(), sizeof(int) * uniq.size(), cudaMemcpyHostToDevice);
        s->n_unique = (int64_t)uniq.size();
      } else {
        cudaGetLastError();
        if (s->d_partner) cudaFree(s->d_partner);
        s->d_partner = nullptr;
        s->d_uniq = nullptr;
        s->n_unique = 0;
      }
    }
  }
  // dense Kronecker matrices K[q][q'] = prod_a F_a[k_a][k'_a] (F_a = M_a on
  // transformed axes, I elsewhere; C-order q) for the tensor-core path
  if (!is_complex && s->P <= kKronMax) {
    const int64_t P = s->P;
    std::vector<int> axis_mode(ntrail, -1);
    for (int k = 0; k < nmodes; ++k) axis_mode[axes[k]] = k;
    // [K | K_lo]: K_lo = round-to-tf32(K - trunc-to-tf32(K)) from the double
    // values, the precomputed lo operand of the 3xTF32 split (ltb_tc_gemm.cu)
    std::vector<float> kron((size_t)2 * P * P);
    auto tf32_trunc = [](float x) {
      uint32_t u;
      std::memcpy(&u, &x, 4);
      u &= 0xFFFFE000u;
      std::memcpy(&x, &u, 4);
      return x;
    };
    auto tf32_round = [](float x) {
      uint32_t u;
      std::memcpy(&u, &x, 4);
      u = (u + 0x1000u) & 0xFFFFE000u;
      std::memcpy(&x, &u, 4);
      return x;
    };
    std::vector<int> qi(ntrail), qj(ntrail);
    for (int dir = 0; dir < 2; ++dir) {
      const double* src = dir == 0 ? h_fwd : h_inv;
      for (int64_t i = 0; i < P; ++i) {
        int64_t r = i;
        for (int a = ntrail - 1; a >= 0; --a) {
          qi[a] = (int)(r % trail_dims[a]);
          r /= trail_dims[a];
        }
        for (int64_t j = 0; j < P; ++j) {
          int64_t c = j;
          double v = 1.0;
          for (int a = ntrail - 1; a >= 0 && v != 0.0; --a) {
            qj[a] = (int)(c % trail_dims[a]);
            c /= trail_dims[a];
            const int k = axis_mode[a];
            if (k < 0) {
              v = (qi[a] == qj[a]) ? v : 0.0;
            } else {
              const int n = s->sizes[k];
              v *= src[s->mat_off[k] + (int64_t)qi[a] * n + qj[a]];
            }
          }
          const float f = (float)v;
          kron[(size_t)i * P + j] = f;
          kron[(size_t)(P + i) * P + j] = tf32_round((float)(v - (double)tf32_trunc(f)));
        }
      }
      if (cudaMalloc(&s->d_kron[dir], sizeof(float) * 2 * P * P) != cudaSuccess) {
        cudaGetLastError();
        s->d_kron[dir] = nullptr;
        break;
      }
      cudaMemcpy(s->d_kron[dir], kron.data(), sizeof(float) * 2 * P * P, cudaMemcpyHostToDevice);
    }
    if (!s->d_kron[0] || !s->d_kron[1]) {
      for (int d = 0; d < 2; ++d)
        if (s->d_kron[d]) cudaFree(s->d_kron[d]);
      s->d_kron[0] = s->d_kron[1] = nullptr;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete s;
    return ltb_set_error(ctx, LTB_ECUDA, "spec upload: %s", cudaGetErrorString(e));
  }
  *out = s;
  return LTB_OK;
}

void ltb_spec_destroy(ltb_spec* s) {
  if (!s) return;
  for (int p = 0; p < 2; ++p)
    for (int d = 0; d < 2; ++d)
      if (s->d_mats[p][d]) cudaFree(s->d_mats[p][d]);
  for (int d = 0; d < 2; ++d)
    if (s->d_kron[d]) cudaFree(s->d_kron[d]);
  if (s->d_uniq) cudaFree(s->d_uniq);
  if (s->d_partner) cudaFree(s->d_partner);
  delete s;
}

int ltb_transform(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in, int layout_in,
                  const void* d_in, int dtype_out, int layout_out, void* d_out, double* h_sumsq) {
  double* d_sum = h_sumsq ? ctx->d_scratch : nullptr;
  LTB_TRY(ltb_transform_impl(ctx, spec, ntubes, inverse, dtype_in, layout_in, d_in, dtype_out, layout_out, d_out,
                             d_sum));
  if (h_sumsq) {
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scratch, d_sum, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    h_sumsq[0] = ctx->h_scratch[0];
    h_sumsq[1] = ctx->h_scratch[1];
  }
  return LTB_OK;
}

int ltb_transform_pair(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in, int layout_in,
                       const void* d_in0, const void* d_in1, int dtype_out, int layout_out, void* d_out0,
                       void* d_out1) {
  return ltb_transform_pair_impl(ctx, spec, ntubes, inverse, dtype_in, layout_in, d_in0, d_in1, dtype_out,
                                 layout_out, d_out0, d_out1);
}

int ltb_slice_gemm(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int64_t k, int op_a,
                   const void* d_a, int64_t lda, int64_t stride_a, int op_b, const void* d_b, int64_t ldb,
                   int64_t stride_b, void* d_c, int64_t ldc, int64_t stride_c) {
  return ltb_gemm_impl(ctx, dtype, batch, m, n, k, op_a, d_a, lda, stride_a, op_b, d_b, ldb, stride_b, d_c, ldc,
                       stride_c, nullptr, nullptr, nullptr, nullptr, nullptr);
}

int ltb_slice_svt(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, const void* d_a, double tau,
                  void* d_out) {
  if (!(tau >= 0)) return ltb_set_error(ctx, LTB_EPARAM, "tau must be >= 0, got %g", tau);
  return ltb_svt_impl(ctx, dtype, batch, m, n, d_a, tau, nullptr, d_out, nullptr);
}

int ltb_slice_svt_carry(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* d_a, double tau,
                        float* d_out, float* d_v, int warm) {
  if (!(tau >= 0)) return ltb_set_error(ctx, LTB_EPARAM, "tau must be >= 0, got %g", tau);
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svt_carry: negative extent");
  if (batch == 0 || I1 == 0 || I2 == 0) return LTB_OK;
  const int st = ltb_svt_carry_impl(ctx, batch, I1, I2, d_a, tau, d_out, d_v, warm, nullptr);
  if (st == LTB_EUNSUPPORTED)
    return ltb_set_error(ctx, LTB_EUNSUPPORTED, "svt_carry: min(I1, I2) = %lld < 32",
                         (long long)std::min(I1, I2));
  return st;
}

int ltb_slice_svt_carry_c64(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const void* d_a, double tau,
                            void* d_out, void* d_vt, int warm) {
  if (!(tau >= 0)) return ltb_set_error(ctx, LTB_EPARAM, "tau must be >= 0, got %g", tau);
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svt_carry_c64: negative extent");
  if (batch == 0 || I1 == 0 || I2 == 0) return LTB_OK;
  const int st = ltb_svt_carry_c64_impl(ctx, batch, I1, I2, d_a, tau, d_out, d_vt, warm, nullptr);
  if (st == LTB_EUNSUPPORTED)
    return ltb_set_error(ctx, LTB_EUNSUPPORTED,
                         "svt_carry_c64: needs I1 >= I2 >= 32, I2 even, and slices beyond the shared-memory tier");
  return st;
}

int ltb_reduce_sumsq_device(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y, double* d_out) {
  return ltb_reduce_sumsq_dev(ctx, dtype, n, d_x, d_y, d_out);
}

int ltb_reduce_sumsq(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y, double* h_out) {
  LTB_TRY(ltb_reduce_sumsq_dev(ctx, dtype, n, d_x, d_y, ctx->d_scratch));
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scratch, ctx->d_scratch, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  h_out[0] = ctx->h_scratch[0];
  h_out[1] = ctx->h_scratch[1];
  return LTB_OK;
}

}  // extern "C"
