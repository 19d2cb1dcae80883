// Host -> device uploads of caller-owned (pageable) host arrays.
//
// The drop-in callers pass plain numpy arrays (reference core.py:287-311
// `chebyshev_filter(H, Y, spec)`, core.py:385 `chfsi_solve(H, ...)`): pageable memory,
// which the CUDA driver copies through its own small staging buffers at a fraction of
// PCIe bandwidth. Page-locking the caller's buffer (cudaHostRegister) costs ~0.6 s per
// GB on the B200 host -- longer than the filter call it would feed. Instead the handle
// owns a ring of pinned staging slots: host threads copy column chunks of the source
// into a free slot (the copy is split over a persistent worker pool, so host memory
// bandwidth, not one core's memcpy, sets the rate) while the DMA engine drains the
// previous slot to HBM; a slot is reused once its copy-out event has completed.
// Pinned (page-locked) sources take one direct cudaMemcpy2DAsync.
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "internal.h"

namespace chfsi {

// Persistent worker pool: run(fn) calls fn(t, T) on T threads (the caller is t = 0)
// and returns when all are done.
class Pool {
 public:
  explicit Pool(int n) : n_(std::max(1, n)) {
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int, int)>& fn) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      job_ = &fn;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, n_);
    std::unique_lock<std::mutex> lock(mu_);
    done_.wait(lock, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int t) {
    int seen = 0;
    for (;;) {
      const std::function<void(int, int)>* job;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(t, n_);
      {
        std::lock_guard<std::mutex> lock(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  int pending_ = 0, gen_ = 0;
  bool stop_ = false;
};

struct Stager {
  static constexpr int kSlots = 4;
  size_t slot_bytes = 0;
  void* slot[kSlots] = {nullptr};
  cudaEvent_t free_ev[kSlots] = {nullptr};
  int next = 0;
  Pool* pool = nullptr;
};

namespace {

size_t env_slot_bytes() {
  const char* e = getenv("CHFSI_STAGE_MB");
  const long long mb = e ? atoll(e) : 64;
  return (size_t)std::max(4LL, mb) << 20;
}

int pool_threads() {
  const char* e = getenv("CHFSI_STAGE_THREADS");
  if (e) return std::max(1, atoi(e));
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::min(16u, std::max(1u, hc));
}

int ensure_stager(Handle* h) {
  if (h->stager) return OK;
  auto* s = new Stager();
  s->slot_bytes = env_slot_bytes();
  for (int i = 0; i < Stager::kSlots; ++i) {
    if (cudaHostAlloc(&s->slot[i], s->slot_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->free_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      for (int j = 0; j <= i; ++j) {
        if (s->slot[j]) cudaFreeHost(s->slot[j]);
        if (s->free_ev[j]) cudaEventDestroy(s->free_ev[j]);
      }
      delete s;
      set_error("staging: cudaHostAlloc of the pinned ring failed");
      return ERR_NOMEM;
    }
  }
  s->pool = new Pool(pool_threads());
  h->stager = s;
  return OK;
}

}  // namespace

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
         a.type == cudaMemoryTypeManaged;
}

int upload_2d(Handle* h, const double2* host, long long ldh, long long rows, long long cols,
              double2* dev, long long ldd, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return OK;
  if (ldh < rows || ldd < rows) {
    set_error("upload_2d: leading dimensions must be >= rows");
    return ERR_ARG;
  }
  const size_t col_bytes = (size_t)rows * sizeof(double2);
  // CHFSI_STAGE=0: the driver's own pageable path (A/B measurement only)
  static const bool staging_on = [] {
    const char* e = getenv("CHFSI_STAGE");
    return !(e && atoi(e) == 0);
  }();
  if (host_is_pinned(host) || !staging_on) {
    CHFSI_CUDA(cudaMemcpy2DAsync(dev, (size_t)ldd * sizeof(double2), host,
                                 (size_t)ldh * sizeof(double2), col_bytes, (size_t)cols,
                                 cudaMemcpyHostToDevice, stream));
    return OK;
  }
  CHFSI_TRY(ensure_stager(h));
  Stager* s = h->stager;
  if (col_bytes > s->slot_bytes) {
    set_error("upload_2d: one column exceeds a staging slot (raise CHFSI_STAGE_MB)");
    return ERR_ARG;
  }
  const long long chunk = (long long)(s->slot_bytes / col_bytes);
  for (long long c0 = 0; c0 < cols; c0 += chunk) {
    const long long nc = std::min(chunk, cols - c0);
    const int k = s->next;
    s->next = (k + 1) % Stager::kSlots;
    CHFSI_CUDA(cudaEventSynchronize(s->free_ev[k]));  // the slot's last copy-out is done
    auto* dst = static_cast<char*>(s->slot[k]);
    const char* src = reinterpret_cast<const char*>(host + c0 * ldh);
    const size_t src_stride = (size_t)ldh * sizeof(double2);
    // split the chunk's bytes evenly over the workers (whole columns when contiguous)
    s->pool->run([&](int t, int T) {
      if (ldh == rows) {
        const size_t total = col_bytes * (size_t)nc;
        const size_t b0 = total * t / T, b1 = total * (t + 1) / T;
        std::memcpy(dst + b0, src + b0, b1 - b0);
      } else {
        const long long j0 = nc * t / T, j1 = nc * (t + 1) / T;
        for (long long j = j0; j < j1; ++j)
          std::memcpy(dst + (size_t)j * col_bytes, src + (size_t)j * src_stride, col_bytes);
      }
    });
    CHFSI_CUDA(cudaMemcpy2DAsync(dev + c0 * ldd, (size_t)ldd * sizeof(double2), dst, col_bytes,
                                 col_bytes, (size_t)nc, cudaMemcpyHostToDevice, stream));
    CHFSI_CUDA(cudaEventRecord(s->free_ev[k], stream));
  }
  return OK;
}

void destroy_stager(Handle* h) {
  Stager* s = h->stager;
  if (!s) return;
  for (int i = 0; i < Stager::kSlots; ++i) {
    if (s->free_ev[i]) {
      cudaEventSynchronize(s->free_ev[i]);
      cudaEventDestroy(s->free_ev[i]);
    }
    if (s->slot[i]) cudaFreeHost(s->slot[i]);
  }
  delete s->pool;
  delete s;
  h->stager = nullptr;
}

}  // namespace chfsi
