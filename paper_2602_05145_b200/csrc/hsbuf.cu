// HiddenStateBuffer: device-resident ring of captured training signals.
//
// Implements the ingestion seam of the reference: SignalGeometry
// (SPEC.md:237-241), extract_signals byte accounting with the 64 MiB flush
// rule and record_sample.
// Records of one sample stay contiguous (modulo the ring wrap); when the ring
// is full the oldest samples are evicted.  Host appends go through pinned
// staging and one H2D copy, then a 16-byte-vectorised pack kernel
// interleaves the tapped layers into [n, layers*H] rows; device appends
// (capture on the same GPU) pack straight from the layer tensors.
#include <algorithm>
#include <atomic>
#include <cstring>

#include "common.h"
#include "handles.h"
#include "kernels.h"
#include "specsim/draft_trainer.hpp"

namespace specsim {

namespace {
constexpr int64_t kDefaultFlush = 64ll << 20;

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    SPECSIM_CUDA(cudaGetDevice(&prev));
    if (prev != dev) SPECSIM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

HiddenStateBuffer::HiddenStateBuffer(const SignalGeometry& g, int64_t capacity_tokens,
                                     int64_t flush_threshold, int device)
    : geom_(g),
      cap_(capacity_tokens),
      flush_threshold_(flush_threshold > 0 ? flush_threshold : kDefaultFlush),
      device_(device) {
  static std::atomic<uint64_t> next_serial{1};
  serial_ = next_serial.fetch_add(1);
  geom_.validate();
  Problems p("invalid hidden-state buffer");
  p.check(capacity_tokens > 0, "capacity_tokens must be > 0");
  p.check(geom_.bytes_per_element == 2, "only bf16 signals (bytes_per_element = 2) are trainable");
  p.check(geom_.hidden_dim % 8 == 0, "hidden_dim must be a multiple of 8 (16-byte rows)");
  p.throw_if_any();
  DeviceGuard dg(device_);
  cudaStream_t s;
  SPECSIM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  stream_ = s;
  const size_t row = static_cast<size_t>(geom_.bytes_per_token());
  // + mirrored rows (kMirrorRows), zero-filled: rows a step reads past the end
  // of a short sample (masked, zero gradient) are then always finite
  SPECSIM_CUDA(cudaMalloc(&ring_feat_, row * (cap_ + kMirrorRows)));
  SPECSIM_CUDA(cudaMemsetAsync(ring_feat_, 0, row * (cap_ + kMirrorRows), s));
  SPECSIM_CUDA(cudaMalloc(&ring_ids_, sizeof(int32_t) * cap_));
  SPECSIM_CUDA(cudaMemsetAsync(ring_ids_, 0, sizeof(int32_t) * cap_, s));
  for (int i = 0; i < kEventRing; ++i) {
    cudaEvent_t ev;
    SPECSIM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    events_.push_back(ev);
  }
}

void HiddenStateBuffer::record_append(void* stream) {
  const int64_t seq = ++append_seq_;
  cudaEvent_t ev = static_cast<cudaEvent_t>(events_[seq % kEventRing]);
  // the slot last held append seq - kEventRing: make sure it has landed so
  // event_for() can report anything that old as complete
  if (seq > kEventRing) SPECSIM_CUDA(cudaEventSynchronize(ev));
  SPECSIM_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
  samples_.at(open_id_).last_seq = seq;
}

// Rows [0, kMirrorRows) written by an append of n rows at ring row pos (two
// segments when it wraps) are copied to their mirror rows past the end.
void HiddenStateBuffer::mirror(int64_t pos, int64_t n, void* stream) {
  const int64_t lim = std::min<int64_t>(kMirrorRows, cap_);
  const size_t row = static_cast<size_t>(geom_.bytes_per_token());
  uint8_t* ring = static_cast<uint8_t*>(ring_feat_);
  auto copy = [&](int64_t lo, int64_t hi) {  // ring rows [lo, hi) of [0, lim)
    lo = std::max<int64_t>(lo, 0);
    hi = std::min<int64_t>(hi, lim);
    if (hi > lo)
      SPECSIM_CUDA(cudaMemcpyAsync(ring + (cap_ + lo) * row, ring + lo * row, (hi - lo) * row,
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  };
  const int64_t first = std::min<int64_t>(n, cap_ - pos);
  copy(pos, pos + first);
  if (first < n) copy(0, n - first);
  if (cap_ < kMirrorRows) {
    // tiny rings: rows [cap, cap + 128) repeat the ring cyclically
    for (int64_t r = lim; r < kMirrorRows; r += cap_) {
      const int64_t c = std::min<int64_t>(cap_, kMirrorRows - r);
      SPECSIM_CUDA(cudaMemcpyAsync(ring + (cap_ + r) * row, ring, c * row,
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
    }
  }
}

void* HiddenStateBuffer::event_for(int64_t seq) const {
  if (seq <= 0 || append_seq_ - seq >= kEventRing) return nullptr;  // known complete
  return events_[static_cast<size_t>(seq % kEventRing)];
}

HiddenStateBuffer::~HiddenStateBuffer() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
  cudaFree(ring_feat_);
  cudaFree(ring_ids_);
  cudaFree(staging_dev_);
  cudaFreeHost(staging_host_);
  for (void* e : events_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

void HiddenStateBuffer::sync() const {
  SPECSIM_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)));
}

const HiddenStateBuffer::Sample& HiddenStateBuffer::sample(int64_t id) const {
  auto it = samples_.find(id);
  if (it == samples_.end())
    throw std::out_of_range("sample " + std::to_string(id) + " is not resident in the buffer");
  return it->second;
}

void HiddenStateBuffer::account(int n) {
  // extract_signals: records and bytes grow; bytes beyond the threshold
  // are flushed to cumulative storage as one event.
  stats_.records += n;
  stats_.bytes += static_cast<int64_t>(n) * geom_.bytes_per_token();
  if (stats_.bytes > flush_threshold_) {
    stats_.cumulative_bytes += stats_.bytes;
    stats_.bytes = 0;
    stats_.flushes += 1;
  }
}

void HiddenStateBuffer::open_sample(int64_t sample_id, double alpha) {
  if (sample_id == open_id_) {
    samples_.at(sample_id).alpha = alpha;
    return;
  }
  if (samples_.count(sample_id))
    throw std::invalid_argument("sample " + std::to_string(sample_id) +
                                " was already closed; records of a sample must be contiguous");
  Sample s;
  s.start = head_;
  s.length = 0;
  s.alpha = alpha;
  samples_.emplace(sample_id, s);
  order_.push_back(sample_id);
  open_id_ = sample_id;
  stats_.samples += 1;  // record_sample
}

void HiddenStateBuffer::reserve(int n) {
  if (n > cap_) throw std::invalid_argument("append larger than the buffer capacity");
  while (head_ + n - tail_ > cap_) {
    if (order_.empty() || order_.front() == open_id_)
      throw std::invalid_argument("open sample exceeds the buffer capacity");
    const Sample& oldest = samples_.at(order_.front());
    tail_ = oldest.start + oldest.length;
    samples_.erase(order_.front());
    order_.pop_front();
  }
}

void HiddenStateBuffer::append(int64_t sample_id, double alpha, const void* const* layer_ptrs,
                               int64_t rows, int64_t ld, const int32_t* token_ids,
                               const int32_t* accepted_idx, int n, bool on_device) {
  Problems p("hsbuf_append");
  p.check(n >= 0, "n must be >= 0");
  p.check(layer_ptrs != nullptr || n == 0, "layer_ptrs is null");
  p.check(token_ids != nullptr || n == 0, "token_ids is null");
  p.check(ld >= geom_.hidden_dim && ld % 8 == 0, "ld must be >= hidden_dim and a multiple of 8");
  p.check(alpha >= 0.0 && alpha <= 1.0, "alpha must be in [0,1]");
  p.throw_if_any();
  if (accepted_idx)
    for (int i = 0; i < n; ++i)
      if (accepted_idx[i] < 0 || accepted_idx[i] >= rows)
        throw std::invalid_argument("accepted_idx out of range");
  if (!accepted_idx && n > rows) throw std::invalid_argument("n > rows");
  open_sample(sample_id, alpha);
  if (n == 0) return;
  reserve(n);
  DeviceGuard dg(device_);
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  const int H = geom_.hidden_dim, L = geom_.layers_tapped;
  const size_t row_bytes = static_cast<size_t>(H) * 2;
  const size_t feat_bytes = row_bytes * L * n;
  const size_t need = feat_bytes + sizeof(int32_t) * 2 * n + 256;
  if (need > staging_bytes_) {
    SPECSIM_CUDA(cudaStreamSynchronize(s));
    cudaFree(staging_dev_);
    cudaFreeHost(staging_host_);
    staging_bytes_ = std::max(need, staging_bytes_ * 2);
    SPECSIM_CUDA(cudaMalloc(&staging_dev_, staging_bytes_));
    SPECSIM_CUDA(cudaMallocHost(&staging_host_, staging_bytes_));
  }
  uint8_t* hst = static_cast<uint8_t*>(staging_host_);
  uint8_t* dst = static_cast<uint8_t*>(staging_dev_);
  kern::LayerPtrs lp{};
  const int32_t* d_idx = nullptr;
  long long src_ld = ld;
  if (!on_device) {
    // stage the accepted rows per layer: [L][n][H] (what a D2H capture into
    // a pinned host buffer produces), one H2D copy, pack on the device.
    for (int l = 0; l < L; ++l) {
      const uint8_t* src = static_cast<const uint8_t*>(layer_ptrs[l]);
      for (int i = 0; i < n; ++i) {
        const int64_t r = accepted_idx ? accepted_idx[i] : i;
        std::memcpy(hst + (static_cast<size_t>(l) * n + i) * row_bytes, src + r * ld * 2,
                    row_bytes);
      }
    }
    std::memcpy(hst + feat_bytes, token_ids, sizeof(int32_t) * n);
    SPECSIM_CUDA(cudaMemcpyAsync(dst, hst, feat_bytes + sizeof(int32_t) * n,
                                 cudaMemcpyHostToDevice, s));
    for (int l = 0; l < L; ++l)
      lp.p[l] = reinterpret_cast<const __nv_bfloat16*>(dst + static_cast<size_t>(l) * n * row_bytes);
    src_ld = H;
  } else {
    for (int l = 0; l < L; ++l) lp.p[l] = static_cast<const __nv_bfloat16*>(layer_ptrs[l]);
    std::memcpy(hst + feat_bytes, token_ids, sizeof(int32_t) * n);
    if (accepted_idx) std::memcpy(hst + feat_bytes + sizeof(int32_t) * n, accepted_idx,
                                  sizeof(int32_t) * n);
    SPECSIM_CUDA(cudaMemcpyAsync(dst + feat_bytes, hst + feat_bytes, sizeof(int32_t) * 2 * n,
                                 cudaMemcpyHostToDevice, s));
    if (accepted_idx) d_idx = reinterpret_cast<const int32_t*>(dst + feat_bytes + sizeof(int32_t) * n);
  }
  const int64_t pos = head_ % cap_;
  kern::pack_signals(lp, L, src_ld, H, d_idx, n, static_cast<__nv_bfloat16*>(ring_feat_), cap_,
                     pos, s);
  SPECSIM_CHECK_LAUNCH();
  // ids: at most two contiguous ring segments
  const int32_t* d_ids = reinterpret_cast<const int32_t*>(dst + feat_bytes);
  const int64_t first = std::min<int64_t>(n, cap_ - pos);
  SPECSIM_CUDA(cudaMemcpyAsync(ring_ids_ + pos, d_ids, sizeof(int32_t) * first,
                               cudaMemcpyDeviceToDevice, s));
  if (first < n)
    SPECSIM_CUDA(cudaMemcpyAsync(ring_ids_, d_ids + first, sizeof(int32_t) * (n - first),
                                 cudaMemcpyDeviceToDevice, s));
  mirror(pos, n, s);
  record_append(s);
  SPECSIM_CUDA(cudaStreamSynchronize(s));  // staging reuse
  head_ += n;
  samples_.at(open_id_).length += n;
  stats_.resident_tokens = head_ - tail_;
  account(n);
}

void HiddenStateBuffer::append_packed(int64_t sample_id, double alpha, const uint16_t* features,
                                      const int32_t* token_ids, int n, int mode) {
  const bool on_device = mode == 1;
  const bool async_pinned = mode == 2;
  Problems p("hsbuf_append_packed");
  p.check(n >= 0, "n must be >= 0");
  p.check(features != nullptr || n == 0, "features is null");
  p.check(token_ids != nullptr || n == 0, "token_ids is null");
  p.check(alpha >= 0.0 && alpha <= 1.0, "alpha must be in [0,1]");
  p.check(mode >= 0 && mode <= 2, "mode must be 0 (host), 1 (device) or 2 (pinned host, async)");
  p.throw_if_any();
  if (async_pinned) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, features) != cudaSuccess || a.type != cudaMemoryTypeHost ||
        cudaPointerGetAttributes(&a, token_ids) != cudaSuccess || a.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      throw std::invalid_argument("mode 2 needs page-locked (pinned) host buffers");
    }
  }
  open_sample(sample_id, alpha);
  if (n == 0) return;
  reserve(n);
  DeviceGuard dg(device_);
  cudaStream_t s = static_cast<cudaStream_t>(stream_);
  const int W = geom_.hidden_dim * geom_.layers_tapped;
  const int64_t pos = head_ % cap_;
  const int64_t first = std::min<int64_t>(n, cap_ - pos);
  const size_t row = static_cast<size_t>(W) * 2;
  uint8_t* ring = static_cast<uint8_t*>(ring_feat_);
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // packed rows are already [n, W]: DMA straight into the ring (two segments)
  SPECSIM_CUDA(cudaMemcpyAsync(ring + pos * row, features, row * first, kind, s));
  if (first < n)
    SPECSIM_CUDA(cudaMemcpyAsync(ring, reinterpret_cast<const uint8_t*>(features) + row * first,
                                 row * (n - first), kind, s));
  SPECSIM_CUDA(cudaMemcpyAsync(ring_ids_ + pos, token_ids, sizeof(int32_t) * first, kind, s));
  if (first < n)
    SPECSIM_CUDA(cudaMemcpyAsync(ring_ids_, token_ids + first, sizeof(int32_t) * (n - first),
                                 kind, s));
  mirror(pos, n, s);
  // consumers (trainer steps) order themselves after this event instead of a
  // host sync; pinned-host appends return immediately so the DMA overlaps
  // the step that is running
  record_append(s);
  if (!async_pinned) SPECSIM_CUDA(cudaStreamSynchronize(s));
  head_ += n;
  samples_.at(open_id_).length += n;
  stats_.resident_tokens = head_ - tail_;
  account(n);
}

void HiddenStateBuffer::read_sample(int64_t id, uint16_t* features, int32_t* ids) const {
  const Sample& sm = sample(id);
  DeviceGuard dg(device_);
  sync();  // async appends land on the buffer's own stream
  const int W = geom_.hidden_dim * geom_.layers_tapped;
  const size_t row = static_cast<size_t>(W) * 2;
  const int64_t pos = sm.start % cap_;
  const int64_t first = std::min<int64_t>(sm.length, cap_ - pos);
  const uint8_t* ring = static_cast<const uint8_t*>(ring_feat_);
  if (features) {
    SPECSIM_CUDA(cudaMemcpy(features, ring + pos * row, row * first, cudaMemcpyDeviceToHost));
    if (first < sm.length)
      SPECSIM_CUDA(cudaMemcpy(reinterpret_cast<uint8_t*>(features) + row * first, ring,
                              row * (sm.length - first), cudaMemcpyDeviceToHost));
  }
  if (ids) {
    SPECSIM_CUDA(cudaMemcpy(ids, ring_ids_ + pos, sizeof(int32_t) * first, cudaMemcpyDeviceToHost));
    if (first < sm.length)
      SPECSIM_CUDA(cudaMemcpy(ids + first, ring_ids_, sizeof(int32_t) * (sm.length - first),
                              cudaMemcpyDeviceToHost));
  }
}

}  // namespace specsim

// ================================================================== C ABI
using namespace specsim;


extern "C" {

int specsim_hsbuf_create(const specsim_signal_geometry* g, int64_t capacity_tokens,
                         int64_t flush_threshold_bytes, int device, specsim_hsbuf** out) {
  return guard([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    SignalGeometry geo{g->hidden_dim, g->layers_tapped, g->bytes_per_element};
    *out = new specsim_hsbuf{new HiddenStateBuffer(geo, capacity_tokens, flush_threshold_bytes,
                                                   device)};
  });
}

int specsim_hsbuf_destroy(specsim_hsbuf* b) {
  return guard([&] {
    if (!b) return;
    delete b->b;
    delete b;
  });
}

int specsim_hsbuf_append(specsim_hsbuf* b, int64_t sample_id, double alpha,
                         const void* const* layer_ptrs, int64_t rows, int64_t ld,
                         const int32_t* token_ids, const int32_t* accepted_idx, int32_t n,
                         int on_device) {
  return guard([&] {
    if (!b) throw std::invalid_argument("null buffer");
    b->b->append(sample_id, alpha, layer_ptrs, rows, ld, token_ids, accepted_idx, n,
                 on_device != 0);
  });
}

int specsim_hsbuf_append_packed(specsim_hsbuf* b, int64_t sample_id, double alpha,
                                const uint16_t* features, const int32_t* token_ids, int32_t n,
                                int mode) {
  return guard([&] {
    if (!b) throw std::invalid_argument("null buffer");
    b->b->append_packed(sample_id, alpha, features, token_ids, n, mode);
  });
}

int specsim_hsbuf_sync(specsim_hsbuf* b) {
  return guard([&] {
    if (!b) throw std::invalid_argument("null buffer");
    b->b->sync();
  });
}

int specsim_hsbuf_stats_get(const specsim_hsbuf* b, specsim_hsbuf_stats* out) {
  return guard([&] {
    if (!b || !out) throw std::invalid_argument("null argument");
    const auto s = b->b->stats();
    *out = specsim_hsbuf_stats{s.records, s.bytes, s.flushes, s.cumulative_bytes, s.samples,
                               s.resident_tokens};
  });
}

int specsim_hsbuf_sample_info(const specsim_hsbuf* b, int64_t sample_id, int32_t* length,
                              double* alpha) {
  return guard([&] {
    if (!b) throw std::invalid_argument("null buffer");
    const auto& s = b->b->sample(sample_id);
    if (length) *length = s.length;
    if (alpha) *alpha = s.alpha;
  });
}

int specsim_hsbuf_read_sample(const specsim_hsbuf* b, int64_t sample_id, uint16_t* features,
                              int32_t* token_ids) {
  return guard([&] {
    if (!b) throw std::invalid_argument("null buffer");
    b->b->read_sample(sample_id, features, token_ids);
  });
}

}  // extern "C"

namespace specsim {
HiddenStateBuffer* hsbuf_unwrap(specsim_hsbuf* b) {
  if (!b) throw std::invalid_argument("null buffer");
  return b->b;
}
}  // namespace specsim
