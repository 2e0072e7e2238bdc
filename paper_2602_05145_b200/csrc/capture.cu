// Capture side of the signal path ("overlap
// both the device-to-host memory transfer ... with the next verification
// step", SPEC.md:267-275 extract_signals, SPEC.md:293 64 MiB flush):
// accepted-token hidden states are packed on the serving stream into a device
// staging segment, copied D2H on the capture stream into a pinned host
// segment (two segments, double-buffered), and flushed by a writer thread to
// "TIDESIG1" shard files (format in proj/include/specsim/draft_trainer.hpp).
// load_shards() is the training side's reader into the HBM ring.
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <fstream>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "common.h"
#include "handles.h"
#include "kernels.h"
#include "specsim/draft_trainer.hpp"

namespace specsim {

namespace {
constexpr int64_t kDefaultFlush = 64ll << 20;
constexpr char kMagic[8] = {'T', 'I', 'D', 'E', 'S', 'I', 'G', '1'};
constexpr uint32_t kVersion = 1;

#pragma pack(push, 1)
struct FileHeader {
  char magic[8];
  uint32_t version, layers, hidden, bytes_per_element;
  uint64_t n_records, payload_bytes;
};
struct RecordHeader {
  int64_t sample_id;
  double alpha;
  int32_t n, width;
  int64_t flags;  // 1 = sample complete (end_sample)
};
#pragma pack(pop)
static_assert(sizeof(FileHeader) == 40 && sizeof(RecordHeader) == 32, "shard layout");

size_t align16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    SPECSIM_CUDA(cudaGetDevice(&prev));
    if (prev != dev) SPECSIM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};
}  // namespace

struct SignalCapture::Impl {
  struct Segment {
    uint8_t* host = nullptr;  // pinned
    uint8_t* dev = nullptr;   // device staging, same byte layout
    size_t cap = 0, used = 0;
    uint64_t n_records = 0;
    cudaEvent_t done = nullptr;  // last D2H into this segment
    bool busy = false;           // queued for / being written by the writer
    int32_t* idx_host = nullptr;  // pinned accepted-row indices (H2D source), same lifetime
    size_t idx_cap = 0, idx_used = 0;
  };

  SignalGeometry geom;
  std::string dir;
  int64_t threshold;
  int device;
  cudaStream_t cstream = nullptr;
  cudaEvent_t packed = nullptr;
  Segment seg[2];
  int cur = 0;
  Stats st;
  std::vector<std::string> paths;
  int64_t next_file = 0;
  bool closed = false;

  mutable std::mutex mu;
  std::condition_variable cv;
  std::deque<int> queue;
  bool stop = false;
  std::exception_ptr writer_error;
  std::thread writer;

  Impl(const SignalGeometry& g, const std::string& d, int64_t thr, int dev)
      : geom(g), dir(d), threshold(thr > 0 ? thr : kDefaultFlush), device(dev) {
    geom.validate();
    Problems p("invalid signal capture");
    p.check(geom.bytes_per_element == 2, "only bf16 signals (bytes_per_element = 2)");
    p.check(geom.hidden_dim % 8 == 0, "hidden_dim must be a multiple of 8 (16-byte rows)");
    p.check(geom.layers_tapped <= 8, "at most 8 tapped layers");
    p.check(!dir.empty(), "directory is empty");
    p.throw_if_any();
    {
      // the directory must exist and be writable: probe with a temp file
      const std::string probe = dir + "/.tidesig_probe";
      std::ofstream f(probe, std::ios::binary);
      if (!f) throw std::invalid_argument("capture directory not writable: " + dir);
      f.close();
      std::remove(probe.c_str());
    }
    DeviceGuard dg(device);
    SPECSIM_CUDA(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
    SPECSIM_CUDA(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
    for (auto& s : seg) {
      SPECSIM_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
      // room for the records behind threshold bytes of features (ids, headers,
      // one more batch) so a SPEC flush, not a full segment, ends a shard
      grow(s, static_cast<size_t>(threshold) + static_cast<size_t>(threshold) / 4 + (16u << 20));
    }
    writer = std::thread([this] { writer_loop(); });
  }

  ~Impl() {
    try {
      close();
    } catch (...) {
    }
    cudaSetDevice(device);
    for (auto& s : seg) {
      cudaFreeHost(s.host);
      cudaFreeHost(s.idx_host);
      cudaFree(s.dev);
      if (s.done) cudaEventDestroy(s.done);
    }
    if (packed) cudaEventDestroy(packed);
    if (cstream) cudaStreamDestroy(cstream);
  }

  void grow(Segment& s, size_t cap) {
    if (s.host) SPECSIM_CUDA(cudaFreeHost(s.host));
    if (s.dev) SPECSIM_CUDA(cudaFree(s.dev));
    s.host = nullptr;
    s.dev = nullptr;
    SPECSIM_CUDA(cudaMallocHost(&s.host, cap));
    SPECSIM_CUDA(cudaMalloc(&s.dev, cap));
    s.cap = cap;
    // one index per captured row at most: rows are >= 16 bytes of features
    if (s.idx_host) SPECSIM_CUDA(cudaFreeHost(s.idx_host));
    s.idx_cap = cap / 16;
    SPECSIM_CUDA(cudaMallocHost(&s.idx_host, sizeof(int32_t) * s.idx_cap));
    s.idx_used = 0;
  }

  // stage accepted-row indices in the segment's pinned arena so the H2D on
  // the serving stream is a true async DMA (reused only after the segment
  // has been written out, like the segment itself)
  const int32_t* stage_idx(Segment& s, const int32_t* idx, int n) {
    int32_t* p = s.idx_host + s.idx_used;
    std::memcpy(p, idx, sizeof(int32_t) * n);
    s.idx_used += static_cast<size_t>(n);
    return p;
  }

  void check_writer() {
    std::lock_guard<std::mutex> lk(mu);
    if (writer_error) std::rethrow_exception(writer_error);
  }

  // hand the current segment to the writer and switch to the other one
  void hand_off() {
    Segment& s = seg[cur];
    if (s.used == 0) return;
    {
      std::lock_guard<std::mutex> lk(mu);
      s.busy = true;
      queue.push_back(cur);
    }
    cv.notify_all();
    cur ^= 1;
  }

  // a free segment with room for `bytes` more
  Segment& room(size_t bytes) {
    for (;;) {
      Segment& s = seg[cur];
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return !s.busy || writer_error; });
        if (writer_error) std::rethrow_exception(writer_error);
      }
      if (s.used + bytes <= s.cap) return s;
      if (s.used == 0) {  // a single record larger than the segment
        grow(s, std::max(bytes, 2 * s.cap));
        return s;
      }
      hand_off();
    }
  }

  void writer_loop() {
    cudaSetDevice(device);
    for (;;) {
      int i;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || !queue.empty(); });
        if (queue.empty()) return;
        i = queue.front();
      }
      Segment& s = seg[i];
      try {
        SPECSIM_CUDA(cudaEventSynchronize(s.done));  // every D2H of the segment landed
        char name[64];
        int64_t idx;
        {
          std::lock_guard<std::mutex> lk(mu);
          idx = next_file++;
        }
        std::snprintf(name, sizeof(name), "/shard_%06lld.tsig", static_cast<long long>(idx));
        const std::string path = dir + name;
        FileHeader h{};
        std::memcpy(h.magic, kMagic, 8);
        h.version = kVersion;
        h.layers = static_cast<uint32_t>(geom.layers_tapped);
        h.hidden = static_cast<uint32_t>(geom.hidden_dim);
        h.bytes_per_element = 2;
        h.n_records = s.n_records;
        h.payload_bytes = s.used;
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        f.write(reinterpret_cast<const char*>(&h), sizeof(h));
        f.write(reinterpret_cast<const char*>(s.host), static_cast<std::streamsize>(s.used));
        f.close();
        if (!f) throw std::runtime_error("failed to write shard " + path);
        std::lock_guard<std::mutex> lk(mu);
        paths.push_back(path);
        st.files += 1;
        st.file_bytes += static_cast<int64_t>(sizeof(h) + s.used);
        s.used = 0;
        s.n_records = 0;
        s.idx_used = 0;
        s.busy = false;
        queue.pop_front();
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        writer_error = std::current_exception();
        s.busy = false;
        queue.pop_front();
      }
      cv.notify_all();
    }
  }

  void capture(int64_t sample_id, const void* const* layer_ptrs, int64_t rows, int64_t ld,
               const int32_t* ids, const int32_t* idx, int n, cudaStream_t stream) {
    if (closed) throw std::invalid_argument("capture is closed");
    const int H = geom.hidden_dim, L = geom.layers_tapped, W = H * L;
    Problems p("capture_append");
    p.check(n >= 0, "n must be >= 0");
    p.check(layer_ptrs != nullptr || n == 0, "layer_ptrs is null");
    p.check(ids != nullptr || n == 0, "token_ids is null");
    p.check(ld >= H && ld % 8 == 0, "ld must be >= hidden_dim and a multiple of 8");
    p.throw_if_any();
    for (int i = 0; i < n && idx; ++i)
      if (idx[i] < 0 || idx[i] >= rows) throw std::invalid_argument("accepted_idx out of range");
    if (!idx && n > rows) throw std::invalid_argument("n > rows");
    if (n > 0)
      for (int l = 0; l < L; ++l)
        if (!layer_ptrs[l]) throw std::invalid_argument("layer pointer is null");
    check_writer();
    if (n == 0) return;
    DeviceGuard dg(device);
    const size_t feat = static_cast<size_t>(n) * W * 2;
    const size_t rec = align16(sizeof(RecordHeader) + feat + sizeof(int32_t) * n);
    Segment& s = room(rec);
    uint8_t* h = s.host + s.used;
    uint8_t* d = s.dev + s.used;
    RecordHeader rh{sample_id, -1.0, n, W, 0};
    std::memcpy(h, &rh, sizeof(rh));
    std::memcpy(h + sizeof(rh) + feat, ids, sizeof(int32_t) * n);
    std::memset(h + sizeof(rh) + feat + sizeof(int32_t) * n, 0,
                rec - sizeof(rh) - feat - sizeof(int32_t) * n);
    kern::LayerPtrs lp{};
    for (int l = 0; l < L; ++l) lp.p[l] = static_cast<const __nv_bfloat16*>(layer_ptrs[l]);
    const int32_t* d_idx = nullptr;
    if (idx) {
      // accepted rows -> the device copy of this record's id slot (pageable
      // source: staged by the driver before the call returns)
      d_idx = reinterpret_cast<const int32_t*>(d + sizeof(rh) + feat);
      SPECSIM_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(d_idx), stage_idx(s, idx, n),
                                   sizeof(int32_t) * n, cudaMemcpyHostToDevice, stream));
    }
    // pack on the serving stream (reads the layer tensors while they are
    // valid), then the D2H on the capture stream overlaps what follows
    kern::pack_signals(lp, L, ld, H, d_idx, n,
                       reinterpret_cast<__nv_bfloat16*>(d + sizeof(rh)), n, 0, stream);
    SPECSIM_CHECK_LAUNCH();
    SPECSIM_CUDA(cudaEventRecord(packed, stream));
    SPECSIM_CUDA(cudaStreamWaitEvent(cstream, packed, 0));
    SPECSIM_CUDA(cudaMemcpyAsync(h + sizeof(rh), d + sizeof(rh), feat, cudaMemcpyDeviceToHost,
                                 cstream));
    SPECSIM_CUDA(cudaEventRecord(s.done, cstream));
    s.used += rec;
    s.n_records += 1;
    // extract_signals accounting: flush past the threshold
    account(n);
  }

  // One serving iteration: request r's accepted rows are
  // rows[offsets[r] .. offsets[r+1]) of the layer matrices.  One pack kernel
  // and one D2H for the whole batch; stored as a batch record (flags 2):
  // header, i64 sample_ids[n_req], i32 counts[n_req] (padded to 16 B),
  // features[total][W], i32 ids[total], padding to 16 B.
  void capture_batch(const int64_t* sample_ids, int n_req, const int32_t* offsets,
                     const int32_t* rows_idx, const void* const* layer_ptrs, int64_t rows,
                     int64_t ld, const int32_t* ids, cudaStream_t stream) {
    if (closed) throw std::invalid_argument("capture is closed");
    const int H = geom.hidden_dim, L = geom.layers_tapped, W = H * L;
    Problems p("capture_batch");
    p.check(n_req >= 0, "n_req must be >= 0");
    p.check((sample_ids && offsets) || n_req == 0, "sample_ids / offsets is null");
    p.check(ld >= H && ld % 8 == 0, "ld must be >= hidden_dim and a multiple of 8");
    p.throw_if_any();
    if (n_req == 0) return;
    if (offsets[0] != 0) throw std::invalid_argument("offsets[0] must be 0");
    for (int r = 0; r < n_req; ++r)
      if (offsets[r + 1] < offsets[r]) throw std::invalid_argument("offsets must be non-decreasing");
    const int total = offsets[n_req];
    if (total > 0) {
      if (!rows_idx || !ids || !layer_ptrs) throw std::invalid_argument("null rows / ids / layers");
      for (int i = 0; i < total; ++i)
        if (rows_idx[i] < 0 || rows_idx[i] >= rows)
          throw std::invalid_argument("accepted row out of range");
      for (int l = 0; l < L; ++l)
        if (!layer_ptrs[l]) throw std::invalid_argument("layer pointer is null");
    }
    check_writer();
    DeviceGuard dg(device);
    const size_t meta = align16(sizeof(int64_t) * n_req + sizeof(int32_t) * n_req);
    const size_t feat = static_cast<size_t>(total) * W * 2;
    const size_t rec = align16(sizeof(RecordHeader) + meta + feat + sizeof(int32_t) * total);
    Segment& s = room(rec);
    uint8_t* h = s.host + s.used;
    uint8_t* d = s.dev + s.used;
    RecordHeader rh{-1, static_cast<double>(n_req), total, W, 2};  // alpha slot = n_req
    std::memcpy(h, &rh, sizeof(rh));
    uint8_t* m = h + sizeof(rh);
    std::memcpy(m, sample_ids, sizeof(int64_t) * n_req);
    for (int r = 0; r < n_req; ++r) {
      const int32_t cnt = offsets[r + 1] - offsets[r];
      std::memcpy(m + sizeof(int64_t) * n_req + sizeof(int32_t) * r, &cnt, sizeof(cnt));
    }
    std::memset(m + sizeof(int64_t) * n_req + sizeof(int32_t) * n_req, 0,
                meta - sizeof(int64_t) * n_req - sizeof(int32_t) * n_req);
    const size_t f_off = sizeof(rh) + meta;
    std::memcpy(h + f_off + feat, ids, sizeof(int32_t) * total);
    std::memset(h + f_off + feat + sizeof(int32_t) * total, 0,
                rec - f_off - feat - sizeof(int32_t) * total);
    if (total > 0) {
      int32_t* d_idx = reinterpret_cast<int32_t*>(d + f_off + feat);
      SPECSIM_CUDA(cudaMemcpyAsync(d_idx, stage_idx(s, rows_idx, total), sizeof(int32_t) * total,
                                   cudaMemcpyHostToDevice, stream));
      kern::LayerPtrs lp{};
      for (int l = 0; l < L; ++l) lp.p[l] = static_cast<const __nv_bfloat16*>(layer_ptrs[l]);
      kern::pack_signals(lp, L, ld, H, d_idx, total,
                         reinterpret_cast<__nv_bfloat16*>(d + f_off), total, 0, stream);
      SPECSIM_CHECK_LAUNCH();
      SPECSIM_CUDA(cudaEventRecord(packed, stream));
      SPECSIM_CUDA(cudaStreamWaitEvent(cstream, packed, 0));
      SPECSIM_CUDA(cudaMemcpyAsync(h + f_off, d + f_off, feat, cudaMemcpyDeviceToHost, cstream));
      SPECSIM_CUDA(cudaEventRecord(s.done, cstream));
    }
    s.used += rec;
    s.n_records += 1;
    account(total);
  }

  void account(int n) {
    std::unique_lock<std::mutex> lk(mu);
    st.records += n;
    st.bytes += static_cast<int64_t>(n) * geom.bytes_per_token();
    if (st.bytes > threshold) {
      st.cumulative_bytes += st.bytes;
      st.bytes = 0;
      st.flushes += 1;
      lk.unlock();
      hand_off();
    }
  }

  void end_sample(int64_t sample_id, double alpha) {
    if (closed) throw std::invalid_argument("capture is closed");
    if (!(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("alpha must be in [0,1]");
    check_writer();
    Segment& s = room(sizeof(RecordHeader));
    RecordHeader rh{sample_id, alpha, 0, geom.hidden_dim * geom.layers_tapped, 1};
    std::memcpy(s.host + s.used, &rh, sizeof(rh));
    s.used += sizeof(rh);
    s.n_records += 1;
    std::lock_guard<std::mutex> lk(mu);
    st.samples += 1;
  }

  void drain() {
    hand_off();
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return (queue.empty() && !seg[0].busy && !seg[1].busy) || writer_error; });
    if (writer_error) std::rethrow_exception(writer_error);
  }

  void close() {
    if (closed) return;
    closed = true;
    std::exception_ptr err;
    try {
      drain();
    } catch (...) {
      err = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (writer.joinable()) writer.join();
    if (err) std::rethrow_exception(err);
  }
};

SignalCapture::SignalCapture(const SignalGeometry& g, const std::string& directory,
                             int64_t flush_threshold, int device)
    : impl_(new Impl(g, directory, flush_threshold, device)) {}
SignalCapture::~SignalCapture() = default;
void SignalCapture::capture(int64_t sample_id, const void* const* layer_ptrs, int64_t rows,
                            int64_t ld, const int32_t* token_ids, const int32_t* accepted_idx,
                            int n, void* stream) {
  impl_->capture(sample_id, layer_ptrs, rows, ld, token_ids, accepted_idx, n,
                 static_cast<cudaStream_t>(stream));
}
void SignalCapture::capture_batch(const int64_t* sample_ids, int n_req, const int32_t* offsets,
                                  const int32_t* accepted_rows, const void* const* layer_ptrs,
                                  int64_t rows, int64_t ld, const int32_t* token_ids,
                                  void* stream) {
  impl_->capture_batch(sample_ids, n_req, offsets, accepted_rows, layer_ptrs, rows, ld, token_ids,
                       static_cast<cudaStream_t>(stream));
}
void SignalCapture::end_sample(int64_t sample_id, double alpha) {
  impl_->end_sample(sample_id, alpha);
}
void SignalCapture::flush() {
  if (impl_->closed) throw std::invalid_argument("capture is closed");
  impl_->drain();
}
void SignalCapture::close() { impl_->close(); }
SignalCapture::Stats SignalCapture::stats() const {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->st;
}
std::vector<std::string> SignalCapture::files() const {
  std::lock_guard<std::mutex> lk(impl_->mu);
  return impl_->paths;
}

namespace {
// Rows of samples whose end_sample record has not been read yet, per buffer
// (HiddenStateBuffer::serial): a request that straddles a flush has its rows
// and its completion record in different shard files, which a caller may load
// one call at a time as they appear.
struct Carried {
  std::vector<uint16_t> feat;
  std::vector<int32_t> ids;
};
std::mutex g_carry_mu;
std::unordered_map<uint64_t, std::pair<std::vector<int64_t>, std::unordered_map<int64_t, Carried>>>
    g_carry;
}  // namespace

int64_t load_shards(HiddenStateBuffer& buf, const std::vector<std::string>& paths) {
  const SignalGeometry& g = buf.geometry();
  const int W = g.hidden_dim * g.layers_tapped;
  struct Chunk {
    const uint16_t* feat;
    const int32_t* ids;
    int n;
  };
  struct Acc {
    std::vector<Chunk> chunks;
    double alpha = 0.0;
    int64_t total = 0;
    bool complete = false;
  };
  std::vector<std::vector<char>> files;
  std::unordered_map<int64_t, Acc> acc;
  std::vector<int64_t> order;
  // unfinished samples of earlier calls come first (first-appearance order)
  std::vector<int64_t> carried_order;
  std::unordered_map<int64_t, Carried> carried;
  {
    std::lock_guard<std::mutex> lk(g_carry_mu);
    auto it = g_carry.find(buf.serial());
    if (it != g_carry.end()) {
      carried_order = std::move(it->second.first);
      carried = std::move(it->second.second);
      g_carry.erase(it);
    }
  }
  for (int64_t id : carried_order) {
    const Carried& c = carried.at(id);
    Acc& a = acc[id];
    a.chunks.push_back({c.feat.data(), c.ids.data(), static_cast<int>(c.ids.size())});
    a.total = static_cast<int64_t>(c.ids.size());
    order.push_back(id);
  }
  for (const auto& path : paths) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw std::invalid_argument("cannot open shard " + path);
    const std::streamsize size = f.tellg();
    f.seekg(0);
    files.emplace_back(static_cast<size_t>(size));
    std::vector<char>& b = files.back();
    if (!f.read(b.data(), size)) throw std::invalid_argument("cannot read shard " + path);
    Problems p("invalid shard " + path);
    FileHeader h{};
    p.check(size >= static_cast<std::streamsize>(sizeof(h)), "truncated header");
    p.throw_if_any();
    std::memcpy(&h, b.data(), sizeof(h));
    p.check(std::memcmp(h.magic, kMagic, 8) == 0, "bad magic (not a TIDESIG1 shard)");
    p.check(h.version == kVersion, "unsupported version");
    p.check(h.layers == static_cast<uint32_t>(g.layers_tapped) &&
                h.hidden == static_cast<uint32_t>(g.hidden_dim) && h.bytes_per_element == 2,
            "signal geometry does not match the buffer");
    p.check(h.payload_bytes + sizeof(h) == static_cast<uint64_t>(size), "payload size mismatch");
    p.throw_if_any();
    size_t off = sizeof(h);
    for (uint64_t r = 0; r < h.n_records; ++r) {
      RecordHeader rh{};
      if (off + sizeof(rh) > static_cast<size_t>(size))
        throw std::invalid_argument("truncated record in shard " + path);
      std::memcpy(&rh, b.data() + off, sizeof(rh));
      if (rh.n < 0 || rh.width != W) throw std::invalid_argument("bad record in shard " + path);
      if (rh.flags & 2) {  // batch record: n_req = sample count, n = total rows
        const char* m = b.data() + off + sizeof(rh);
        // n_req travels as a double: bound it by the bytes left (12 per request)
        // before any size arithmetic
        const double room = static_cast<double>(static_cast<size_t>(size) - off - sizeof(rh));
        if (!(rh.alpha >= 0.0) || rh.alpha * 12.0 > room || rh.alpha != std::floor(rh.alpha))
          throw std::invalid_argument("bad batch record (request count) in shard " + path);
        const int64_t n_req = static_cast<int64_t>(rh.alpha);
        const size_t meta = align16(sizeof(int64_t) * n_req + sizeof(int32_t) * n_req);
        const size_t feat = static_cast<size_t>(rh.n) * W * 2;
        const size_t rec = align16(sizeof(rh) + meta + feat + sizeof(int32_t) * rh.n);
        if (off + rec > static_cast<size_t>(size))
          throw std::invalid_argument("truncated batch record in shard " + path);
        const char* fp = m + meta;
        const char* ip = fp + feat;
        int64_t row = 0;
        for (int64_t r = 0; r < n_req; ++r) {
          int64_t sid;
          int32_t cnt;
          std::memcpy(&sid, m + sizeof(int64_t) * r, sizeof(sid));
          std::memcpy(&cnt, m + sizeof(int64_t) * n_req + sizeof(int32_t) * r, sizeof(cnt));
          if (cnt < 0 || row + cnt > rh.n)
            throw std::invalid_argument("bad batch record in shard " + path);
          auto it = acc.find(sid);
          if (it == acc.end()) {
            it = acc.emplace(sid, Acc{}).first;
            order.push_back(sid);
          }
          if (cnt > 0) {
            it->second.chunks.push_back(
                {reinterpret_cast<const uint16_t*>(fp + static_cast<size_t>(row) * W * 2),
                 reinterpret_cast<const int32_t*>(ip + sizeof(int32_t) * row), cnt});
            it->second.total += cnt;
          }
          row += cnt;
        }
        off += rec;
        continue;
      }
      const size_t feat = static_cast<size_t>(rh.n) * W * 2;
      const size_t rec = rh.n ? align16(sizeof(rh) + feat + sizeof(int32_t) * rh.n) : sizeof(rh);
      if (off + rec > static_cast<size_t>(size))
        throw std::invalid_argument("truncated record in shard " + path);
      auto it = acc.find(rh.sample_id);
      if (it == acc.end()) {
        it = acc.emplace(rh.sample_id, Acc{}).first;
        order.push_back(rh.sample_id);
      }
      if (rh.n > 0) {
        it->second.chunks.push_back(
            {reinterpret_cast<const uint16_t*>(b.data() + off + sizeof(rh)),
             reinterpret_cast<const int32_t*>(b.data() + off + sizeof(rh) + feat), rh.n});
        it->second.total += rh.n;
      }
      if (rh.flags & 1) {
        it->second.alpha = rh.alpha;
        it->second.complete = true;
      }
      off += rec;
    }
  }
  std::vector<uint16_t> feat;
  std::vector<int32_t> ids;
  std::vector<int64_t> keep_order;
  std::unordered_map<int64_t, Carried> keep;
  int64_t appended = 0;
  for (int64_t id : order) {
    const Acc& a = acc.at(id);
    if (!a.complete) {  // completion record not read yet: carry the rows over
      Carried& c = keep[id];
      c.feat.resize(static_cast<size_t>(a.total) * W);
      c.ids.resize(static_cast<size_t>(a.total));
      size_t r = 0;
      for (const Chunk& ch : a.chunks) {
        std::memcpy(c.feat.data() + r * W, ch.feat, sizeof(uint16_t) * ch.n * W);
        std::memcpy(c.ids.data() + r, ch.ids, sizeof(int32_t) * ch.n);
        r += ch.n;
      }
      keep_order.push_back(id);
      continue;
    }
    ++appended;
    if (a.total == 0) throw std::invalid_argument("sample " + std::to_string(id) + " has no rows");
    if (a.chunks.size() == 1) {
      buf.append_packed(id, a.alpha, a.chunks[0].feat, a.chunks[0].ids, a.chunks[0].n, 0);
      continue;
    }
    feat.resize(static_cast<size_t>(a.total) * W);
    ids.resize(static_cast<size_t>(a.total));
    size_t r = 0;
    for (const Chunk& c : a.chunks) {
      std::memcpy(feat.data() + r * W, c.feat, sizeof(uint16_t) * c.n * W);
      std::memcpy(ids.data() + r, c.ids, sizeof(int32_t) * c.n);
      r += c.n;
    }
    buf.append_packed(id, a.alpha, feat.data(), ids.data(), static_cast<int>(a.total), 0);
  }
  if (!keep_order.empty()) {
    std::lock_guard<std::mutex> lk(g_carry_mu);
    g_carry[buf.serial()] = {std::move(keep_order), std::move(keep)};
  }
  return appended;
}

}  // namespace specsim

// ================================================================== C ABI
using namespace specsim;

struct specsim_capture {
  SignalCapture* c;
};

extern "C" {

int specsim_capture_create(const specsim_signal_geometry* g, const char* directory,
                           int64_t flush_threshold_bytes, int device, specsim_capture** out) {
  return guard([&] {
    if (!g || !directory || !out) throw std::invalid_argument("null argument");
    SignalGeometry geo{g->hidden_dim, g->layers_tapped, g->bytes_per_element};
    *out = new specsim_capture{new SignalCapture(geo, directory, flush_threshold_bytes, device)};
  });
}
int specsim_capture_destroy(specsim_capture* c) {
  if (!c) return SPECSIM_OK;
  const int r = guard([&] { c->c->close(); });
  delete c->c;
  delete c;
  return r;
}
int specsim_capture_append(specsim_capture* c, int64_t sample_id, const void* const* layer_ptrs,
                           int64_t rows, int64_t ld, const int32_t* token_ids,
                           const int32_t* accepted_idx, int32_t n, void* stream) {
  return guard([&] {
    c->c->capture(sample_id, layer_ptrs, rows, ld, token_ids, accepted_idx, n, stream);
  });
}
int specsim_capture_append_batch(specsim_capture* c, const int64_t* sample_ids, int32_t n_req,
                                 const int32_t* offsets, const int32_t* accepted_rows,
                                 const void* const* layer_ptrs, int64_t rows, int64_t ld,
                                 const int32_t* token_ids, void* stream) {
  return guard([&] {
    c->c->capture_batch(sample_ids, n_req, offsets, accepted_rows, layer_ptrs, rows, ld,
                        token_ids, stream);
  });
}
int specsim_capture_end_sample(specsim_capture* c, int64_t sample_id, double alpha) {
  return guard([&] { c->c->end_sample(sample_id, alpha); });
}
int specsim_capture_flush(specsim_capture* c) {
  return guard([&] { c->c->flush(); });
}
int specsim_capture_close(specsim_capture* c) {
  return guard([&] { c->c->close(); });
}
int specsim_capture_stats_get(const specsim_capture* c, specsim_capture_stats* out) {
  return guard([&] {
    const SignalCapture::Stats s = c->c->stats();
    *out = specsim_capture_stats{s.records, s.bytes,   s.flushes,   s.cumulative_bytes,
                                 s.samples, s.files, s.file_bytes};
  });
}
int specsim_capture_file(const specsim_capture* c, int64_t i, char* buf, int64_t cap) {
  return guard([&] {
    const auto f = c->c->files();
    if (i < 0 || i >= static_cast<int64_t>(f.size()))
      throw std::invalid_argument("file index out of range");
    if (static_cast<int64_t>(f[static_cast<size_t>(i)].size()) + 1 > cap)
      throw std::invalid_argument("buffer too small");
    std::memcpy(buf, f[static_cast<size_t>(i)].c_str(), f[static_cast<size_t>(i)].size() + 1);
  });
}
int specsim_hsbuf_load_shards(specsim_hsbuf* buf, const char* const* paths, int32_t n_paths,
                              int64_t* samples) {
  return guard([&] {
    if (!buf || (!paths && n_paths > 0)) throw std::invalid_argument("null argument");
    std::vector<std::string> p;
    for (int i = 0; i < n_paths; ++i) p.emplace_back(paths[i]);
    const int64_t n = load_shards(*buf->b, p);
    if (samples) *samples = n;
  });
}

}  // extern "C"
