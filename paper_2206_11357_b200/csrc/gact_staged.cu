// gact_staged.cu — the staged (host-buffer) forms of include/gact.h: the paper's "Parallel
// Swap and Prefetch" as one blocking call. Host buffers are cut into pieces of
// whole lcm(G, 4096)-element blocks and staged through GACT_STAGED_SLOTS rotating workspace slots;
// the host->device copies run on an internal swap-in stream, the batched kernels on the
// caller's stream, the device->host copies on an internal swap-out stream, and CUDA events
// order the three ("two new streams (swap in/out) ... the CUDA event").
//
// A piece starting at element `off` of its tensor is quantized with the Philox block counter
// off / 16 (QTensor::ctr0), so every result is bit-identical to the batch forms.
#include <cstring>
#include <vector>

#include "gact.h"
#include "gact_internal.h"

namespace {

constexpr int kSlots = GACT_STAGED_SLOTS;
// Piece boundaries: multiples of 4096 (every power-of-two group size, and 512 for the Philox
// block offset off / 16) and of G: lcm(G, 4096) elements.
int64_t piece_elems(int32_t G) {
  int64_t a = 4096, b = G;
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return 4096 / a * G;
}
constexpr uint64_t kAlign = 256;

uint64_t align_up(uint64_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
int elem_bytes(int32_t dtype) { return dtype == GACT_F32 ? 4 : 2; }

// Internal swap-in / swap-out streams and the per-slot events, once per thread and device.
struct Engine {
  int device = -1;
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t start = nullptr;
  cudaEvent_t in_done[kSlots], comp_done[kSlots], out_done[kSlots];
};

Engine* engine_for_current_device() {
  static thread_local std::vector<Engine> engines;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  for (Engine& e : engines)
    if (e.device == dev) return &e;
  Engine e;
  e.device = dev;
  const unsigned ef = cudaEventDisableTiming;
  bool ok = cudaStreamCreateWithFlags(&e.in, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&e.out, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&e.start, ef) == cudaSuccess;
  for (int j = 0; ok && j < kSlots; ++j)
    ok = cudaEventCreateWithFlags(&e.in_done[j], ef) == cudaSuccess &&
         cudaEventCreateWithFlags(&e.comp_done[j], ef) == cudaSuccess &&
         cudaEventCreateWithFlags(&e.out_done[j], ef) == cudaSuccess;
  if (!ok) return nullptr;
  engines.push_back(e);
  return &engines.back();
}

// Host memory (page-locked or pageable) vs device memory (device / managed).
bool is_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

// One of a tensor's four buffers: the bytes of a piece [off, off + m) and where they live.
enum Kind { ELEMS, WORDS, GROUPS };
struct Buf {
  char* base;
  bool host;
  bool input;  // read by the kernel (host -> device) or written (device -> host)
  Kind kind;
};
struct Shape {
  int32_t es, bits, G;
};
uint64_t buf_offset(Kind k, const Shape& s, int64_t off) {
  switch (k) {
    case ELEMS: return (uint64_t)off * s.es;
    case WORDS: return (uint64_t)(off / 32 * s.bits) * 4;  // off is a multiple of 4096
    default: return (uint64_t)(off / s.G) * 4;
  }
}
uint64_t buf_bytes(Kind k, const Shape& s, int64_t m) {
  switch (k) {
    case ELEMS: return (uint64_t)m * s.es;
    case WORDS: return (uint64_t)ceil_div(m * s.bits, 32) * 4;
    default: return (uint64_t)ceil_div(m, s.G) * 4;
  }
}

struct Copy {
  void* dst;
  const void* src;
  uint64_t bytes;
};

// The pipeline: pieces are appended to the current chunk until its slot is full, then the
// chunk is issued (copies in -> kernels -> copies out) and the next slot is taken.
template <typename Item>
class Pipeline {
 public:
  Pipeline(Engine* e, char* ws, uint64_t ws_bytes, cudaStream_t s, int32_t G,
           cudaError_t (*enqueue)(const Item*, int32_t, int32_t, cudaStream_t))
      : e_(e), ws_(ws), slot_bytes_((ws_bytes / kSlots) & ~(kAlign - 1)), s_(s), G_(G),
        piece_(piece_elems(G)), enqueue_(enqueue) {}

  cudaError_t begin() {
    cudaError_t r = cudaEventRecord(e_->start, s_);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(e_->in, e_->start, 0);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(e_->out, e_->start, 0);
    return r;
  }

  // Bytes the staged buffers of piece [off, off + m) need in a slot.
  static uint64_t need(const Buf* b, int nb, const Shape& s, int64_t m) {
    uint64_t t = 0;
    for (int i = 0; i < nb; ++i)
      if (b[i].host) t += align_up(buf_bytes(b[i].kind, s, m));
    return t;
  }

  // Adds tensor [0, n) with buffers b[0..nb); make(ptrs, off, m) builds the piece's item
  // from the four (device) pointers in b's order.
  template <typename Make>
  cudaError_t add(const Buf* b, int nb, const Shape& s, int64_t n, Make make) {
    bool any_host = false;
    for (int i = 0; i < nb; ++i) any_host = any_host || b[i].host;
    if (!any_host) {  // all device: one in-place item, no staging
      void* p[4];
      for (int i = 0; i < nb; ++i) p[i] = b[i].base;
      items_.push_back(make(p, 0, n));
      return cudaSuccess;
    }
    int64_t off = 0;
    while (off < n) {
      const uint64_t room = slot_bytes_ - used_;
      // the largest piece (whole lcm(G, 4096)-blocks, or the tensor's rest) that fits the room
      int64_t lo = 0, hi = ceil_div(n - off, piece_);
      while (lo < hi) {
        const int64_t k = (lo + hi + 1) / 2;
        const int64_t m = k * piece_ < n - off ? k * piece_ : n - off;
        if (need(b, nb, s, m) <= room) lo = k; else hi = k - 1;
      }
      if (lo == 0) {
        if (used_ == 0) return cudaErrorInvalidValue;  // cannot happen above the minimum
        cudaError_t r = flush();
        if (r != cudaSuccess) return r;
        continue;
      }
      const int64_t m = lo * piece_ < n - off ? lo * piece_ : n - off;
      char* slot = ws_ + (uint64_t)slot_ * slot_bytes_;
      void* p[4];
      for (int i = 0; i < nb; ++i) {
        const uint64_t o = buf_offset(b[i].kind, s, off), bytes = buf_bytes(b[i].kind, s, m);
        if (!b[i].host) {
          p[i] = b[i].base + o;
          continue;
        }
        p[i] = slot + used_;
        if (b[i].input) cin_.push_back(Copy{p[i], b[i].base + o, bytes});
        else cout_.push_back(Copy{b[i].base + o, p[i], bytes});
        used_ += align_up(bytes);
      }
      items_.push_back(make(p, off, m));
      off += m;
    }
    return cudaSuccess;
  }

  // Issues the current chunk on the current slot and moves to the next slot.
  cudaError_t flush() {
    if (items_.empty()) return cudaSuccess;
    const int j = slot_;
    cudaError_t r = cudaSuccess;
    if (used_slot_[j]) r = cudaStreamWaitEvent(e_->in, e_->out_done[j], 0);  // slot free again
    for (const Copy& c : cin_)
      if (r == cudaSuccess) r = cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, e_->in);
    if (r == cudaSuccess) r = cudaEventRecord(e_->in_done[j], e_->in);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(s_, e_->in_done[j], 0);
    if (r == cudaSuccess) r = enqueue_(items_.data(), (int32_t)items_.size(), G_, s_);
    if (r == cudaSuccess) r = cudaEventRecord(e_->comp_done[j], s_);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(e_->out, e_->comp_done[j], 0);
    for (const Copy& c : cout_)
      if (r == cudaSuccess) r = cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToHost, e_->out);
    if (r == cudaSuccess) r = cudaEventRecord(e_->out_done[j], e_->out);
    used_slot_[j] = true;
    items_.clear();
    cin_.clear();
    cout_.clear();
    used_ = 0;
    slot_ = (slot_ + 1) % kSlots;
    return r;
  }

  // Flushes and waits for every copy and kernel of the call.
  cudaError_t finish() {
    cudaError_t r = flush();
    const cudaError_t a = cudaStreamSynchronize(e_->out);
    const cudaError_t b = cudaStreamSynchronize(e_->in);
    const cudaError_t c = cudaStreamSynchronize(s_);
    if (r == cudaSuccess) r = a;
    if (r == cudaSuccess) r = b;
    if (r == cudaSuccess) r = c;
    return r;
  }

 private:
  Engine* e_;
  char* ws_;
  uint64_t slot_bytes_;
  cudaStream_t s_;
  int32_t G_;
  int64_t piece_;
  cudaError_t (*enqueue_)(const Item*, int32_t, int32_t, cudaStream_t);
  int slot_ = 0;
  uint64_t used_ = 0;
  bool used_slot_[kSlots] = {};
  std::vector<Item> items_;
  std::vector<Copy> cin_, cout_;
};

// Bytes one whole piece needs in a slot in the worst case (fp32, b = 8, all four buffers
// staged): the workspace must hold one per slot.
uint64_t max_piece_bytes(int32_t G) {
  const int64_t m = piece_elems(G);
  return align_up((uint64_t)m * 4) + align_up((uint64_t)m) + 2 * align_up((uint64_t)(m / G) * 4);
}

// Validation shared by both directions (the batch forms' rules plus the workspace).
gact_status check_common(const gact_tensor_desc* d, int32_t count, int32_t G, const void* ws,
                         uint64_t ws_bytes) {
  if (count < 0 || (count > 0 && !d)) return GACT_ERR_INVALID_ARG;
  for (int32_t i = 0; i < count; ++i) {
    const gact_tensor_desc& t = d[i];
    if (!(t.bits == 1 || t.bits == 2 || t.bits == 4 || t.bits == 8)) return GACT_ERR_UNSUPPORTED_BITS;
    if (t.n < 0 || t.dtype < GACT_F32 || t.dtype > GACT_F16) return GACT_ERR_INVALID_ARG;
    if (t.n == 0) continue;
    if (!t.data || !t.packed || !t.group_min || !t.group_scale) return GACT_ERR_INVALID_ARG;
    if (!aligned(t.data, 16) || !aligned(t.packed, 8) || !aligned(t.group_min, 4) ||
        !aligned(t.group_scale, 4))
      return GACT_ERR_ALIGNMENT;
  }
  if (gact::group_log2(G) < -1) return GACT_ERR_GROUP_SIZE;
  if (!ws || ws_bytes < GACT_STAGED_MIN_WORKSPACE || !aligned(ws, kAlign)) return GACT_ERR_INVALID_ARG;
  if (((ws_bytes / kSlots) & ~(kAlign - 1)) < max_piece_bytes(G)) return GACT_ERR_INVALID_ARG;
  return GACT_OK;
}

}  // namespace

extern "C" {

gact_status gact_quantize_pack_staged(const gact_tensor_desc* descs, int32_t count,
                                      int32_t group_size, void* workspace,
                                      uint64_t workspace_bytes, void* stream) {
  gact_status st = check_common(descs, count, group_size, workspace, workspace_bytes);
  if (st != GACT_OK) return st;
  Engine* e = engine_for_current_device();
  if (!e) return GACT_ERR_CUDA;
  Pipeline<gact::QItem> pipe(e, static_cast<char*>(workspace), workspace_bytes,
                             static_cast<cudaStream_t>(stream), group_size, gact::enqueue_quantize);
  cudaError_t r = pipe.begin();
  for (int32_t i = 0; i < count && r == cudaSuccess; ++i) {
    const gact_tensor_desc& d = descs[i];
    if (d.n == 0) continue;
    const Buf b[4] = {{static_cast<char*>(d.data), is_host(d.data), true, ELEMS},
                      {reinterpret_cast<char*>(d.packed), is_host(d.packed), false, WORDS},
                      {reinterpret_cast<char*>(d.group_min), is_host(d.group_min), false, GROUPS},
                      {reinterpret_cast<char*>(d.group_scale), is_host(d.group_scale), false, GROUPS}};
    const Shape s{elem_bytes(d.dtype), d.bits, group_size};
    r = pipe.add(b, 4, s, d.n, [&](void* const* p, int64_t off, int64_t m) {
      gact::QItem it;
      it.t.x = p[0];
      it.t.packed = static_cast<uint32_t*>(p[1]);
      it.t.group_min = static_cast<float*>(p[2]);
      it.t.group_scale = static_cast<float*>(p[3]);
      it.t.n = m;
      it.t.nwords = ceil_div(m * d.bits, 32);
      it.t.seed = d.seed;
      it.t.ctr0 = (uint64_t)off / 16;  // R3: off is a multiple of 512, 16 elements per block
      it.dtype = d.dtype;
      it.bits = d.bits;
      return it;
    });
  }
  const cudaError_t f = pipe.finish();
  return (r == cudaSuccess && f == cudaSuccess) ? GACT_OK : GACT_ERR_CUDA;
}

gact_status gact_unpack_dequantize_staged(const gact_tensor_desc* descs, int32_t count,
                                          int32_t group_size, void* workspace,
                                          uint64_t workspace_bytes, void* stream) {
  gact_status st = check_common(descs, count, group_size, workspace, workspace_bytes);
  if (st != GACT_OK) return st;
  Engine* e = engine_for_current_device();
  if (!e) return GACT_ERR_CUDA;
  Pipeline<gact::DItem> pipe(e, static_cast<char*>(workspace), workspace_bytes,
                             static_cast<cudaStream_t>(stream), group_size, gact::enqueue_dequantize);
  cudaError_t r = pipe.begin();
  for (int32_t i = 0; i < count && r == cudaSuccess; ++i) {
    const gact_tensor_desc& d = descs[i];
    if (d.n == 0) continue;
    const Buf b[4] = {{static_cast<char*>(d.data), is_host(d.data), false, ELEMS},
                      {reinterpret_cast<char*>(d.packed), is_host(d.packed), true, WORDS},
                      {reinterpret_cast<char*>(d.group_min), is_host(d.group_min), true, GROUPS},
                      {reinterpret_cast<char*>(d.group_scale), is_host(d.group_scale), true, GROUPS}};
    const Shape s{elem_bytes(d.dtype), d.bits, group_size};
    r = pipe.add(b, 4, s, d.n, [&](void* const* p, int64_t, int64_t m) {
      gact::DItem it;
      it.t.y = p[0];
      it.t.packed = static_cast<const uint32_t*>(p[1]);
      it.t.group_min = static_cast<const float*>(p[2]);
      it.t.group_scale = static_cast<const float*>(p[3]);
      it.t.n = m;
      it.dtype = d.dtype;
      it.bits = d.bits;
      return it;
    });
  }
  const cudaError_t f = pipe.finish();
  return (r == cudaSuccess && f == cudaSuccess) ? GACT_OK : GACT_ERR_CUDA;
}

}  // extern "C"
