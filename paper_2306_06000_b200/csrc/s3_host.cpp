// s3_host.cpp -- host control plane behind include/s3.h.
//
// Owns the request pool, the first-fit-decreasing scheduler
// (PAPER.md:164-166), the supervisor's bookkeeping (free
// capacity, eviction, doubling) and the host mirror of the slot table.  All
// device work goes to the kernels in s3_kernels.cu on cfg.stream; eviction
// D2H copies ride a side stream.  One host synchronisation per step: the
// keep-scan report readback in s3_evict_compact.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/s3.h"
#include "s3_internal.h"

using namespace s3;

namespace {

constexpr int64_t kAlign = 256;
constexpr int32_t kMaxFeedChunks = 64;    // s3_decode_step_host pipeline depth limit

// cuStreamWriteValue32 through the runtime's driver entry point (no -lcuda)
// cuStreamWriteValue32 / cuStreamWaitValue32 (same signature)
typedef int (*StreamValue32Fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
StreamValue32Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (StreamValue32Fn)p;
}
StreamValue32Fn write_value32() {
  static StreamValue32Fn fn = driver_fn("cuStreamWriteValue32");
  return fn;
}
StreamValue32Fn wait_value32() {
  static StreamValue32Fn fn = driver_fn("cuStreamWaitValue32");
  return fn;
}
constexpr unsigned kWaitGeq = 0x0;   // CU_STREAM_WAIT_VALUE_GEQ: (int32_t)(*addr - value) >= 0
inline int64_t align_up(int64_t x, int64_t a = kAlign) { return (x + a - 1) / a * a; }

// FFD order: reservation (cap) descending, then req_id ascending (R7).
struct Key {
  int64_t cap, req;
  bool operator<(const Key& o) const { return cap != o.cap ? cap > o.cap : req < o.req; }
};

struct EventBox {
  cudaEvent_t ev = nullptr;
  EventBox() { cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); }
  ~EventBox() { if (ev) cudaEventDestroy(ev); }
};

struct Item {
  int64_t req;
  int32_t prompt, gen, cap;
  int32_t evicted;          // 1: KV lives in host_store
  int64_t host_off, host_bytes;
  int32_t host_rows;
  std::shared_ptr<EventBox> ready;   // D2H completion
  const uint8_t* stage_src = nullptr;  // its rows in the eviction staging buffer, valid during
  uint64_t evict_seq = 0;              // the s3_evict_compact call that staged them
};

using Pool = std::map<Key, Item>;

// One-pass FFD with skip-and-continue, implemented as "repeatedly take the
// first item in FFD order that fits": an item skipped once never fits later
// because free capacity only shrinks.  fits(cap) -> bin index or -1;
// max_fit() -> the largest cap any bin can take now.
template <class MaxFit, class Fit, class Take>
int64_t ffd_scan(Pool& pool, MaxFit max_fit, Fit fit, Take take) {
  int64_t count = 0;
  for (;;) {
    const int64_t mf = max_fit();
    if (mf <= 0) break;
    auto it = pool.lower_bound(Key{mf, INT64_MIN});
    if (it == pool.end()) break;
    const int bin = fit(it->first.cap);
    if (bin < 0) break;   // cannot happen: max_fit bounds it
    Item item = it->second;
    pool.erase(it);
    take(bin, item);
    ++count;
  }
  return count;
}

// Multi-bin placement (R26): the rank with the most free rows among
// the ranks with a free slot (ties: lowest rank), or -1 if the item does not
// fit there.  Worst fit spreads the freed rows evenly, so the lockstep step --
// as long as the busiest rank's attention pass -- stays balanced.
int worst_fit(int world, const int64_t* free_rows, const int64_t* free_slots, int64_t cap) {
  int best = -1;
  for (int r = 0; r < world; ++r)
    if (free_slots[r] > 0 && (best < 0 || free_rows[r] > free_rows[best])) best = r;
  return best >= 0 && cap <= free_rows[best] ? best : -1;
}

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> free_events;
  struct Pending { cudaEvent_t a, b; double bytes; int kind; };
  std::vector<Pending> pending;
  int64_t attn_launches = 0, move_launches = 0, fused_steps = 0, d2h_copies = 0, h2d_copies = 0, prep_launches = 0;
  double attn_ms = 0, move_ms = 0, attn_bytes = 0, move_bytes = 0, fused_move_bytes = 0, prep_ms = 0;
  double d2h_ms = 0, d2h_bytes = 0, h2d_ms = 0, h2d_bytes = 0;
  // absolute intervals (ms after `ref`) of attention launches and eviction copies, for the
  // overlap evidence: how much of the side-stream D2H ran while an attention kernel ran
  cudaEvent_t ref = nullptr;
  std::vector<std::pair<double, double>> attn_iv, d2h_iv;
  cudaEvent_t get() {
    if (!free_events.empty()) { cudaEvent_t e = free_events.back(); free_events.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

}  // namespace

struct s3_ctx {
  s3_config cfg{};
  Shape sh{};
  int32_t C = 512;
  int64_t S = 32768;
  s3_buffers buf{};
  cudaStream_t st = nullptr, side = nullptr;
  int num_sms = 148;
  int grid_attn = 148, grid_combine = 592, grid_move = 592;
  // device carve
  DSlot* slots[2] = {nullptr, nullptr};
  int cur = 0;
  Unit* units = nullptr;
  Split* splits = nullptr;
  float* partials = nullptr;
  int32_t* ctrl = nullptr;
  int64_t* ctrl64 = nullptr;
  MoveEntry* entries = nullptr;
  int32_t* key_chunk0 = nullptr;
  int32_t* key_src = nullptr;
  DepDesc* desc = nullptr;
  unsigned long long* progress = nullptr;
  uint32_t attn_epoch = 0;
  bool fused_pending = false;   // the pending statuses came from a fused decode step
  uint32_t* flags = nullptr;
  uint8_t* report_dev = nullptr;
  unsigned long long* verify_count = nullptr;
  // host-fed steps (s3_decode_step_host): copy stream, per-chunk ready words
  uint32_t* ready = nullptr;
  uint32_t* done = nullptr;                 // per-chunk finished-warp counters (device out + CE D2H)
  uint32_t* evdone = nullptr;               // per-evictee staged-row counters (fused eviction D2H)
  std::vector<uint32_t> ev_target;          // their cumulative targets
  uint8_t* prep_scratch = nullptr;          // multi-CTA k_prep: totals, flags, header partials, done counter
  uint32_t prep_epoch = 0;
  uint32_t done_target[kMaxFeedChunks] = {};  // cumulative values the D2H stream waits for
  cudaStream_t hio = nullptr, d2h = nullptr;
  cudaEvent_t ev_hio_start = nullptr, ev_hio_done = nullptr, ev_comb = nullptr, ev_d2h_done = nullptr;
  uint32_t feed_epoch = 0;
  Feed feed;                    // set only for the duration of a host-fed decode call
  // pinned host
  uint8_t* h_report = nullptr;
  uint8_t* h_report_dev = nullptr;          // the same pinned buffer as seen by kernels (UVA mapping)
  uint8_t* h_upload = nullptr;
  int64_t upload_cap = 0, upload_used = 0;
  // host mirror (arena order)
  std::vector<DSlot> slots_h;
  int64_t tail = 0;
  // pools
  Pool pool;        // world == 1: everything; world > 1: the shared fresh pool
  Pool home;        // world > 1: this rank's evicted requests
  std::unordered_set<int64_t> live;   // req ids queued, running or evicted (not yet finished)
  std::unordered_map<int64_t, std::shared_ptr<EventBox>> evict_done;   // req -> its eviction D2H's completion
  int64_t n_evicted_waiting = 0;
  // host store allocator (first fit) + deferred frees
  std::map<int64_t, int64_t> free_blocks;
  struct Deferred { int64_t off, bytes; std::shared_ptr<EventBox> done; };
  std::vector<Deferred> deferred_free;      // host-store ranges freed once their reload H2D completed
  cudaEvent_t ev_report = nullptr;          // after the fused step's report readback
  // eviction staging, double-buffered when it holds two maximal evictions: a step's
  // evictees go to one half while the other half's D2H (previous step) is still running
  bool stage_dbl = false;
  int stage_next = 0, stage_cur = 0;
  std::shared_ptr<EventBox> stage_d2h[2];
  // state
  bool status_pending = false;
  uint64_t evict_seq = 0;       // s3_evict_compact calls (staging of the current call is reusable)
  uint32_t epoch = 0;
  int64_t finished_total = 0, evicted_total = 0, tokens_total = 0;
  int64_t launches = 0;     // kernels launched by this context
  bool poisoned = false;
  const char* err = "ok";
  Prof prof;
  // (a8) library-owned NCCL communicator for the per-step counter all-reduce
  ncclComm_t comm = nullptr;
  cudaStream_t xs = nullptr;                // its stream (highest priority, non-blocking)
  int64_t* x_dev = nullptr;                 // [world][S3_NCOUNTERS] device matrix
  int64_t* x_host = nullptr;                // pinned staging of the same
  std::vector<int64_t> x_last;              // the last exchanged matrix
  int32_t exchanges = 0;
};

namespace {

s3_status fail(s3_ctx* c, s3_status s, const char* msg) {
  if (c) {
    c->err = msg;
    if (s == S3_E_CUDA || s == S3_E_NCCL) c->poisoned = true;
  }
  return s;
}

// NCCL, resolved at run time: the library loads without it, and in a torch process
// "libnccl.so.2" is torch's already-loaded copy
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
};
const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy;
    return a;
  }();
  return api;
}
static_assert(sizeof(ncclUniqueId) == S3_NCCL_ID_BYTES, "ncclUniqueId size");

#define CK(expr, msg)                                             \
  do {                                                            \
    cudaError_t e__ = (expr);                                     \
    if (e__ != cudaSuccess) return fail(ctx, S3_E_CUDA, msg);     \
  } while (0)

bool validate(const s3_config* c) {
  if (!c) return false;
  if (c->num_layers < 1 || c->num_heads < 1) return false;
  if (c->head_dim != 64 && c->head_dim != 128 && c->head_dim != 256) return false;
  if ((int64_t)c->num_heads * c->head_dim > 4096) return false;   // <= 16 head warps per attention CTA
  if (c->num_kv_heads < 0 || (c->num_kv_heads > 0 && c->num_heads % c->num_kv_heads)) return false;
  if (c->max_seq_len < 1 || c->arena_rows < c->max_seq_len) return false;
  if (c->arena_rows > INT32_MAX) return false;
  if (c->max_running < 1 || c->max_running > 65535) return false;
  if (c->chunk_rows < 0 || c->chunk_rows > 32768 || c->move_chunk_bytes < 0 || c->move_chunk_bytes % 16) return false;
  if (c->move_chunk_bytes > 0 && (c->move_chunk_bytes < 1024 || c->move_chunk_bytes > 36864)) return false;
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return false;
  if (c->attn_variant < 0 || c->attn_variant > 2) return false;
  if (c->compact_mode < 0 || c->compact_mode > 1) return false;
  if (c->compact_policy < 0 || c->compact_policy > 1) return false;
  if (c->reserve_sms < -1 || c->reserve_sms > 64) return false;
  return true;
}

Shape make_shape(const s3_config* c) {
  Shape s;
  s.L = c->num_layers; s.H = c->num_heads; s.D = c->head_dim; s.max_len = c->max_seq_len;
  s.Hkv = c->num_kv_heads > 0 ? c->num_kv_heads : c->num_heads;
  s.pad = 0;
  s.row_elems = 2LL * s.L * s.Hkv * s.D;
  s.kvpt = 4LL * s.L * s.Hkv * s.D;
  return s;
}

struct Carve {
  int64_t slots, units, splits, partials, ctrl, ctrl64, entries, keys, desc, progress, flags, report, verify, ready,
      done, evdone, prep, total;
};

Carve carve(const s3_config* c) {
  const Shape sh = make_shape(c);
  const int64_t C = c->chunk_rows ? c->chunk_rows : 512;
  const int64_t S = c->move_chunk_bytes ? c->move_chunk_bytes : 32768;
  const int64_t R = c->arena_rows, Bm = c->max_running;
  const int64_t units_max = R / C + Bm + 2;
  const int64_t parts_max = 2 * (R / C) + 2;
  const int64_t flags_max = (R * sh.kvpt) / S + Bm + 2;
  Carve k;
  int64_t o = 0;
  k.slots = o;    o += align_up(2 * Bm * (int64_t)sizeof(DSlot));
  k.units = o;    o += align_up(units_max * (int64_t)sizeof(Unit));
  k.splits = o;   o += align_up(Bm * (int64_t)sizeof(Split));
  k.partials = o; o += align_up(parts_max * sh.L * sh.H * (int64_t)(sh.D + 4) * 4);
  k.ctrl = o;     o += align_up(CTRL_WORDS * 4);
  k.ctrl64 = o;   o += align_up(CTRL64_WORDS * 8);
  k.entries = o;  o += align_up((Bm + 1) * (int64_t)sizeof(MoveEntry));
  k.keys = o;     o += align_up(2 * (Bm + 2) * 4);
  k.desc = o;     o += align_up((R / AT_RPS + units_max + 2) * (int64_t)sizeof(DepDesc));
  k.progress = o; o += align_up(units_max * sh.L * 8);
  k.flags = o;    o += align_up(flags_max * 4);
  k.report = o;   o += align_up(report_bytes((int32_t)Bm));
  k.verify = o;   o += align_up(8);
  k.ready = o;    o += align_up(kMaxFeedChunks * 4);
  k.done = o;     o += align_up(kMaxFeedChunks * 4);
  k.evdone = o;   o += align_up(Bm * 4);
  k.prep = o;     o += align_up(PREP_MAX_CTAS * (PREP_NX + 1 + 4) * 8 + 8);
  k.total = o;
  return k;
}

// ---- host store allocator -------------------------------------------------
int64_t hs_alloc(s3_ctx* c, int64_t n) {
  n = align_up(n);
  for (auto it = c->free_blocks.begin(); it != c->free_blocks.end(); ++it) {
    if (it->second >= n) {
      const int64_t off = it->first, sz = it->second;
      c->free_blocks.erase(it);
      if (sz > n) c->free_blocks[off + n] = sz - n;
      return off;
    }
  }
  return -1;
}

void hs_free(s3_ctx* c, int64_t off, int64_t n) {
  n = align_up(n);
  auto it = c->free_blocks.emplace(off, n).first;
  auto nx = std::next(it);
  if (nx != c->free_blocks.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    c->free_blocks.erase(nx);
  }
  if (it != c->free_blocks.begin()) {
    auto pv = std::prev(it);
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      c->free_blocks.erase(it);
    }
  }
}

void flush_deferred(s3_ctx* c) {   // free host-store ranges whose reload copy has completed
  std::vector<s3_ctx::Deferred> keep;
  for (auto& d : c->deferred_free) {
    if (d.done && cudaEventQuery(d.done->ev) != cudaSuccess) { keep.push_back(d); continue; }
    hs_free(c, d.off, d.bytes);
  }
  c->deferred_free.swap(keep);
}

void prof_collect(s3_ctx* c) {     // call when cfg.stream is idle; side-stream pairs may still run
  std::vector<Prof::Pending> keep;
  for (auto& p : c->prof.pending) {
    if (cudaEventQuery(p.b) != cudaSuccess) { keep.push_back(p); continue; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    if (c->prof.ref && (p.kind == 0 || p.kind == 2)) {
      float t0 = 0.f, t1 = 0.f;
      if (cudaEventElapsedTime(&t0, c->prof.ref, p.a) == cudaSuccess &&
          cudaEventElapsedTime(&t1, c->prof.ref, p.b) == cudaSuccess)
        (p.kind == 0 ? c->prof.attn_iv : c->prof.d2h_iv).emplace_back(t0, t1);
      else
        cudaGetLastError();
    }
    if (p.kind == 0) { c->prof.attn_ms += ms; c->prof.attn_bytes += p.bytes; c->prof.attn_launches++; }
    else if (p.kind == 1) { c->prof.move_ms += ms; c->prof.move_bytes += p.bytes; c->prof.move_launches++; }
    else if (p.kind == 2) { c->prof.d2h_ms += ms; c->prof.d2h_bytes += p.bytes; c->prof.d2h_copies++; }
    else if (p.kind == 4) { c->prof.prep_ms += ms; c->prof.prep_launches++; }
    else { c->prof.h2d_ms += ms; c->prof.h2d_bytes += p.bytes; c->prof.h2d_copies++; }
    c->prof.free_events.push_back(p.a);
    c->prof.free_events.push_back(p.b);
  }
  c->prof.pending.swap(keep);
}

uint8_t* upload_reserve(s3_ctx* c, int64_t n) {
  n = align_up(n, 64);
  if (c->upload_used + n > c->upload_cap) {
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return nullptr;
    c->upload_used = 0;
  }
  uint8_t* p = c->h_upload + c->upload_used;
  c->upload_used += n;
  return p;
}

// Place admitted items at the tail (appended in scan order, R9):
// fresh -> prompt rows by k_fill; evicted -> H2D reload after its D2H event.
s3_status place_items(s3_ctx* ctx, const std::vector<Item>& items, s3_admit_report* rep,
                      int64_t* admitted_ids) {
  s3_admit_report r{};
  if (!items.empty()) {
    const int32_t B0 = (int32_t)ctx->slots_h.size();
    const int32_t n = (int32_t)items.size();
    uint8_t* up = upload_reserve(ctx, (int64_t)n * sizeof(DSlot) + (int64_t)n * 4 + 64);
    if (!up) return fail(ctx, S3_E_CUDA, "upload sync failed");
    DSlot* rec = reinterpret_cast<DSlot*>(up);
    int32_t* fill = reinterpret_cast<int32_t*>(up + align_up((int64_t)n * sizeof(DSlot), 64));
    int32_t n_fill = 0, max_prompt = 0;
    for (int32_t i = 0; i < n; ++i) {
      const Item& it = items[i];
      DSlot s;
      s.req = it.req; s.prompt = it.prompt; s.cap = it.cap; s.off = (int32_t)ctx->tail; s.status = 0;
      if (it.evicted) {
        s.gen = it.gen;
        s.len = it.host_rows;
        ctx->evict_done.erase(it.req);   // re-admitted: its host copy is no longer waited for
        uint8_t* dst = (uint8_t*)ctx->buf.arena + (int64_t)s.off * ctx->sh.kvpt;
        if (it.stage_src && it.evict_seq == ctx->evict_seq) {
          // re-admitted in the step that evicted it (R10): its rows are still in the
          // staging buffer (stream-ordered after the attention pass that staged them),
          // so the reload is an HBM copy and PCIe stays off the critical path; the host
          // copy is made all the same (the eviction D2H is already queued)
          CK(cudaMemcpyAsync(dst, it.stage_src, it.host_bytes, cudaMemcpyDeviceToDevice, ctx->st), "reload D2D");
          r.stage_reload_bytes += it.host_bytes;
        } else {
          CK(cudaStreamWaitEvent(ctx->st, it.ready->ev, 0), "wait D2H event");
          cudaEvent_t e0 = nullptr, e1 = nullptr;
          if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->st); }
          CK(cudaMemcpyAsync(dst, (uint8_t*)ctx->buf.host_store + it.host_off, it.host_bytes,
                             cudaMemcpyHostToDevice, ctx->st), "reload H2D");
          if (ctx->prof.on) {
            cudaEventRecord(e1, ctx->st);
            ctx->prof.pending.push_back({e0, e1, (double)it.host_bytes, 3});
          }
          r.h2d_bytes += it.host_bytes;
        }
        ctx->deferred_free.push_back({it.host_off, it.host_bytes, nullptr});
        ctx->n_evicted_waiting--;
        r.n_reloaded++;
      } else {
        s.gen = 0;
        s.len = it.prompt;
        fill[n_fill++] = B0 + i;
        max_prompt = std::max(max_prompt, it.prompt);
        r.n_fresh++;
        r.fill_bytes += (int64_t)it.prompt * ctx->sh.kvpt;
      }
      rec[i] = s;
      ctx->slots_h.push_back(s);
      ctx->tail += it.cap;
      if (admitted_ids) admitted_ids[i] = it.req;
    }
    if (r.n_reloaded) {              // the reloads' host ranges may be reused once this event fires
      auto done = std::make_shared<EventBox>();
      CK(cudaEventRecord(done->ev, ctx->st), "event");
      for (auto& d : ctx->deferred_free)
        if (!d.done) d.done = done;
    }
    DSlot* dst = ctx->slots[ctx->cur] + B0;
    CK(cudaMemcpyAsync(dst, rec, (size_t)n * sizeof(DSlot), cudaMemcpyHostToDevice, ctx->st), "slot upload");
    if (n_fill) {
      int32_t* dfill = reinterpret_cast<int32_t*>(ctx->units);   // units are rebuilt every decode step
      CK(cudaMemcpyAsync(dfill, fill, (size_t)n_fill * 4, cudaMemcpyHostToDevice, ctx->st), "fill upload");
      CK(launch_fill(ctx->sh, ctx->cfg.synth_seed, ctx->slots[ctx->cur], dfill, n_fill, max_prompt,
                     (uint16_t*)ctx->buf.arena, ctx->st), "k_fill");
      ctx->launches += 1;
    }
    r.n_admitted = n;
  }
  r.n_batch = (int32_t)ctx->slots_h.size();
  r.tail_rows = ctx->tail;
  if (rep) *rep = r;
  return S3_OK;
}

s3_status check_ctx(s3_ctx* ctx) {
  if (!ctx) return S3_E_INVAL;
  if (ctx->poisoned) return S3_E_CUDA;
  return S3_OK;
}

int64_t stage_bytes(const s3_ctx* c) {
  if (!c->buf.staging) return 0;
  return c->stage_dbl ? c->buf.staging_bytes / 2 / 256 * 256 : c->buf.staging_bytes;
}
uint8_t* stage_ptr(const s3_ctx* c, int half) {
  return (uint8_t*)c->buf.staging + (c->stage_dbl ? (int64_t)half * stage_bytes(c) : 0);
}

// Per-evictee staged-row counters: the fused attention kernels count each
// evictee's rows as they become final in staging, and the eviction D2H of
// that evictee waits for its count (cuStreamWaitValue32) instead of for the
// end of the attention pass.  Needs the stream memory operations.
uint32_t* ev_counters(const s3_ctx* c) { return wait_value32() ? c->evdone : nullptr; }

// R27 at admission: under the on-demand policy a step whose pool was empty left
// its holes in place; when requests wait again (a later s3_submit), shift the
// survivors up before the FFD so it sees the free rows of the every-step
// policy.  A keep-scan with every slot RUNNING and the ordered k_move.
s3_status compact_holes(s3_ctx* ctx, int64_t* moved) {
  *moved = 0;
  const int32_t B = (int32_t)ctx->slots_h.size();
  int64_t sum_cap = 0;
  for (const DSlot& sl : ctx->slots_h) sum_cap += sl.cap;
  if (sum_cap == ctx->tail) return S3_OK;        // no holes
  const Shape& sh = ctx->sh;
  CK(launch_keep_scan(sh, ctx->slots[ctx->cur], ctx->slots[1 - ctx->cur], B, ctx->S, ctx->report_dev, ctx->entries,
                      ctx->key_chunk0, ctx->key_src, ctx->ctrl64, 0, 1, ctx->st), "k_keep_scan");
  ctx->launches += 1;
  CK(cudaMemcpyAsync(ctx->h_report, ctx->report_dev, (size_t)report_bytes(B), cudaMemcpyDeviceToHost, ctx->st),
     "report D2H");
  CK(cudaStreamSynchronize(ctx->st), "report sync");
  const DReportHeader* h = reinterpret_cast<const DReportHeader*>(ctx->h_report);
  if (h->n_before != B || h->n_kept != B || h->tail != sum_cap)
    return fail(ctx, S3_E_CUDA, "admit: inconsistent compaction report");
  if (h->n_chunks > 0) {
    ctx->epoch++;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->st); }
    const int grid = (int)std::min<int64_t>((h->n_chunks + 2 * 3 - 1) / (2 * 3), ctx->grid_move);
    CK(launch_move((uint8_t*)ctx->buf.arena, (uint8_t*)ctx->buf.staging, ctx->entries, ctx->key_chunk0,
                   ctx->key_src, h->n_entries, h->n_chunks, ctx->S, sh.kvpt, ctx->ctrl64, ctx->flags, ctx->epoch, 0,
                   grid, ctx->st), "k_move");
    ctx->launches += 1;
    if (ctx->prof.on) {
      cudaEventRecord(e1, ctx->st);
      ctx->prof.pending.push_back({e0, e1, 2.0 * (double)h->moved_bytes, 1});
    }
  }
  int64_t run = 0;
  for (DSlot& sl : ctx->slots_h) { sl.off = (int32_t)run; run += sl.cap; }
  ctx->tail = run;
  ctx->cur = 1 - ctx->cur;
  *moved = h->moved_bytes;
  return S3_OK;
}

}  // namespace

// ===========================================================================
// ABI
// ===========================================================================
extern "C" {

s3_status s3_workspace_query(const s3_config* cfg, int64_t* arena_b, int64_t* ws_b, int64_t* staging_min,
                             int64_t* host_min) {
  if (!validate(cfg)) return S3_E_INVAL;
  const Shape sh = make_shape(cfg);
  // + 8 guard rows: the tensor-core kernel loads whole 8-row groups, up to 7 rows past a slot's end
  if (arena_b) *arena_b = (cfg->arena_rows + 8) * sh.kvpt;
  if (ws_b) *ws_b = carve(cfg).total;
  if (staging_min) *staging_min = (int64_t)cfg->max_seq_len * sh.kvpt;
  if (host_min) *host_min = align_up((int64_t)cfg->max_seq_len * sh.kvpt);
  return S3_OK;
}

s3_status s3_kv_init(const s3_config* cfg, const s3_buffers* b, s3_ctx** out) {
  if (!out || !b || !validate(cfg)) return S3_E_INVAL;
  *out = nullptr;
  const Shape sh = make_shape(cfg);
  const Carve k = carve(cfg);
  if (!b->arena || b->arena_bytes < (cfg->arena_rows + 8) * sh.kvpt) return S3_E_NOMEM;
  if (!b->workspace || b->workspace_bytes < k.total) return S3_E_NOMEM;
  if (((uintptr_t)b->arena | (uintptr_t)b->workspace) % kAlign) return S3_E_INVAL;
  if (b->staging && ((uintptr_t)b->staging % 16)) return S3_E_INVAL;
  if (!b->host_store || b->host_store_bytes < 1) return S3_E_NOMEM;
  s3_ctx* ctx = new (std::nothrow) s3_ctx();
  if (!ctx) return S3_E_NOMEM;
  ctx->cfg = *cfg;
  ctx->sh = sh;
  ctx->C = cfg->chunk_rows ? cfg->chunk_rows : 512;
  ctx->S = cfg->move_chunk_bytes ? cfg->move_chunk_bytes : 32768;
  ctx->buf = *b;
  ctx->st = (cudaStream_t)cfg->stream;
  auto bail = [&](const char* m) { ctx->err = m; s3_kv_destroy(ctx); return S3_E_CUDA; };
  if (cudaSetDevice(cfg->device) != cudaSuccess) return bail("cudaSetDevice");
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess) return bail("side stream");
  if (cudaEventCreateWithFlags(&ctx->ev_report, cudaEventDisableTiming) != cudaSuccess) return bail("event");
  int dev = cfg->device;
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev);
  int occ = 1;
  const void* ka = attn_kernel_ptr(sh);
  if (!ka) return bail("head_dim");
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ka, attn_block_threads(sh), 0);
  ctx->grid_attn = ctx->num_sms * std::max(1, occ);
  if (cfg->attn_variant == 2) {
    if (!attn_tc_supported(sh)) return bail("attn_variant 2 needs head_dim 128 and 2..16 query heads per KV head");
    for (int nc : {8, 16})
      for (bool pack : {false, true})
        for (bool feed : {false, true})
          for (bool r33 : {false, true})
            if (cudaFuncSetAttribute(attn_tc_kernel_ptr(nc, pack, feed, r33),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, attn_tc_smem(nc)) != cudaSuccess)
              return bail("attn_tc smem attribute");
    ctx->grid_attn = ctx->num_sms;
  }
  if (cfg->attn_variant == 0 && attn_tma_stages(sh) >= 2) {
    const int smem = attn_tma_smem(sh, attn_tma_stages(sh));
    if (cudaFuncSetAttribute(attn_tma_kernel_ptr(sh), cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return bail("attn smem attribute");
    int occ2 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, attn_tma_kernel_ptr(sh), attn_block_threads(sh) + 64, smem);
    ctx->grid_attn = ctx->num_sms * std::max(1, occ2);
  }
  // persistent attention grids leave `reserve` SMs free for other streams' kernels (the
  // multi-GPU counter all-reduce must not queue behind the whole attention pass)
  {
    const int reserve = cfg->reserve_sms > 0 ? cfg->reserve_sms : (cfg->reserve_sms == 0 && cfg->world > 1 ? 4 : 0);
    const int per_sm = std::max(1, ctx->grid_attn / ctx->num_sms);
    if (reserve >= ctx->num_sms / 2) return bail("reserve_sms too large");
    ctx->grid_attn = (ctx->num_sms - reserve) * per_sm;
  }
  ctx->grid_combine = ctx->num_sms * 4;
  cudaFuncSetAttribute(move_kernel_ptr(), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  ctx->grid_move = ctx->num_sms;   // one CTA per SM (its buffers fill most of shared memory)
  uint8_t* ws = (uint8_t*)b->workspace;
  ctx->slots[0] = reinterpret_cast<DSlot*>(ws + k.slots);
  ctx->slots[1] = ctx->slots[0] + cfg->max_running;
  ctx->units = reinterpret_cast<Unit*>(ws + k.units);
  ctx->splits = reinterpret_cast<Split*>(ws + k.splits);
  ctx->partials = reinterpret_cast<float*>(ws + k.partials);
  ctx->ctrl = reinterpret_cast<int32_t*>(ws + k.ctrl);
  ctx->ctrl64 = reinterpret_cast<int64_t*>(ws + k.ctrl64);
  ctx->entries = reinterpret_cast<MoveEntry*>(ws + k.entries);
  ctx->key_chunk0 = reinterpret_cast<int32_t*>(ws + k.keys);
  ctx->key_src = ctx->key_chunk0 + (cfg->max_running + 2);
  ctx->desc = reinterpret_cast<DepDesc*>(ws + k.desc);
  ctx->progress = reinterpret_cast<unsigned long long*>(ws + k.progress);
  ctx->flags = reinterpret_cast<uint32_t*>(ws + k.flags);
  ctx->report_dev = ws + k.report;
  ctx->verify_count = reinterpret_cast<unsigned long long*>(ws + k.verify);
  ctx->ready = reinterpret_cast<uint32_t*>(ws + k.ready);
  ctx->done = reinterpret_cast<uint32_t*>(ws + k.done);
  ctx->evdone = reinterpret_cast<uint32_t*>(ws + k.evdone);
  ctx->prep_scratch = ws + k.prep;
  ctx->ev_target.assign((size_t)cfg->max_running, 0u);
  if (cudaMemsetAsync(ws + k.ready, 0, (size_t)(k.total - k.ready), ctx->st) != cudaSuccess) return bail("memset");
  if (cudaMemsetAsync(ws + k.ctrl, 0, CTRL_WORDS * 4, ctx->st) != cudaSuccess) return bail("memset");
  if (cudaMemsetAsync(ws + k.flags, 0, (size_t)(k.report - k.flags), ctx->st) != cudaSuccess) return bail("memset");
  if (cudaMemsetAsync(ws + k.progress, 0, (size_t)(k.flags - k.progress), ctx->st) != cudaSuccess) return bail("memset");
  const int64_t rb = report_bytes(cfg->max_running) + 64;
  if (cudaHostAlloc((void**)&ctx->h_report, (size_t)rb, cudaHostAllocMapped) != cudaSuccess) return bail("pinned");
  if (cudaHostGetDevicePointer((void**)&ctx->h_report_dev, ctx->h_report, 0) != cudaSuccess) return bail("mapped");
  ctx->upload_cap = align_up(4 * ((int64_t)cfg->max_running * (sizeof(DSlot) + 4) + 4096));
  if (cudaHostAlloc((void**)&ctx->h_upload, (size_t)ctx->upload_cap, cudaHostAllocDefault) != cudaSuccess)
    return bail("pinned");
  ctx->free_blocks[0] = b->host_store_bytes / kAlign * kAlign;
  ctx->stage_dbl = b->staging && b->staging_bytes / 2 / 256 * 256 >= (int64_t)cfg->max_seq_len * sh.kvpt;
  if (cudaStreamSynchronize(ctx->st) != cudaSuccess) return bail("sync");
  *out = ctx;
  return S3_OK;
}

s3_status s3_kv_destroy(s3_ctx* ctx) {
  if (!ctx) return S3_E_INVAL;
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  ctx->pool.clear();
  ctx->home.clear();
  ctx->stage_d2h[0].reset();
  ctx->stage_d2h[1].reset();
  for (auto& p : ctx->prof.pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : ctx->prof.free_events) cudaEventDestroy(e);
  ctx->deferred_free.clear();
  if (ctx->prof.ref) cudaEventDestroy(ctx->prof.ref);
  if (ctx->ev_report) cudaEventDestroy(ctx->ev_report);
  if (ctx->hio) { cudaStreamSynchronize(ctx->hio); cudaStreamDestroy(ctx->hio); }
  if (ctx->d2h) { cudaStreamSynchronize(ctx->d2h); cudaStreamDestroy(ctx->d2h); }
  if (ctx->ev_comb) cudaEventDestroy(ctx->ev_comb);
  if (ctx->ev_d2h_done) cudaEventDestroy(ctx->ev_d2h_done);
  if (ctx->ev_hio_start) cudaEventDestroy(ctx->ev_hio_start);
  if (ctx->ev_hio_done) cudaEventDestroy(ctx->ev_hio_done);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->h_report) cudaFreeHost(ctx->h_report);
  if (ctx->h_upload) cudaFreeHost(ctx->h_upload);
  if (ctx->comm) nccl_api().comm_destroy(ctx->comm);
  if (ctx->xs) { cudaStreamSynchronize(ctx->xs); cudaStreamDestroy(ctx->xs); }
  if (ctx->x_dev) cudaFree(ctx->x_dev);
  if (ctx->x_host) cudaFreeHost(ctx->x_host);
  delete ctx;
  return S3_OK;
}

const char* s3_last_error(const s3_ctx* ctx) { return ctx ? ctx->err : "null context"; }

s3_status s3_submit(s3_ctx* ctx, const s3_request* reqs, int32_t n) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (n < 0 || (n > 0 && !reqs)) return fail(ctx, S3_E_INVAL, "submit: bad arguments");
  for (int32_t i = 0; i < n; ++i) {
    const s3_request& r = reqs[i];
    if (r.prompt_len < 0 || r.alloc_out < 1 || (int64_t)r.prompt_len + r.alloc_out > ctx->cfg.max_seq_len)
      return fail(ctx, S3_E_INVAL, "submit: bad request");
    if ((int64_t)r.prompt_len + r.alloc_out > ctx->cfg.arena_rows)
      return fail(ctx, S3_E_UNSCHEDULABLE, "submit: reservation larger than the arena");
  }
  {  // a req id may be live only once: not already queued / running / evicted, not twice in this call
    std::unordered_set<int64_t> seen;
    seen.reserve((size_t)n);
    for (int32_t i = 0; i < n; ++i)
      if (ctx->live.count(reqs[i].req_id) || !seen.insert(reqs[i].req_id).second)
        return fail(ctx, S3_E_INVAL, "submit: duplicate request id");
  }
  for (int32_t i = 0; i < n; ++i) {
    const s3_request& r = reqs[i];
    Item it{};
    it.req = r.req_id; it.prompt = r.prompt_len; it.gen = 0; it.cap = r.prompt_len + r.alloc_out;
    it.evicted = 0; it.host_off = -1;
    ctx->pool.emplace(Key{it.cap, it.req}, it);
    ctx->live.insert(it.req);
  }
  return S3_OK;
}

s3_status s3_decode_step(s3_ctx* ctx, int32_t l0, int32_t nl, const void* q, const void* k_new,
                         const void* v_new, const uint8_t* eos, float* out) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (ctx->status_pending) return fail(ctx, S3_E_STATE, "decode_step: statuses not consumed");
  if (l0 < 0 || nl < 1 || l0 + nl > ctx->sh.L) return fail(ctx, S3_E_INVAL, "decode_step: layer range");
  const bool finalize = (l0 + nl == ctx->sh.L);
  const int32_t B = (int32_t)ctx->slots_h.size();
  if (l0 == 0)   // the append row off+len must lie inside the slot (R28 stops sequences at max_len)
    for (const DSlot& s : ctx->slots_h)
      if (s.len >= s.cap) return fail(ctx, S3_E_STATE, "decode_step: a slot has no free row (len >= cap)");
  // fuse the row shift into this attention pass when the step is whole
  const bool fuse = finalize && l0 == 0 && ctx->cfg.compact_mode == 0 && B > 0 &&
                    ((ctx->cfg.attn_variant == 0 && attn_tma_stages(ctx->sh) >= 2) || ctx->cfg.attn_variant == 2);
  if (B > 0) {
    if (!q || !k_new || !v_new || !out || (finalize && !eos)) return fail(ctx, S3_E_INVAL, "decode_step: null");
    if (fuse) {
      // this step's evictees go to staging half `stage_next`: the D2H that last read it must be done
      ctx->stage_cur = ctx->stage_next;
      if (ctx->stage_d2h[ctx->stage_cur])
        CK(cudaStreamWaitEvent(ctx->st, ctx->stage_d2h[ctx->stage_cur]->ev, 0), "wait staging");
    }
    if (ctx->cfg.attn_variant == 2 && !ctx->feed.ready) {   // the tensor-core kernel reads the new row from the arena
      CK(launch_append(ctx->sh, ctx->slots[ctx->cur], B, l0, nl, (const uint16_t*)k_new, (const uint16_t*)v_new,
                       (uint16_t*)ctx->buf.arena, ctx->st), "k_append");
      ctx->launches += 1;
    }
    PrepArgs pa;
    pa.sh = ctx->sh; pa.slots = ctx->slots[ctx->cur]; pa.next = ctx->slots[1 - ctx->cur]; pa.B = B; pa.C = ctx->C;
    pa.eos = eos; pa.finalize = finalize ? 1 : 0; pa.fuse = fuse ? 1 : 0;
    pa.compact_policy = ctx->cfg.compact_policy;
    pa.pool_nonempty = (ctx->pool.size() + ctx->home.size()) > 0 ? 1 : 0;
    // fuse the evictions only when their rows also fit the host store: the largest free
    // block takes every evictee, so s3_evict_compact cannot run out of host store after
    // the kernel has already moved them out of the arena
    flush_deferred(ctx);
    int64_t largest = 0;
    for (const auto& fb : ctx->free_blocks) largest = std::max(largest, fb.second);
    pa.staging_bytes = std::min(stage_bytes(ctx), largest);
    pa.units = ctx->units; pa.splits = ctx->splits; pa.ctrl = ctx->ctrl;
    pa.xagg = reinterpret_cast<long long*>(ctx->prep_scratch);
    pa.xflag = reinterpret_cast<unsigned long long*>(pa.xagg + PREP_MAX_CTAS * PREP_NX);
    pa.xpart = reinterpret_cast<long long*>(pa.xflag + PREP_MAX_CTAS);
    pa.xdone = reinterpret_cast<int32_t*>(pa.xpart + PREP_MAX_CTAS * 4);
    pa.epoch = ++ctx->prep_epoch;
    // fused: k_prep writes the keep-scan report straight into pinned host memory, so the
    // host's eviction bookkeeping and FFD start as soon as k_prep ends (overlapping the
    // attention kernel) and no copy engine is involved -- a report copy would queue
    // behind the previous step's eviction D2H on the copy engine and hold up attention
    static const int devrep = [] { const char* e = getenv("S3_PREP_DEVREPORT"); return e ? atoi(e) : 0; }();  // A/B
    pa.report = fuse && !devrep ? ctx->h_report_dev : ctx->report_dev;
    pa.fused_out = fuse ? reinterpret_cast<int32_t*>(ctx->h_report_dev + report_bytes(B)) : nullptr;
    cudaEvent_t p0 = nullptr, p1 = nullptr;
    if (ctx->prof.on) { p0 = ctx->prof.get(); p1 = ctx->prof.get(); cudaEventRecord(p0, ctx->st); }
    CK(launch_prep(pa, ctx->st), "k_prep");
    ctx->launches += 1;
    if (ctx->prof.on) {
      cudaEventRecord(p1, ctx->st);
      ctx->prof.pending.push_back({p0, p1, 0.0, 4});
    }
    if (fuse && devrep)
      CK(cudaMemcpyAsync(ctx->h_report, ctx->report_dev, (size_t)report_bytes(B), cudaMemcpyDeviceToHost, ctx->st),
         "report D2H");
    if (fuse) {
      CK(cudaEventRecord(ctx->ev_report, ctx->st), "event");
      CK(launch_deps(ctx->units, ctx->ctrl, ctx->desc, ctx->cfg.attn_variant == 2 ? 1 : 0, ctx->num_sms * 4,
                     ctx->st), "k_deps");
      ctx->launches += 1;
    }
    ctx->attn_epoch++;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->st); }
    // the tensor-core kernel picks its ring shape per launch from the step's mean rows per
    // slot, and its softmax width from the tile counts the two widths would give: NC = 16
    // packs up to 16 / G KV heads of a short unit into one 128-row tile (8 / G with NC = 8)
    // at ~4 % more per tile (tools/attn_sweep.py: equal-tile cases 0.876 / 0.915 at 45 rows,
    // 0.929 / 0.952 at 105), so it is launched when it needs < 1 / 1.04 of NC = 8's tiles
    int32_t mean_rows = 0, nc_pick = 8;
    if (ctx->cfg.attn_variant == 2 && B > 0) {
      const int G = ctx->sh.H / ctx->sh.Hkv, Hkv = ctx->sh.Hkv;
      auto tiles = [&](int pmax, int r) -> int64_t {   // one (slot, layer): the kernel's packing rules
        const int rg = (r + 7) & ~7;
        if (pmax > 1 && 2 * rg <= 128) {                 // short unit: heads packed
          const int np = std::min(std::min(pmax, 128 / rg), Hkv);
          return (Hkv + np - 1) / np;
        }
        const int tl = r % 128, tg = (tl + 7) & ~7;
        if (pmax > 1 && tl > 0 && 2 * tg <= 128) {       // long unit: full tiles + packed tails
          const int np = std::min(std::min(pmax, 128 / tg), Hkv);
          if (np > 1) return (int64_t)Hkv * (r / 128) + (Hkv + np - 1) / np;
        }
        return (int64_t)Hkv * ((r + 127) / 128);
      };
      int64_t rows = 0, t8 = 0, t16 = 0;
      for (const DSlot& sl : ctx->slots_h) {
        const int r = sl.len + 1;
        rows += r;
        if (G <= 8) { t8 += tiles(8 / G, r); t16 += tiles(16 / G, r); }
      }
      mean_rows = (int32_t)std::min<int64_t>((rows + B - 1) / B, 1 << 30);
      nc_pick = G > 8 || (double)t16 * 1.04 < (double)t8 ? 16 : 8;
    }
    if (ctx->cfg.attn_variant == 2)
      CK(launch_attn_tc(ctx->sh, (const uint16_t*)q, (const uint16_t*)k_new, (const uint16_t*)v_new,
                        (uint16_t*)ctx->buf.arena, ctx->cfg.arena_rows,
                        ctx->buf.staging ? stage_ptr(ctx, ctx->stage_cur) : nullptr, stage_bytes(ctx), out, ctx->partials,
                        ctx->units, ctx->splits, ctx->desc, ctx->progress, ctx->attn_epoch, ctx->ctrl, B, l0, nl,
                        ctx->grid_attn, ctx->grid_combine, ctx->feed, ev_counters(ctx), mean_rows, nc_pick, ctx->st),
         "k_attn_tc");
    else
      CK(launch_attn(ctx->sh, (const uint16_t*)q, (const uint16_t*)k_new, (const uint16_t*)v_new,
                     (uint16_t*)ctx->buf.arena, ctx->buf.staging ? stage_ptr(ctx, ctx->stage_cur) : nullptr, out,
                     ctx->partials, ctx->units,
                     ctx->splits, ctx->desc, ctx->progress, ctx->attn_epoch, ctx->ctrl, B, l0, nl, ctx->grid_attn,
                     ctx->grid_combine, ctx->cfg.attn_variant, ctx->feed, ev_counters(ctx), ctx->st), "k_attn");
    ctx->launches += 2;   // attention, combine
    if (ctx->prof.on) {
      cudaEventRecord(e1, ctx->st);
      int64_t sum_len = 0;
      for (const DSlot& s : ctx->slots_h) sum_len += s.len;
      const double HD = (double)ctx->sh.H * ctx->sh.D, KD = (double)ctx->sh.Hkv * ctx->sh.D;
      // algorithmic bytes: prior rows K+V (KV heads), new row
      // write, k_new+v_new read, q read (bf16, query heads), out write (fp32)
      const double bytes = nl * (KD * (4.0 * (double)sum_len + 4.0 * B + 4.0 * B) + HD * (2.0 * B + 4.0 * B));
      ctx->prof.pending.push_back({e0, e1, bytes, 0});
    }
  }
  ctx->fused_pending = fuse;
  if (finalize) {
    for (DSlot& s : ctx->slots_h) { s.len += 1; s.gen += 1; }
    ctx->tokens_total += B;
    ctx->status_pending = true;
  }
  return S3_OK;
}

namespace {
bool is_pinned_host(const void* p, void** dev_ptr = nullptr) {
  cudaPointerAttributes at{};
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  if (at.type != cudaMemoryTypeHost) return false;
  if (dev_ptr) *dev_ptr = at.devicePointer;
  return at.devicePointer != nullptr;
}
}  // namespace

s3_status s3_decode_step_host(s3_ctx* ctx, const s3_host_io* io) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!io) return fail(ctx, S3_E_INVAL, "decode_step_host: null io");
  if (ctx->status_pending) return fail(ctx, S3_E_STATE, "decode_step: statuses not consumed");
  const int32_t B = (int32_t)ctx->slots_h.size();
  const int32_t L = ctx->sh.L;
  if (B == 0) return s3_decode_step(ctx, 0, L, nullptr, nullptr, nullptr, nullptr, nullptr);
  void* out_dev = nullptr;
  if (!is_pinned_host(io->q) || !is_pinned_host(io->k_new) || !is_pinned_host(io->v_new) ||
      !is_pinned_host(io->eos) || !is_pinned_host(io->out, &out_dev))
    return fail(ctx, S3_E_INVAL, "decode_step_host: host buffers must be pinned");
  if (!io->q_dev || !io->k_new_dev || !io->v_new_dev || !io->eos_dev)
    return fail(ctx, S3_E_INVAL, "decode_step_host: null device landing buffer");
  if (io->chunks < 0) return fail(ctx, S3_E_INVAL, "decode_step_host: chunks < 0");
  if (!ctx->hio) {
    CK(cudaStreamCreateWithFlags(&ctx->hio, cudaStreamNonBlocking), "copy stream");
    CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking), "copy stream");
    CK(cudaEventCreateWithFlags(&ctx->ev_hio_start, cudaEventDisableTiming), "event");
    CK(cudaEventCreateWithFlags(&ctx->ev_hio_done, cudaEventDisableTiming), "event");
    CK(cudaEventCreateWithFlags(&ctx->ev_comb, cudaEventDisableTiming), "event");
    CK(cudaEventCreateWithFlags(&ctx->ev_d2h_done, cudaEventDisableTiming), "event");
  }
  // the detection in k_prep reads eos first: a tiny in-stream copy
  CK(cudaMemcpyAsync(io->eos_dev, io->eos, (size_t)B, cudaMemcpyHostToDevice, ctx->st), "eos H2D");
  // the landing buffers are free once the previous step's kernels (earlier on cfg.stream) are done
  CK(cudaEventRecord(ctx->ev_hio_start, ctx->st), "event");
  CK(cudaStreamWaitEvent(ctx->hio, ctx->ev_hio_start, 0), "wait");
  StreamValue32Fn wv = write_value32(), wt = wait_value32();
  // the TMA-ring and tensor-core kernels wait on ready words; the register-streaming one cannot
  const bool pipe = wv && ((ctx->cfg.attn_variant == 0 && attn_tma_stages(ctx->sh) >= 2) || ctx->cfg.attn_variant == 2);
  // device out + per-chunk D2H overlapped with the kernel (counters in k_attn_tma's consumers)
  const bool ce_out = pipe && wt && io->out_dev && ctx->cfg.attn_variant == 0;
  int32_t nch = pipe ? std::min(io->chunks ? io->chunks : 16, kMaxFeedChunks) : 1;
  nch = std::max(1, std::min(nch, B));
  const int32_t cb = (B + nch - 1) / nch;
  nch = (B + cb - 1) / cb;
  const uint32_t epoch = ++ctx->feed_epoch;
  const size_t wq = (size_t)ctx->sh.H * ctx->sh.D * 2, wk = (size_t)ctx->sh.Hkv * ctx->sh.D * 2;
  for (int32_t c = 0; c < nch; ++c) {
    const int32_t b0 = c * cb, nb = std::min(B, b0 + cb) - b0;
    // [L][B][heads][D]: one strided copy per tensor covers slots [b0, b0+nb) of every layer
    CK(cudaMemcpy2DAsync((uint8_t*)io->q_dev + b0 * wq, B * wq, (const uint8_t*)io->q + b0 * wq, B * wq, nb * wq,
                         (size_t)L, cudaMemcpyHostToDevice, ctx->hio), "q H2D");
    CK(cudaMemcpy2DAsync((uint8_t*)io->k_new_dev + b0 * wk, B * wk, (const uint8_t*)io->k_new + b0 * wk, B * wk,
                         nb * wk, (size_t)L, cudaMemcpyHostToDevice, ctx->hio), "k_new H2D");
    CK(cudaMemcpy2DAsync((uint8_t*)io->v_new_dev + b0 * wk, B * wk, (const uint8_t*)io->v_new + b0 * wk, B * wk,
                         nb * wk, (size_t)L, cudaMemcpyHostToDevice, ctx->hio), "v_new H2D");
    if (pipe && wv(ctx->hio, (unsigned long long)(uintptr_t)(ctx->ready + c), epoch, 0) != 0)
      return fail(ctx, S3_E_CUDA, "decode_step_host: stream write");
  }
  CK(cudaEventRecord(ctx->ev_hio_done, ctx->hio), "event");
  if (!pipe) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_hio_done, 0), "wait");
  if (pipe) { ctx->feed.ready = ctx->ready; ctx->feed.cb = cb; ctx->feed.epoch = epoch; }
  if (ce_out) ctx->feed.done = ctx->done;
  // split-K slots (len + 1 > C, k_prep's rule) get their out rows from k_combine, after the kernel
  std::vector<int32_t> split_slots;
  uint32_t expect[kMaxFeedChunks] = {};
  if (ce_out) {
    const uint32_t warps = (uint32_t)(attn_block_threads(ctx->sh) / 32);
    for (int32_t b = 0; b < B; ++b) {
      if (ctx->slots_h[b].len + 1 > ctx->C) split_slots.push_back(b);
      else expect[b / cb] += warps * (uint32_t)L;
    }
  }
  // pipelined without counters: the kernels store `out` to mapped host memory as items finish
  const bool dev_out = io->out_dev && (ce_out || !pipe);
  float* kout = static_cast<float*>(dev_out ? io->out_dev : out_dev);
  const s3_status rc = s3_decode_step(ctx, 0, L, io->q_dev, io->k_new_dev, io->v_new_dev, io->eos_dev, kout);
  ctx->feed = Feed{};
  if (rc != S3_OK) return rc;
  const size_t wo = (size_t)ctx->sh.H * ctx->sh.D * 4;
  if (dev_out) {
    // enqueued after the attention and combine launches, so a wait here can never hold them up
    cudaStream_t ds = ce_out ? ctx->d2h : ctx->st;
    if (ce_out) {
      CK(cudaStreamWaitEvent(ds, ctx->ev_hio_start, 0), "wait");
      for (int32_t c = 0; c < nch; ++c) {
        if (!expect[c]) continue;
        ctx->done_target[c] += expect[c];
        if (wt(ds, (unsigned long long)(uintptr_t)(ctx->done + c), ctx->done_target[c], kWaitGeq) != 0)
          return fail(ctx, S3_E_CUDA, "decode_step_host: stream wait");
        const int32_t b0 = c * cb, nb = std::min(B, b0 + cb) - b0;
        CK(cudaMemcpy2DAsync((uint8_t*)io->out + b0 * wo, B * wo, (const uint8_t*)io->out_dev + b0 * wo, B * wo,
                             nb * wo, (size_t)L, cudaMemcpyDeviceToHost, ds), "out D2H");
      }
      CK(cudaEventRecord(ctx->ev_comb, ctx->st), "event");
      CK(cudaStreamWaitEvent(ds, ctx->ev_comb, 0), "wait");
      for (int32_t b : split_slots)
        CK(cudaMemcpy2DAsync((uint8_t*)io->out + b * wo, B * wo, (const uint8_t*)io->out_dev + b * wo, B * wo, wo,
                             (size_t)L, cudaMemcpyDeviceToHost, ds), "out D2H");
      CK(cudaEventRecord(ctx->ev_d2h_done, ds), "event");
      CK(cudaStreamWaitEvent(ctx->st, ctx->ev_d2h_done, 0), "wait");
    } else {
      CK(cudaMemcpyAsync(io->out, io->out_dev, (size_t)L * B * wo, cudaMemcpyDeviceToHost, ds), "out D2H");
    }
  }
  // completion of cfg.stream implies the copies are done too
  CK(cudaStreamWaitEvent(ctx->st, ctx->ev_hio_done, 0), "wait");
  return S3_OK;
}

s3_status s3_evict_compact(s3_ctx* ctx, s3_evict_report* rep, int32_t* perm, s3_evicted* evicted,
                           int64_t* finished_ids) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!rep) return fail(ctx, S3_E_INVAL, "evict_compact: null report");
  if (!ctx->status_pending) return fail(ctx, S3_E_STATE, "evict_compact: no completed decode step");
  const int32_t B = (int32_t)ctx->slots_h.size();
  ctx->evict_seq++;
  s3_evict_report r{};
  r.n_before = B;
  r.first_hole = B;
  if (B == 0) {
    ctx->status_pending = false;
    *rep = r;
    return S3_OK;
  }
  const Shape& sh = ctx->sh;
  const DReportHeader* h = reinterpret_cast<const DReportHeader*>(ctx->h_report);
  bool fused = false;
  if (ctx->fused_pending) {
    // the decode step ran the keep-scan and copied its report back before the
    // attention kernel: wait for that copy only, not for the attention pass
    CK(cudaEventSynchronize(ctx->ev_report), "report sync");
    fused = *reinterpret_cast<const int32_t*>(ctx->h_report + report_bytes(B)) == 1;
  }
  if (!fused) {
    CK(launch_keep_scan(sh, ctx->slots[ctx->cur], ctx->slots[1 - ctx->cur], B, ctx->S, ctx->report_dev,
                        ctx->entries, ctx->key_chunk0, ctx->key_src, ctx->ctrl64, ctx->cfg.compact_policy,
                        (ctx->pool.size() + ctx->home.size()) > 0 ? 1 : 0, ctx->st), "k_keep_scan");
    ctx->launches += 1;
    CK(cudaMemcpyAsync(ctx->h_report, ctx->report_dev, (size_t)report_bytes(B), cudaMemcpyDeviceToHost, ctx->st),
       "report D2H");
    CK(cudaStreamSynchronize(ctx->st), "report sync");
  }
  ctx->fused_pending = false;
  flush_deferred(ctx);
  prof_collect(ctx);
  ctx->upload_used = 0;
  const int32_t* dperm = reinterpret_cast<const int32_t*>(ctx->h_report + report_perm_off(B));
  const DEvicted* dev = reinterpret_cast<const DEvicted*>(ctx->h_report + report_ev_off(B));
  const int64_t* dfin = reinterpret_cast<const int64_t*>(ctx->h_report + report_fin_off(B));
  if (h->n_before != B || h->n_kept + h->n_finished + h->n_evicted != B)
    return fail(ctx, S3_E_CUDA, "evict_compact: inconsistent device report");

  // host store for every evictee (before any device move is enqueued)
  std::vector<int64_t> hoff(h->n_evicted);
  for (int32_t i = 0; i < h->n_evicted; ++i) {
    hoff[i] = hs_alloc(ctx, (int64_t)dev[i].len * sh.kvpt);
    if (hoff[i] < 0) {               // ranges still pinned by in-flight reloads: drain them and retry
      CK(cudaStreamSynchronize(ctx->st), "sync");
      flush_deferred(ctx);
      hoff[i] = hs_alloc(ctx, (int64_t)dev[i].len * sh.kvpt);
    }
    if (hoff[i] < 0) {
      for (int32_t j = 0; j < i; ++j) hs_free(ctx, hoff[j], (int64_t)dev[j].len * sh.kvpt);
      if (fused) {   // the decode step already took the evictees' rows out of the arena
        ctx->poisoned = true;
        return fail(ctx, S3_E_NOMEM, "evict_compact: host store exhausted after a fused step (context poisoned)");
      }
      return fail(ctx, S3_E_NOMEM, "evict_compact: host store too small for this step's evictions");
    }
  }
  // the fused step already wrote its evictees to half stage_cur; the k_move path takes the next half
  if (!fused) ctx->stage_cur = ctx->stage_next;
  const bool staged = h->n_evicted > 0 && ctx->buf.staging && h->d2h_bytes <= stage_bytes(ctx);
  uint8_t* stage = ctx->buf.staging ? stage_ptr(ctx, ctx->stage_cur) : nullptr;
  if (fused && ctx->prof.on) {
    ctx->prof.fused_steps++;
    ctx->prof.fused_move_bytes += (double)h->moved_bytes + (double)h->d2h_bytes;
  }
  std::shared_ptr<EventBox> d2h_done;
  std::vector<std::shared_ptr<EventBox>> per_ev;   // staged path: one completion event per evictee
  if (h->n_evicted > 0) {
    d2h_done = std::make_shared<EventBox>();
    if (!staged) {
      // synchronous fallback: copy straight from the arena before rows move
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->st); }
      for (int32_t i = 0; i < h->n_evicted; ++i) {
        const DSlot& s = ctx->slots_h[dev[i].b];
        CK(cudaMemcpyAsync((uint8_t*)ctx->buf.host_store + hoff[i],
                           (uint8_t*)ctx->buf.arena + (int64_t)s.off * sh.kvpt, (size_t)dev[i].len * sh.kvpt,
                           cudaMemcpyDeviceToHost, ctx->st), "evict D2H (sync)");
      }
      if (ctx->prof.on) {
        cudaEventRecord(e1, ctx->st);
        ctx->prof.pending.push_back({e0, e1, (double)h->d2h_bytes, 2});
      }
      CK(cudaEventRecord(d2h_done->ev, ctx->st), "event");
    } else if (ctx->stage_d2h[ctx->stage_cur] && !fused) {
      // k_move rewrites this staging half: the D2H that last read it must be done
      CK(cudaStreamWaitEvent(ctx->st, ctx->stage_d2h[ctx->stage_cur]->ev, 0), "wait staging");
    }
  }
  if (!fused && h->n_chunks > 0) {
    ctx->epoch++;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->st); }
    const int grid = (int)std::min<int64_t>((h->n_chunks + 2 * 3 - 1) / (2 * 3), ctx->grid_move);
    CK(launch_move((uint8_t*)ctx->buf.arena, stage, ctx->entries, ctx->key_chunk0,
                   ctx->key_src, h->n_entries, h->n_chunks, ctx->S, sh.kvpt, ctx->ctrl64, ctx->flags, ctx->epoch,
                   staged ? 1 : 0, grid, ctx->st), "k_move");
    ctx->launches += 1;
    if (ctx->prof.on) {
      cudaEventRecord(e1, ctx->st);
      const double bytes = 2.0 * (double)h->moved_bytes + (staged ? 2.0 * (double)h->d2h_bytes : 0.0);
      ctx->prof.pending.push_back({e0, e1, bytes, 1});
    }
  }
  if (staged) {
    // fused step: each evictee's copy starts as soon as the attention kernel has
    // staged all its rows (per-evictee counters), overlapping the rest of the pass;
    // otherwise (k_move staging) after the staging pass
    StreamValue32Fn wt = wait_value32();
    const bool counted = fused && ev_counters(ctx) != nullptr;
    if (!counted) {
      cudaEvent_t k4;
      CK(cudaEventCreateWithFlags(&k4, cudaEventDisableTiming), "event");
      CK(cudaEventRecord(k4, ctx->st), "event");
      CK(cudaStreamWaitEvent(ctx->side, k4, 0), "side wait");
      cudaEventDestroy(k4);
    } else {
      // the staging half must not be read before this step's k_prep wrote its plan
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_report, 0), "side wait");
    }
    const int nwc = attn_block_threads(sh) / 32;    // CUDA-core kernel: consumer warps that append the new row
    per_ev.resize(h->n_evicted);
    for (int32_t i = 0; i < h->n_evicted; ++i) {
      if (counted) {
        // rows each kernel counts for this evictee over the step's L layers
        const uint32_t target = ctx->cfg.attn_variant == 2
                                    ? (uint32_t)((int64_t)sh.L * sh.Hkv * dev[i].len)
                                    : (uint32_t)((int64_t)sh.L * ((dev[i].len - 1) + nwc));
        ctx->ev_target[i] += target;
        if (wt(ctx->side, (unsigned long long)(uintptr_t)(ctx->evdone + i), ctx->ev_target[i], kWaitGeq) != 0)
          return fail(ctx, S3_E_CUDA, "evict_compact: stream wait");
      }
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (ctx->prof.on) { e0 = ctx->prof.get(); e1 = ctx->prof.get(); cudaEventRecord(e0, ctx->side); }
      CK(cudaMemcpyAsync((uint8_t*)ctx->buf.host_store + hoff[i], stage + dev[i].stage_off,
                         (size_t)dev[i].len * sh.kvpt, cudaMemcpyDeviceToHost, ctx->side), "evict D2H");
      if (ctx->prof.on) {
        cudaEventRecord(e1, ctx->side);
        ctx->prof.pending.push_back({e0, e1, (double)dev[i].len * sh.kvpt, 2});
      }
      per_ev[i] = std::make_shared<EventBox>();   // this evictee's host copy (s3_evict_wait_req, reload gate)
      CK(cudaEventRecord(per_ev[i]->ev, ctx->side), "event");
    }
    CK(cudaEventRecord(d2h_done->ev, ctx->side), "event");
    ctx->stage_d2h[ctx->stage_cur] = d2h_done;
    if (ctx->stage_dbl) ctx->stage_next = 1 - ctx->stage_cur;   // the next evictions use the other half
  }
  // requeue evicted requests with doubled reservation (R5), in batch order
  int64_t pcie = 0;
  for (int32_t i = 0; i < h->n_evicted; ++i) {
    const DEvicted& e = dev[i];
    Item it{};
    it.req = e.req; it.prompt = e.prompt; it.gen = e.gen;
    it.cap = std::min<int64_t>(2LL * e.cap, ctx->cfg.max_seq_len);
    it.evicted = 1;
    it.host_off = hoff[i];
    it.host_bytes = (int64_t)e.len * sh.kvpt;
    it.host_rows = e.len;
    it.ready = (size_t)i < per_ev.size() ? per_ev[i] : d2h_done;
    ctx->evict_done[e.req] = it.ready;
    if (staged) { it.stage_src = stage + e.stage_off; it.evict_seq = ctx->evict_seq; }
    pcie += 2LL * e.cap * sh.kvpt;
    (ctx->cfg.world > 1 ? ctx->home : ctx->pool).emplace(Key{it.cap, it.req}, it);
    ctx->n_evicted_waiting++;
    if (evicted) {
      s3_evicted& o = evicted[i];
      o.req_id = e.req; o.batch_index = e.b; o.prompt_len = e.prompt; o.gen_len = e.gen; o.len = e.len;
      o.cap_rows = e.cap; o.new_cap_rows = it.cap; o.host_off = hoff[i];
    }
  }
  // host mirror: stable compaction
  std::vector<DSlot> kept;
  kept.reserve(h->n_kept);
  int64_t run = 0;
  for (int32_t b = 0; b < B; ++b) {
    if (dperm[b] >= 0) {
      DSlot s = ctx->slots_h[b];
      if (h->compacted) {
        s.off = (int32_t)run;
        run += s.cap;
      } else {
        run = (int64_t)s.off + s.cap;            // holes stay (R27); tail = end of the last slot
      }
      kept.push_back(s);
    }
    if (perm) perm[b] = dperm[b];
  }
  if (run != h->tail || (int32_t)kept.size() != h->n_kept)
    return fail(ctx, S3_E_CUDA, "evict_compact: host/device mirror mismatch");
  ctx->slots_h.swap(kept);
  ctx->tail = run;
  ctx->cur = 1 - ctx->cur;
  ctx->status_pending = false;
  if (finished_ids) std::memcpy(finished_ids, dfin, sizeof(int64_t) * (size_t)h->n_finished);
  for (int32_t i = 0; i < h->n_finished; ++i) ctx->live.erase(dfin[i]);
  ctx->finished_total += h->n_finished;
  ctx->evicted_total += h->n_evicted;
  r.n_finished = h->n_finished;
  r.n_evicted = h->n_evicted;
  r.n_kept = h->n_kept;
  r.tail_rows = h->tail;
  r.d2h_bytes = h->d2h_bytes;
  r.moved_bytes = h->moved_bytes;
  r.paper_pcie_bytes = pcie;
  r.paper_hbm_bytes = h->hbm_bytes;
  r.first_hole = h->first_hole;
  r.sync_evict = (h->n_evicted > 0 && !staged) ? 1 : 0;
  *rep = r;
  return S3_OK;
}

s3_status s3_evict_wait(s3_ctx* ctx) {
  if (s3_status s = check_ctx(ctx)) return s;
  CK(cudaStreamSynchronize(ctx->side), "side sync");
  CK(cudaStreamSynchronize(ctx->st), "sync");
  flush_deferred(ctx);
  ctx->evict_done.clear();
  return S3_OK;
}

s3_status s3_evict_wait_req(s3_ctx* ctx, int64_t req_id) {
  if (s3_status s = check_ctx(ctx)) return s;
  auto it = ctx->evict_done.find(req_id);
  if (it == ctx->evict_done.end()) return S3_OK;   // no host copy pending for this request
  CK(cudaEventSynchronize(it->second->ev), "evict wait");
  ctx->evict_done.erase(it);
  return S3_OK;
}

s3_status s3_admit(s3_ctx* ctx, s3_admit_report* rep, int64_t* admitted_ids) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (ctx->status_pending) return fail(ctx, S3_E_STATE, "admit: statuses not consumed");
  if (ctx->cfg.world != 1) return fail(ctx, S3_E_STATE, "admit: world > 1 uses admit_home/admit_shared");
  int64_t moved = 0;
  if (ctx->cfg.compact_policy == 1 && !ctx->pool.empty())
    if (s3_status s = compact_holes(ctx, &moved)) return s;
  int64_t free_rows = ctx->cfg.arena_rows - ctx->tail;
  int64_t slots_left = ctx->cfg.max_running - (int64_t)ctx->slots_h.size();
  std::vector<Item> taken;
  ffd_scan(
      ctx->pool, [&] { return slots_left > 0 ? free_rows : 0; },
      [&](int64_t cap) { return cap <= free_rows ? 0 : -1; },
      [&](int, const Item& it) { free_rows -= it.cap; slots_left--; taken.push_back(it); });
  const s3_status st = place_items(ctx, taken, rep, admitted_ids);
  if (rep) rep->moved_bytes = moved;
  return st;
}

s3_status s3_admit_home(s3_ctx* ctx, s3_admit_report* rep, int64_t* admitted_ids) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (ctx->status_pending) return fail(ctx, S3_E_STATE, "admit_home: statuses not consumed");
  int64_t moved = 0;   // before the counters are exchanged: free rows = R - tail
  if (ctx->cfg.compact_policy == 1 && (!ctx->pool.empty() || !ctx->home.empty()))
    if (s3_status s = compact_holes(ctx, &moved)) return s;
  int64_t free_rows = ctx->cfg.arena_rows - ctx->tail;
  int64_t slots_left = ctx->cfg.max_running - (int64_t)ctx->slots_h.size();
  std::vector<Item> taken;
  ffd_scan(
      ctx->home, [&] { return slots_left > 0 ? free_rows : 0; },
      [&](int64_t cap) { return cap <= free_rows ? 0 : -1; },
      [&](int, const Item& it) { free_rows -= it.cap; slots_left--; taken.push_back(it); });
  const s3_status st = place_items(ctx, taken, rep, admitted_ids);
  if (rep) rep->moved_bytes = moved;
  return st;
}

s3_status s3_admit_shared(s3_ctx* ctx, const int64_t* counters_all, s3_admit_report* rep,
                          int64_t* admitted_ids) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (ctx->status_pending) return fail(ctx, S3_E_STATE, "admit_shared: statuses not consumed");
  if (!counters_all) return fail(ctx, S3_E_INVAL, "admit_shared: null counters");
  const int W = ctx->cfg.world;
  std::vector<int64_t> fr(W), sl(W);
  for (int r = 0; r < W; ++r) { fr[r] = counters_all[r * S3_NCOUNTERS + 0]; sl[r] = counters_all[r * S3_NCOUNTERS + 2]; }
  if (fr[ctx->cfg.rank] != ctx->cfg.arena_rows - ctx->tail)
    return fail(ctx, S3_E_STATE, "admit_shared: counters do not match this rank");
  std::vector<Item> taken;
  ffd_scan(
      ctx->pool,
      [&] {
        int64_t m = 0;
        for (int r = 0; r < W; ++r) if (sl[r] > 0) m = std::max(m, fr[r]);
        return m;
      },
      [&](int64_t cap) { return worst_fit(W, fr.data(), sl.data(), cap); },
      [&](int bin, const Item& it) {
        fr[bin] -= it.cap;
        sl[bin]--;
        if (bin == ctx->cfg.rank) taken.push_back(it);
      });
  return place_items(ctx, taken, rep, admitted_ids);
}

s3_status s3_counters_local(const s3_ctx* ctx, int64_t row[S3_NCOUNTERS]) {
  if (!ctx || !row) return S3_E_INVAL;
  row[0] = ctx->cfg.arena_rows - ctx->tail;
  row[1] = (int64_t)ctx->slots_h.size();
  row[2] = ctx->cfg.max_running - (int64_t)ctx->slots_h.size();
  row[3] = ctx->n_evicted_waiting;
  row[4] = (int64_t)ctx->pool.size() - (ctx->cfg.world > 1 ? 0 : ctx->n_evicted_waiting);
  row[5] = ctx->finished_total;
  row[6] = ctx->evicted_total;
  row[7] = ctx->tokens_total;
  return S3_OK;
}

s3_status s3_nccl_get_unique_id(uint8_t id[S3_NCCL_ID_BYTES]) {
  if (!id) return S3_E_INVAL;
  const NcclApi& api = nccl_api();
  if (!api.ok) return S3_E_NCCL;
  ncclUniqueId u;
  if (api.get_unique_id(&u) != ncclSuccess) return S3_E_NCCL;
  std::memcpy(id, &u, sizeof(u));
  return S3_OK;
}

s3_status s3_comm_init(s3_ctx* ctx, const uint8_t id[S3_NCCL_ID_BYTES]) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!id) return fail(ctx, S3_E_INVAL, "comm_init: null id");
  if (ctx->comm) return fail(ctx, S3_E_STATE, "comm_init: communicator already bound");
  if (ctx->cfg.world > S3_MAX_RANKS) return fail(ctx, S3_E_INVAL, "comm_init: world > S3_MAX_RANKS");
  const NcclApi& api = nccl_api();
  if (!api.ok) return S3_E_NCCL;   // not loadable: nothing bound, the context stays usable
  CK(cudaSetDevice(ctx->cfg.device), "cudaSetDevice");
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
  CK(cudaStreamCreateWithPriority(&ctx->xs, cudaStreamNonBlocking, hi), "exchange stream");
  const size_t bytes = sizeof(int64_t) * S3_NCOUNTERS * (size_t)ctx->cfg.world;
  CK(cudaMalloc(&ctx->x_dev, bytes), "exchange buffer");
  CK(cudaHostAlloc(&ctx->x_host, bytes, cudaHostAllocDefault), "exchange host buffer");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  if (api.comm_init_rank(&ctx->comm, ctx->cfg.world, u, ctx->cfg.rank) != ncclSuccess) {
    ctx->comm = nullptr;
    return fail(ctx, S3_E_NCCL, "ncclCommInitRank");
  }
  return S3_OK;
}

s3_status s3_exchange_counters(s3_ctx* ctx, int64_t* counters_all) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!counters_all) return fail(ctx, S3_E_INVAL, "exchange_counters: null output");
  if (!ctx->comm) return fail(ctx, S3_E_STATE, "exchange_counters: no communicator (s3_comm_init)");
  const int W = ctx->cfg.world;
  const size_t n = (size_t)S3_NCOUNTERS * W, bytes = n * sizeof(int64_t);
  std::memset(ctx->x_host, 0, bytes);
  s3_counters_local(ctx, ctx->x_host + (size_t)ctx->cfg.rank * S3_NCOUNTERS);
  CK(cudaMemcpyAsync(ctx->x_dev, ctx->x_host, bytes, cudaMemcpyHostToDevice, ctx->xs), "exchange H2D");
  if (nccl_api().all_reduce(ctx->x_dev, ctx->x_dev, n, ncclInt64, ncclSum, ctx->comm, ctx->xs) != ncclSuccess)
    return fail(ctx, S3_E_NCCL, "ncclAllReduce");
  CK(cudaMemcpyAsync(ctx->x_host, ctx->x_dev, bytes, cudaMemcpyDeviceToHost, ctx->xs), "exchange D2H");
  CK(cudaStreamSynchronize(ctx->xs), "exchange sync");
  std::memcpy(counters_all, ctx->x_host, bytes);
  ctx->x_last.assign(ctx->x_host, ctx->x_host + n);
  ctx->exchanges++;
  return S3_OK;
}

s3_status s3_counters_get(const s3_ctx* ctx, s3_counters* c) {
  if (!ctx || !c) return S3_E_INVAL;
  *c = s3_counters{};
  std::vector<int64_t> m = ctx->x_last;
  int W = ctx->cfg.world;
  if (m.empty()) {   // no exchange yet: this rank's row alone
    W = 1;
    m.assign(S3_NCOUNTERS, 0);
    s3_counters_local(ctx, m.data());
  }
  c->world = W;
  c->exchanges = ctx->exchanges;
  for (int r = 0; r < W && r < S3_MAX_RANKS; ++r) {
    const int64_t* row = m.data() + (size_t)r * S3_NCOUNTERS;
    c->rank_free_rows[r] = row[0];
    c->rank_running[r] = row[1];
    c->free_rows_total += row[0];
    c->running_total += row[1];
    c->evicted_waiting_total += row[3];
    c->finished_total += row[5];
    c->evicted_total += row[6];
    c->tokens_total += row[7];
  }
  c->fresh_waiting = m[4];   // the shared pool is replicated on every rank
  return S3_OK;
}

int32_t s3_plan_ffd(int32_t n, const int64_t* cap, const int64_t* req_id, int64_t free_rows, int32_t max_items,
                    uint8_t* admitted) {
  Pool pool;
  std::map<int64_t, int32_t> idx;
  for (int32_t i = 0; i < n; ++i) {
    Item it{};
    it.req = req_id[i]; it.cap = (int32_t)cap[i];
    pool.emplace(Key{cap[i], req_id[i]}, it);
    idx[req_id[i]] = i;
    admitted[i] = 0;
  }
  int64_t left = max_items;
  return (int32_t)ffd_scan(
      pool, [&] { return left > 0 ? free_rows : 0; }, [&](int64_t c) { return c <= free_rows ? 0 : -1; },
      [&](int, const Item& it) { free_rows -= it.cap; left--; admitted[idx[it.req]] = 1; });
}

int32_t s3_plan_ffd_multibin(int32_t n, const int64_t* cap, const int64_t* req_id, int32_t world,
                             int64_t* free_rows, int64_t* free_slots, int32_t* rank) {
  Pool pool;
  std::map<int64_t, int32_t> idx;
  for (int32_t i = 0; i < n; ++i) {
    Item it{};
    it.req = req_id[i]; it.cap = (int32_t)cap[i];
    pool.emplace(Key{cap[i], req_id[i]}, it);
    idx[req_id[i]] = i;
    rank[i] = -1;
  }
  return (int32_t)ffd_scan(
      pool,
      [&] {
        int64_t m = 0;
        for (int r = 0; r < world; ++r) if (free_slots[r] > 0) m = std::max(m, free_rows[r]);
        return m;
      },
      [&](int64_t c) { return worst_fit(world, free_rows, free_slots, c); },
      [&](int bin, const Item& it) {
        free_rows[bin] -= it.cap;
        free_slots[bin]--;
        rank[idx[it.req]] = bin;
      });
}

s3_status s3_batch_size(const s3_ctx* ctx, int32_t* B) {
  if (!ctx || !B) return S3_E_INVAL;
  *B = (int32_t)ctx->slots_h.size();
  return S3_OK;
}

s3_status s3_batch_view(const s3_ctx* ctx, s3_slot* slots, int32_t* B) {
  if (!ctx || !B) return S3_E_INVAL;
  *B = (int32_t)ctx->slots_h.size();
  if (slots)
    for (int32_t i = 0; i < *B; ++i) {
      const DSlot& s = ctx->slots_h[i];
      slots[i].req_id = s.req; slots[i].prompt_len = s.prompt; slots[i].gen_len = s.gen;
      slots[i].len = s.len; slots[i].cap_rows = s.cap; slots[i].off = s.off;
    }
  return S3_OK;
}

s3_status s3_profile_enable(s3_ctx* ctx, int32_t on) {
  if (s3_status s = check_ctx(ctx)) return s;
  CK(cudaStreamSynchronize(ctx->st), "sync");
  CK(cudaStreamSynchronize(ctx->side), "side sync");
  prof_collect(ctx);
  ctx->prof.on = on != 0;
  ctx->prof.attn_iv.clear();
  ctx->prof.d2h_iv.clear();
  if (!ctx->prof.ref) CK(cudaEventCreate(&ctx->prof.ref), "event");
  CK(cudaEventRecord(ctx->prof.ref, ctx->st), "event");
  ctx->prof.attn_launches = ctx->prof.move_launches = ctx->prof.fused_steps = 0;
  ctx->prof.attn_ms = ctx->prof.move_ms = ctx->prof.attn_bytes = ctx->prof.move_bytes = 0;
  ctx->prof.fused_move_bytes = 0;
  ctx->prof.d2h_copies = ctx->prof.h2d_copies = 0;
  ctx->prof.d2h_ms = ctx->prof.d2h_bytes = ctx->prof.h2d_ms = ctx->prof.h2d_bytes = 0;
  ctx->prof.prep_launches = 0;
  ctx->prof.prep_ms = 0;
  return S3_OK;
}

s3_status s3_profile_get(s3_ctx* ctx, s3_profile* p) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!p) return fail(ctx, S3_E_INVAL, "profile_get: null");
  CK(cudaStreamSynchronize(ctx->st), "sync");
  CK(cudaStreamSynchronize(ctx->side), "side sync");
  prof_collect(ctx);
  p->kernel_launches = ctx->launches;
  p->attn_launches = ctx->prof.attn_launches;
  p->move_launches = ctx->prof.move_launches;
  p->attn_ms = ctx->prof.attn_ms;
  p->move_ms = ctx->prof.move_ms;
  p->attn_bytes = ctx->prof.attn_bytes;
  p->move_bytes = ctx->prof.move_bytes;
  p->fused_steps = ctx->prof.fused_steps;
  p->fused_move_bytes = ctx->prof.fused_move_bytes;
  p->d2h_copies = ctx->prof.d2h_copies; p->h2d_copies = ctx->prof.h2d_copies;
  p->d2h_ms = ctx->prof.d2h_ms; p->d2h_bytes = ctx->prof.d2h_bytes;
  p->h2d_ms = ctx->prof.h2d_ms; p->h2d_bytes = ctx->prof.h2d_bytes;
  double ov = 0;
  for (const auto& d : ctx->prof.d2h_iv)
    for (const auto& k : ctx->prof.attn_iv) ov += std::max(0.0, std::min(d.second, k.second) - std::max(d.first, k.first));
  p->d2h_overlap_ms = ov;
  p->prep_launches = ctx->prof.prep_launches;
  p->prep_ms = ctx->prof.prep_ms;
  return S3_OK;
}

s3_status s3_synth_inputs(s3_ctx* ctx, int32_t l0, int32_t nl, const int32_t* out_len_by_req, int64_t n_req,
                          void* q, void* k_new, void* v_new, uint8_t* eos) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (l0 < 0 || nl < 1 || l0 + nl > ctx->sh.L) return fail(ctx, S3_E_INVAL, "synth: layer range");
  const int32_t B = (int32_t)ctx->slots_h.size();
  if (B == 0) return S3_OK;
  if (!q || !k_new || !v_new || !eos || !out_len_by_req) return fail(ctx, S3_E_INVAL, "synth: null");
  CK(launch_synth(ctx->sh, ctx->cfg.synth_seed, ctx->slots[ctx->cur], B, l0, nl, out_len_by_req, n_req,
                  (uint16_t*)q, (uint16_t*)k_new, (uint16_t*)v_new, eos, ctx->st), "k_synth");
  ctx->launches += 1;
  return S3_OK;
}

s3_status s3_verify_resident(s3_ctx* ctx, int64_t* bad) {
  if (s3_status s = check_ctx(ctx)) return s;
  if (!bad) return fail(ctx, S3_E_INVAL, "verify: null");
  const int32_t B = (int32_t)ctx->slots_h.size();
  CK(cudaMemsetAsync(ctx->verify_count, 0, 8, ctx->st), "memset");
  CK(launch_verify(ctx->sh, ctx->cfg.synth_seed, ctx->slots[ctx->cur], B, (const uint16_t*)ctx->buf.arena,
                   ctx->verify_count, ctx->st), "k_verify");
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&v, ctx->verify_count, 8, cudaMemcpyDeviceToHost, ctx->st), "D2H");
  CK(cudaStreamSynchronize(ctx->st), "sync");
  *bad = (int64_t)v;
  return S3_OK;
}

s3_status s3_gemm(void* stream, const s3_gemm_args* g) {
  if (!g) return S3_E_INVAL;
  GemmCall c;
  c.a = g->a; c.w = g->w; c.c = g->c;
  for (int i = 0; i < 3; ++i) c.d[i] = g->d[i];
  c.M = g->M; c.N = g->N; c.K = g->K; c.seg_cols = g->seg_cols; c.epi = g->epi;
  c.workspace = g->workspace; c.workspace_bytes = g->workspace_bytes;
  const cudaError_t e = launch_gemm(c, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue) return S3_E_INVAL;
  return e == cudaSuccess ? S3_OK : S3_E_CUDA;
}

s3_status s3_gemm_workspace(const s3_gemm_args* g, int64_t* bytes) {
  if (!g || !bytes) return S3_E_INVAL;
  GemmCall c{};
  c.M = g->M; c.N = g->N; c.K = g->K; c.seg_cols = g->seg_cols; c.epi = g->epi;
  const int64_t b = gemm_workspace_bytes(c);
  if (b < 0) return S3_E_INVAL;
  *bytes = b;
  return S3_OK;
}

s3_status s3_cast_bf16(void* stream, const float* src, void* dst, int64_t n) {
  if (n < 0 || (n > 0 && (!src || !dst))) return S3_E_INVAL;
  const cudaError_t e = launch_cast_bf16(src, dst, n, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue) return S3_E_INVAL;
  return e == cudaSuccess ? S3_OK : S3_E_CUDA;
}

}  // extern "C"
