// server.cu — request-coalescing server over one cold_ctx (host-side C++ runtime; include/cold.h
// "request coalescing server").
//
// The paper's serving lesson (§3.3, P:690-692 Doc C): after Float16, each inference query was too
// small to fill the GPU and launch overhead dominated; MPS let several queries share the GPU. On B200
// the same problem has a batching answer: requests that arrive while the GPU is busy are concatenated
// into ONE scoring call (cold_score_batch + cold_topk over all of them), so a burst of small queries
// costs one pass of the hot path instead of one per query. Requests are independent, so the
// scores and the per-request top-K of a coalesced call are exactly those of separate calls.
//
// One dispatcher thread owns the ctx (a ctx is externally synchronized). Pipeline of two slots: while
// the GPU scores batch b, the thread collects and stages batch b + 1, then waits for b and publishes its
// results (idx / key copied into each request's output, then done_ns[r] = completion time, stored with
// release semantics).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cold.h"

// cold_api.cu: the schema and capacities of a ctx (the server sizes its staging from them)
extern "C" void cold_ctx_describe(const cold_ctx* ctx, int* num_groups, const cold_group** groups, int* max_requests,
                                  int64_t* max_ads, int* device);

namespace {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct ReqRec {
  const cold_batch* b;   // caller-owned host batch (alive until cold_server_drain returns)
  int32_t r;             // request index inside b
  int32_t n;             // its ads
  int32_t* idx;          // caller-owned outputs [K]
  float* key;
  int64_t* done_ns;
};

// growable pinned host buffer (only resized by the dispatcher while its slot is idle)
struct Pinned {
  void* p = nullptr;
  size_t cap = 0;
  bool reserve(size_t bytes) {
    if (bytes <= cap) return true;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t c = std::max<size_t>(bytes, 4096) * 3 / 2;
    if (cudaHostAlloc(&p, c, cudaHostAllocDefault) != cudaSuccess) { cudaGetLastError(); return false; }
    cap = c;
    return true;
  }
  ~Pinned() { if (p) cudaFreeHost(p); }
};

struct Slot {
  std::vector<ReqRec> recs;
  Pinned h_in;                             // one contiguous pinned image of the batch: ao | per group offs, ids
  void* d_in = nullptr;                    // its device copy (one H2D per call)
  size_t d_in_cap = 0;
  std::vector<const int32_t*> ids_dev, offs_dev, offs_host;
  const int32_t* ao_host = nullptr;
  const int32_t* ao_dev = nullptr;
  float* d_scores = nullptr;
  int32_t* d_idx = nullptr;
  float* d_key = nullptr;
  Pinned h_res;                            // [B * K] idx then [B * K] key
  cudaEvent_t done = nullptr;
  bool inflight = false;
};

}  // namespace

struct cold_server {
  cold_ctx* ctx = nullptr;
  cold_server_config cfg{};
  std::vector<cold_group> groups;
  int device = 0;
  cudaStream_t stream = nullptr;
  Slot slot[2];
  std::mutex m;
  std::condition_variable cv, cv_drain;
  std::deque<ReqRec> q;
  std::atomic<int64_t> queued{0};          // q.size(), readable without the lock (the idle spin)
  std::atomic<bool> stopping{false};
  int64_t submitted = 0, completed = 0;
  bool stop = false;
  cold_status first_error = COLD_OK;
  std::string error_text;
  std::thread worker;
  // statistics (written by the dispatcher, read by cold_server_drain)
  std::atomic<int64_t> batches{0}, batched_requests{0};

  cold_status assemble(Slot& s);
  void run();
};

// concatenate the slot's requests into one batch: a single pinned image [ad offsets | per group: offsets,
// ids] (16 B aligned segments), copied to the device with ONE cudaMemcpyAsync; the call then takes the
// device-batch path (no per-group staging copies inside the library), with host copies of the offsets
// from the pinned image
cold_status cold_server::assemble(Slot& s) {
  const int B = (int)s.recs.size();
  const int M = (int)groups.size();
  auto al = [](size_t x) { return (x + 15) / 16 * 16; };
  // sizes
  int64_t n_ads = 0;
  for (const ReqRec& q : s.recs) n_ads += q.n;
  std::vector<size_t> off_bytes(M, 0), id_bytes(M, 0);
  size_t total = al(sizeof(int32_t) * (B + 1));
  for (int g = 0; g < M; g++) {
    const cold_group& G = groups[g];
    if (G.side == COLD_CROSS || !s.recs[0].b->ids[g]) continue;
    if (G.side == COLD_USER || G.pooled) {
      const int64_t rows = G.side == COLD_USER ? B : n_ads;
      size_t nid = 0;
      for (const ReqRec& q : s.recs) {
        const int32_t* o = q.b->offs_host[g];
        const int32_t* aoq = q.b->ad_offsets_host;
        const int lo = G.side == COLD_USER ? q.r : aoq[q.r], hi = G.side == COLD_USER ? q.r + 1 : aoq[q.r + 1];
        nid += (size_t)(o[hi] - o[lo]);
      }
      off_bytes[g] = al(sizeof(int32_t) * (rows + 1));
      id_bytes[g] = al(sizeof(int32_t) * std::max<size_t>(nid, 1));
    } else {
      id_bytes[g] = al(sizeof(int32_t) * (size_t)n_ads);
    }
    total += off_bytes[g] + id_bytes[g];
  }
  if (!s.h_in.reserve(total)) return COLD_ERR_OOM;
  if (total > s.d_in_cap) {
    if (s.d_in) cudaFree(s.d_in);
    s.d_in = nullptr;
    s.d_in_cap = 0;
    if (cudaMalloc(&s.d_in, total * 3 / 2) != cudaSuccess) { cudaGetLastError(); return COLD_ERR_OOM; }
    s.d_in_cap = total * 3 / 2;
  }
  uint8_t* hbase = (uint8_t*)s.h_in.p;
  uint8_t* dbase = (uint8_t*)s.d_in;
  size_t pos = 0;
  int32_t* ao = (int32_t*)hbase;
  ao[0] = 0;
  for (int i = 0; i < B; i++) ao[i + 1] = ao[i] + s.recs[i].n;
  s.ao_host = ao;
  s.ao_dev = (const int32_t*)dbase;
  pos += al(sizeof(int32_t) * (B + 1));
  s.ids_dev.assign(M, nullptr);
  s.offs_dev.assign(M, nullptr);
  s.offs_host.assign(M, nullptr);
  for (int g = 0; g < M; g++) {
    const cold_group& G = groups[g];
    if (G.side == COLD_CROSS || !s.recs[0].b->ids[g]) continue;
    if (G.side == COLD_USER || G.pooled) {
      // CSR bags: offsets over requests (USER) or ads (AD pooled), ids concatenated in order
      int32_t* oo = (int32_t*)(hbase + pos);
      int32_t* ii = (int32_t*)(hbase + pos + off_bytes[g]);
      s.offs_host[g] = oo;
      s.offs_dev[g] = (const int32_t*)(dbase + pos);
      s.ids_dev[g] = (const int32_t*)(dbase + pos + off_bytes[g]);
      int64_t row = 0;
      oo[0] = 0;
      for (const ReqRec& q : s.recs) {
        const int32_t* o = q.b->offs_host[g];
        const int32_t* aoq = q.b->ad_offsets_host;
        const int lo = G.side == COLD_USER ? q.r : aoq[q.r], hi = G.side == COLD_USER ? q.r + 1 : aoq[q.r + 1];
        const int32_t* src = q.b->ids[g];
        const int32_t len_all = o[hi] - o[lo];
        memcpy(ii + oo[row], src + o[lo], sizeof(int32_t) * (size_t)len_all);   // the rows' bags are contiguous
        const int32_t shift = oo[row] - o[lo];
        for (int j = lo; j < hi; j++, row++) oo[row + 1] = o[j + 1] + shift;
      }
    } else {   // single-valued AD group: the request's ad slice
      int32_t* ii = (int32_t*)(hbase + pos);
      s.ids_dev[g] = (const int32_t*)(dbase + pos);
      for (int i = 0; i < B; i++) {
        const ReqRec& q = s.recs[i];
        memcpy(ii + ao[i], q.b->ids[g] + q.b->ad_offsets_host[q.r], sizeof(int32_t) * (size_t)q.n);
      }
    }
    pos += off_bytes[g] + id_bytes[g];
  }
  if (cudaMemcpyAsync(s.d_in, s.h_in.p, total, cudaMemcpyHostToDevice, stream) != cudaSuccess) return COLD_ERR_CUDA;
  return COLD_OK;
}

void cold_server::run() {
  cudaSetDevice(device);
  const int K = cfg.top_k;
  int cur = 0;
  auto fail_slot = [&](Slot& s, cold_status st) {
    std::lock_guard<std::mutex> lk(m);
    if (first_error == COLD_OK) { first_error = st; error_text = cold_last_error(); }
    for (const ReqRec& r : s.recs) __atomic_store_n(r.done_ns, (int64_t)-1, __ATOMIC_RELEASE);
    completed += (int64_t)s.recs.size();
    s.recs.clear();
    cv_drain.notify_all();
  };
  for (;;) {
    Slot& s = slot[cur];
    Slot& o = slot[cur ^ 1];
    {
      std::unique_lock<std::mutex> lk(m);
      if (!o.inflight) {
        if (q.empty() && !stop) {   // idle: spin up to 200 us for the next request (no wake-up latency), then block
          lk.unlock();
          const int64_t t_end = now_ns() + 200000;
          while (queued.load(std::memory_order_acquire) == 0 && !stopping.load(std::memory_order_relaxed) &&
                 now_ns() < t_end) {
          }
          lk.lock();
        }
        cv.wait(lk, [&] { return stop || !q.empty(); });
        if (q.empty() && stop) break;
        // optional short wait for a fuller batch when the GPU is idle
        if (cfg.max_wait_us > 0 && (int)q.size() < cfg.max_batch_requests)
          cv.wait_for(lk, std::chrono::microseconds(cfg.max_wait_us),
                      [&] { return stop || (int)q.size() >= cfg.max_batch_requests; });
      }
      int64_t ads = 0;
      while (!q.empty() && (int)s.recs.size() < cfg.max_batch_requests && ads + q.front().n <= cfg.max_batch_ads) {
        ads += q.front().n;
        s.recs.push_back(q.front());
        q.pop_front();
        queued.fetch_sub(1, std::memory_order_relaxed);
      }
    }
    if (!s.recs.empty()) {
      const int B = (int)s.recs.size();
      cold_status st = assemble(s);
      if (st == COLD_OK) {
        cold_batch db;
        memset(&db, 0, sizeof(db));
        db.num_requests = B;
        db.ad_offsets = s.ao_dev;
        db.ad_offsets_host = s.ao_host;
        db.ids = s.ids_dev.data();
        db.offs = s.offs_dev.data();
        db.offs_host = s.offs_host.data();
        st = cold_score_batch(ctx, &db, s.d_scores, stream);
        if (st == COLD_OK) st = cold_topk(ctx, s.d_scores, s.ao_dev, s.ao_host, B, K, nullptr, s.d_idx, s.d_key, stream);
        int32_t* hi = (int32_t*)s.h_res.p;
        float* hk = (float*)(hi + (size_t)cfg.max_batch_requests * K);
        if (st == COLD_OK &&
            (cudaMemcpyAsync(hi, s.d_idx, sizeof(int32_t) * (size_t)B * K, cudaMemcpyDeviceToHost, stream) ||
             cudaMemcpyAsync(hk, s.d_key, sizeof(float) * (size_t)B * K, cudaMemcpyDeviceToHost, stream) ||
             cudaEventRecord(s.done, stream)))
          st = COLD_ERR_CUDA;
      }
      if (st != COLD_OK) fail_slot(s, st);
      else {
        s.inflight = true;
        batches++;
        batched_requests += B;
      }
    }
    if (o.inflight) {   // publish the previous batch while this one runs
      const cudaError_t e = cudaEventSynchronize(o.done);
      o.inflight = false;
      if (e != cudaSuccess) {
        fail_slot(o, COLD_ERR_CUDA);
      } else {
        const int32_t* hi = (const int32_t*)o.h_res.p;
        const float* hk = (const float*)(hi + (size_t)cfg.max_batch_requests * K);
        const int64_t t = now_ns();
        for (size_t i = 0; i < o.recs.size(); i++) {
          const ReqRec& r = o.recs[i];
          memcpy(r.idx, hi + i * K, sizeof(int32_t) * K);
          memcpy(r.key, hk + i * K, sizeof(float) * K);
          __atomic_store_n(r.done_ns, t, __ATOMIC_RELEASE);
        }
        std::lock_guard<std::mutex> lk(m);
        completed += (int64_t)o.recs.size();
        o.recs.clear();
        cv_drain.notify_all();
      }
    }
    if (s.inflight) cur ^= 1;
  }
}

extern "C" cold_status cold_server_create(cold_ctx* ctx, const cold_server_config* cfg, cold_server** out) {
  if (!ctx || !cfg || !out) return COLD_ERR_INVALID_ARG;
  *out = nullptr;
  int M = 0, max_req = 0, device = 0;
  int64_t max_ads = 0;
  const cold_group* groups = nullptr;
  cold_ctx_describe(ctx, &M, &groups, &max_req, &max_ads, &device);
  if (cfg->max_batch_requests < 1 || cfg->max_batch_requests > max_req) return COLD_ERR_CAPACITY;
  if (cfg->max_batch_ads < 1 || cfg->max_batch_ads > max_ads) return COLD_ERR_CAPACITY;
  if (cfg->top_k < 1 || cfg->top_k > 4096) return COLD_ERR_K_RANGE;
  if (cfg->max_wait_us < 0) return COLD_ERR_INVALID_ARG;
  cold_server* s = new cold_server();
  s->ctx = ctx;
  s->cfg = *cfg;
  s->groups.assign(groups, groups + M);
  s->device = device;
  cudaSetDevice(device);
  bool ok = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) == cudaSuccess;
  const size_t K = (size_t)cfg->top_k, B = (size_t)cfg->max_batch_requests;
  for (Slot& sl : s->slot) {
    ok = ok && cudaMalloc(&sl.d_scores, sizeof(float) * (size_t)cfg->max_batch_ads) == cudaSuccess;
    ok = ok && cudaMalloc(&sl.d_idx, sizeof(int32_t) * B * K) == cudaSuccess;
    ok = ok && cudaMalloc(&sl.d_key, sizeof(float) * B * K) == cudaSuccess;
    ok = ok && sl.h_res.reserve(8 * B * K);
    ok = ok && cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    cold_server_destroy(s);
    return COLD_ERR_OOM;
  }
  s->worker = std::thread([s] { s->run(); });
  *out = s;
  return COLD_OK;
}

extern "C" void cold_server_destroy(cold_server* s) {
  if (!s) return;
  if (s->worker.joinable()) {
    {
      std::lock_guard<std::mutex> lk(s->m);
      s->stop = true;
      s->stopping.store(true);
    }
    s->cv.notify_all();
    s->worker.join();
  }
  cudaSetDevice(s->device);
  for (Slot& sl : s->slot) {
    if (sl.d_scores) cudaFree(sl.d_scores);
    if (sl.d_in) cudaFree(sl.d_in);
    if (sl.d_idx) cudaFree(sl.d_idx);
    if (sl.d_key) cudaFree(sl.d_key);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

extern "C" cold_status cold_server_submit(cold_server* s, const cold_batch* reqs, const int64_t* arrival_ns,
                                          int32_t* idx_out, float* key_out, int64_t* done_ns) {
  if (!s || !reqs || !idx_out || !key_out || !done_ns || !reqs->ad_offsets_host || !reqs->ids || !reqs->offs)
    return COLD_ERR_INVALID_ARG;
  const int R = reqs->num_requests;
  if (R < 1) return COLD_ERR_INVALID_ARG;
  const int32_t* ao = reqs->ad_offsets_host;
  const int K = s->cfg.top_k;
  if (ao[0] != 0) return COLD_ERR_INVALID_ARG;
  for (int r = 0; r < R; r++) {
    const int n = ao[r + 1] - ao[r];
    if (n < 1) return COLD_ERR_INVALID_ARG;
    if (n < K) return COLD_ERR_K_RANGE;
    if (n > s->cfg.max_batch_ads) return COLD_ERR_CAPACITY;
  }
  {   // the dispatcher copies the requests' slices on the CPU: every array must be host memory
    auto on_device = [](const void* p) {
      cudaPointerAttributes at;
      if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
      return at.type == cudaMemoryTypeDevice;
    };
    for (size_t g = 0; g < s->groups.size(); g++)
      if (on_device(reqs->ids[g]) || on_device(reqs->offs[g])) return COLD_ERR_INVALID_ARG;
  }
  for (size_t g = 0; g < s->groups.size(); g++) {   // bag groups need host offsets (the server copies slices)
    const cold_group& G = s->groups[g];
    if (reqs->ids[g] && (G.side == COLD_USER || (G.side == COLD_AD && G.pooled)) &&
        (!reqs->offs_host || !reqs->offs_host[g]))
      return COLD_ERR_INVALID_ARG;
  }
  for (int r = 0; r < R; r++) __atomic_store_n(done_ns + r, (int64_t)0, __ATOMIC_RELAXED);
  for (int r = 0; r < R; r++) {
    if (arrival_ns)   // open-loop replay: enqueue request r at its arrival time (monotonic clock)
      while (now_ns() < arrival_ns[r]) {
      }
    {
      std::lock_guard<std::mutex> lk(s->m);
      s->q.push_back(ReqRec{reqs, r, ao[r + 1] - ao[r], idx_out + (size_t)r * K, key_out + (size_t)r * K, done_ns + r});
      s->submitted++;
      s->queued.fetch_add(1, std::memory_order_release);
    }
    s->cv.notify_one();
  }
  return COLD_OK;
}

extern "C" cold_status cold_server_drain(cold_server* s, int64_t* batches, int64_t* requests) {
  if (!s) return COLD_ERR_INVALID_ARG;
  std::unique_lock<std::mutex> lk(s->m);
  s->cv_drain.wait(lk, [&] { return s->completed >= s->submitted; });
  if (batches) *batches = s->batches.load();
  if (requests) *requests = s->batched_requests.load();
  return s->first_error;
}
