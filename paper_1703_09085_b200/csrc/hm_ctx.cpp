// Context, device arena, profiling and matrix bookkeeping of libhm.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "hm_internal.h"

namespace hm {

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("HM_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

void* Ctx::pinned(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (pin_used + bytes > pin_cap) {
    // recycle: wait until every copy from the staging buffer has completed and
    // every kernel (auxiliary streams too) has read its in-place descriptors
    HM_CUDA(cudaDeviceSynchronize());
    pin_used = 0;
    if (bytes > pin_cap) {
      if (pin) cudaFreeHost(pin);
      pin = nullptr;
      size_t cap = std::max(bytes, (size_t)256 << 20);
      HM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pin), cap, cudaHostAllocMapped | cudaHostAllocPortable));
      pin_cap = cap;
    }
  }
  void* p = pin + pin_used;
  pin_used += bytes;
  return p;
}

int* Ctx::rank_alloc(size_t n) {
  static const bool off = [] { const char* e = std::getenv("HM_RANK_HOST"); return e && e[0] == '0'; }();
  if (off || n > 4096) return nullptr;
  if (!rank_host) {
    rank_cap = (size_t)1 << 16;
    HM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&rank_host), rank_cap * sizeof(int),
                          cudaHostAllocMapped | cudaHostAllocPortable));
  }
  if (rank_used + n > rank_cap) return nullptr;
  int* p = rank_host + rank_used;
  rank_used += n;
  return p;
}

void Ctx::trim(bool captures) {
  HM_CUDA(cudaStreamSynchronize(stream));
  if (captures) cap_free();
  if (ws) dfree(ws, ws_cap * sizeof(double));
  ws = nullptr;
  ws_cap = 0;
  if (sp) dfree(sp, sp_cap);
  sp = nullptr;
  sp_cap = 0;
  sp_top = 0;
  HM_CUDA(cudaStreamSynchronize(stream));
  if (pool) cudaMemPoolTrimTo(pool, 0);
}

void Ctx::cap_free() {
  for (auto& L : cap)
    if (L.data) dfree(L.data, L.ndoubles * sizeof(double));
  cap.clear();
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  cap_free();
  if (ws) dfree(ws, ws_cap * sizeof(double));
  if (sp) dfree(sp, sp_cap);
  cudaStreamSynchronize(stream);
  for (int i = 0; i < kAux; i++) {
    if (aux[i]) { cudaStreamSynchronize(aux[i]); cudaStreamDestroy(aux[i]); }
    if (ev_join[i]) cudaEventDestroy(ev_join[i]);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (pin) cudaFreeHost(pin);
  if (pool) cudaMemPoolDestroy(pool);
  if (plog) std::fclose(plog);
  if (rank_host) cudaFreeHost(rank_host);
}

double* Ctx::stack_ws(size_t ndoubles) {
  if (ndoubles > ws_cap) {
    if (ws) dfree(ws, ws_cap * sizeof(double));
    ws = nullptr;
    ws_cap = 0;
    const size_t cap = std::max(ndoubles + ndoubles / 8, (size_t)1 << 24);
    ws = static_cast<double*>(dmalloc(cap * sizeof(double)));   // throws HM_ENOMEM
    ws_cap = cap;
  }
  return ws;
}

void* Ctx::dmalloc(size_t bytes) {
  if (bytes == 0) bytes = 8;
  void* p = nullptr;
  if (has_alloc) {
    p = alloc.alloc(bytes, stream, alloc.user);
    if (!p) throw Error(HM_ENOMEM, "device allocation hook failed (" + std::to_string(bytes) + " B)");
    return p;
  }
  cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, bytes, pool, stream) : cudaMallocAsync(&p, bytes, stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(HM_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  return p;
}

void Ctx::dfree(void* p, size_t bytes) {
  if (!p) return;
  if (has_alloc) {
    alloc.free(p, bytes, stream, alloc.user);
    return;
  }
  cudaFreeAsync(p, stream);
}

cudaEvent_t Ctx::get_event() {
  if (!free_events.empty()) {
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  HM_CUDA(cudaEventCreate(&e));
  return e;
}

bool Ctx::multi_stream() {
  static const bool on = [] { const char* e = std::getenv("HM_STREAMS"); return !(e && e[0] == '0'); }();
  return on;
}

cudaStream_t Ctx::fork(int i) {
  if (!multi_stream()) return stream;
  if (!aux[i]) {
    HM_CUDA(cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking));
    HM_CUDA(cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming));
  }
  if (!ev_fork) HM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  HM_CUDA(cudaEventRecord(ev_fork, stream));
  HM_CUDA(cudaStreamWaitEvent(aux[i], ev_fork, 0));
  return aux[i];
}

void Ctx::join(int i) {
  if (!multi_stream() || !aux[i]) return;
  HM_CUDA(cudaEventRecord(ev_join[i], aux[i]));
  HM_CUDA(cudaStreamWaitEvent(stream, ev_join[i], 0));
}

void Ctx::prof_begin(int cls, cudaEvent_t* a, cudaStream_t st) {
  (void)cls;
  if (!prof) return;
  *a = get_event();
  HM_CUDA(cudaEventRecord(*a, st ? st : stream));
  if (plog && !pbase) {
    HM_CUDA(cudaEventCreate(&pbase));
    HM_CUDA(cudaEventRecord(pbase, stream));
  }
}

void Ctx::prof_end(int cls, cudaEvent_t a, double fl, double by, cudaStream_t st) {
  if (!prof || !a) return;
  cudaEvent_t b = get_event();
  cudaEventRecord(b, st ? st : stream);
  pend.push_back(Pending{cls, a, b, fl, by, std::move(note)});
  note.clear();
  if (pend.size() > 4096) prof_collect();
}

void Ctx::prof_collect() {
  for (auto& p : pend) {
    cudaEventSynchronize(p.b);
    float ms_ = 0.f;
    cudaEventElapsedTime(&ms_, p.a, p.b);
    ms[p.cls] += ms_;
    if (plog) {
      float t0 = 0.f;
      if (pbase) cudaEventElapsedTime(&t0, pbase, p.a);
      std::fprintf(plog, "%d %.4f %.4f %s\n", p.cls, t0, ms_, p.note.c_str());
    }
    launches[p.cls] += 1;
    flops[p.cls] += p.flops;
    bytes[p.cls] += p.bytes;
    free_events.push_back(p.a);
    free_events.push_back(p.b);
  }
  pend.clear();
}

void Ctx::sp_prepare() {
  if (sp_hwm > sp_cap) {
    if (sp) dfree(sp, sp_cap);
    sp = nullptr;
    sp_cap = 0;
    const size_t cap = sp_hwm + sp_hwm / 8;
    try {
      sp = static_cast<char*>(dmalloc(cap));
      sp_cap = cap;
    } catch (const Error&) {   // the arenas fall back to per-chunk allocations
      sp = nullptr;
    }
  }
  sp_top = 0;
  sp_hwm = 0;
}

void* Arena::alloc_bytes(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (stack_mode) {
    const size_t need = ctx->sp_top + bytes;
    ctx->sp_hwm = std::max(ctx->sp_hwm, need);
    if (need <= ctx->sp_cap) {
      void* p = ctx->sp + ctx->sp_top;
      ctx->sp_top = need;
      return p;
    }
    ctx->sp_top = need;   // account the overflow so the next operation sizes the pool
    void* p = ctx->dmalloc(bytes);
    blocks.push_back({p, bytes});
    return p;
  }
  if (bytes > cur_left) {
    if (bytes >= chunk_min) {   // large request: its own block, keep the current chunk
      void* p = ctx->dmalloc(bytes);
      blocks.push_back({p, bytes});
      return p;
    }
    const size_t sz = chunk_min;
    chunk_min = std::min(chunk_min * 2, (size_t)1 << 30);
    cur = static_cast<char*>(ctx->dmalloc(sz));
    blocks.push_back({cur, sz});
    cur_left = sz;
  }
  void* p = cur;
  cur += bytes;
  cur_left -= bytes;
  return p;
}

void Arena::release() {
  for (auto& b : blocks) ctx->dfree(b.first, b.second);
  blocks.clear();
  cur = nullptr;
  cur_left = 0;
  if (stack_mode && ctx->sp_top > mark) ctx->sp_top = mark;
}

void Mat::free_all(Ctx* c) {
  c->dfree(fpool.first, fpool.second);
  c->dfree(dpool.first, dpool.second);
  fpool = {nullptr, 0};
  dpool = {nullptr, 0};
}

std::vector<LeafDesc> leaf_table(const Mat& M) {
  const Tree& T = *M.tree;
  std::vector<LeafDesc> v(T.leaf_order.size());
  for (size_t i = 0; i < T.leaf_order.size(); i++) {
    const int b = T.leaf_order[i];
    LeafDesc& d = v[i];
    d.kind = T.bl_kind[b];
    d.row0 = T.cl_start[T.bl_row[b]];
    d.col0 = T.cl_start[T.bl_col[b]];
    d.m = T.cl_size[T.bl_row[b]];
    d.n = T.cl_size[T.bl_col[b]];
    d.k = (d.kind == HM_BLOCK_ADM) ? M.rank[b] : 0;
    d.A = M.pA[b];
    d.B = M.pB[b];
  }
  return v;
}

}  // namespace hm
