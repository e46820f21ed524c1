// Rebuild-and-swap FIB store on the GPU (SPEC update-engine; paper
// §3.6).
//
// The reference's FibStore keeps one active Snapshot {epoch, fib, tree}, a list
// of pending UpdateOps and retired snapshots awaiting reclamation.
// Here a snapshot's tree is a device FIB (lpm6cu_fib) and the whole rebuild —
// interval sweep and layout — runs on the GPU (build.cu) on the store's own
// stream, so lookups on other streams keep running during a commit. Publication
// is a pointer swap under a mutex held for a few instructions; readers pin with
// acquire/release and never wait on a rebuild.
//
// Reclamation is stream-ordered, which the CPU reference does not need: a
// reader's release only says the HOST is done with the snapshot, while lookups
// it queued may still be running. Release therefore records an event on the
// reader's stream, and a retired snapshot is freed only when no reader holds it
// and every such event has completed ("no reclamation-before-release").
#include <cuda_runtime.h>

#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "capi_internal.hpp"
#include "capi_util.hpp"
#include "lpm6/fib.hpp"
#include "lpm6/update.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// Re-throw a C ABI status as lpm6::Error (its message is the thread's last error).
void ck_status(int st) {
  if (st != 0) throw Error(static_cast<Errc>(st - 1), lpm6cu_last_error());
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    ck(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DevGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

std::vector<Prefix> to_rules(const lpm6cu_prefix* rules, uint64_t n) {
  std::vector<Prefix> out(n);
  if (n) std::memcpy(static_cast<void*>(out.data()), rules, n * sizeof(Prefix));  // same 32-byte layout
  return out;
}

FibTable table_of(const std::vector<Prefix>& rules, u32 default_nh) {
  FibTable t(default_nh);
  for (const Prefix& p : rules) t.insert(p);
  return t;
}

UpdateOp op_of(const lpm6_update_op& o) {
  UpdateOp op;
  op.kind = static_cast<UpdateKind>(o.kind);
  std::memcpy(static_cast<void*>(&op.prefix), &o.prefix, sizeof(Prefix));
  return op;
}

// Stage ops onto `view` in order; invalid ops are skipped and reported.
uint64_t stage_into(FibTable& view, const lpm6_update_op* ops, uint64_t n, int32_t* op_status,
                    std::vector<UpdateOp>* log) {
  uint64_t staged = 0;
  for (uint64_t i = 0; i < n; ++i) {
    int32_t st = 0;
    try {
      const UpdateOp op = op_of(ops[i]);
      apply_update(view, op);
      if (log) log->push_back(op);
      ++staged;
    } catch (const Error& e) {
      st = capi::status_of(e.code());
    }
    if (op_status) op_status[i] = st;
  }
  return staged;
}

}  // namespace

struct lpm6cu_snapshot {
  lpm6cu_store* store = nullptr;
  uint64_t epoch = 0;
  lpm6cu_fib* fib = nullptr;
  std::vector<Prefix> rules;
  // Guarded by store->mu. At most one fence per reader stream: events on one
  // stream complete in order, so a release re-records that stream's fence.
  struct Fence {
    cudaStream_t stream;
    cudaEvent_t event;
  };
  uint64_t refs = 0;
  std::vector<Fence> fences;

  // Only reclaim() deletes snapshots, after their fences completed (store_destroy
  // waits for them): no lookup can still read the FIB.
  ~lpm6cu_snapshot() {
    if (fib) capi::fib_destroy_quiesced(fib);
  }
};

struct lpm6cu_store {
  int device = 0;
  u32 default_nh = 0;
  lpm6cu_build_opts opts{};
  cudaStream_t build_stream = nullptr;

  std::mutex commit_mu;  // one committer at a time

  std::mutex stage_mu;  // staged view = active rules + pending ops, in order
  FibTable view;
  std::vector<UpdateOp> pending;

  std::mutex mu;  // active pointer, refs, fences, retired list (held briefly)
  lpm6cu_snapshot* active = nullptr;
  std::vector<lpm6cu_snapshot*> retired;
  std::vector<cudaEvent_t> event_pool;
  lpm6cu_store_stats stats{};

  // Detach retired snapshots that no reader holds and whose fences completed.
  std::vector<lpm6cu_snapshot*> collect(bool wait) {  // under mu
    std::vector<lpm6cu_snapshot*> dead;
    for (size_t i = 0; i < retired.size();) {
      lpm6cu_snapshot* s = retired[i];
      bool done = s->refs == 0;
      for (size_t f = 0; done && f < s->fences.size(); ++f) {
        const cudaError_t q = wait ? cudaEventSynchronize(s->fences[f].event) : cudaEventQuery(s->fences[f].event);
        if (q == cudaErrorNotReady) done = false;
        else if (q != cudaSuccess) cudaGetLastError();  // a failed fence cannot become ready; treat as done
      }
      if (!done) {
        ++i;
        continue;
      }
      for (const auto& f : s->fences) event_pool.push_back(f.event);
      s->fences.clear();
      dead.push_back(s);
      retired[i] = retired.back();
      retired.pop_back();
      ++stats.reclaimed;
    }
    stats.retired = retired.size();
    return dead;
  }

  void reclaim(bool wait) {
    std::vector<lpm6cu_snapshot*> dead;
    {
      std::lock_guard<std::mutex> lk(mu);
      dead = collect(wait);
    }
    for (lpm6cu_snapshot* s : dead) delete s;  // cudaFree outside the lock
  }

  lpm6cu_snapshot* build(std::vector<Prefix> rules, uint64_t epoch) {
    auto snap = std::make_unique<lpm6cu_snapshot>();
    snap->store = this;
    snap->epoch = epoch;
    const auto t0 = std::chrono::steady_clock::now();
    ck_status(lpm6cu_fib_build_device(device, reinterpret_cast<const lpm6cu_prefix*>(rules.data()), rules.size(),
                                      default_nh, &opts, build_stream, &snap->fib));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    snap->rules = std::move(rules);
    std::lock_guard<std::mutex> lk(mu);
    stats.last_build_ms = ms;
    return snap.release();
  }
};

extern "C" {

int lpm6_parse_update(const char* line, lpm6_update_op* op) {
  return guard([&] {
    if (!line || !op) throw Error(Errc::InvalidArgument, "NULL argument");
    const UpdateOp u = parse_update(line);
    std::memset(op, 0, sizeof *op);
    op->kind = static_cast<uint32_t>(u.kind);
    std::memcpy(&op->prefix, &u.prefix, sizeof(Prefix));
  });
}

int lpm6_apply_updates(const lpm6cu_prefix* rules, uint64_t n, const lpm6_update_op* ops, uint64_t n_ops,
                       lpm6cu_prefix* out, uint64_t cap, uint64_t* out_n, uint64_t* staged, int32_t* op_status) {
  return guard([&] {
    if ((n && !rules) || (n_ops && !ops) || !out_n) throw Error(Errc::InvalidArgument, "NULL argument");
    FibTable view = table_of(to_rules(rules, n), 0);
    const uint64_t k = stage_into(view, ops, n_ops, op_status, nullptr);
    if (staged) *staged = k;
    *out_n = view.size();
    if (!out) return;
    if (cap < view.size()) throw Error(Errc::InvalidArgument, "output capacity below the resulting rule count");
    std::memcpy(out, view.entries().data(), view.size() * sizeof(Prefix));
  });
}

int lpm6cu_store_create(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                        const lpm6cu_build_opts* opts, lpm6cu_store** out) {
  return guard([&] {
    if ((n && !rules) || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    auto s = std::make_unique<lpm6cu_store>();
    s->device = device;
    s->default_nh = default_nh;
    s->opts.merge_adjacent = 1;
    if (opts) s->opts = *opts;
    std::vector<Prefix> r = to_rules(rules, n);
    s->view = table_of(r, default_nh);  // DuplicatePrefix / ReservedNextHop as FibTable::insert
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw Error(Errc::CudaError, "no CUDA device " + std::to_string(device));
    DevGuard dg(device);
    ck(cudaStreamCreateWithFlags(&s->build_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    try {
      s->active = s->build(std::move(r), 1);  // acquire with no updates ever -> epoch 1
    } catch (...) {
      cudaStreamDestroy(s->build_stream);
      throw;
    }
    // Reserve room for the next snapshot's line array too: every commit builds a new
    // array while the active one is still alive, and growing the pool maps device
    // memory through the driver (tens of ms in a process that holds a lot of it).
    // The pool keeps freed memory, so the first commit then allocates from it.
    {
      lpm6cu_geometry g{};
      if (lpm6cu_fib_geometry(s->active->fib, &g) == LPM6CU_OK && g.total_words) {
        void* spare = nullptr;
        const size_t bytes = static_cast<size_t>(g.total_words) * 8 + (static_cast<size_t>(g.total_words) * 8) / 4;
        if (cudaMallocFromPoolAsync(&spare, bytes, capi::fib_line_pool(device), s->build_stream) == cudaSuccess) {
          cudaFreeAsync(spare, s->build_stream);
          cudaStreamSynchronize(s->build_stream);
        } else {
          cudaGetLastError();  // only a warm-up: the first commit grows the pool instead
        }
      }
    }
    s->stats.epoch = 1;
    s->stats.active_rules = s->active->rules.size();
    *out = s.release();
  });
}

int lpm6cu_store_destroy(lpm6cu_store* s) {
  return guard([&] {
    if (!s) return;
    DevGuard dg(s->device);
    {
      std::lock_guard<std::mutex> lk(s->mu);
      if (s->active->refs) throw Error(Errc::InvalidArgument, "store destroyed while a snapshot is acquired");
      for (lpm6cu_snapshot* r : s->retired)
        if (r->refs) throw Error(Errc::InvalidArgument, "store destroyed while a snapshot is acquired");
      s->retired.push_back(s->active);
      s->active = nullptr;
    }
    s->reclaim(true);
    for (cudaEvent_t e : s->event_pool) cudaEventDestroy(e);
    cudaStreamDestroy(s->build_stream);
    delete s;
  });
}

int lpm6cu_store_stage(lpm6cu_store* s, const lpm6_update_op* ops, uint64_t n, uint64_t* staged,
                       int32_t* op_status) {
  return guard([&] {
    if (!s || (n && !ops)) throw Error(Errc::InvalidArgument, "NULL argument");
    std::lock_guard<std::mutex> lk(s->stage_mu);
    const uint64_t k = stage_into(s->view, ops, n, op_status, &s->pending);
    if (staged) *staged = k;
  });
}

int lpm6cu_store_commit(lpm6cu_store* s, uint64_t* epoch) {
  return guard([&] {
    if (!s) throw Error(Errc::InvalidArgument, "NULL store");
    std::lock_guard<std::mutex> ck_(s->commit_mu);
    std::vector<Prefix> rules;
    size_t taken = 0;
    {
      std::lock_guard<std::mutex> lk(s->stage_mu);
      taken = s->pending.size();
      if (taken) rules = s->view.entries();  // = active rules with the first `taken` pending ops applied
    }
    uint64_t cur = 0;
    {
      std::lock_guard<std::mutex> lk(s->mu);
      cur = s->active->epoch;
    }
    if (taken == 0) {  // empty pending -> same epoch, same active handle
      if (epoch) *epoch = cur;
      return;
    }
    DevGuard dg(s->device);
    // Rebuild off the lookup path; a failure leaves the active snapshot and the
    // pending ops untouched.
    lpm6cu_snapshot* next = s->build(std::move(rules), cur + 1);
    {
      // The new FIB inherits the active one's kernel config (shape and the tuned
      // line path, lpm6cu_fib_tune_line_path); the staged levels are re-resolved
      // for the new tree. Only commits retire the active snapshot, and this one
      // holds commit_mu, so reading it here is safe.
      const lpm6cu_fib* prev = nullptr;
      {
        std::lock_guard<std::mutex> lk(s->mu);
        prev = s->active->fib;
      }
      lpm6cu_kernel_config c{};
      if (lpm6cu_fib_kernel_config(prev, &c) == LPM6CU_OK) {
        c.smem_levels = 0xFF;
        if (lpm6cu_fib_set_kernel_config(next->fib, &c) != LPM6CU_OK) {
          lpm6cu_kernel_config d{};
          d.smem_levels = 0xFF;
          lpm6cu_fib_set_kernel_config(next->fib, &d);  // shape not available for this tree: defaults
        }
      }
    }
    {
      std::lock_guard<std::mutex> lk(s->stage_mu);
      s->pending.erase(s->pending.begin(), s->pending.begin() + static_cast<std::ptrdiff_t>(taken));
    }
    {
      const auto t0 = std::chrono::steady_clock::now();
      std::lock_guard<std::mutex> lk(s->mu);
      s->retired.push_back(s->active);  // "atomic swap": one pointer replacement
      s->active = next;
      s->stats.last_publish_us =
          std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      s->stats.epoch = next->epoch;
      s->stats.active_rules = next->rules.size();
      ++s->stats.commits;
    }
    capi::BuildTrace tr("store commit");
    s->reclaim(false);
    tr.mark("reclaim");
    if (epoch) *epoch = next->epoch;
  });
}

int lpm6cu_store_acquire(lpm6cu_store* s, lpm6cu_snapshot** snap) {
  return guard([&] {
    if (!s || !snap) throw Error(Errc::InvalidArgument, "NULL argument");
    std::lock_guard<std::mutex> lk(s->mu);
    ++s->active->refs;
    *snap = s->active;
  });
}

int lpm6cu_store_release(lpm6cu_snapshot* snap, void* stream) {
  return guard([&] {
    if (!snap) throw Error(Errc::InvalidArgument, "NULL snapshot");
    lpm6cu_store* s = snap->store;
    DevGuard dg(s->device);
    bool retired = false;
    {
      std::lock_guard<std::mutex> lk(s->mu);
      if (snap->refs == 0) throw Error(Errc::InvalidArgument, "snapshot released more often than acquired");
      --snap->refs;  // before anything that can fail: a failed fence must not pin the snapshot
      retired = snap != s->active;
      const auto st = static_cast<cudaStream_t>(stream);
      // Recycle fences that have completed; re-record this stream's fence if it has one.
      bool mine = false;
      cudaEvent_t e = nullptr;
      for (size_t i = 0; i < snap->fences.size();) {
        auto& f = snap->fences[i];
        if (f.stream == st) {
          mine = true;
          e = f.event;
        } else if (cudaEventQuery(f.event) == cudaSuccess) {
          s->event_pool.push_back(f.event);
          f = snap->fences.back();
          snap->fences.pop_back();
          continue;
        }
        ++i;
      }
      cudaGetLastError();  // a query of a failed stream's event reports its error; it stays a fence
      if (!e) {
        e = s->event_pool.empty() ? nullptr : s->event_pool.back();
        if (e) s->event_pool.pop_back();
        else if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
      }
      if (!e || cudaEventRecord(e, st) != cudaSuccess) {
        // No fence available: wait for this reader's stream instead (rare; never unsafe).
        if (e && !mine) s->event_pool.push_back(e);
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize (release without a fence)");
      } else if (!mine) {
        snap->fences.push_back({st, e});
      }
    }
    if (retired) s->reclaim(false);
  });
}

int lpm6cu_snapshot_info(const lpm6cu_snapshot* snap, uint64_t* epoch, const lpm6cu_fib** fib, uint64_t* n_rules) {
  return guard([&] {
    if (!snap) throw Error(Errc::InvalidArgument, "NULL snapshot");
    if (epoch) *epoch = snap->epoch;
    if (fib) *fib = snap->fib;
    if (n_rules) *n_rules = snap->rules.size();
  });
}

int lpm6cu_snapshot_rules(const lpm6cu_snapshot* snap, lpm6cu_prefix* out, uint64_t cap) {
  return guard([&] {
    if (!snap || (!out && !snap->rules.empty())) throw Error(Errc::InvalidArgument, "NULL argument");
    if (cap < snap->rules.size()) throw Error(Errc::InvalidArgument, "capacity below the snapshot's rule count");
    if (!snap->rules.empty()) std::memcpy(out, snap->rules.data(), snap->rules.size() * sizeof(Prefix));
  });
}

int lpm6cu_store_lookup_batch(lpm6cu_store* s, const void* addrs, uint64_t n, void* out, void* stream,
                              uint64_t* epoch) {
  lpm6cu_snapshot* snap = nullptr;
  int st = lpm6cu_store_acquire(s, &snap);
  if (st) return st;
  st = lpm6cu_lookup_batch(snap->fib, addrs, n, out, stream);
  if (epoch) *epoch = snap->epoch;
  const std::string msg = st ? lpm6cu_last_error() : "";
  const int rs = lpm6cu_store_release(snap, stream);
  if (st) lpm6::capi::set_error(msg);  // report the lookup's failure, not the release's
  return st ? st : rs;
}

int lpm6cu_store_reclaim(lpm6cu_store* s) {
  return guard([&] {
    if (!s) throw Error(Errc::InvalidArgument, "NULL store");
    DevGuard dg(s->device);
    s->reclaim(false);
  });
}

int lpm6cu_store_stats_get(lpm6cu_store* s, lpm6cu_store_stats* out) {
  return guard([&] {
    if (!s || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    {
      std::lock_guard<std::mutex> lk(s->mu);
      *out = s->stats;
      out->fences = s->active->fences.size();
      for (const lpm6cu_snapshot* r : s->retired) out->fences += r->fences.size();
    }
    std::lock_guard<std::mutex> lk(s->stage_mu);
    out->pending_ops = s->pending.size();
  });
}

}  // extern "C"
