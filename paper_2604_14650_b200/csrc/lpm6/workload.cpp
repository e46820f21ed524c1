// Seeded generators for the five BASELINE workloads.
//
// Pinned choices (DESIGN.md §3 repeats them):
//  * C0: 1,000 prefixes, lengths U[/16,/64]; each prefix after the first is, with
//    p = 0.2, a more-specific of a random earlier prefix (extra bits random);
//    plus ::/0. Next hops U[1,255].
//  * C1 (also C3): 200,000 prefixes = 2,000 aggregates (/16-/24 blocks in
//    2000::/3) + 198,000 routes with lengths 45% /48, 20% /32-/40, 25% /41-/47,
//    10% /49-/64. A route is, with p = 0.3, a more-specific of a random earlier
//    route (nesting depth <= 4 below its aggregate); otherwise it sits in a
//    random aggregate. Plus ::/0. Next hops U[1,255].
//  * C2 (also C4): 1,000,000 prefixes, 10,000 aggregates, C1's length shares
//    with the /32-/40 bucket widened to /16-/40, nesting depth <= 6, next hops
//    U[1,65535], no ::/0 (uniform queries exercise no-match -> default 0).
//  * Rules whose range would put a boundary on the sentinel key are redrawn.
#include "lpm6/workload.hpp"

#include <cmath>
#include <thread>

namespace lpm6 {

namespace {

struct Rng {
  u64 s;
  explicit Rng(u64 seed) : s(seed) {}
  u64 next() { return mix64(s += 0x9E3779B97F4A7C15ull); }
  u64 below(u64 n) { return next() % n; }
  int range(int lo, int hi) { return lo + static_cast<int>(below(static_cast<u64>(hi - lo + 1))); }
  double unit() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
};

inline u64 keep_mask(int len) { return len == 0 ? 0ull : (~0ull << (64 - len)); }

struct Node {
  u64 top;
  int len;
  int depth;
};

struct Builder {
  FibTable fib;
  std::vector<Node> nodes;

  bool add(u64 top, int len, u32 nh, int depth) {
    top &= keep_mask(len);
    const u128 end = u128(top) + (u128(1) << (64 - len));
    if (top == kSentinelKey || end == u128(kSentinelKey)) return false;  // sentinel collision
    if (fib.find(u128(top) << 64, len)) return false;
    fib.insert(Prefix{u128(top) << 64, len, nh});
    nodes.push_back(Node{top, len, depth});
    return true;
  }
};

FibTable gen_c0(u64 seed) {
  Rng r(seed);
  Builder b;
  b.fib.insert(Prefix{0, 0, static_cast<u32>(r.range(1, 255))});  // ::/0
  size_t placed = 0;
  while (placed < 1000) {
    int len;
    u64 top;
    if (!b.nodes.empty() && r.unit() < 0.2) {
      const Node& p = b.nodes[r.below(b.nodes.size())];
      if (p.len >= 64) continue;
      len = r.range(p.len + 1 > 16 ? p.len + 1 : 16, 64);
      top = p.top | (r.next() & ~keep_mask(p.len));
    } else {
      len = r.range(16, 64);
      top = r.next();
    }
    if (b.add(top, len, static_cast<u32>(r.range(1, 255)), 0)) ++placed;
  }
  return std::move(b.fib);
}

// Backbone-like generator shared by C1 (200K) and C2 (1M).
FibTable gen_backbone(u64 seed, size_t n_total, size_t n_agg, int low_bucket_min, int max_depth,
                      u32 max_nh, bool default_route) {
  Rng r(seed);
  Builder b;
  b.nodes.reserve(n_total);
  auto nh = [&] { return static_cast<u32>(1 + r.below(max_nh)); };
  if (default_route) b.fib.insert(Prefix{0, 0, nh()});
  const u64 block = 1ull << 61;  // 2000::/3
  while (b.nodes.size() < n_agg) b.add(block | (r.next() >> 3), r.range(16, 24), nh(), 0);
  const size_t first_route = b.nodes.size();
  while (b.nodes.size() < n_total) {
    const double u = r.unit();
    const int len = u < 0.45 ? 48 : u < 0.65 ? r.range(low_bucket_min, 40) : u < 0.90 ? r.range(41, 47)
                                                                                       : r.range(49, 64);
    u64 top = 0;
    int depth = -1;
    if (b.nodes.size() > first_route && r.unit() < 0.3) {  // more-specific of an earlier route
      for (int t = 0; t < 8 && depth < 0; ++t) {
        const Node& p = b.nodes[first_route + r.below(b.nodes.size() - first_route)];
        if (p.len < len && p.depth < max_depth) {
          top = p.top | (r.next() & ~keep_mask(p.len));
          depth = p.depth + 1;
        }
      }
    }
    for (int t = 0; t < 8 && depth < 0; ++t) {  // inside a random aggregate
      const Node& a = b.nodes[r.below(first_route)];
      if (a.len < len) {
        top = a.top | (r.next() & ~keep_mask(a.len));
        depth = 1;
      }
    }
    if (depth < 0) {  // no shorter aggregate found: a free-standing route in 2000::/3
      top = block | (r.next() >> 3);
      depth = 1;
    }
    b.add(top, len, nh(), depth);
  }
  return std::move(b.fib);
}

}  // namespace

WorkloadConfig workload_config(int id) {
  WorkloadConfig c;
  c.id = id;
  switch (id) {
    case kC0:
      c.name = "C0";
      c.fib_kind = 0;
      c.n_queries = 1ull << 20;
      c.query_seed = 0xC0C0;
      c.in_prefix_frac = 0.7;
      c.uniform_kind = kUniform128;
      c.value_bytes = 1;
      break;
    case kC1:
      c.name = "C1";
      c.fib_kind = 1;
      c.n_queries = 1ull << 28;
      c.query_seed = 0xC1C1;
      c.in_prefix_frac = 0.9;
      c.uniform_kind = kUniform2000;
      c.value_bytes = 1;
      break;
    case kC2:
      c.name = "C2";
      c.fib_kind = 2;
      c.n_queries = 1ull << 30;
      c.query_seed = 0xC2C2;
      c.in_prefix_frac = 0.5;
      c.uniform_kind = kUniform128;
      c.value_bytes = 2;
      break;
    case kC3a:
      c.name = "C3a";
      c.fib_kind = 1;
      c.n_queries = 1ull << 28;
      c.query_seed = 0xC3A0;
      c.in_prefix_frac = 0.0;
      c.uniform_kind = kUniform128;
      c.value_bytes = 1;
      break;
    case kC3b:
      c.name = "C3b";
      c.fib_kind = 1;
      c.n_queries = 1ull << 28;
      c.query_seed = 0xC3B0;
      c.in_prefix_frac = 1.0;
      c.pick = kPickZipf;
      c.zipf_s = 1.1;
      c.value_bytes = 1;
      break;
    case kC4:
      c.name = "C4";
      c.fib_kind = 2;
      c.n_queries = 1ull << 33;
      c.chunk = 1ull << 26;
      c.query_seed = 0xC4C4;
      c.in_prefix_frac = 0.5;
      c.uniform_kind = kUniform128;
      c.value_bytes = 2;
      break;
    default:
      throw Error(Errc::InvalidArgument, "unknown workload id " + std::to_string(id));
  }
  return c;
}

FibTable make_fib(int fib_kind) {
  switch (fib_kind) {
    case 0:
      return gen_c0(0x5EED0000C0ull);
    case 1:
      return gen_backbone(0x5EED0000C1ull, 200000, 2000, 32, 4, 255, true);
    case 2:
      return gen_backbone(0x5EED0000C2ull, 1000000, 10000, 16, 6, 65535, false);
    default:
      throw Error(Errc::InvalidArgument, "unknown fib kind " + std::to_string(fib_kind));
  }
}

QueryTables make_query_tables(std::span<const Prefix> e, const WorkloadConfig& cfg) {
  QueryTables t;
  t.top.resize(e.size());
  t.len.resize(e.size());
  for (size_t i = 0; i < e.size(); ++i) {
    t.top[i] = e[i].top64();
    t.len[i] = static_cast<u8>(e[i].length);
  }
  if (cfg.pick == kPickZipf && !e.empty()) {
    const size_t n = e.size();
    t.cdf.resize(n);
    double acc = 0;
    for (size_t r = 0; r < n; ++r) acc += std::pow(static_cast<double>(r + 1), -cfg.zipf_s);
    double run = 0;
    for (size_t r = 0; r < n; ++r) {
      run += std::pow(static_cast<double>(r + 1), -cfg.zipf_s);
      t.cdf[r] = run / acc;
    }
    t.cdf[n - 1] = 1.0;
    t.perm.resize(n);
    for (size_t i = 0; i < n; ++i) t.perm[i] = static_cast<u32>(i);
    Rng rng(cfg.query_seed ^ 0x217F);
    for (size_t i = n - 1; i > 0; --i) std::swap(t.perm[i], t.perm[rng.below(i + 1)]);
  }
  return t;
}

QuerySpec make_query_spec(const WorkloadConfig& cfg, const QueryTables& t) {
  QuerySpec s{};
  s.seed = cfg.query_seed;
  s.in_prefix_thr = cfg.in_prefix_frac >= 1.0 ? (1ull << 53)
                                               : static_cast<u64>(cfg.in_prefix_frac * 9007199254740992.0);
  s.uniform_kind = cfg.uniform_kind;
  s.pick = cfg.pick;
  s.n_prefixes = t.top.size();
  s.pfx_top = t.top.data();
  s.pfx_len = t.len.data();
  s.zipf_cdf = t.cdf.empty() ? nullptr : t.cdf.data();
  s.zipf_perm = t.perm.empty() ? nullptr : t.perm.data();
  return s;
}

void gen_queries_host(const QuerySpec& spec, u64 first, u64 n, u64* out, int threads) {
  auto work = [&](u64 lo, u64 hi) {
    for (u64 i = lo; i < hi; ++i) gen_query(spec, first + i, &out[2 * i], &out[2 * i + 1]);
  };
  if (threads <= 1 || n < (1u << 16)) {
    work(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const u64 chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const u64 lo = std::min<u64>(n, t * chunk), hi = std::min<u64>(n, lo + chunk);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
}

}  // namespace lpm6
