#include "lpm6/snapshot.hpp"

#include <bit>
#include <cstdio>
#include <cstring>
#include <fstream>

namespace lpm6 {

static_assert(std::endian::native == std::endian::little, "snapshot I/O assumes a little-endian host");

namespace {

[[noreturn]] void bad(const std::string& why) { throw Error(Errc::BadSnapshotFile, "PBT1 snapshot: " + why); }

template <class T>
T get(const unsigned char* p) {
  T v;
  std::memcpy(&v, p, sizeof v);
  return v;
}

template <class T>
void put(std::vector<unsigned char>& out, T v) {
  const auto* p = reinterpret_cast<const unsigned char*>(&v);
  out.insert(out.end(), p, p + sizeof v);
}

// Separator j (0-based) of node n at internal level l: first key of child n*b + j + 1
// (decision S:244), or the sentinel past the m real keys.
u64 ref_separator(const RefGeometry& g, const u64* boundaries, u64 span_child, u64 n, u32 j) {
  const u64 idx = (n * g.b + j + 1) * span_child;
  return idx < g.num_keys ? boundaries[idx] : kSentinelKey;
}

}  // namespace

RefGeometry plan_ref_geometry(u64 m, u32 k) {
  if (k < 2) throw Error(Errc::InvalidArgument, "k must be >= 2");
  RefGeometry g;
  g.k = k;
  g.b = k + 1;
  g.num_keys = m;
  u64 cap = k;
  while (cap < m) {
    cap *= g.b;
    ++g.depth;
  }
  g.level_start.resize(g.depth + 1);
  u64 start = 0, nodes = 1;
  for (u32 l = 0; l <= g.depth; ++l) {  // level_start(i) = k (b^i - 1) / (b - 1)
    g.level_start[l] = start;
    start += nodes * k;
    nodes *= g.b;
  }
  g.leaf_start = g.level_start[g.depth];
  g.allocated_leaf_nodes = (m + k - 1) / k;
  return g;
}

std::vector<unsigned char> save_snapshot(const IntervalMap& map, u32 k) {
  const u64 m = map.size();
  if (m == 0) throw Error(Errc::InvalidArgument, "an interval map has at least one boundary");
  if (k > 0xFFFF) throw Error(Errc::InvalidArgument, "k must fit in u16");
  for (u64 i = 0; i < m; ++i)
    if (map.boundaries[i] == kSentinelKey) throw Error(Errc::SentinelCollision, "boundary equals the sentinel key");
  const RefGeometry g = plan_ref_geometry(m, k);
  std::vector<unsigned char> out;
  out.reserve(kSnapshotHeaderBytes + g.total_key_slots() * 8 + g.allocated_leaf_nodes * k * 4);
  out.insert(out.end(), {'P', 'B', 'T', '1'});
  put<u16>(out, kSnapshotVersion);
  put<u16>(out, static_cast<u16>(k));
  put<u16>(out, static_cast<u16>(g.depth));
  put<u64>(out, m);
  put<u64>(out, g.allocated_leaf_nodes);
  // internal levels, fully allocated (b^l nodes each)
  u64 nodes = 1, span_child = k;
  for (u32 l = 1; l < g.depth; ++l) span_child *= g.b;  // leaf keys under a child of a level-0 node
  for (u32 l = 0; l < g.depth; ++l) {
    for (u64 n = 0; n < nodes; ++n)
      for (u32 j = 0; j < k; ++j) put<u64>(out, ref_separator(g, map.boundaries.data(), span_child, n, j));
    nodes *= g.b;
    span_child /= g.b;
  }
  const u64 slots = g.allocated_leaf_nodes * k;
  for (u64 i = 0; i < slots; ++i) put<u64>(out, i < m ? map.boundaries[i] : kSentinelKey);
  for (u64 i = 0; i < slots; ++i) put<u32>(out, map.next_hops[i < m ? i : m - 1]);
  return out;
}

LoadedSnapshot load_snapshot(const void* data, u64 size, u32 default_next_hop) {
  const auto* p = static_cast<const unsigned char*>(data);
  if (!p || size < kSnapshotHeaderBytes) bad("truncated header");
  if (std::memcmp(p, "PBT1", 4) != 0) bad("bad magic");
  const u16 version = get<u16>(p + 4), k = get<u16>(p + 6), depth = get<u16>(p + 8);
  const u64 m = get<u64>(p + 10), alloc = get<u64>(p + 18);
  if (version != kSnapshotVersion) bad("unsupported version " + std::to_string(version));
  if (k < 2) bad("k < 2");
  if (m == 0) bad("no keys");
  if (m > size / 8) bad("key count exceeds the file size");
  const RefGeometry g = plan_ref_geometry(m, k);
  if (g.depth != depth) bad("depth " + std::to_string(depth) + " does not match m and k (" + std::to_string(g.depth) + ")");
  if (alloc != g.allocated_leaf_nodes) bad("allocated_leaf_nodes != ceil(m / k)");
  const u64 slots = alloc * k;
  if (size != kSnapshotHeaderBytes + g.total_key_slots() * 8 + slots * 4) bad("size does not match the geometry");
  const unsigned char* keys = p + kSnapshotHeaderBytes;
  const unsigned char* vals = keys + g.total_key_slots() * 8;
  auto key = [&](u64 i) { return get<u64>(keys + 8 * i); };
  auto val = [&](u64 i) { return get<u32>(vals + 4 * i); };

  LoadedSnapshot out;
  out.geometry = g;
  IntervalMap& map = out.map;
  map.default_next_hop = default_next_hop;
  map.boundaries.resize(m);
  map.next_hops.resize(m);
  for (u64 i = 0; i < m; ++i) {
    map.boundaries[i] = key(g.leaf_start + i);
    map.next_hops[i] = val(i);
    if (map.next_hops[i] == kUnresolved) bad("reserved next hop in the value array");
    if (i > 0 && map.boundaries[i] <= map.boundaries[i - 1]) bad("leaf keys not strictly increasing");
  }
  if (map.boundaries[0] != 0) bad("first boundary is not 0");
  if (map.boundaries[m - 1] == kSentinelKey) bad("boundary equals the sentinel key");
  for (u64 i = m; i < slots; ++i) {
    if (key(g.leaf_start + i) != kSentinelKey) bad("leaf padding is not the sentinel");
    if (val(i) != map.next_hops[m - 1]) bad("value padding does not replicate the last value");
  }
  u64 nodes = 1, span_child = k;
  for (u32 l = 1; l < g.depth; ++l) span_child *= g.b;
  for (u32 l = 0; l < g.depth; ++l) {
    for (u64 n = 0; n < nodes; ++n)
      for (u32 j = 0; j < k; ++j)
        if (key(g.level_start[l] + n * k + j) != ref_separator(g, map.boundaries.data(), span_child, n, j))
          bad("internal separator mismatch at level " + std::to_string(l));
    nodes *= g.b;
    span_child /= g.b;
  }
  return out;
}

std::vector<unsigned char> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw Error(Errc::Io, "cannot open " + path);
  const std::streamoff n = in.tellg();
  std::vector<unsigned char> buf(static_cast<size_t>(n));
  in.seekg(0);
  if (n > 0 && !in.read(reinterpret_cast<char*>(buf.data()), n)) throw Error(Errc::Io, "cannot read " + path);
  return buf;
}

void write_file(const std::string& path, const void* data, u64 size) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Error(Errc::Io, "cannot create " + path);
  if (size && !out.write(static_cast<const char*>(data), static_cast<std::streamsize>(size)))
    throw Error(Errc::Io, "cannot write " + path);
}

u64 trace_header_count(const unsigned char* p, u64 header_bytes, u64 size) {
  if (!p || header_bytes < kTraceHeaderBytes || size < kTraceHeaderBytes)
    throw Error(Errc::BadTraceFile, "PBTR trace: truncated header");
  if (std::memcmp(p, "PBTR", 4) != 0) throw Error(Errc::BadTraceFile, "PBTR trace: bad magic");
  if (get<u16>(p + 4) != kTraceVersion) throw Error(Errc::BadTraceFile, "PBTR trace: unsupported version");
  const u64 n = get<u64>(p + 8);
  if (n > (size - kTraceHeaderBytes) / 8 || size != kTraceHeaderBytes + n * 8)
    throw Error(Errc::BadTraceFile, "PBTR trace: size does not match the key count");
  return n;
}

std::vector<unsigned char> save_trace(const u64* keys, u64 n) {
  std::vector<unsigned char> out;
  out.reserve(kTraceHeaderBytes + n * 8);
  out.insert(out.end(), {'P', 'B', 'T', 'R'});
  put<u16>(out, kTraceVersion);
  put<u16>(out, 0);
  put<u64>(out, n);
  const auto* b = reinterpret_cast<const unsigned char*>(keys);
  out.insert(out.end(), b, b + n * 8);
  return out;
}

}  // namespace lpm6
