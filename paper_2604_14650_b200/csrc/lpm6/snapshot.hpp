// Reference file formats on the lookup path's input side.
//
// PBT1 — the reference's binary tree snapshot (tree.hpp:90-96):
//   "PBT1", u16 version = 1, u16 k, u16 depth, u64 m, u64 allocated_leaf_nodes,
//   then the key array (u64 LE) and the value array (u32 LE) of its LinearizedTree:
//   k-key nodes (b = k + 1), internal levels fully allocated breadth-first, then
//   ceil(m/k) leaves of boundaries + sentinel padding; one value per leaf slot,
//   padding replicating the last. Header fields are written back to
//   back (26 bytes), little-endian.
//
// The B200 layout is different (128-byte lines, compact levels), so a snapshot
// is not an image of device memory: loading one validates it and takes the m
// leaf keys and values — the interval map — which the device layout fill turns
// into a FIB with no interval sweep (lpm6cu_fib_load_snapshot). Saving writes
// the reference's layout byte for byte from an interval map, so the reference
// CLI can read what this side writes.
//
// PBTR — the reference's key trace: "PBTR", u16 version = 1,
// u16 reserved, u64 count, then count u64 LE keys (16-byte header).
#pragma once

#include <string>
#include <vector>

#include "lpm6/intervals.hpp"

namespace lpm6 {

inline constexpr u16 kSnapshotVersion = 1;
inline constexpr u64 kSnapshotHeaderBytes = 26;
inline constexpr u16 kTraceVersion = 1;
inline constexpr u64 kTraceHeaderBytes = 16;

// The reference's TreeGeometry (tree.hpp:18-33) for m keys at k keys per node.
struct RefGeometry {
  u32 k = 8, b = 9, depth = 0;
  u64 num_keys = 0, allocated_leaf_nodes = 0, leaf_start = 0;
  std::vector<u64> level_start;  // depth + 1 entries
  u64 total_key_slots() const { return leaf_start + allocated_leaf_nodes * k; }
};
RefGeometry plan_ref_geometry(u64 m, u32 k);

// Bytes of the PBT1 snapshot of `map` at k keys per node (reference layout).
std::vector<unsigned char> save_snapshot(const IntervalMap& map, u32 k = 8);

struct LoadedSnapshot {
  IntervalMap map;  // boundaries = the m real leaf keys, next_hops = their values
  RefGeometry geometry;
};

// Parse and validate a PBT1 image; BadSnapshotFile on any inconsistency (magic,
// version, sizes, geometry, key order, sentinel padding, value replication,
// internal separators). default_next_hop is not stored in the format; the
// loaded map carries `default_next_hop` (lookups never read it: the intervals
// cover the whole key space).
LoadedSnapshot load_snapshot(const void* data, u64 size, u32 default_next_hop = 0);

std::vector<unsigned char> read_file(const std::string& path);   // Io on failure
void write_file(const std::string& path, const void* data, u64 size);

// PBTR: check the 16-byte header against the total file size; returns the key
// count (BadTraceFile on a bad magic, version or size).
u64 trace_header_count(const unsigned char* header, u64 header_bytes, u64 file_size);
inline u64 trace_key_count(const void* data, u64 size) {
  return trace_header_count(static_cast<const unsigned char*>(data), size, size);
}
std::vector<unsigned char> save_trace(const u64* keys, u64 n);

}  // namespace lpm6
