// Route updates for the rebuild-and-swap FIB store (SPEC update-engine).
//
// An update is an Insert, Delete or Modify of one (value, length) rule,
// plus Announce — the trace's "A" line, insert-or-modify. Staging
// validates each op against the FIB as it will be after every op staged before
// it ("stage delete of absent prefix -> staged=0, 1 error"; an insert
// and a delete of the same prefix in one batch are both staged), so the store
// keeps that view and commit builds exactly it.
#pragma once

#include <istream>
#include <string_view>
#include <vector>

#include "lpm6/fib.hpp"

namespace lpm6 {

enum class UpdateKind : u32 { Insert = 0, Delete = 1, Modify = 2, Announce = 3 };

struct UpdateOp {
  UpdateKind kind = UpdateKind::Insert;
  u32 reserved = 0;
  Prefix prefix;  // next_hop ignored for Delete
};
static_assert(sizeof(UpdateOp) == 48, "UpdateOp is lpm6_update_op (include/lpm6cu.h)");

// "A <ipv6>/<len> <next_hop>" or "W <ipv6>/<len> [next_hop]". Host bits
// are masked as in parse_prefix (fib.cpp:72-105); /65+ -> UnsupportedPrefixLength.
UpdateOp parse_update(std::string_view line);

struct UpdateTraceStats {
  u64 lines = 0, ops = 0, errors = 0;
};

// One op per line; '#' comments and blank lines skipped. Lines that fail to
// parse are counted in stats.errors and skipped (routing feeds are noisy).
std::vector<UpdateOp> load_update_trace(std::istream& in, UpdateTraceStats* stats = nullptr);

// Validate `op` against `view` and apply it. Throws, leaving `view`
// unchanged: UnknownPrefix (Delete/Modify of an absent rule), DuplicatePrefix
// (Insert of a present one), ReservedNextHop, UnsupportedPrefixLength,
// InvalidArgument (host bits set / unknown kind).
void apply_update(FibTable& view, const UpdateOp& op);

}  // namespace lpm6
