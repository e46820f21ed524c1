#include "lpm6/update.hpp"

#include <string>

namespace lpm6 {

namespace {

std::string_view trim(std::string_view s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string_view::npos) return {};
  const auto e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

}  // namespace

UpdateOp parse_update(std::string_view line) {
  const std::string_view s = trim(line);
  if (s.size() < 2 || (s[0] != 'A' && s[0] != 'W') || (s[1] != ' ' && s[1] != '\t'))
    throw Error(Errc::MalformedAddress, "update line must start with 'A ' or 'W ': '" + std::string(s) + "'");
  UpdateOp op;
  std::string body(trim(s.substr(2)));
  if (s[0] == 'W') {
    op.kind = UpdateKind::Delete;
    if (body.find_first_of(" \t") == std::string::npos) body += " 0";  // next hop optional on withdraw
  } else {
    op.kind = UpdateKind::Announce;
  }
  op.prefix = parse_prefix(body).prefix;
  if (op.kind == UpdateKind::Delete) op.prefix.next_hop = 0;
  return op;
}

std::vector<UpdateOp> load_update_trace(std::istream& in, UpdateTraceStats* stats) {
  std::vector<UpdateOp> ops;
  UpdateTraceStats st;
  std::string line;
  while (std::getline(in, line)) {
    std::string_view s(line);
    if (auto h = s.find('#'); h != std::string_view::npos) s = s.substr(0, h);
    if (trim(s).empty()) continue;
    ++st.lines;
    try {
      ops.push_back(parse_update(s));
      ++st.ops;
    } catch (const Error&) {
      ++st.errors;
    }
  }
  if (stats) *stats = st;
  return ops;
}

void apply_update(FibTable& view, const UpdateOp& op) {
  const Prefix& p = op.prefix;
  if (p.length < 0 || p.length > 64)
    throw Error(Errc::UnsupportedPrefixLength, "unsupported prefix length /" + std::to_string(p.length));
  const u128 mask = p.length == 0 ? u128(0) : ~u128(0) << (128 - p.length);
  if ((p.value & mask) != p.value)
    throw Error(Errc::InvalidArgument, "non-canonical prefix (host bits set): " + format_ipv6(p.value) + "/" +
                                           std::to_string(p.length));
  switch (op.kind) {
    case UpdateKind::Insert:
      view.insert(p);  // ReservedNextHop / DuplicatePrefix (fib.cpp:120-127)
      return;
    case UpdateKind::Delete:
      view.erase(p.value, p.length);  // UnknownPrefix (fib.cpp:141-152)
      return;
    case UpdateKind::Modify:
      view.modify(p.value, p.length, p.next_hop);  // ReservedNextHop / UnknownPrefix (fib.cpp:153-161)
      return;
    case UpdateKind::Announce:
      view.insert_or_replace(p);  // ReservedNextHop (fib.cpp:129-139)
      return;
  }
  throw Error(Errc::InvalidArgument, "unknown update kind " + std::to_string(static_cast<u32>(op.kind)));
}

}  // namespace lpm6
