"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the update engine's
staging rule, the checker for csrc/lpm6/update.cpp and csrc/store.cpp.

Follows the reference FibTable mutators and the SPEC's FibStore contract:
  * insert: ReservedNextHop, then DuplicatePrefix        (fib.cpp:120-127)
  * insert_or_replace ("A" lines): ReservedNextHop        (fib.cpp:129-139)
  * erase: UnknownPrefix; swap-with-last removal          (fib.cpp:141-152)
  * modify: ReservedNextHop, then UnknownPrefix           (fib.cpp:153-161)
  * stage validates each op against the FIB after all earlier staged ops and
    skips invalid ones; commit applies them in order.
  * trace line "A|W <ipv6>/<len> [next_hop]"

Only tests/ use this module.
"""
from __future__ import annotations

import ipaddress

INSERT, DELETE, MODIFY, ANNOUNCE = 0, 1, 2, 3
UNRESOLVED = 0xFFFFFFFF
MASK128 = (1 << 128) - 1


class OracleFib:
    """Ordered rule list + index with the reference's removal order."""

    def __init__(self, rules=()):
        self.entries: list[tuple[int, int, int]] = []  # (value128, length, next_hop)
        self.index: dict[tuple[int, int], int] = {}
        for v, ln, nh in rules:
            self.insert(v, ln, nh)

    def insert(self, v, ln, nh):
        if nh == UNRESOLVED:
            raise KeyError("ReservedNextHop")
        if (v, ln) in self.index:
            raise KeyError("DuplicatePrefix")
        self.index[(v, ln)] = len(self.entries)
        self.entries.append((v, ln, nh))

    def insert_or_replace(self, v, ln, nh):
        if nh == UNRESOLVED:
            raise KeyError("ReservedNextHop")
        i = self.index.get((v, ln))
        if i is None:
            self.index[(v, ln)] = len(self.entries)
            self.entries.append((v, ln, nh))
        else:
            self.entries[i] = (v, ln, nh)

    def erase(self, v, ln):
        i = self.index.pop((v, ln), None)
        if i is None:
            raise KeyError("UnknownPrefix")
        last = self.entries.pop()
        if i < len(self.entries):
            self.entries[i] = last
            self.index[(last[0], last[1])] = i

    def modify(self, v, ln, nh):
        if nh == UNRESOLVED:
            raise KeyError("ReservedNextHop")
        i = self.index.get((v, ln))
        if i is None:
            raise KeyError("UnknownPrefix")
        self.entries[i] = (v, ln, nh)


def apply_op(fib: OracleFib, kind: int, v: int, ln: int, nh: int) -> str | None:
    """Apply one op; returns None or the Errc name of the rejection (fib unchanged)."""
    if ln < 0 or ln > 64:
        return "UnsupportedPrefixLength"
    mask = 0 if ln == 0 else (MASK128 << (128 - ln)) & MASK128
    if v & ~mask & MASK128:
        return "InvalidArgument"
    try:
        if kind == INSERT:
            fib.insert(v, ln, nh)
        elif kind == DELETE:
            fib.erase(v, ln)
        elif kind == MODIFY:
            fib.modify(v, ln, nh)
        elif kind == ANNOUNCE:
            fib.insert_or_replace(v, ln, nh)
        else:
            return "InvalidArgument"
    except KeyError as e:
        return e.args[0]
    return None


def stage(fib: OracleFib, ops) -> tuple[int, list[str | None]]:
    errs = [apply_op(fib, *op) for op in ops]
    return sum(e is None for e in errs), errs


def parse_update_line(line: str):
    """(kind, value128, length, next_hop) of an "A"/"W" trace line."""
    tok = line.split()
    if len(tok) < 2 or tok[0] not in ("A", "W"):
        raise ValueError("MalformedAddress")
    addr, ln = tok[1].rsplit("/", 1)
    ln = int(ln)
    if ln > 64:
        raise ValueError("UnsupportedPrefixLength")
    v = int(ipaddress.IPv6Address(addr))
    mask = 0 if ln == 0 else (MASK128 << (128 - ln)) & MASK128
    if tok[0] == "W":
        return DELETE, v & mask, ln, 0
    if len(tok) < 3:
        raise ValueError("MissingNextHop")
    return ANNOUNCE, v & mask, ln, int(tok[2])
