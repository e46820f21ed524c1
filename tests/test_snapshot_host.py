"""Reference file formats on the host (no GPU): PBT1 snapshots in the reference's
tree layout (checked against the oracle's restatement of build_tree)
and PBTR key traces; every malformed input maps to the reference's Errc."""
import struct

import numpy as np
import pytest

from _util import random_fib_rules

SENT = 0xFFFFFFFFFFFFFFFF


def spec_map(lpm):
    """The 5-interval map of S:212 (A=2001:db8::/32 -> 1, B=2001:db8:1::/48 -> 2)."""
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    from _util import rules_array
    rules = rules_array([(0x20010DB8 << 96, 32, 1), ((0x20010DB8 << 96) | (1 << 80), 48, 2)], PREFIX_DTYPE)
    return lpm.build_intervals(lpm.FibTable(0, rules))


def maps(lpm):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    out = [("spec5", spec_map(lpm)), ("c0", lpm.build_intervals(lpm.workload_fib(0)))]
    for n in (0, 3, 7, 8, 9, 50, 2000):
        rng = np.random.default_rng(n)
        rules = random_fib_rules(rng, n, PREFIX_DTYPE, True)
        out.append((f"rand{n}", lpm.build_intervals(lpm.FibTable(0, rules))))
    return out


def header(data):
    magic, ver, k, depth, m, alloc = struct.unpack_from("<4sHHHQQ", data, 0)
    return magic, ver, k, depth, m, alloc


@pytest.mark.parametrize("k", [8, 16, 4, 2])
def test_snapshot_matches_reference_layout(lpm, orc, k):
    for name, imap in maps(lpm):
        data = lpm.encode_snapshot(imap, k)
        g, keys, values = orc.build_tree(imap.boundaries, imap.next_hops, k)
        total = g.leaf_start + g.allocated_leaf_nodes * k
        magic, ver, hk, depth, m, alloc = header(data)
        assert (magic, ver, hk, depth, m, alloc) == (b"PBT1", 1, k, g.depth, len(imap), g.allocated_leaf_nodes), name
        assert len(data) == 26 + total * 8 + alloc * k * 4
        got_keys = np.frombuffer(data, np.uint64, total, 26)
        got_vals = np.frombuffer(data, np.uint32, alloc * k, 26 + total * 8)
        np.testing.assert_array_equal(got_keys, keys[:total], err_msg=name)
        np.testing.assert_array_equal(got_vals, values, err_msg=name)
        back, bk = lpm.decode_snapshot(data)
        assert bk == k
        np.testing.assert_array_equal(back.boundaries, imap.boundaries)
        np.testing.assert_array_equal(back.next_hops, imap.next_hops)


def test_snapshot_spec_examples(lpm):
    # 5-interval map, k=8 -> depth 0: keys [0, A, B, Bend, Aend, S, S, S], values [def,1,2,1,def,def,def,def]
    imap = spec_map(lpm)
    data = lpm.encode_snapshot(imap, 8)
    a, b = 0x20010DB8 << 32, (0x20010DB8 << 32) | (1 << 16)
    keys = np.frombuffer(data, np.uint64, 8, 26)
    assert list(keys) == [0, a, b, b + (1 << 16), a + (1 << 32), SENT, SENT, SENT]
    assert list(np.frombuffer(data, np.uint32, 8, 26 + 64)) == [0, 1, 2, 1, 0, 0, 0, 0]
    # m=100, k=8 -> depth 2, level_start [0, 8, 80], keys length 80 + 13*8 = 184
    big = lpm.IntervalMap(np.arange(100, dtype=np.uint64) * 3, np.arange(100, dtype=np.uint32) % 7, 0)
    data = lpm.encode_snapshot(big, 8)
    _, _, _, depth, m, alloc = header(data)
    assert (depth, m, alloc) == (2, 100, 13)
    assert len(data) == 26 + 184 * 8 + 13 * 8 * 4
    keys = np.frombuffer(data, np.uint64, 184, 26)
    # level-1 node 0 separators = first keys of children 1..8 = boundaries[8*1 .. 8*8]
    assert list(keys[8:16]) == [int(big.boundaries[8 * j]) for j in range(1, 9)]


def test_snapshot_file_roundtrip(lpm, tmp_path):
    imap = lpm.build_intervals(lpm.workload_fib(0))
    p = tmp_path / "c0.pbt1"
    lpm.save_snapshot(imap, p)
    assert p.read_bytes() == lpm.encode_snapshot(imap)  # byte-identical for identical trees
    back, k = lpm.decode_snapshot(p.read_bytes())
    assert k == 8
    np.testing.assert_array_equal(back.boundaries, imap.boundaries)


def corrupt_cases(data):
    _, _, k, depth, m, alloc = header(data)
    total = (len(data) - 26 - alloc * k * 4) // 8
    leaf = total - alloc * k
    d = bytearray(data)

    def at(fn):
        c = bytearray(d)
        fn(c)
        return bytes(c)

    def setkey(c, i, v):
        struct.pack_into("<Q", c, 26 + 8 * i, v)

    def setval(c, i, v):
        struct.pack_into("<I", c, 26 + 8 * total + 4 * i, v)

    return {
        "magic": at(lambda c: c.__setitem__(slice(0, 4), b"PBT2")),
        "version": at(lambda c: struct.pack_into("<H", c, 4, 2)),
        "k<2": at(lambda c: struct.pack_into("<H", c, 6, 1)),
        "depth": at(lambda c: struct.pack_into("<H", c, 8, depth + 1)),
        "m=0": at(lambda c: struct.pack_into("<Q", c, 10, 0)),
        "alloc": at(lambda c: struct.pack_into("<Q", c, 18, alloc + 1)),
        "truncated": bytes(d[:-1]),
        "extra": bytes(d) + b"\0",
        "header": bytes(d[:20]),
        "unsorted": at(lambda c: setkey(c, leaf + 2, 0)),
        "first!=0": at(lambda c: setkey(c, leaf, 1)),
        "padding": at(lambda c: setkey(c, leaf + m, 12345) if m < alloc * k else setkey(c, leaf + 1, 0)),
        "value_pad": at(lambda c: setval(c, alloc * k - 1, 999) if m < alloc * k else setval(c, 0, 0xFFFFFFFF)),
        "reserved_value": at(lambda c: setval(c, 0, 0xFFFFFFFF)),
        "separator": at(lambda c: setkey(c, 0, 7)) if depth > 0 else at(lambda c: setkey(c, leaf + 1, 0)),
    }


def test_snapshot_corruption_is_bad_snapshot_file(lpm):
    from paper_2604_14650_b200.fib import PREFIX_DTYPE
    rules = random_fib_rules(np.random.default_rng(5), 300, PREFIX_DTYPE, True)
    imap = lpm.build_intervals(lpm.FibTable(0, rules))
    data = lpm.encode_snapshot(imap, 8)
    assert len(imap) % 8 != 0  # so the padding cases hit padding
    for name, bad in corrupt_cases(data).items():
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.decode_snapshot(bad)
        assert e.value.code == "BadSnapshotFile", name


def test_snapshot_encode_errors(lpm):
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.encode_snapshot(lpm.IntervalMap(np.zeros(0, np.uint64), np.zeros(0, np.uint32), 0))
    assert e.value.code == "InvalidArgument"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.encode_snapshot(lpm.IntervalMap(np.array([0, SENT], np.uint64), np.array([1, 2], np.uint32), 0))
    assert e.value.code == "SentinelCollision"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.encode_snapshot(spec_map(lpm), 1)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(lpm.Lpm6Error) as e:
        lpm.save_snapshot(spec_map(lpm), "/nonexistent-dir/x.pbt1")
    assert e.value.code == "Io"


def test_trace_format(lpm, tmp_path):
    keys = np.random.default_rng(0).integers(0, 2**64, 1000, dtype=np.uint64)
    p = tmp_path / "t.pbtr"
    lpm.save_trace(keys, p)
    data = p.read_bytes()
    assert data[:4] == b"PBTR" and struct.unpack_from("<HHQ", data, 4) == (1, 0, 1000)
    assert len(data) == 16 + 8000
    np.testing.assert_array_equal(np.frombuffer(data, np.uint64, 1000, 16), keys)
    assert lpm.trace_count(data) == 1000
    lpm.save_trace(np.zeros(0, np.uint64), p)
    assert lpm.trace_count(p.read_bytes()) == 0  # zero-length trace is a valid file
    bad = {
        "magic": b"PBTX" + data[4:],
        "version": data[:4] + struct.pack("<H", 2) + data[6:],
        "truncated": data[:-3],
        "count": data[:8] + struct.pack("<Q", 1001) + data[16:],
        "header": data[:10],
    }
    for name, b in bad.items():
        with pytest.raises(lpm.Lpm6Error) as e:
            lpm.trace_count(b)
        assert e.value.code == "BadTraceFile", name


def test_memory_footprint(lpm):
    # full depth-5 tree, m = 472,392, k = 8: leaf 3,779,136 B, internal 472,384 B
    f = lpm.ref_memory_footprint(472392, 8)
    assert f["leaf_bytes"] == 3779136 and f["internal_bytes"] == 472384
    assert f["value_bytes"] == 472392 * 4 and f["total_bytes"] == 3779136 + 472384 + 472392 * 4
    assert abs(f["bytes_per_interval_value8"] - 18.0) / 18.0 < 0.10  # the paper's "18 bytes"
    # m = 5 -> 64 B of keys + value bytes
    f5 = lpm.ref_memory_footprint(5, 8)
    assert f5["leaf_bytes"] + f5["internal_bytes"] == 64 and f5["total_bytes"] == 64 + 32
    # the reference footprint equals the bytes of its PBT1 snapshot minus the 26-byte header
    imap = lpm.build_intervals(lpm.workload_fib(0))
    assert lpm.ref_memory_footprint(len(imap))["total_bytes"] == len(lpm.encode_snapshot(imap)) - 26
    # B200 layout: every byte of the line array accounted for
    tree = lpm.build_tree(imap)
    g = tree.geometry
    b = g.memory_footprint()
    assert b["total_bytes"] == g.total_words * 8 == b["internal_bytes"] + b["leaf_bytes"] + b["image_bytes"]
    assert b["bytes_per_interval"] == b["total_bytes"] / len(imap)
