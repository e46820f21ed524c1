#!/usr/bin/env python
"""bench.py — batched IPv6 LPM throughput on B200 (BASELINE.json metric).

A step = one pass of the lookup over one batch of synthetic queries (default:
workload C2 = the 1M-prefix projected FIB, 1,073,741,824 queries per GPU and
16-bit next hops, BASELINE.json configs[2] — the largest configuration that fits
one GPU; BASELINE quotes its metric on no single config). Prints ONE JSON line
(rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2]
  python bench.py --impl reference ...   # the reference's CPU lookup on host cores

Multi-GPU (N > 1) is launched by torchrun: rank 0 builds the FIB on the host,
NCCL broadcasts keys/values to every GPU, each GPU generates and looks up its own
query batch (no inter-GPU traffic during lookups; weak scaling), device time is
the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "IPv6 lookups/sec (G/s) per B200 and at 1/2/4/8 GPUs; % of roofline"
UNIT = "G lookups/s"
HBM_FALLBACK_GBS = 6650.0
CPU_SAMPLE = 1 << 26  # bounded CPU-baseline sample (67.1M queries; SURVEY §8d asks >= 64M)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C2",
                    help="BASELINE config: C0..C4; default C2, the largest single-GPU config (1M-prefix FIB, "
                         "1,073,741,824 queries, 16-bit next hops)")
    ap.add_argument("--lanes", type=int, default=0, help="lanes per query (4/8/16), 0 = auto")
    ap.add_argument("--smem-levels", type=int, default=None, help="levels staged in smem, default auto")
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--queries-per-lane", type=int, default=0, help="32-query tiles per warp iteration (1/2/4)")
    ap.add_argument("--plane-levels", type=int, default=0,
                    help="split-plane descent of staged levels 1..P-1 (with a fixed --line-path; the tuner picks its own)")
    ap.add_argument("--min-ctas", type=int, default=0, help="register cap: min CTAs/SM launch bound")
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (256/512/1024)")
    ap.add_argument("--queries", type=int, default=0, help="override queries per GPU (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="also time every kernel shape (extra key)")
    ap.add_argument("--no-extras", action="store_true", help="skip the key/packet-input and store timings")
    ap.add_argument("--line-path", choices=["tune", "lsu", "tex", "split", "tex-split", "tex-select"], default="tune",
                    help="L2 lines through the LSU or the texture pipe (lpm6cu_kernel_config.line_path 0-4); tune = time all on the step's "
                         "batch before the warm-up (lpm6cu_fib_tune_line_path) and keep the faster")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay each step's launch from a CUDA graph (auto: batches under 2^24 queries, "
                         "where the host launch path would otherwise bound the step)")
    return ap.parse_args()


# ---- distributed plumbing ------------------------------------------------------------

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shared_gpu_mode():
    """LPM6_BENCH_SHARED_GPU=1: a harness check of the torchrun path on a box with fewer
    GPUs than ranks — ranks share devices (local rank mod device count) and the
    collectives run over gloo (NCCL refuses two ranks on one GPU). The ranks' kernels
    never wait on one another (lookups shard with no exchange), but they contend for
    the same SMs, so the numbers of such a run are not bench values; the line says so."""
    return os.environ.get("LPM6_BENCH_SHARED_GPU", "") not in ("", "0")


def force_dist_mode():
    """LPM6_BENCH_FORCE_DIST=1: create the process group at world size 1 too, so that a
    one-GPU box runs every collective of the multi-rank path (the line-array broadcast,
    the MAX reductions, the gathers and barriers) through NCCL itself. The line says so."""
    return os.environ.get("LPM6_BENCH_FORCE_DIST", "") not in ("", "0")


def init_dist(ws, local, backend="nccl"):
    import torch
    import torch.distributed as dist
    force = force_dist_mode()
    if (ws > 1 or force) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if ws == 1:  # forced: a standalone rendezvous when not under torchrun
            os.environ.setdefault("MASTER_PORT", "29537")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return dist if (ws > 1 or force) else None


# ---- clocks ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---- roofline -----------------------------------------------------------------------------

def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback"


def device_build_ms(lpm, fib, device, vb, reps=3):
    """Wall time of the GPU FIB build (rules on the host -> ready device FIB), best of reps."""
    import torch
    lpm.Fib.build_device(fib, device, value_bytes=vb).close()  # warm-up (module load, allocator)
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lpm.Fib.build_device(fib, device, value_bytes=vb).close()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


def _time_ms(torch, fn, stream, reps=3):
    fn()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(reps):
        fn()
    a1.record(stream)
    torch.cuda.synchronize()
    return a0.elapsed_time(a1) / reps


def time_extras(lpm, torch, fdev, fib, addrs, n, vb, stream, device):
    """The same workload through the other inputs (8-byte keys; 64-byte Ethernet+IPv6
    frames) and the update store's commit latency. Each result is checked against
    the address path's output."""
    out = {}
    ref = fdev.lookup_batch(addrs, None, stream)
    keys = addrs[:, 8:16].contiguous().view(torch.int64).reshape(-1)
    ko = torch.empty_like(ref)
    ms = _time_ms(torch, lambda: fdev.lookup_keys(keys, ko, stream), stream)
    out["keys8"] = {"value": n / ms / 1e6, "unit": UNIT, "ms": ms, "dram_bytes_per_query": 8 + vb,
                    "matches_address_path": bool(torch.equal(ko, ref))}
    # the same keys from pinned host memory through the C ABI: 8 + vb bytes over PCIe per query
    hk = torch.empty(n, dtype=torch.int64, pin_memory=True)
    hk.copy_(keys)
    ho = torch.empty(n * vb, dtype=torch.uint8, pin_memory=True)
    hk_np, ho_np = hk.numpy(), ho.numpy()
    fdev.lookup_keys(hk_np, ho_np)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        fdev.lookup_keys(hk_np, ho_np)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out["keys8_e2e"] = {"value": n / ms / 1e6, "unit": UNIT, "ms": ms, "h2d_bytes_per_step": n * 8,
                        "d2h_bytes_per_step": n * vb,
                        "matches_address_path": bool(np.array_equal(ho_np, ref.view(torch.uint8).cpu().numpy())),
                        "path": "lpm6cu_lookup_keys(host pinned buffers)"}
    del keys, ko, hk, ho
    m = min(n, 1 << 26)
    frames = torch.zeros((m, 64), dtype=torch.uint8, device=addrs.device)
    frames[:, 12] = 0x86  # EtherType 0x86DD
    frames[:, 13] = 0xDD
    frames[:, 14] = 0x60  # IPv6 version
    frames[:, 38:54] = torch.flip(addrs[:m], dims=[1])  # destination, network byte order
    frames = frames.reshape(-1)
    po = torch.empty(m * vb, dtype=torch.uint8, device=addrs.device)
    ms = _time_ms(torch, lambda: fdev.lookup_packets(frames, m, 64, 38, po, stream), stream)
    out["packets64"] = {"value": m / ms / 1e6, "unit": UNIT, "frames": m, "stride": 64, "dst_offset": 38, "ms": ms,
                        "matches_address_path": bool(torch.equal(po, ref.view(torch.uint8)[: m * vb]))}
    del frames, po
    # serving-size batches through the C ABI (device buffers): back-to-back calls and call-to-result
    small = []
    for b in (256, 4096, 65536):
        if b > n:
            continue
        sub, so = addrs[:b], torch.empty(b * vb, dtype=torch.uint8, device=addrs.device)
        ms = _time_ms(torch, lambda: fdev.lookup_batch(sub, so, stream), stream, reps=200)
        lat = []
        for _ in range(50):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fdev.lookup_batch(sub, so, stream)
            torch.cuda.synchronize()
            lat.append((time.perf_counter() - t0) * 1e6)
        small.append({"batch": b, "us_per_call_back_to_back": ms * 1e3, "us_call_to_result_median": float(np.median(lat)),
                      "glps_back_to_back": b / ms / 1e6})
    out["small_batches"] = small
    # the same batch sizes from page-locked host buffers (zero-copy up to 2^16 queries:
    # one launch + one sync, the kernel reads addresses / writes next hops over PCIe)
    small_h = []
    for b in (256, 4096, 65536):
        if b > n:
            continue
        ha = addrs[:b].cpu().pin_memory().numpy()
        ho = torch.empty(b * vb, dtype=torch.uint8).pin_memory().numpy()
        fdev.lookup_batch(ha, ho)
        lat = []
        for _ in range(100):
            t0 = time.perf_counter()
            fdev.lookup_batch(ha, ho)  # synchronous for host buffers
            lat.append((time.perf_counter() - t0) * 1e6)
        small_h.append({"batch": b, "us_call_to_result_median": float(np.median(lat)),
                        "us_call_to_result_p99": float(np.percentile(lat, 99)),
                        "matches_device_path": bool(np.array_equal(ho, ref.view(torch.uint8)[: b * vb].cpu().numpy()))})
    out["small_batches_host_pinned"] = small_h
    # store: create (device build) + commits of 1,000 announces each
    from paper_2604_14650_b200.fib import Prefix
    st = lpm.FibStore(fib, device, value_bytes=vb)
    rng = np.random.default_rng(1)
    rules = fib.rules
    commits = []
    for _ in range(3):
        idx = rng.integers(0, len(rules), 1000)
        ops = [lpm.UpdateOp(3, Prefix(int(rules[i]["value_hi"]) << 64, int(rules[i]["length"]),
                                      int(rng.integers(1, 255)))) for i in idx]
        st.stage(ops)
        t0 = time.perf_counter()
        st.commit()
        commits.append((time.perf_counter() - t0) * 1e3)
    s = st.stats
    out["store_commit"] = {"ops_per_commit": 1000, "commit_ms": commits, "device_build_ms": s.last_build_ms,
                           "publish_us": s.last_publish_us, "epoch": s.epoch,
                           "note": "stage 1,000 announces, rebuild the whole FIB on the GPU, publish; "
                                   "paper quotes 850 ms for a 1M-prefix rebuild (P:1334-1335)"}
    st.close()
    return out


NCU_METRICS = ROOT / "profiles" / "r02_ncu_metrics.json"


def ncu_metrics(workload):
    """Per-query figures of the committed `ncu --set full` capture of this workload's
    bench kernel (profiles/r02_ncu_metrics.json, tools/ncu_metrics.py); C3a falls back
    to C1's packed-key capture and C4 to C2's (same FIB and kernel)."""
    try:
        t = json.loads(NCU_METRICS.read_text())
    except Exception:
        return None
    return t.get(workload) or t.get({"C3a": "C1_packed", "C3b": "C1", "C4": "C2"}.get(workload, workload))


def roofline_object(geom, vb, cfg, lps, l2_gbs, smem_gbs, hbm_gbs, hbm_src, workload, n_per_launch, sm_mhz):
    """The bench line's `roofline`: SURVEY §8d's model evaluated at the shared-memory
    split the kernel actually runs (T = its staged levels) — `bound`, `achieved`,
    `peak`, `frac` — plus the max-over-T form §8d states (`frac_best_T`), the HBM
    fraction, the DRAM traffic of one launch from the committed ncu capture, and the
    kernel's own ceiling from that capture: one L1 data-pipe wavefront per SM per
    clock divided by the measured wavefronts per query."""
    T = min(int(cfg["smem_levels"]), geom.depth + 1)
    at = roofline(geom, vb, l2_gbs, smem_gbs, hbm_gbs, only_T=T)
    best = roofline(geom, vb, l2_gbs, smem_gbs, hbm_gbs)
    bpq = at["bytes_per_query"][at["bound"]]
    peak = {"hbm": hbm_gbs, "smem": smem_gbs, "l2": l2_gbs}[at["bound"]]
    m = ncu_metrics(workload)
    obj = {"bound": at["bound"], "achieved": lps * bpq / 1e9, "peak": peak, "unit": "GB/s",
           "frac": lps * bpq / 1e9 / peak,
           "traffic": m["dram_bytes_per_query"] * n_per_launch if m else None,
           "model": "SURVEY §8d at the kernel's split: bytes/query hbm 16+w, smem 128*T, l2 128*(d+1-T)+w",
           "T": T, "lps_achieved_per_gpu": lps / 1e9, "lps_roofline_per_gpu": at["lps"] / 1e9,
           "terms_glps": at["terms_glps"], "bytes_per_query": at["bytes_per_query"],
           "frac_best_T": lps / best["lps"], "best_T": best["T"], "lps_roofline_best_T": best["lps"] / 1e9,
           "hbm_frac": lps * (16 + vb) / 1e9 / hbm_gbs,
           "peak_sources": {"hbm": hbm_src,
                            "smem": "probe in this run: shared-memory read kernel on this device (not in MEASURED_PEAKS.json)",
                            "l2": "probe in this run: random 128-B line gathers over a tree-sized buffer (not in MEASURED_PEAKS.json)"},
           "measured": {"l2_gather_gbs": l2_gbs, "smem_gbs": smem_gbs, "hbm_gbs": hbm_gbs}}
    if m:
        clk = sm_mhz or m["sm_clock_mhz"]
        # both L1TEX data pipes move one wavefront per SM per clock
        ceil_lsu = 148 * clk * 1e6 / m["lsu_wavefronts_per_query"] / 1e9
        ceil_tex = 148 * clk * 1e6 / m["tex_wavefronts_per_query"] / 1e9 if m["tex_wavefronts_per_query"] else None
        ceil = min(c for c in (ceil_lsu, ceil_tex) if c)
        obj.update({"limiter_ncu": f"L1 LSU data pipe {m['lsu_data_pipe_pct']:.1f}% of peak, texture data pipe "
                                   f"{m['tex_data_pipe_pct']:.1f}%, issue {m['issue_active_pct']:.1f}% ({m['capture']})",
                    "l1_wavefront_ceiling_glps": ceil, "frac_of_l1_ceiling": lps / 1e9 / ceil,
                    "l1_ceilings_glps": {"lsu": ceil_lsu, "tex": ceil_tex},
                    "lsu_wavefronts_per_query": m["lsu_wavefronts_per_query"],
                    "tex_wavefronts_per_query": m["tex_wavefronts_per_query"],
                    "traffic_per_query": m["dram_bytes_per_query"], "ncu_capture": m["capture"]})
    return obj


def roofline(geom, w, l2_gbs, smem_gbs, hbm_gbs, smem_cap=232448, only_T=None):
    """roofline_lps = max_T min(HBM/(16+w), SMEM/(128 T), L2/(128 (d+1-T) + w));
    with only_T, the term at that split alone."""
    d = geom.depth
    levels = d + 1
    best = None
    for T in range(0, levels + 1):
        if only_T is not None and T != only_T:
            continue
        staged = (geom.total_words if T >= levels else geom.level_start[T]) * 8 if T else 0
        if staged > smem_cap and only_T is None:
            break
        terms = {"hbm": hbm_gbs * 1e9 / (16 + w)}
        if T:
            terms["smem"] = smem_gbs * 1e9 / (128 * T)
        l2_bytes = 128 * (levels - T) + w
        terms["l2"] = l2_gbs * 1e9 / l2_bytes
        bound = min(terms, key=terms.get)
        cand = {"T": T, "lps": terms[bound], "bound": bound, "terms_glps": {k: v / 1e9 for k, v in terms.items()},
                "bytes_per_query": {"hbm": 16 + w, "smem": 128 * T, "l2": l2_bytes}}
        if best is None or cand["lps"] > best["lps"]:
            best = cand
    return best


# ---- reference arm ---------------------------------------------------------------------------

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    """'<model name>, <nproc> CPUs, avx512f yes/no' (SURVEY §8d asks for all three)."""
    name, avx512 = "unknown", False
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and name == "unknown":
                name = line.split(":", 1)[1].strip()
            if line.startswith("flags"):
                avx512 = avx512 or " avx512f" in line
    except Exception:
        pass
    return f"{name}, {os.cpu_count()} CPUs, avx512f {'yes' if avx512 else 'no'}"


def time_reference_cpu(fib, addrs, threads, repeats=1):
    """The reference's own lpm6::lookup_interval_oracle (oracle/_ref, intervals.cpp:142-145)
    on `threads` std::threads over one shared IntervalMap (SURVEY §8d baseline A). No
    fallback: without oracle/_ref (built from /root/reference) this raises."""
    from oracle.oracle import REF_SO, RefOracle
    if not REF_SO.exists():
        raise FileNotFoundError(f"{REF_SO} is not built; build() compiles it from /root/reference")
    keys = np.ascontiguousarray(addrs[:, 1])
    r = RefOracle()
    st, rmap = r.build_intervals(fib.rules, fib.default_next_hop)
    assert st == 0, r.error()
    rmap.lookup(keys[: 1 << 16], threads)  # warm-up
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        rmap.lookup(keys, threads)
        times.append(time.perf_counter() - t0)
    return times, "reference", "oracle/_ref lpm6::lookup_interval_oracle (reference fib.cpp+intervals.cpp)"


def oracle_check(fib, host_addrs, gpu_out, vb, threads, extra=None):
    """Part of the CPU-baseline leg (the only place bench.py runs oracle/): the CPU
    oracle's answers for a sample of the timed run's addresses, compared with the
    GPU's output for them. A checker only; nothing measured comes from here."""
    from oracle.oracle import Oracle
    o = Oracle()
    st, b, nh = o.build_intervals(fib.rules, fib.default_next_hop)
    want, _ = o.lookup_batch(0, b, nh, host_addrs, threads=threads)
    got = gpu_out.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[vb]).astype(np.uint32)
    res = {"checked": int(len(want)), "mismatches": int(np.count_nonzero(got != want)),
           "oracle": "oracle/lpm6_oracle.c interval oracle"}
    if extra:
        res.update(extra)
    return res


def time_restated_planb(fib, addrs, threads):
    """Restated PlanB AVX-512 Listing 1 + B=16 batched search, k=8 (oracle/lpm6_oracle_avx512.c)."""
    from oracle.oracle import Oracle
    o = Oracle()
    st, b, nh = o.build_intervals(fib.rules, fib.default_next_hop)
    tree = o.build_tree(b, nh, 8)
    o.lookup_batch(2, b, nh, addrs[: 1 << 16], threads, tree=tree)
    t0 = time.perf_counter()
    _, ran = o.lookup_batch(2, b, nh, addrs, threads, tree=tree)
    dt = time.perf_counter() - t0
    return dt, {2: "avx512_batch16", 1: "branchfree_scalar"}[ran]


def single_thread_baselines(fib, addrs, n1=1 << 22):
    """SURVEY §8d asks for the CPU baselines on one thread as well as on all cores:
    the reference's lookup_interval_oracle and the restated PlanB search on the first
    n1 queries of the sample, one thread each."""
    a = addrs[:n1]
    out = {"sample": f"first {len(a)} queries, 1 thread"}
    times, kind, _ = time_reference_cpu(fib, a, 1, repeats=1)
    out["reference_oracle"] = {"value": len(a) / times[0] / 1e9, "unit": UNIT, "cores": 1, "kind": kind}
    try:
        dt, variant = time_restated_planb(fib, a, 1)
        out["restated_planb"] = {"value": len(a) / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                                 "variant": variant}
    except Exception as e:  # extra context only
        out["restated_planb"] = {"error": str(e)}
    return out


def shared_config(info, fib_len, n_per_gpu, ws):
    """The `config` object of both arms (identical keys and values for the same
    workload and GPU count; each arm's own details live outside it)."""
    if info.chunk and n_per_gpu == info.n_queries:
        return {"workload": info.name, "fib_prefixes": fib_len, "queries_total": info.n_queries,
                "chunk": info.chunk, "value_bytes": info.value_bytes, "parallelism": f"dp{ws}",
                "scaling": "strong"}
    return {"workload": info.name, "fib_prefixes": fib_len, "queries_per_gpu": n_per_gpu,
            "value_bytes": info.value_bytes, "parallelism": f"dp{ws}", "scaling": "weak"}


def product_mapped():
    """Product-library mappings of this process (the reference arm must have none)."""
    try:
        return sorted({ln.split()[-1] for ln in open("/proc/self/maps")
                       if "paper_2604_14650_b200" in ln or "liblpm6cu" in ln})
    except OSError:
        return []


def run_reference(args):
    """--impl reference: the reference's own CPU lookup (lookup_interval_oracle from
    oracle/_ref, compiled from /root/reference's fib.cpp + intervals.cpp) on every host
    thread, over the same workload and config as our arm. Each step looks up a bounded,
    different slice of the workload's query stream (CPU_SAMPLE queries: slice i of the
    stream for step i), generated before its timer starts. The FIB and queries come
    from oracle/liblpm6work.so (our generator compiled alone), so this process never
    maps the product library; rank 0 alone runs under torchrun."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import REF_SO, RefOracle
    from oracle.workload import Workloads
    if not REF_SO.exists():
        raise FileNotFoundError(f"{REF_SO} is not built; build() compiles it from /root/reference")
    wl = Workloads()
    threads = cpu_threads()
    info = wl.info(args.workload)
    fib = wl.fib(info.fib_kind)
    n_full = args.queries or info.n_queries
    sample = min(n_full, CPU_SAMPLE)
    r = RefOracle()
    t0 = time.perf_counter()
    st, rmap = r.build_intervals(fib.rules, fib.default_next_hop)
    build_s = time.perf_counter() - t0
    assert st == 0, r.error()
    step_s = []
    first_q = wl.queries(args.workload, fib, 0, 1 << 16, threads)
    rmap.lookup(np.ascontiguousarray(first_q[:, 1]), threads)  # warm-up pass
    for i in range(args.warmup + args.steps):
        first = (i * sample) % max(n_full - sample + 1, 1)
        keys = np.ascontiguousarray(wl.queries(args.workload, fib, first, sample, threads)[:, 1])
        t0 = time.perf_counter()
        rmap.lookup(keys, threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            step_s.append(dt)
    total = sum(step_s)
    value = sample * len(step_s) / total / 1e9
    mapped = product_mapped()
    assert not mapped, f"reference arm mapped the product library: {mapped}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / len(step_s) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "impl": "reference",
        "data": f"synthetic seeded {info.name} workload (oracle/liblpm6work.so, bit-identical to our arm's "
                f"generator); step i looks up queries [i*{sample}, (i+1)*{sample}) of the stream",
        "config": shared_config(info, len(fib), n_full, args.gpus),
        "sample": {"queries_per_step": sample, "of_workload_queries": n_full,
                   "why": "bounded CPU sample per step so the run ends within minutes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{sample} queries of {info.name} per step ({len(step_s)} steps)",
                         "what": "oracle/_ref lpm6::lookup_interval_oracle (reference fib.cpp+intervals.cpp)",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_intervals_ms": build_s * 1e3,
        "step_ms": [x * 1e3 for x in step_s],
        "product_library_mapped": mapped,
    }
    print(json.dumps(line), flush=True)
    return 0


def output_digest(torch, gen, fdev, addrs, out, c0, nc, chunk, stream, dist):
    """sha256 over (chunk index, per-chunk hash) for all chunks in order
    (dispatch.combine_digests); the per-chunk hash is computed on the device
    (dispatch.chunk_hash)."""
    from paper_2604_14650_b200 import dispatch
    mine = {}
    for c in range(c0, c0 + nc):
        gen.run(c * chunk, chunk, addrs, stream)
        fdev.lookup_batch(addrs, out, stream)
        mine[c] = dispatch.chunk_hash(out)
    return dispatch.combine_digests(mine, dist)


def gather_block_hashes(torch, out, dist):
    from paper_2604_14650_b200 import dispatch
    h = f"{dispatch.chunk_hash(out):016x}"
    if dist is None:
        return [h]
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, h)
    return parts


def gather_per_rank(ms, dist):
    """Every rank's summed device time of the timed steps (rank order), for the
    balance check in multi-GPU lines; [ms] at one rank."""
    if dist is None:
        return [ms]
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, float(ms))
    return allv


def choose_line_path(args, fdev, addrs, out, stream):
    """Leaf path for the timed steps: fixed by --line-path, or measured on this batch
    (untimed, before the warm-up) by the library's tuner. Returns the kernel config."""
    if args.line_path == "tune":
        fdev.tune_line_path(addrs, out, stream)
    else:
        c = fdev.kernel_config()
        fdev.set_kernel_config(lanes_per_query=c["lanes_per_query"], smem_levels=c["smem_levels"],
                               ctas_per_sm=c["ctas_per_sm"], threads_per_cta=c["threads_per_cta"],
                               queries_per_lane=c["queries_per_lane"], min_ctas_per_sm=c["min_ctas_per_sm"],
                               line_path={"lsu": 0, "tex": 1, "split": 2, "tex-split": 3, "tex-select": 4}[args.line_path],
                               plane_levels=args.plane_levels)
    cfg = fdev.kernel_config()
    cfg["line_path_choice"] = args.line_path
    return cfg


# ---- C4: fixed total, 64M-address chunks partitioned across GPUs ---------------------------------

def run_chunked(args, lpm, dispatch, fdev, fib, info, geom, cfg, ws, rank, dev_index, dist, build_ms, bcast_ms):
    """C4 (BASELINE configs[4]): info.n_queries addresses in info.chunk-sized chunks, chunk c
    seeded by its index (any GPU can generate any chunk), chunks split contiguously over the
    ranks (strong scaling). Each chunk is generated on the device untimed, then looked up
    between CUDA events; a step = one pass over this rank's chunks; device time = max over
    ranks of the summed lookup times."""
    import torch
    chunk, vb = info.chunk, info.value_bytes
    total_chunks = info.n_queries // chunk
    c0, nc = dispatch.shard(rank, ws, 0, total=total_chunks)
    addrs = torch.empty((chunk, 16), dtype=torch.uint8, device="cuda")
    out = torch.empty(chunk * vb, dtype=torch.uint8, device="cuda")
    gen = lpm.QueryGen(args.workload, fib, dev_index)
    stream = torch.cuda.current_stream()
    l2_gbs = lpm.probe_l2_gather(dev_index, max(geom.tree_bytes, 1 << 22), 128)
    smem_gbs = lpm.probe_smem(dev_index)
    hbm_gbs, hbm_src = hbm_peak()

    gen.run(c0 * chunk, chunk, addrs, stream)
    cfg = choose_line_path(args, fdev, addrs, out, stream)

    def one_pass():
        evs = []
        for c in range(c0, c0 + nc):
            gen.run(c * chunk, chunk, addrs, stream)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fdev.lookup_batch(addrs, out, stream)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    for _ in range(max(args.warmup, 0)):
        one_pass()
    if dist is not None:
        dist.barrier()
    with ClockSampler(dev_index) as clk:
        step_ms = [one_pass() for _ in range(args.steps)]
    total_ms = dispatch.max_over_ranks(sum(step_ms), dist, "cuda")
    per_rank_ms = gather_per_rank(sum(step_ms), dist)
    value = info.n_queries * args.steps / (total_ms * 1e-3) / 1e9
    # Output digest (untimed pass): a hash of every chunk's next hops, combined in chunk
    # order over all ranks — identical for every GPU count if sharding changes nothing.
    digest = output_digest(torch, gen, fdev, addrs, out, c0, nc, chunk, stream, dist)
    parity = None
    if rank == 0:  # CPU-baseline leg: the oracle checks a sample of chunk c0's output
        gen.run(c0 * chunk, 1 << 20, addrs, stream)
        fdev.lookup_batch(addrs[: 1 << 20], out[: (1 << 20) * vb], stream)
        torch.cuda.synchronize()
        ha = addrs[: 1 << 20].cpu().numpy().view(np.uint64).reshape(-1, 2)
        parity = oracle_check(fib, ha, out[: (1 << 20) * vb].cpu().numpy(), vb, cpu_threads(), {"chunk": c0})
    if rank != 0:
        if dist is not None:
            dist.barrier()
        return 0
    lps_gpu = nc * chunk * args.steps / (sum(step_ms) * 1e-3)
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64",
        "data": f"synthetic: seeded {info.name} FIB ({len(fib)} prefixes); {info.n_queries} queries in "
                f"{total_chunks} chunks of {chunk}, chunk c seeded by c, generated on device (untimed)",
        "config": shared_config(info, len(fib), info.n_queries, ws),
        "layout": {"intervals": geom.num_keys, "tree_depth": geom.depth, "chunks_per_gpu": nc,
                   "sharding": "contiguous chunk ranges; FIB replicated by NCCL broadcast"},
        "kernel": cfg,
        "l2_flush": f"not needed: each chunk streams {chunk * 16 / 1e9:.1f} GB of addresses (> 126 MB L2)",
        "roofline": roofline_object(geom, vb, cfg, lps_gpu, l2_gbs, smem_gbs, hbm_gbs, hbm_src, info.name, chunk,
                                    clocks.get("sm_mhz")),
        "cpu_baseline": None, "e2e": None,
        "gpu_launches": 2 * nc * args.steps,
        "clocks": clocks, "parity_sample": parity,
        "fib_build_ms": build_ms, "fib_build_device_ms": device_build_ms(lpm, fib, dev_index, vb),
        "fib_broadcast_ms": bcast_ms, "step_ms": step_ms, "per_rank_total_ms": per_rank_ms,
        "output_digest": digest,
    }
    if ws > 1 and shared_gpu_mode():
        line["harness_check"] = "LPM6_BENCH_SHARED_GPU: ranks shared GPUs over gloo; not a bench value"
    if ws == 1 and force_dist_mode():
        line["harness_check"] = "LPM6_BENCH_FORCE_DIST: the multi-rank collectives ran through NCCL at world size 1"
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
    return 0


# ---- our arm ------------------------------------------------------------------------------------

def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = dist_env()
    shared = ws > 1 and shared_gpu_mode()
    if shared:
        local = local % torch.cuda.device_count()
    dist = init_dist(ws, local, "gloo" if shared else "nccl")
    torch.cuda.set_device(local)
    dev_index = local
    import paper_2604_14650_b200 as lpm

    info = lpm.workload_info(args.workload)
    fib = lpm.workload_fib(info.fib_kind)
    n = args.queries or info.n_queries
    vb = info.value_bytes

    # -- FIB: host build on rank 0, NCCL broadcast to the others -----------------------------
    from paper_2604_14650_b200 import dispatch
    t0 = time.perf_counter()
    tree = dispatch.build_on_root(fib, rank, vb)
    build_ms = (time.perf_counter() - t0) * 1e3
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    geom, lines_t = dispatch.replicate_tree(tree, dist, torch.device("cuda", dev_index))
    e1.record()
    torch.cuda.synchronize()
    bcast_ms = dispatch.max_over_ranks(e0.elapsed_time(e1), dist, "cuda") if dist is not None else 0.0
    fdev = lpm.Fib.wrap_device(geom, lines_t, dev_index)
    cfg = fdev.set_kernel_config(lanes_per_query=args.lanes, smem_levels=args.smem_levels,
                                 ctas_per_sm=args.ctas_per_sm, queries_per_lane=args.queries_per_lane,
                                 min_ctas_per_sm=args.min_ctas, threads_per_cta=args.threads)
    if info.chunk and not args.queries:
        return run_chunked(args, lpm, dispatch, fdev, fib, info, geom, cfg, ws, rank, dev_index, dist,
                           build_ms, bcast_ms)

    # -- queries: this rank's slice, generated on the device ------------------------------------
    addrs = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    out = torch.empty(n * vb, dtype=torch.uint8, device="cuda")
    gen = lpm.QueryGen(args.workload, fib, dev_index)
    first, _ = dispatch.shard(rank, ws, n)
    gen.run(first, n, addrs)
    torch.cuda.synchronize()

    # -- roofline denominators measured on this device --------------------------------------------
    tree_bytes = geom.tree_bytes
    l2_gbs = lpm.probe_l2_gather(dev_index, max(tree_bytes, 1 << 22), 128)
    smem_gbs = lpm.probe_smem(dev_index)
    hbm_gbs, hbm_src = hbm_peak()

    stream = torch.cuda.current_stream()

    cfg = choose_line_path(args, fdev, addrs, out, stream)

    def launch(s=stream):
        fdev.lookup_batch(addrs, out, s)

    step = launch
    use_graph = args.graph == "on" or (args.graph == "auto" and n < (1 << 24))
    if use_graph:
        launch()  # resolves and caches the launch plan outside the capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):  # captured on torch's side stream, replayed on the current one
            launch(torch.cuda.current_stream())
        step = graph.replay

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev_index) as clk:
        if use_graph and hasattr(torch.cuda, "_sleep"):
            # Launch-bound steps (~12 us): hold the stream in an untimed device sleep
            # while the host enqueues all K replays, so host submission gaps never
            # land between the timing events (the sleep itself is before ev[0]).
            torch.cuda._sleep(int(2e6 + 2e5 * args.steps))
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = dispatch.max_over_ranks(sum(step_ms), dist, "cuda")
    per_rank_ms = gather_per_rank(sum(step_ms), dist)
    # Rank r always resolves queries [r*n, (r+1)*n): its block's hash is the same at any GPU count.
    block_hashes = gather_block_hashes(torch, out, dist)
    ms_per_step = total_ms / args.steps
    value = ws * n * args.steps / (total_ms * 1e-3) / 1e9  # aggregate G lookups/s
    lps_gpu = n / (ms_per_step * 1e-3)

    # -- sample of the timed output, checked against the oracle in the CPU-baseline leg ------------
    m_s = min(n, 1 << 20)
    sample_addrs = addrs[:m_s].cpu().numpy().view(np.uint64).reshape(-1, 2) if rank == 0 else None
    sample_out = out[: m_s * vb].cpu().numpy() if rank == 0 else None

    # -- end to end through the C ABI with host buffers -------------------------------------------
    e2e = None
    if not args.no_e2e:
        # N > 1: every rank pins its own host buffers at once, so each rank uses the
        # first 2^26 of its queries (1 GiB of addresses) to bound pinned host memory.
        n_e = n if ws == 1 else min(n, 1 << 26)
        h_addrs = torch.empty((n_e, 16), dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(n_e * vb, dtype=torch.uint8, pin_memory=True)
        h_addrs.copy_(addrs[:n_e])
        torch.cuda.synchronize()
        ha_np, ho_np = h_addrs.numpy(), h_out.numpy()
        fdev.lookup_batch(ha_np, ho_np)  # warm-up: allocates the staging pipeline
        if dist is not None:
            dist.barrier()
        k_e2e = max(1, min(args.steps, 5))
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(k_e2e):
            fdev.lookup_batch(ha_np, ho_np)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = dispatch.max_over_ranks(s0.elapsed_time(s1), dist, "cuda")
        e2e = {"value": ws * n_e * k_e2e / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": ws * n_e * 16,
               "d2h_bytes_per_step": ws * n_e * vb, "steps": k_e2e, "queries_per_rank": n_e,
               "path": "lpm6cu_lookup_batch(host pinned buffers): " + (
                   "zero-copy, the kernel reads the addresses and writes the next hops over PCIe"
                   if n_e <= (1 << 20) else "8M-address chunks, H2D/kernel/D2H on 3 streams")}
        same = bool(np.array_equal(ho_np[: 1 << 20], out[: 1 << 20].cpu().numpy()))
        e2e["matches_device_path"] = same
        del h_addrs, h_out

    # -- optional shape sweep --------------------------------------------------------------------------
    sweep = None
    if args.sweep and rank == 0:
        sweep = []
        shapes = [(1, 256, 0), (1, 256, 4), (2, 256, 0), (1, 512, 2), (1, 1024, 1)]
        for t_lv in range(max(0, geom.depth - 2), geom.depth + 1 + geom.leaf_image):
            for qpl, thr, minb in shapes:
                try:
                    fdev.set_kernel_config(smem_levels=t_lv, queries_per_lane=qpl, threads_per_cta=thr,
                                           min_ctas_per_sm=minb)
                except Exception:
                    continue
                # launch() directly, never the captured graph: a graph replays the kernel
                # and parameters captured before the sweep changed the config
                for _ in range(2):
                    launch()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(3):
                    launch()
                a1.record(stream)
                torch.cuda.synchronize()
                ms = a0.elapsed_time(a1) / 3
                sweep.append({"smem_levels": t_lv, "queries_per_lane": qpl, "threads": thr, "min_ctas_per_sm": minb,
                              "ms": ms, "glps": n / ms / 1e6})
        fdev.set_kernel_config(lanes_per_query=args.lanes, smem_levels=args.smem_levels,
                               ctas_per_sm=args.ctas_per_sm, queries_per_lane=args.queries_per_lane,
                               min_ctas_per_sm=args.min_ctas, threads_per_cta=args.threads,
                               line_path=cfg["line_path"], plane_levels=cfg.get("plane_levels", 0))

    # -- other inputs and the update store (rank 0; extra keys, not the headline) ---------------------
    extras = None
    if rank == 0 and not args.no_extras:
        extras = time_extras(lpm, torch, fdev, fib, addrs, n, vb, stream, dev_index)

    # -- CPU baseline (rank 0, N = 1) ---------------------------------------------------------------------
    # -- CPU-baseline leg (rank 0): oracle check of the timed sample; oracle timing at N = 1 ------------
    cpu = None
    parity = oracle_check(fib, sample_addrs, sample_out, vb, cpu_threads()) if rank == 0 else None
    if rank == 0 and ws == 1 and not args.no_cpu:
        threads = cpu_threads()
        m_cpu = min(n, CPU_SAMPLE)
        ha = lpm.workload_queries_host(args.workload, fib, 0, m_cpu, threads=threads)
        times, kind, what = time_reference_cpu(fib, ha, threads, repeats=1)
        cpu = {"value": m_cpu / times[0] / 1e9, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"first {m_cpu} queries of {info.name}", "what": what, "cpu": cpu_model()}
        try:
            dt, variant = time_restated_planb(fib, ha, threads)
            cpu["restated_planb"] = {"value": m_cpu / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
                                     "variant": variant}
        except Exception as e:
            cpu["restated_planb"] = {"error": str(e)}
        cpu["single_thread"] = single_thread_baselines(fib, ha)

    if rank != 0:
        if dist is not None:
            dist.barrier()
        return 0

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64",
        "data": f"synthetic: seeded {info.name} FIB ({len(fib)} prefixes) and query generator, "
                f"{n} queries per GPU generated on device",
        "config": shared_config(info, len(fib), n, ws),
        "layout": {"intervals": geom.num_keys, "tree_depth": geom.depth, "node_keys": geom.k,
                   "leaf_keys": geom.leaf_keys, "tree_bytes": tree_bytes,
                   "sharding": "query batches; FIB replicated by NCCL broadcast"},
        "kernel": cfg,
        "l2_flush": f"not needed: each step streams {n * 16 / 1e9:.1f} GB of addresses (> 126 MB L2)",
        "roofline": roofline_object(geom, vb, cfg, lps_gpu, l2_gbs, smem_gbs, hbm_gbs, hbm_src, info.name, n,
                                    clocks.get("sm_mhz")),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "cuda_graph": use_graph,
        "clocks": clocks,
        "parity_sample": parity,
        "fib_build_ms": build_ms,
        "fib_build_device_ms": device_build_ms(lpm, fib, dev_index, vb),
        "fib_broadcast_ms": bcast_ms,
        "step_ms": step_ms,
        "ms_per_step_median": float(np.median(step_ms)),
        "per_rank_total_ms": per_rank_ms,
        "output_digest": {"per_rank_block_hash": block_hashes,
                          "note": "rank r's block = queries [r*n, (r+1)*n); equal across GPU counts"},
    }
    if sweep is not None:
        line["sweep"] = sweep
    if extras is not None:
        line["extras"] = extras
        if "keys8_e2e" in extras:
            # the same lookups from host buffers of 8-byte keys — the input of the reference's
            # batched search (search_batch) — i.e. half the PCIe bytes of `e2e`
            k = extras["keys8_e2e"]
            line["e2e_keys"] = {"value": k["value"], "unit": k["unit"], "h2d_bytes_per_step": k["h2d_bytes_per_step"],
                                "d2h_bytes_per_step": k["d2h_bytes_per_step"], "path": k["path"],
                                "matches_address_path": k["matches_address_path"]}
    if ws > 1 and shared_gpu_mode():
        line["harness_check"] = "LPM6_BENCH_SHARED_GPU: ranks shared GPUs over gloo; not a bench value"
    if ws == 1 and force_dist_mode():
        line["harness_check"] = "LPM6_BENCH_FORCE_DIST: the multi-rank collectives ran through NCCL at world size 1"
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
