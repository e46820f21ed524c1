"""Summarise an ncu report: time, pipe utilisation, wavefronts per query, stall reasons."""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def f(d, k):
    try:
        return float(d[k][1].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


def main(rep, queries):
    d = raw(rep)
    sms = 148
    t = f(d, "gpu__time_duration.sum")
    print(f"{rep}: {t:.3f} ms, {queries / (t * 1e-3) / 1e9:.2f} G lookups/s")
    for k in ["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread", "launch__occupancy_limit_registers"]:
        print(f"  {k:70s} {f(d, k):10.2f}")
    per_q = lambda v: v / queries
    wf = f(d, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg") * sms
    wl = f(d, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg") * sms
    ws = f(d, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg") * sms
    print(f"  data-pipe wavefronts/query: total {per_q(wf):.2f}  global {per_q(wl):.2f}  shared+shfl {per_q(ws):.2f}")
    print(f"  instructions/query: {per_q(f(d, 'smsp__inst_executed.sum')):.2f}   "
          f"shared ld/query {per_q(f(d, 'smsp__sass_inst_executed_op_shared_ld.sum')):.3f}   "
          f"bank conflicts/query {per_q(f(d, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')):.2f}")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    dram = sum(f(d, k) * scale.get(d.get(k, ("byte", ""))[0], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"  dram bytes/query: {per_q(dram):.2f}")
    st = {k.split("stalled_")[1]: f(d, k) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued")}
    tot = sum(v for v in st.values() if v == v)
    top = sorted(st.items(), key=lambda kv: -kv[1])[:7]
    print("  stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 268435456)
