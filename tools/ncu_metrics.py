"""Per-query figures from one `ncu --set full` capture's raw page (CSV), merged into
profiles/r02_ncu_metrics.json under a workload label; bench.py reads them for the
roofline object (DRAM traffic, L1 data-pipe wavefronts -> the kernel's own ceiling).
    python tools/ncu_metrics.py <raw.csv> <queries> <label> <capture-name>"""
import csv
import json
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parents[1] / "profiles" / "r02_ncu_metrics.json"


def main(raw, queries, label, capture):
    rows = list(csv.reader(open(raw)))
    d = {h: v for h, v in zip(rows[0], rows[2])}
    f = lambda k: float(d[k].replace(",", ""))
    sms = f("device__attribute_multiprocessor_count") if "device__attribute_multiprocessor_count" in d else 148
    q = float(queries)
    lsu = f("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg") * sms / q
    shared = f("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg") * sms / q
    shared_ld = f("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum") / q
    dram_r = f("dram__bytes_read.sum") * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[rows[1][rows[0].index("dram__bytes_read.sum")]]
    dram_w = f("dram__bytes_write.sum") * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[rows[1][rows[0].index("dram__bytes_write.sum")]]
    e = {"l1_wavefront_ceiling_glps": None,
        "capture": capture, "queries": int(q), "gpu_time_ms": f("gpu__time_duration.sum"),
        "lsu_data_pipe_pct": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "tex_data_pipe_pct": f("l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "lsu_wavefronts_per_query": lsu, "shared_ld_wavefronts_per_query": shared_ld,
        "shuffle_wavefronts_per_query": shared - shared_ld, "lgds_wavefronts_per_query": lsu - shared,
        "tex_wavefronts_per_query": f("l1tex__t_output_wavefronts_pipe_tex_mem_texture.sum") / q,
        "bank_conflicts_per_query": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") / q,
        "instructions_per_query": f("smsp__inst_executed.sum") / q,
        "dram_read_bytes": dram_r, "dram_write_bytes": dram_w, "dram_bytes_per_query": (dram_r + dram_w) / q,
        "sm_clock_mhz": f("sm__cycles_elapsed.avg.per_second") * 1e3,  # reported in GHz
    }
    # the kernel's own ceiling: one L1 data-pipe wavefront per SM per clock
    e["l1_wavefront_ceiling_glps"] = sms * e["sm_clock_mhz"] * 1e6 / lsu / 1e9
    allm = json.loads(OUT.read_text()) if OUT.exists() else {}
    allm[label] = e
    OUT.write_text(json.dumps(allm, indent=1) + "\n")
    print(json.dumps(e, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
