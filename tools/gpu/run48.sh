# C1 / C3a / C3b bench lines again, now that profiles/r02_ncu_metrics.json holds the v20 captures
# (their roofline objects cite the capture of the kernel they ran).
cd $GRAFT_REPO_ROOT
O=gpurun_out
for w in C1 C3a C3b; do
  timeout 900 python bench.py --workload $w > $O/r48_bench_$w.json 2> $O/r48_bench_$w.err
done
python - <<'PY'
import json
for w in ("C1","C3a","C3b"):
    d=json.loads(open(f"gpurun_out/r48_bench_{w}.json").read().strip().splitlines()[-1]); k=d["kernel"]; r=d["roofline"]
    print(w, round(d["value"],2), "lp",k["line_path"],"tiles",k["queries_per_lane"],"planes",k["plane_levels"],"l1ceil",round(r["l1_wavefront_ceiling_glps"],1),"frac_l1",round(r["frac_of_l1_ceiling"],3), r["ncu_capture"], "e2e", round(d["e2e"]["value"],3), d["parity_sample"]["mismatches"])
PY
