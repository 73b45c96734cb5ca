# Copy the outputs of tools/gpu/r02h.sh (gpurun_out/) into profiles/ as the
# round-2 evidence files and refresh profiles/traffic.json.
#   bash tools/collect_r02.sh
set -e
G=gpurun_out; P=profiles
cp $G/bench.json $P/r02_bench_c4.json; cp $G/bench_ref.json $P/r02_bench_ref_c4.json
cp $G/bench_noahead.json $P/r02_bench_c4_noahead.json
cp $G/bench_c4u.json $P/r02_bench_c4_uncolored.json; cp $G/bench_c2_rmat20.json $P/r02_bench_c2_rmat20.json
cp $G/bench_c2u.json $P/r02_bench_c2_uncolored.json
cp $G/bench_c3_grid.json $P/r02_bench_c3_grid.json; cp $G/bench_c1_sbm.json $P/r02_bench_c1_sbm.json
python tools/iter_summary.py $G/iterw_c4_colored.csv 25 > $P/r02_iter_c4_colored_warm.txt
python tools/iter_summary.py $G/iterw_c4_uncolored.csv 25 > $P/r02_iter_c4_uncolored_warm.txt
python tools/prof_summary.py $G/launches.csv > $P/r02_launches_summary.txt 2>&1
cp $G/tl_c4c.txt $P/r02_timeline_c4_colored.txt; cp $G/tl_c4u.txt $P/r02_timeline_c4_uncolored.txt
cp $G/tl_c2c.txt $P/r02_timeline_c2_colored.txt
cp $G/ktrace_c4_ah.txt $P/r02_ktrace_c4_ahead_pass.txt; cp $G/ahead_stats_c4.txt $P/r02_ahead_stats_c4.txt
[ -f $G/l2_gather.txt ] && cp $G/l2_gather.txt $P/r02_l2_gather.txt
for c in c2_rmat20 c3_grid c4_chung_lu; do cp $G/rp_$c.txt $P/r02_run_profile_$c.txt; done
cp $G/rk_c4.txt $P/r02_run_kernels_c4.txt
[ -f $G/capped_c3_p4.txt ] && cp $G/capped_c3_p4.txt $P/r02_capped_c3_phase4.txt
python tools/ncu_full_summary.py $G/c4_ah_pass_full.ncu-rep "C4 coloured, ahead pass of a tail stage (k_ah_pass, launch 250 of the iteration), ncu --set full" > $P/r02_c4_ah_pass_full.txt
python tools/ncu_full_summary.py $G/c4_ah_accum_full.ncu-rep "C4 coloured, ahead accumulation of the window (k_ah_accum), ncu --set full" > $P/r02_c4_ah_accum_full.txt
python tools/ncu_full_summary.py $G/c4_t0_stage1_full.ncu-rep "C4 coloured, tier-0 decide of stage 1 (k_decide_t0, general path), ncu --set full" > $P/r02_c4_t0_stage1_full.txt
python - <<'PY'
import csv, json
DEC = ("k_decide_", "k_hub_accum", "k_hub_pass", "k_single_", "k_ah_accum", "k_ah_pass")
def decide_bytes(path):
    rows = list(csv.reader(open(path))); hdr = None; tot = 0.0
    for r in rows:
        if "Kernel Name" in r:
            hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and any(k in d["Kernel Name"] for k in DEC):
                tot += float(d["Metric Value"].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["Metric Unit"]]
    return tot
t = json.load(open("profiles/traffic.json"))
t["c4_chung_lu/colored"] = decide_bytes("gpurun_out/iterw_c4_colored.csv")
t["c4_chung_lu/uncolored"] = decide_bytes("gpurun_out/iterw_c4_uncolored.csv")
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
print("traffic", t["c4_chung_lu/colored"] / 1e9, t["c4_chung_lu/uncolored"] / 1e9)
PY
