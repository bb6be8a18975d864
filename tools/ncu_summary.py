"""Summaries of an ncu launch list (csv) and a full-set report (.ncu-rep) for profiles/.
usage: python tools/ncu_summary.py TAG   (reads gpurun_out/launches_TAG.csv, gpurun_out/prof_TAG.ncu-rep)"""
import collections, csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "profiles")


def short(name):
    name = name.replace("void ", "").replace("sphg::", "").replace("(anonymous namespace)::", "")
    name = name.replace("<unnamed>::", "").replace("unnamed>::", "")
    return name.split("(")[0]


rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv"))))
i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[i]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
agg, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[i + 1:]:
    if len(r) > mv:
        try:
            v = float(r[mv].replace(",", ""))
        except ValueError:
            continue
        agg[short(r[kn])] += v / 1e6
        cnt[short(r[kn])] += 1
tot = sum(agg.values())
launch = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 5 --warmup 3 "
                    "--no-e2e --no-cpu-baseline (C5 64M, 1x B200); cold-cache serialised launches: compare shares",
          "total_ms": round(tot, 3),
          "kernels": [{"kernel": k, "launches": cnt[k], "ms_total": round(v, 3), "ms_per_launch": round(v / cnt[k], 3),
                       "share": round(v / tot, 4)} for k, v in sorted(agg.items(), key=lambda x: -x[1])]}
json.dump(launch, open(os.path.join(out, f"{tag}_launches_64m.json"), "w"), indent=1)
full = []
for rep in (os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep"),
            os.path.join(ROOT, "gpurun_out", f"prof_{tag}_build.ncu-rep"),     # the Verlet builder
            os.path.join(ROOT, "gpurun_out", f"prof_{tag}_density.ncu-rep")):  # k_density (tools/prof_density.sh)
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units = rr[0], rr[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "smsp__inst_executed.sum"]
    for r in rr[2:]:
        if "nan" in r[hdr.index("dram__bytes_read.sum")].lower():
            continue  # a capture whose metric passes failed (repeated kernel); the other capture is kept
        e = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k in keys:
            if k in hdr:
                e[k] = (r[hdr.index(k)] + " " + units[hdr.index(k)]).strip()
        st = {}
        for j, hh in enumerate(hdr):
            if hh.startswith("smsp__pcsamp_warps_issue_stalled_") and not hh.endswith("not_issued"):
                try:
                    st[hh.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[j].replace(",", ""))
                except ValueError:
                    pass
        s = sum(st.values()) or 1.0
        e["stalls_pct"] = {k: round(100 * v / s, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        full.append(e)
if full:
    json.dump(full, open(os.path.join(out, f"{tag}_ncu_full_64m.json"), "w"), indent=1)
print("ok", tag)
