"""Turn one round's ncu outputs (gpurun_out/) into the tracked summaries under profiles/.

    python scripts/make_profiles.py TAG MAPS

reads gpurun_out/launches_TAG.csv (the --metrics gpu__time_duration.sum launch
list of `bench.py --maps MAPS --steps 1 --warmup 1`) and gpurun_out/prof_TAG.ncu-rep
(the --set full capture of the two hot kernels), and writes
profiles/TAG_launches.md, profiles/TAG_ncu_full.txt and profiles/ncu_summary.json
(DRAM bytes per launch per map, read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(__file__))
from ncu_summary import summarize  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = re.compile(r"sat_systolic|sat_cluster|sat_cta|fill_sentinel|cert_|cfar_ws|cfar_fused|cfar_integral|cfar_naive|sort_detections|sort_runs|merge_pass|frontend_|rfrm_")


def short(name):
    m = re.search(r"(\w+_kernel)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(tag):
    path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg, order = {}, []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"]) if OURS.search(r["Kernel Name"]) else "(torch: synthetic input generation)"
        ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1)
        if k not in agg:
            agg[k] = [0, 0.0]
            order.append(k)
        agg[k][0] += 1
        agg[k][1] += ns
    return order, agg


def main():
    tag, maps = sys.argv[1], int(sys.argv[2])
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    order, agg = launches(tag)
    ours = {k: v for k, v in agg.items() if not k.startswith("(torch")}
    tot = sum(v[1] for v in ours.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list, `bench.py --maps {maps} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline`\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold-cache launches;\n"
                "compare shares, not absolute times). Two passes (warmup + 1 timed step) over the batch.\n\n")
        f.write("| kernel | launches | total ms | share of library kernels |\n|---|---:|---:|---:|\n")
        for k in order:
            n, ns = agg[k]
            share = f"{100 * ns / tot:.1f}%" if k in ours else "-"
            f.write(f"| `{k}` | {n} | {ns / 1e6:.3f} | {share} |\n")
    # the raw launch list of the library's kernels (ncu CSV rows, unmodified)
    src = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    lines = [l for l in open(src) if l.startswith('"')]
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        f.write(lines[0])
        for l in lines[1:]:
            if OURS.search(l):
                f.write(l)
    full = summarize(os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep"))
    # merge: kernels captured by other runs keep their entries
    summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = json.load(open(summ)) if os.path.exists(summ) else {}
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.txt"), "w") as f:
        f.write(f"# {tag}: ncu --set full --clock-control none, bench.py --maps {maps} (one launch each, cfg3 maps)\n")
        for d in full:
            f.write(f"----- {d['kernel'][:100]}\n")
            for k, v in d.items():
                if k != "kernel":
                    f.write(f"  {k:66s} {v}\n")
            def num(key):
                v, u = d[key].split()[:2] if len(d[key].split()) > 1 else (d[key].split()[0], "")
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(u, 1)
                return float(v.replace(",", "")) * scale
            rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
            name = short(d["kernel"]).split("<")[0]
            js[name] = {"tag": tag, "maps": maps, "dram_read_bytes": rd, "dram_write_bytes": wr,
                        "source": f"ncu --set full of bench.py (config 3, {maps} maps), profiles/{tag}_ncu_full.txt",
                    "dram_bytes_per_launch_per_map": (rd + wr) / maps,
                        "duration": d["gpu__time_duration.sum"]}
    with open(summ, "w") as f:
        json.dump(js, f, indent=1)
    print(json.dumps(js, indent=1))


if __name__ == "__main__":
    main()
