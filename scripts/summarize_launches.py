"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) into profiles/.

    python scripts/summarize_launches.py gpurun_out/r01_c4_launches.csv profiles/r01_c4_launches.txt

Writes a per-kernel table (launches, device time, share, DRAM bytes per launch) and merges the DRAM bytes
per launch of the bench's kernel names into profiles/traffic.json (read by bench.py's roofline "traffic").
ncu times are cold-cache and serialised: compare shares, not absolutes."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH_NAMES = {"gemm3_tc2_kernel": "gemm3_tcgen05", "gemm3_tc_kernel": "gemm3_tcgen05", "gs_pass1_kernel": "gs_pass1",
               "gs_pass2_kernel": "gs_pass2", "upd_p1_kernel": "upd_p1", "upd_p2_tma_kernel": "upd_p2",
               "upd_p2_kernel": "upd_p2", "upd_p3_kernel": "upd_p3", "pack_weights_kernel": "pack_params",
               "colsum_pairs_kernel": "bias_colsum", "ritz_kernel": "extract.ritz",
               "pack_weights_f16_kernel": "pack_params", "split_pair_kernel": "split_pair",
               "ritz_tc_kernel": "extract.ritz"}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    n = n.split("::")[-1]
    return n.split("<")[0]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    hdr, per, units = None, {}, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        units[d["Metric Name"]] = d["Metric Unit"]
        per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
    tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[units.get("gpu__time_duration.sum", "ns")]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for v in per.values():
        a = agg[short(v["name"])]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0) * tscale
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# {os.path.basename(src)}: {len(per)} launches (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none; cold-cache, serialised)",
             f"{'kernel':28s} {'launches':>8s} {'total us':>12s} {'share':>7s} {'DRAM MB/launch':>15s}"]
    traffic = {}
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:28s} {a[0]:8d} {a[1]:12.1f} {100 * a[1] / tot:6.1f}% {a[2] / a[0] / 1e6:15.2f}")
        if n in BENCH_NAMES:
            b = BENCH_NAMES[n]
            t = traffic.setdefault(b, [0.0, 0])
            t[0] += a[2]
            t[1] += a[0]
    open(dst, "w").write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    for b, (byts, cnt) in traffic.items():
        cur[b] = round(byts / cnt, 1)
    cur["_source"] = os.path.basename(dst)
    json.dump(cur, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines[:25]))


if __name__ == "__main__":
    main()
