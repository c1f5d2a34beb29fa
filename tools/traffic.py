"""Per-kernel DRAM traffic of one engine step from an ncu CSV
(ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv
 --profile-from-start off python tools/op_profile.py --op all)  ->  profiles JSON.

    python tools/traffic.py gpurun_out/traffic.csv profiles/r1_step_traffic.json
"""
import csv
import io
import json
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    text = open(src).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    kern = {}
    order = []
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        if key not in kern:
            kern[key] = {}
            order.append(key)
        v = r["Metric Value"].replace(",", "")
        unit = r["Metric Unit"]
        val = float(v)
        if unit in ("Mbyte", "MB"):
            val *= 1e6
        elif unit in ("Kbyte", "KB"):
            val *= 1e3
        elif unit in ("Gbyte", "GB"):
            val *= 1e9
        elif unit in ("usecond", "us"):
            val *= 1e-6
        elif unit in ("msecond", "ms"):
            val *= 1e-3
        elif unit in ("nsecond", "ns"):
            val *= 1e-9
        kern[key][r["Metric Name"]] = val
    out = []
    for key in order:
        m = kern[key]
        out.append({"id": int(key[0]), "kernel": key[1].split("(")[0][:80],
                    "dram_read_bytes": m.get("dram__bytes_read.sum"), "dram_write_bytes": m.get("dram__bytes_write.sum"),
                    "duration_s": m.get("gpu__time_duration.sum")})
    conv = [k for k in out if "conv_tc_kernel" in k["kernel"]]
    summary = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                         "--clock-control none (cold, serialised launches) of one eager step, batch 32, "
                         "tools/op_profile.py --op all",
               "conv_launches": len(conv),
               "conv_dram_bytes": sum((k["dram_read_bytes"] or 0) + (k["dram_write_bytes"] or 0) for k in conv),
               "kernels": out}
    json.dump(summary, open(dst, "w"), indent=1)
    print(len(out), "kernels;", len(conv), "conv launches;", summary["conv_dram_bytes"] / 1e6, "MB conv DRAM traffic")


if __name__ == "__main__":
    main()
