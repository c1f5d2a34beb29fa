"""Per-layer roofline table from a bench.py JSON line.

    python tools/layer_roofline.py gpurun_out/<tag>_bench.log > profiles/<round>_layer_roofline.md

Uses the engine's own per-launch bookkeeping that bench.py records under
roofline.per_layer (FLOPs; algorithmic bytes = each layer's input + weights + outputs
once per step, as engine.CompiledGraph.op_info counts them) -- no name matching -- and
the dense peaks bench.py used (roofline.peaks_tflops: measured tcgen05 MMA burst peaks)
with the HBM bandwidth of MEASURED_PEAKS.json."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    line = next(ln for ln in open(sys.argv[1]) if ln.startswith("{"))
    d = json.loads(line)
    r = d["roofline"]
    peaks = r["peaks_tflops"]
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6535.4
    print(f"Per-layer roofline, {d['config']['workload']} ({d['config'].get('plan')}), one step; peaks (TFLOP/s): "
          f"{peaks}, HBM {hbm} GB/s\n")
    print("| layer | precision | ms / step | TFLOP/s | % dtype peak | GB/s (alg.) | % HBM | bound | time / bound |")
    print("|---|---|---|---|---|---|---|---|---|")
    tot_t = tot_b = 0.0
    for name, e in r["per_layer"].items():
        s = e["ms"] / 1e3
        pk = peaks.get(e["precision"], peaks.get("fp16"))
        t_c, t_m = e["flops"] / (pk * 1e12), e["bytes"] / (hbm * 1e9)
        bound = "tensor" if t_c >= t_m else "hbm"
        tot_t += s
        tot_b += max(t_c, t_m)
        print(f"| {name} | {e['precision']} | {e['ms']:.4f} | {e['flops'] / s / 1e12:.0f} | "
              f"{100 * e['flops'] / s / 1e12 / pk:.0f} | {e['bytes'] / s / 1e9:.0f} | "
              f"{100 * e['bytes'] / s / 1e9 / hbm:.0f} | {bound} | {s / max(t_c, t_m):.2f} |")
    print(f"| **sum** | | {tot_t * 1e3:.4f} | | | | | | {tot_t / tot_b:.2f} |")


if __name__ == "__main__":
    main()
