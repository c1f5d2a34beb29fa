"""Per-layer roofline table from a bench.py JSON line and the engine's op_info.

    python tools/layer_roofline.py profiles/r1_bench_latest.json > profiles/r1_layer_roofline.md
FLOPs and algorithmic bytes (inputs once + outputs once per frame, weights ignored) are
recomputed from the PointPillars shapes; peaks from MEASURED_PEAKS.json (int8 = 2x bf16)."""
import json
import sys

B = 32
H0, W0 = 248, 216  # block-0 / concat resolution
LAYERS = {  # name: (M pixels per frame, N, K, precision, in bytes/elem, out bytes per pixel)
    "conv backbone.blocks.0.0": (H0 * W0, 64, 9 * 64, "fp16", 2, 64),
    "conv backbone.blocks.0.3": (H0 * W0, 64, 9 * 64, "int8", 1, 64),
    "conv backbone.blocks.0.6": (H0 * W0, 64, 9 * 64, "int8", 1, 64),
    "conv backbone.blocks.0.9": (H0 * W0, 64, 9 * 64, "int8", 1, 64 + 128),
    "conv backbone.blocks.1.0": (124 * 108, 128, 9 * 64, "int8", 1, 128),
    "conv backbone.blocks.1.3": (124 * 108, 128, 9 * 128, "int8", 1, 128),
    "conv backbone.blocks.1.6": (124 * 108, 128, 9 * 128, "int8", 1, 128),
    "conv backbone.blocks.1.9": (124 * 108, 128, 9 * 128, "int8", 1, 128),
    "conv backbone.blocks.1.12": (124 * 108, 128, 9 * 128, "int8", 1, 128),
    "conv backbone.blocks.1.15": (124 * 108, 128, 9 * 128, "int8", 1, 128 + 256),
    "conv backbone.blocks.2.0": (62 * 54, 256, 9 * 128, "int8", 1, 256),
    "conv backbone.blocks.2.3": (62 * 54, 256, 9 * 256, "int8", 1, 256),
    "conv backbone.blocks.2.6": (62 * 54, 256, 9 * 256, "int8", 1, 256),
    "conv backbone.blocks.2.9": (62 * 54, 256, 9 * 256, "int8", 1, 256),
    "conv backbone.blocks.2.12": (62 * 54, 256, 9 * 256, "int8", 1, 256),
    "conv backbone.blocks.2.15": (62 * 54, 256, 9 * 256, "int8", 1, 512),
    "conv neck.deblocks.0.0": (H0 * W0, 128, 64, "fp16", 2, 128),
    "conv neck.deblocks.1.0": (124 * 108, 4 * 128, 128, "fp16", 2, 4 * 128),
    "conv neck.deblocks.2.0": (62 * 54, 16 * 128, 256, "fp16", 2, 16 * 128),
    "conv heads(fused)": (H0 * W0, 20, 384, "int8", 1, 80),
}


def main():
    d = json.loads(open(sys.argv[1]).read().splitlines()[0])
    per = d["roofline"]["per_layer_ms"]
    peaks = {"fp16": 1599.3, "int8": 2 * 1599.3}
    hbm = 6535.4
    print("| layer | ms / 32 frames | TFLOP/s | % dtype peak | GB/s (alg.) | % HBM | bound | time / bound |")
    print("|---|---|---|---|---|---|---|---|")
    for name, ms in per.items():
        M, N, K, prec, ein, outb = LAYERS[name]
        flops = 2.0 * B * M * N * K
        cin = K // 9 if name.startswith("conv backbone.") else K
        # exact names (a suffix match would also catch the neck.deblocks.* layers)
        stride2 = name in ("conv backbone.blocks.1.0", "conv backbone.blocks.2.0")
        in_px = M * 4 if stride2 else M  # stride-2 convs read 4x their outputs
        in_bytes = in_px * cin * ein
        if name == "conv backbone.blocks.0.0":
            in_bytes = 16000 * cin * ein  # the gather reads pillar rows, not a canvas
        bytes_ = B * (in_bytes + M * outb)
        t_c, t_m = flops / (peaks[prec] * 1e12), bytes_ / (hbm * 1e9)
        bound = "tensor" if t_c >= t_m else "hbm"
        s = ms / 1e3
        print(f"| {name} | {ms:.4f} | {flops / s / 1e12:.0f} | {100 * flops / s / 1e12 / peaks[prec]:.0f} | "
              f"{bytes_ / s / 1e9:.0f} | {100 * bytes_ / s / 1e9 / hbm:.0f} | {bound} | {s / max(t_c, t_m):.2f} |")


if __name__ == "__main__":
    main()
