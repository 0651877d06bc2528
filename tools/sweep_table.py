"""Markdown table of a tools/sweep.py JSON:
    python tools/sweep_table.py profiles/r02/sweep_r2e.json"""
import json
import sys


def main(path):
    d = json.load(open(path))
    print("| workload | ours FP32 (ms) | fully_fused schedule | cuFFT+cuBLAS (ms) | torch.fft (ms) | speed-up | "
          "3xTF32 (ms) | layer roofline | max rel. err |")
    print("|---|---|---|---|---|---|---|---|---|")
    n15 = 0
    for r in d["rows"]:
        err = max(v for v in r["max_rel_error"].values() if v is not None)
        sched = r["fully_fused_schedule"].replace("|", "\\|")
        n15 += r["speedup_vs_best_unfused"] >= 1.5
        print(f"| {r['workload']} | {r['best_ours_fp32']} | `{sched}` | {r['staged']} | {r.get('torch_fft')} | "
              f"{r['speedup_vs_best_unfused']:.2f}× | {r.get('tf32x3')} | {r['frac_layer_roofline']:.3f} | {err:.1e} |")
    print(f"\n{n15} of {len(d['rows'])} points >= 1.5x")


if __name__ == "__main__":
    main(sys.argv[1])
