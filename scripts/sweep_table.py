"""Markdown table of a bench config sweep: python scripts/sweep_table.py sweep.jsonl tag > profiles/<tag>_config_sweep.md"""
import json
import sys

rows = [json.loads(x) for x in open(sys.argv[1]) if x.strip()]
tag = sys.argv[2] if len(sys.argv) > 2 else "sweep"
print("# Config sweep (1 x B200, `bench.py --steps 10 --warmup 3 --no-cpu`, L2 flushed between steps)\n")
print(f"Raw JSON lines: `profiles/{tag}_config_sweep.jsonl`.  Dense = fastest of cuDNN SDPA / flash-attn 2.8 / "
      "flashinfer on the same shape.\nPer-kernel times are CUDA-event brackets of each launch (include launch gaps).\n")
print("| args | ours (us) | dense best (us) | speed-up | path | Monarch GFLOP | eff. TFLOP/s | kernels (us x launches/step) |")
print("|---|---|---|---|---|---|---|---|")
for d in rows:
    ours = d["value"] * 1000
    dense = d.get("dense_fa_best_ms")
    sp = d.get("speedup_vs_dense")
    ks = "; ".join(f"{k['name']} {k['ms_avg'] * 1000:.1f}x{k['launches_per_step']:g}" for k in d.get("kernels", []))
    gf = d.get("algorithmic", {}).get("flops_per_layer", 0) / 1e9
    print(f"| `{d.get('args', '')}` | {ours:.1f} | {f'{dense * 1000:.1f}' if dense else '-'} | {sp if sp else '-'} | "
          f"{d['config'].get('path', '-')} | {gf:.2f} | {d.get('effective_tflops', '-')} | {ks} |")
