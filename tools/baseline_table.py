"""BASELINE.md §2 table rows from the committed bench lines (profiles/<tag>_bench/*.json).
usage: python tools/baseline_table.py [r02_bench]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r02_bench")
ORDER = [("bench_train8_1m", "train8_1m (8 × 1080p, fwd+bwd)"),
         ("bench_mip360_1m", "mip360_1m (1 × 1080p, fwd)"),
         ("bench_nerfsynth200k", "nerfsynth200k (8 × 800², fwd+bwd)"),
         ("bench_sweep64_3m", "sweep64_3m (64 × 1080p, fwd)"),
         ("bench_train8_1m_dipoles", "train8_1m + dipoles (NEXT-1)"),
         ("bench_nerfsynth200k_detail8", "nerfsynth200k + 8 detail sites (NEXT-2)"),
         ("bench_train8_1m_detail8", "train8_1m + 8 detail sites (NEXT-2)"),
         ("bench_train8_1m_fisheye", "train8_1m, 200° fisheye (NEXT-4)"),
         ("bench_train8_1m_knn", "train8_1m, unfiltered sym-16NN lists (P:236)"),
         ("bench_mip360_1m_trace", "mip360_1m, adjacency-walk tracer (NEXT-4)"),
         ("bench_mip360_1m_trace_fisheye", "mip360_1m, tracer, 200° fisheye")]


def f(x, nd=1):
    return "–" if x is None else f"{x:,.{nd}f}"


print("| config | GPUs | fwd FPS | fwd Mpix/s | fwd+bwd FPS | fwd+bwd Mpix/s | sort HBM | "
      "dominant kernel (frac) | step FP32 / HBM frac | e2e FPS |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name, label in ORDER:
    p = os.path.join(d, name + ".json")
    if not os.path.exists(p):
        continue
    j = json.loads(open(p).read().strip().splitlines()[-1])
    train = j["config"].get("pass") == "fwd+bwd"
    ro = j.get("roofline") or {}
    tr = j.get("trace")
    if tr:
        ro = tr["roofline"]
    kern = ro.get("kernel", "?").split(" ")[0]
    dom = f"{ro['frac']:.3f} {'HBM ' if ro.get('unit') == 'GB/s' else ''}({kern})" if ro else "–"
    st = j.get("roofline_step") or {}
    step = f"{st['fp32_frac']:.3f} / {st['hbm_frac']:.3f}" if st else "–"
    srt = (j.get("sort") or {}).get("hbm_frac")
    e2e = (j.get("e2e") or {}).get("value")
    fwd = j.get("fwd_fps") if train else j["value"]          # render workloads: the headline
    fmp = j.get("fwd_mpix_s") if train else j.get("mpix_s")
    print(f"| {label} | {j['n_gpus']} | {f(fwd)} | {f(fmp, 0)} | "
          f"{('**' + f(j['value']) + '**') if train else 'n/a'} | {f(j.get('mpix_s'), 0) if train else 'n/a'} | "
          f"{f(srt, 2) if srt is not None and not tr else '–'} | {dom} | {step if not tr else '–'} | {f(e2e)} |")
