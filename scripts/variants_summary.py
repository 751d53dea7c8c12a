import json, sys, glob, os
for f in sorted(glob.glob("gpurun_out/var/*.jsonl")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d["kernels"]
        print(f"{os.path.basename(f):14s} {d['value']:9.1f} it/s  " + "  ".join(f"{n}={v['ms_total'] / max(1, v['launches']) * 1e3:7.1f}us" for n, v in k.items()))
    except Exception as e:
        print(f, "failed", e)
