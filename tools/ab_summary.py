import glob, json, sys
tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/ab_{tag}_p*_d*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1][:-6], d["workload"][:10], f"{d['ms_per_step']:.4f} ms", f"{d['achieved_gbs']:.0f} GB/s",
                  f"{d['achieved_tflops']:.0f} TF/s", f"roof {d['roofline_frac']:.3f}")
        elif "Error" in l or "error" in l:
            print(f, l[:200])
