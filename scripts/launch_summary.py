"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv, sys, collections
path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
d = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0][:70]
    v = float(r[iv].replace(",", ""))
    d.setdefault(name, []).append(v)
unit = "ns"
print(f"# ncu launch list {path} (gpu__time_duration.sum, --clock-control none)")
print("# per-launch times are cold-cache and serialised by ncu: compare SHARES of the step, not absolutes")
tot = sum(sum(v) for k, v in d.items() if "k_w4a8_gemm" in k or "k_act_quant" in k)
for k, v in d.items():
    share = f" share_of_ffn_kernels={sum(v) / tot:6.1%}" if ("k_w4a8_gemm" in k or "k_act_quant" in k) and tot else ""
    print(f"{k:72s} launches={len(v):4d} mean_{unit}={sum(v)/len(v):10.0f} min={min(v):10.0f} max={max(v):10.0f}{share}")
