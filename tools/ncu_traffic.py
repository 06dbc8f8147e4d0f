"""Per-launch DRAM traffic of the roofline kernels from one `ncu --set full`
capture of tools/profile_step.py (cfg3): writes profiles/ncu_traffic.json,
which bench.py reads into the `traffic` fields.
Usage: python tools/ncu_traffic.py gpurun_out/prof.ncu-rep [out.json]"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name")
cols = {m: hdr.index(m) for m in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "usecond": 1e-3,
         "msecond": 1, "nsecond": 1e-6}


def val(r, m):
    return float(r[cols[m]].replace(",", "")) * scale.get(units[cols[m]], 1)


launches = []
for r in rows[2:]:
    launches.append((r[ki], val(r, "gpu__time_duration.sum"),
                     val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")))


def pick(sub, count=None):
    sel = [x for x in launches if sub in x[0]]
    return sel[:count] if count else sel


res = {}
sort = pick("k_hist<1>", 1) + pick("k_onesweep", 4)  # the first order-field sort
if len(sort) == 5:
    res["order_sort"] = sum(x[2] for x in sort)
for key, sub in [("classify", "k_classify_zreg<0>"), ("classify_ascent", "k_classify_zreg<1>")]:
    sel = pick(sub, 1)
    if sel:
        res[key] = sel[0][2]
fl = pick("k_big_flood")
if fl:
    res["k_big_flood"] = sum(x[2] for x in fl) / len(fl)
res["_source"] = {"report": rep.split("/")[-1], "unit": "bytes per launch (dram__bytes_read.sum + "
                  "dram__bytes_write.sum); order_sort = k_hist + 4 onesweep passes",
                  "launches": [[n[:60], round(ms, 4), b] for n, ms, b in launches]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "_source"}))
