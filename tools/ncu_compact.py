"""Compact an ncu --csv launch list (one row per metric) into one row per launch:
id,kernel,grid,block,time_us,dram_read_mb,dram_write_mb.

    python tools/ncu_compact.py gpurun_out/launchesNN.csv > profiles/<round>_launches.csv
"""
import collections
import csv
import io
import re
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def main():
    txt = open(sys.argv[1]).read()
    rows = csv.DictReader(io.StringIO(txt[txt.find('"ID"'):]))
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(r["ID"], {"kernel": re.sub(r"\(.*", "", r["Kernel Name"]).replace("unnamed>::", "").replace("void ", ""),
                                     "grid": r["Grid Size"], "block": r["Block Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v * TIME.get(u, 1e-3)
        elif r["Metric Name"] == "dram__bytes_read.sum":
            d["rd"] = v * BYTES.get(u, 1e-6)
        elif r["Metric Name"] == "dram__bytes_write.sum":
            d["wr"] = v * BYTES.get(u, 1e-6)
    w = csv.writer(sys.stdout)
    w.writerow(["id", "kernel", "grid", "block", "time_us", "dram_read_mb", "dram_write_mb"])
    for i, d in per.items():
        w.writerow([i, d["kernel"], d["grid"], d["block"], f"{d.get('us', 0):.2f}", f"{d.get('rd', 0):.2f}",
                    f"{d.get('wr', 0):.2f}"])


if __name__ == "__main__":
    main()
