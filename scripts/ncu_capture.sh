#!/bin/bash
# ncu --set full of one persistent launch of scripts/ncu_pass.py; exports the raw
# metrics CSV and the 60 hottest SASS lines (by warp-stall samples) into gpurun_out/.
# usage: bash scripts/ncu_capture.sh <tag> <inst> <kind> <s> <iters>
tag=$1; shift
mkdir -p gpurun_out
rm -f /tmp/$tag.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hallar -s 1 -c 1 \
  -o /tmp/$tag python scripts/ncu_pass.py "$@" > gpurun_out/$tag.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>>gpurun_out/$tag.log
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > /tmp/${tag}_src.csv 2>>gpurun_out/$tag.log
python3 - "$tag" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/{tag}_src.csv", errors="replace")))
hdr = rows[0]
def col(name):
    for i, h in enumerate(hdr):
        if h.strip() == name:
            return i
    return None
ws = col("Warp Stall Sampling (All Samples)")
if ws is None:
    ws = next((i for i, h in enumerate(hdr) if "Stall Sampling" in h), None)
body = [r for r in rows[1:] if len(r) == len(hdr)]
def val(r):
    try:
        return float(r[ws].replace(",", ""))
    except Exception:
        return 0.0
body.sort(key=val, reverse=True)
with open(f"gpurun_out/{tag}_hot.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(hdr)
    for r in body[:60]:
        w.writerow(r)
PY
ls -la /tmp/$tag.ncu-rep >> gpurun_out/$tag.log
