#!/bin/bash
# bit-identity and timing of the 128-row SYMV epilogue against the 32-row one
mkdir -p gpurun_out
python scripts/epilogue_ab.py gpurun_out/epi_r128.npz
KBLAS_SYMV_EPILOGUE=32 python scripts/epilogue_ab.py gpurun_out/epi_r32.npz
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/epi_r128.npz"), np.load("gpurun_out/epi_r32.npz")
bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=True)]
print("cases", len(a.files), "bit-different", len(bad), bad[:8])
PY
for e in r128 32; do
  if [ $e = 32 ]; then export KBLAS_SYMV_EPILOGUE=32; else unset KBLAS_SYMV_EPILOGUE; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/epi_$e.csv python bench.py --steps 4 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  python - $e <<'PY'
import csv, io, sys, collections
txt = open(f"gpurun_out/epi_{sys.argv[1]}.csv").read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
agg = collections.defaultdict(list)
for r in rows:
    if "symv" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum":
        agg[r["Kernel Name"].split("(")[0][-45:]].append(float(r["Metric Value"].replace(",", "")))
print(sys.argv[1], {k: (len(v), round(sum(v) / len(v) / 1e3, 1)) for k, v in agg.items()})
PY
done
unset KBLAS_SYMV_EPILOGUE
