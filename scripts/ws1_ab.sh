#!/bin/bash
# A/B of the SYMV t1 partial layout (row-block-major default vs tile-major)
# on one box: bench.py blocks (configs[4] D/Z 100k, configs[1]) interleaved.
mkdir -p gpurun_out
for rep in 1 2; do
  for lay in rowblock tile; do
    KBLAS_WS1_LAYOUT=$lay timeout 600 python bench.py --no-cpu --steps 30 > gpurun_out/ws1_ab_${lay}_$rep.log 2>&1
    python - "$lay" "$rep" <<'PY'
import json, sys
for line in open(f"gpurun_out/ws1_ab_{sys.argv[1]}_{sys.argv[2]}.log"):
    if line.startswith("{"):
        d = json.loads(line); z = d["zhemv_100k"]; c1 = d["configs1_dsymv_32768"]
        print(json.dumps({"layout": sys.argv[1], "rep": int(sys.argv[2]), "d100k": d["value"], "d100k_kernel_ms": d["per_rank"]["kernel_ms"][0],
              "d100k_step_ms": d["ms_per_step"], "z100k": z["value"], "z100k_kernel_ms": z["per_rank"]["kernel_ms"][0],
              "z100k_step_ms": z["ms_per_step"], "c1": c1["value"], "c1_step_ms": c1["ms_per_step"],
              "c1_kernel_ms": c1["roofline"]["kernel_avg_ms"], "sm_mhz": d["clocks"]["sm_mhz"]}))
PY
  done
done
