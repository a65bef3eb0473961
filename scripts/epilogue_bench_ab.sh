#!/bin/bash
# step-time A/B of the 128-row SYMV epilogue (default) against the 32-row
# one (KBLAS_SYMV_EPILOGUE=32), interleaved on one box
mkdir -p gpurun_out
for rep in 1 2; do
  for e in r128 32; do
    if [ $e = 32 ]; then export KBLAS_SYMV_EPILOGUE=32; else unset KBLAS_SYMV_EPILOGUE; fi
    timeout 600 python bench.py --no-cpu --steps 30 > gpurun_out/epib_${e}_$rep.log 2>&1
    python - $e $rep <<'PY'
import json, sys
for line in open(f"gpurun_out/epib_{sys.argv[1]}_{sys.argv[2]}.log"):
    if line.startswith("{"):
        d = json.loads(line); z = d["zhemv_100k"]; c1 = d["configs1_dsymv_32768"]
        print(json.dumps({"epilogue": sys.argv[1], "rep": int(sys.argv[2]), "d100k": d["value"],
              "d100k_step_ms": d["ms_per_step"], "d100k_kernel_ms": d["per_rank"]["kernel_ms"][0],
              "z100k": z["value"], "c1": c1["value"], "c1_step_ms": c1["ms_per_step"], "e2e": d["e2e"]["value"]}))
PY
  done
done
unset KBLAS_SYMV_EPILOGUE
