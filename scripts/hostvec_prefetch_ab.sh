mkdir -p gpurun_out
for rep in 1 2; do
for pf in 1 0; do
  echo "== KBLAS_HOSTVEC_PREFETCH=$pf rep $rep"
  for n in 2048 4096 8192; do KBLAS_HOSTVEC_PREFETCH=$pf LD_LIBRARY_PATH=paper_1410_1726_b200 ./scripts/h2d_probe $n | grep -E "n=|kernel only|hostvec"; done
  KBLAS_HOSTVEC_PREFETCH=$pf python scripts/e2e_probe_symv.py 16384 30 | tail -1
done
done
