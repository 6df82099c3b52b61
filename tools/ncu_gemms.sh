out=gpurun_out/ncu1; mkdir -p $out
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -c 7 -o $out/full \
  python bench.py --steps 1 --warmup 0 --mx 0 --sweep 0 --no-cpu-baseline > $out/run.log 2>&1
ncu -i $out/full.ncu-rep --page raw --csv > $out/full_raw.csv 2>/dev/null
ncu -i $out/full.ncu-rep --page details --csv > $out/full_details.csv 2>/dev/null
ls -la $out
