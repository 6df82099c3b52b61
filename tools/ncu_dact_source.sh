# per-SASS-instruction execution counts of the dA kernel (one launch of the bench step)
out=gpurun_out/ncu_src; mkdir -p $out
ncu --clock-control none --kernel-name-base demangled -k regex:"${KRE:-gemm_kernel<\(int\)2,}" -c 1 --section SourceCounters \
  --import-source on -o $out/dact -f python bench.py --steps 1 --warmup 1 --mx 0 --sweep 0 --no-cpu-baseline > $out/run.log 2>&1
ncu -i $out/dact.ncu-rep --page source --csv --print-source sass > $out/dact_sass.csv 2> $out/src.err
ls -la $out; head -3 $out/dact_sass.csv | cut -c1-400
