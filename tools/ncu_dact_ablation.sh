out=gpurun_out/ncu_dact; mkdir -p $out
lib=paper_2511_21431_b200/libmemfine.so
cp $lib $out/.intree.so
for n in ${NAMES:-base noepi nosmem}; do
  cp ab_libs/$n.so $lib
  ncu --clock-control none --kernel-name-base demangled -k regex:"${KRE:-gemm_kernel<\(int\)2,}" -c 1 --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,smsp__inst_executed_pipe_xu.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_elapsed --csv python bench.py --steps 1 --warmup 1 --mx 0 --sweep 0 --no-cpu-baseline > $out/$n.csv 2> $out/$n.err
done
cp $out/.intree.so $lib
for n in ${NAMES:-base noepi nosmem}; do echo "== $n"; grep -v "^==" $out/$n.csv | grep -E "duration|cycles|tensor|inst|wavefronts|tma" | awk -F'","' 'NF>3{print $(NF-3), $(NF-2), $NF}' ; done
