out=gpurun_out/t15; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_contract.py -x -q -k "full_size_sampled or gpu_arm" > $out/tests.log 2>&1; echo "rc=$?" >> $out/tests.log
timeout 600 python bench.py --config qwen3 --ep-emulate 8 --sweep 0 --mx 0 --no-cpu-baseline > $out/q8.json 2>&1
