out=gpurun_out/t7; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "quad" > $out/q.log 2>&1; echo "rc=$?" >> $out/q.log
timeout 2400 python -m pytest tests -m gpu -x -q > $out/all.log 2>&1; echo "rc=$?" >> $out/all.log
