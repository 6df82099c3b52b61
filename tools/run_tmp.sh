out=gpurun_out/t4; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_router.py -x -q > $out/tests.log 2>&1; echo "rc=$?" >> $out/tests.log
bash tools/lib_ab.sh "base W" --mx 0
