out=gpurun_out/t3; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ipc_p2p.py -x -q > $out/ipc.log 2>&1; echo "rc=$?" >> $out/ipc.log
timeout 900 python bench.py --config mixtral --ep-emulate 8 --no-cpu-baseline > $out/cfg_mixtral_ep8.json 2> $out/cfg_mixtral_ep8.err
