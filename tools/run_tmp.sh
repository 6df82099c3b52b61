out=gpurun_out/t16; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_ipc_p2p.py -x -q > $out/ipc.log 2>&1; echo "rc=$?" >> $out/ipc.log
