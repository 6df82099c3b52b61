out=gpurun_out/t5; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_ep_local.py tests/test_gpu_ipc_p2p.py tests/test_gpu_nccl_ep_path.py -x -q > $out/ep.log 2>&1; echo "rc=$?" >> $out/ep.log
