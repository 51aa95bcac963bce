timeout 900 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_protected_quick.py tests/test_gpu_parity.py tests/test_gpu_depthwise.py tests/test_gpu_conv_quick.py -q -x > gpurun_out/t_r02s.log 2>&1
bash tools/_ab.sh A C C2
echo done
