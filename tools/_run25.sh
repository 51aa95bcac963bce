timeout 900 python -m pytest tests/test_gpu_fic_staged.py tests/test_gpu_bench_configs.py tests/test_gpu_depthwise.py tests/test_gpu_protected_quick.py -q -x > gpurun_out/t_r02t.log 2>&1
bash tools/_ab.sh A C3 C4
echo done
