for L in 0 4 8; do for B in 32 1024; do for C in 0 2; do timeout 200 python tools/epi_probe.py --layer $L --batch $B --checks $C --flags 0 >> gpurun_out/epi_probe21.txt 2>&1; done; done; done
timeout 600 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_protected_quick.py -q -x > gpurun_out/t_r02q.log 2>&1
echo done
