timeout 1100 python -m pytest tests -m gpu -q -x > gpurun_out/t_r02aa.log 2>&1
Q="--no-cpu-baseline --skip-vgg --skip-mbv2 --skip-r50net --skip-abft --skip-campaign5 --campaign-trials 10"
timeout 600 python bench.py $Q > gpurun_out/b32_r02aa.json 2>gpurun_out/b32_r02aa.err
echo done
