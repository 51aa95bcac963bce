timeout 900 python bench.py > gpurun_out/bench_r02_full3.json 2>gpurun_out/bench_r02_full3.err
Q="--no-cpu-baseline --skip-vgg --skip-mbv2 --skip-r50net --skip-abft --skip-campaign5 --campaign-trials 10"
timeout 600 python bench.py $Q --global-batch 1024 --steps 5 --warmup 3 > gpurun_out/b1024_r02d.json 2>gpurun_out/b1024_r02d.err
echo done
