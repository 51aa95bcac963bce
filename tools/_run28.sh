timeout 1100 python -m pytest tests -m gpu -q > gpurun_out/t_r02v.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02_full2.json 2>gpurun_out/bench_r02_full2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv_i8_tc|verdict|ic_from|ic_final|icb_scan" -c 400 --csv --log-file gpurun_out/launches_bench_r02b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-vgg --skip-mbv2 --skip-r50net --skip-abft --skip-campaign5 --campaign-trials 4 > /dev/null 2>&1
echo done
