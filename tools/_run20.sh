timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_i8_tc -s 5 -c 3 -o gpurun_out/prof_fic_r02 python tools/profile_step.py --variant fic --only layer1.1.conv2,layer3.1.conv2,layer4.1.conv2 --reps 3 > gpurun_out/prof_fic_r02.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-vgg --skip-mbv2 --skip-r50net --skip-abft --skip-campaign5 --campaign-trials 4 > gpurun_out/launches_bench_r02.log 2>&1
echo done
