# How the committed profiles were produced (run under gpurun from the repo root;
# outputs land in gpurun_out/, summaries are copied to profiles/ by hand).
# Usage: bash tools/profile_recipes.sh <recipe>
set -u
Q="--no-cpu-baseline --skip-vgg --skip-mbv2 --skip-r50net --skip-abft --skip-campaign5 --campaign-trials 4"
case "${1:-}" in
  launches)  # per-launch durations of the bench step (profiles/r02/launches_bench_r02.*)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 $Q > gpurun_out/launches_bench.log 2>&1
    python tools/launch_summary.py gpurun_out/launches_bench.csv ;;
  conv-full)  # one full ncu capture of the FIC conv on three layers (profiles/ncu_summary.json)
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_i8_tc -s 5 -c 3 \
      -o gpurun_out/prof_fic python tools/profile_step.py --variant fic \
      --only layer1.1.conv2,layer3.1.conv2,layer4.1.conv2 --reps 3 > gpurun_out/prof_fic.log 2>&1 ;;
  hbm-full)  # the HBM kernels, one launch each (profiles/r02/hbm_kernels_ncu_r02.txt)
    for k in colsum_i8_tall colsum_i8_wide pack_input_smem; do
      ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 \
        -o gpurun_out/hbm_$k -f python tools/hbm_sweep.py > /dev/null 2>&1
    done ;;
  epi)  # per-layer epilogue attribution (profiles/r02/epi_probe_*.txt)
    for L in 0 4 8 13; do for B in 32 1024; do for C in 0 2; do
      timeout 200 python tools/epi_probe.py --layer $L --batch $B --checks $C --flags 0 >> gpurun_out/epi_probe.txt 2>&1
    done; done; done ;;
  final)  # the round-end sequence: GPU tests, smoke, bench, reference arm
    timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1
    python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/final_smoke.log 2>&1
    timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
    timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err ;;
  *) echo "recipes: launches conv-full hbm-full epi final"; exit 2 ;;
esac
