start=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; echo "tests rc=$? t=$(( $(date +%s) - start ))" >> gpurun_out/final_times.txt
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$? t=$(( $(date +%s) - start ))" >> gpurun_out/final_times.txt
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$? t=$(( $(date +%s) - start ))" >> gpurun_out/final_times.txt
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$? t=$(( $(date +%s) - start ))" >> gpurun_out/final_times.txt
