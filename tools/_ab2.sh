out=gpurun_out/ab_probe.txt; rm -f $out
for L in 0 4 8; do for B in 32 1024; do for C in 0 2; do for V in "$@"; do
  (cd abtmp/$V && echo -n "$V " >> ../../$out && timeout 200 python tools/epi_probe.py --layer $L --batch $B --checks $C --flags 0 >> ../../$out 2>&1)
done; done; done; done
