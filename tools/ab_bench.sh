#!/bin/bash
# A/B on one box: bench of ab_old/ (a previous build) vs the working tree, alternating
for rep in 1 2; do
  for c in ${CONFIGS:-C2 C5}; do
    (cd ab_old && python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e > ../gpurun_out/ab_old_${c}_$rep.log 2>&1)
    python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e > gpurun_out/ab_new_${c}_$rep.log 2>&1
  done
done
