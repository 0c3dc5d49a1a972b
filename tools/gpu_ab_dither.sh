#!/bin/bash
# Dithering-kernel A/B on one box: parity of each candidate build (dither kinds,
# full-size C4), then alternating C4 bench lines of ab_old/ (HEAD build), the
# working tree and ab_magic/ (working tree built with -DBPC_LIN_MAGIC).
mkdir -p gpurun_out
OUT=$PWD/gpurun_out
for v in . ab_magic; do
  tag=$(basename $(cd $v && pwd))
  (cd $v && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_units.py \
     -k "dither or C4" -x -q > $OUT/ab_pytest_$tag.log 2>&1; echo pytest_$tag=$?; tail -2 $OUT/ab_pytest_$tag.log)
done
for rep in 1 2; do
  for v in ab_old . ab_magic; do
    tag=$(basename $(cd $v && pwd))
    (cd $v && timeout 300 python bench.py --config C4 --steps 300 --warmup 10 --no-cpu --no-e2e > $OUT/ab_${tag}_$rep.json 2> $OUT/ab_${tag}_$rep.err)
    tail -1 $OUT/ab_${tag}_$rep.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', $rep, d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})"
  done
done
