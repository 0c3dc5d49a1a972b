#!/bin/bash
# Reducer / unit-counter poll intervals: same-box A/B of the working tree
# (1000 / 512 ns), ab_a/ (200 / 128 ns) and ab_b/ (64 / 64 ns); parity of ab_b.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out
(cd ab_b && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > $OUT/abp_pytest_b.log 2>&1; echo pytest_b=$?; tail -1 $OUT/abp_pytest_b.log)
for rep in 1 2; do
  for c in C4 C5 C2; do
    for v in . ab_a ab_b; do
      tag=$([ $v = . ] && echo head || echo $v)
      (cd $v && timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 > $OUT/abp_${tag}_${c}_$rep.json)
      python -c "import json; d=json.load(open('$OUT/abp_${tag}_${c}_$rep.json')); print('$tag $c $rep', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})"
    done
  done
done
