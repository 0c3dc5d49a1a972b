#!/bin/bash
# Three-way same-box A/B: parity of the working tree and ab_crw3/, then
# alternating bench lines of ab_old/ (HEAD), ab_crw3/ and the working tree.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out
SEL="tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py"
for v in . ab_crw3; do
  tag=$([ $v = . ] && echo new || echo $v)
  (cd $v && timeout 900 python -m pytest $SEL -x -q > $OUT/ab3_pytest_$tag.log 2>&1; echo pytest_$tag=$?; tail -1 $OUT/ab3_pytest_$tag.log)
done
for rep in 1 2; do
  for c in ${CONFIGS:-C4 C5 C2}; do
    for v in ab_old ab_crw3 .; do
      tag=$([ $v = . ] && echo new || echo $v)
      (cd $v && timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 > $OUT/ab3_${tag}_${c}_$rep.json)
      python -c "import json; d=json.load(open('$OUT/ab3_${tag}_${c}_$rep.json')); print('$tag $c $rep', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})"
    done
  done
done
