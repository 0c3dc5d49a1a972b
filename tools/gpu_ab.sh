#!/bin/bash
# Same-box A/B: parity of the working tree (SEL / KSEL), then alternating bench
# lines of ab_old/ (a HEAD build) and the working tree per config.
mkdir -p gpurun_out
OUT=$PWD/gpurun_out
SEL=${SEL:-"tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py"}
timeout 1200 python -m pytest $SEL ${KSEL:+-k "$KSEL"} -x -q > $OUT/ab_pytest.log 2>&1; echo pytest=$?; tail -2 $OUT/ab_pytest.log
for rep in 1 2; do
  for c in ${CONFIGS:-C2 C3 C4 C5}; do
    for v in ab_old .; do
      tag=$([ $v = . ] && echo new || echo old)
      (cd $v && timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 > $OUT/ab_${tag}_${c}_$rep.json)
      python -c "import json; d=json.load(open('$OUT/ab_${tag}_${c}_$rep.json')); print('$tag $c $rep', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()})"
    done
  done
done
