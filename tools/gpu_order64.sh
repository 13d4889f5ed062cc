#!/bin/bash
# launch order x Viterbi layout for the fp64 legs
run() { # label config dtype
  timeout 600 python bench.py --config $2 --no-cpu-baseline --single-dtype --dtype $3 --steps ${4:-20} --warmup 3 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1))"
}
for o in vit_first fb_first; do
  for v in lanes chain16; do
    export LOGHMM_PIPE_ORDER=$o
    if [ $v = lanes ]; then export LOGHMM_VIT_ALGO=lanes; unset LOGHMM_VIT_NW; else export LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=16; fi
    run "c2 f64 $o $v" c2 float64
  done
done
unset LOGHMM_VIT_ALGO LOGHMM_VIT_NW
for o in vit_first fb_first; do
  export LOGHMM_PIPE_ORDER=$o
  run "c3 f64 $o" c3 float64 10
  run "c4 f64 $o" c4 float64 10
  run "c5 f32 $o" c5 float32 3
  run "c5 f64 $o" c5 float64 3
done
