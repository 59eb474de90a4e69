# usage: ab.sh OUT "VAR=val ..." ... ; runs each env setting twice, interleaved (experiments build)
out=$1; shift
for i in 1 2; do for e in "$@"; do
  echo -n "$e : "
  env $e FADE_LIB_PATH=$PWD/build/exp/libfade_b200.so python bench.py --no-cpu-baseline --no-sweep --no-e2e $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']/d['config']['timesteps_per_step']*1000,2),'us', round(d['value'],4), round(d['config']['early_window_ms_per_step']/d['config']['timesteps_per_step']*1000,2), 'us early')"
done; done > gpurun_out/$out 2>&1
