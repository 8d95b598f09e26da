# like ab_libs.sh with extra bench arguments: ab_libs_args.sh "<bench args>" lib1.so lib2.so ...
LIB=paper_2605_20868_b200/libcertkv_b200.so
ARGS="$1"; shift
for v in "$@"; do
  cp "$v" $LIB; touch $LIB
  for i in 1 2; do
    python bench.py --no-cpu-baseline --no-e2e $ARGS 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$ARGS', round(d['ms_per_step'],4), round(d['roofline']['pass_a_ms'],4))"
  done
done
