# ab_env.sh with extra bench arguments: ab_env_args.sh "<bench args>" VAR=value|- ...
python -c "import __graft_entry__ as g; g.build()"
ARGS="$1"; shift
for v in "$@"; do
  for i in 1 2; do
    if [ "$v" = "-" ]; then e=""; else e="$v"; fi
    env $e python bench.py --no-cpu-baseline --no-e2e $ARGS 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$ARGS', round(d['ms_per_step'],4), round(d['roofline']['pass_a_ms'],4))"
  done
done
