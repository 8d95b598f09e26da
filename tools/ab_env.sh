# A/B over environment settings on the same box: each arg is "VAR=value" (or "-" for none)
python -c "import __graft_entry__ as g; g.build()"
for v in "$@"; do
  for i in 1 2; do
    if [ "$v" = "-" ]; then e=""; else e="$v"; fi
    env $e python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['pass_a_ms'],4))"
  done
done
