# A/B over compile flags: for each arg, rebuild with CKV_NVCC_EXTRA=arg and run the bench twice
for v in "$@"; do
  CKV_NVCC_EXTRA="$v" python -c "from paper_2605_20868_b200 import build; build.build(force=True)" || exit 1
  for i in 1 2; do
    python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['pass_a_ms'],4))"
  done
done
