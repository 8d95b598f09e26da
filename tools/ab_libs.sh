# A/B of prebuilt library variants on the same box: for each .so given, install
# it as the in-tree library (newer than the sources, so build() keeps it) and
# run the default bench twice.
LIB=paper_2605_20868_b200/libcertkv_b200.so
for v in "$@"; do
  cp "$v" $LIB; touch $LIB
  for i in 1 2; do
    python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['pass_a_ms'],4))"
  done
done
