# k_select variant sweep (same box): step ms at C3 / kv1 with nb just below and above 8192
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { CKV_SEL=$1 timeout 300 python bench.py $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-variant 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%-8s %-40s %.4f ms' % ('$1', '$2', l['ms_per_step']))"; }
for v in 0:0 32:256 16:512 8:1024; do run $v "--ctx 131040"; done
for v in 0:0 64:256 32:512 16:1024; do run $v "--ctx 131088"; done
for v in 0:0 8:1024 16:512 32:256; do run $v "--ctx 131040 --kv-heads 1"; done
for v in 0:0 16:1024 32:512 64:256; do run $v "--ctx 131088 --kv-heads 1"; done
