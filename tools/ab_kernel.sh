# Per-kernel device time (ncu launch list, gpu__time_duration) of one kernel for
# each prebuilt library variant, on the same box: ab_kernel.sh REGEX lib1.so lib2.so ...
LIB=paper_2605_20868_b200/libcertkv_b200.so
RE=$1; shift
for v in "$@"; do
  cp "$v" $LIB; touch $LIB
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$RE" --csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null |
    python3 -c "
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10 and r[-3] == 'gpu__time_duration.sum']
t = [float(r[-1]) for r in rows][-3:]
print('$v', [round(x, 1) for x in t])"
done
