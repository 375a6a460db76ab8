# per-kernel device times (ncu launch list, serialized) for configs c2 and c5
mkdir -p gpurun_out
for CFG in c2 c5; do
  B="python bench.py --config $CFG --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
  $B > gpurun_out/plain_t_$CFG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pyramid_kernel|gftt_|klt_kernel" --csv --log-file gpurun_out/times_$CFG.csv $B > gpurun_out/ncu_t_$CFG.log 2>&1
  python - "$CFG" <<'PY'
import csv, sys, collections
cfg = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/times_{cfg}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        n = r[ki].split("(")[0].split("::")[-1][:40]
        d.setdefault(n, []).append(float(r[vi].replace(",", "")) / 1e3)
print(cfg, {k: round(sorted(v)[len(v) // 2], 1) for k, v in d.items()})
PY
done
