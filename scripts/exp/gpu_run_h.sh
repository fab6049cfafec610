TESTS="tests/test_gpu_parity.py tests/test_gpu_pins.py" bash scripts/gpu_quick.sh
SAGA_REPLAY_TRACE=1 timeout 900 python scripts/profile_step.py --config C2 > gpurun_out/trace_c2.log 2>&1
python - gpurun_out/trace_c2.log <<'PY'
import re, sys, collections
agg = collections.defaultdict(lambda: [0, 0.0, [0.0] * 8])
for l in open(sys.argv[1]):
    m = re.search(r"pol=(\d+) cap=(\d+) .* Mcycles=([\d.]+) phases=([\d.,]+)", l)
    if m:
        a = agg[int(m.group(1))]
        a[0] += 1; a[1] = max(a[1], float(m.group(3)))
        for i, x in enumerate(m.group(4).split(",")): a[2][i] += float(x)
for p, a in sorted(agg.items()):
    print("pol", p, "items", a[0], "max Mcycles", a[1], "mean phases", [round(x / a[0], 1) for x in a[2]])
PY
CFGS="C1 C3 C4 C5" bash scripts/gpu_configs2.sh
