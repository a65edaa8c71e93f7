# Per-phase bench times of several workloads (no e2e / cpu baseline): bash tools/phases.sh cfg2 cfg4 ...
for wl in "$@"; do
  python bench.py --workload $wl --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ph.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ph.json')); print(sys.argv[1], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})" $wl
done
