# A/B timing of library variants on one workload: bash tools/ab_wl.sh cfg4 lib1.so lib2.so ...
wl=$1; shift
for v in "$@"; do
  EDKM_LIB=$v python bench.py --workload $wl --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items() if not k.startswith('AR')})" $v
done
