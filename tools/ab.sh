# A/B timing of library variants: bash tools/ab.sh lib1.so lib2.so ... (CFG3 bench phases, no e2e)
for v in "$@"; do
  EDKM_LIB=$v python bench.py --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/ab.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items() if not k.startswith('AR')})" $v
done
