# A/B of library variants over several workloads: bash tools/ab_phases.sh "cfg1 cfg2 cfg3" lib1.so lib2.so ...
wls=$1; shift
for wl in $wls; do
  for v in "$@"; do
    EDKM_LIB=$v python bench.py --workload $wl --no-e2e --no-cpu-baseline --no-graph --steps 20 > gpurun_out/ab.json 2> gpurun_out/ab.err \
      || { echo "$wl $v FAILED"; tail -3 gpurun_out/ab.err; continue; }
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(sys.argv[1], sys.argv[2].split('/')[-1], round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['phases_ms'].items() if not k.startswith('AR')})" $wl $v
  done
done
