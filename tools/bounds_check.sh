# Bounds-checking build of libedkm.so (-DEDKM_BOUNDS: device asserts on the table kernels' indexing,
# table_common.cuh) run through the GPU parity, multi-rank and full-size suites and the sanitizer
# step -- the substitute for compute-sanitizer, which this pool has closed.
# Usage (on the GPU box): bash tools/bounds_check.sh > gpurun_out/bounds_check.txt 2>&1
set -u
LIB=paper_2309_00964_b200/libedkm_bounds.so
python -c "from paper_2309_00964_b200 import build as B; B.build(out='$LIB', defines=['EDKM_BOUNDS'])" || exit 1
echo "checking build: $LIB ($(nm -D $LIB | grep -c ' T edkm_') exported edkm_ symbols)"
EDKM_LIB=$LIB python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -q 2>&1 | tail -3
EDKM_LIB=$LIB python tools/sanitize_step.py && echo "sanitize_step: ok"
for wl in cfg3 cfg4; do
  EDKM_LIB=$LIB python bench.py --workload $wl --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-clocks \
      > /dev/null 2>&1 && echo "bench $wl under the checking build: ok" || echo "bench $wl under the checking build: FAILED"
done
