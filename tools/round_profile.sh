# Round-end evidence on one B200 (run under gpurun): GPU tests, the bench line (with e2e and
# cpu_baseline), the reference arm, per-workload phases, the N=2 gloo check-mode bench line, the
# ncu launch list of the bench command, one `--set full` capture of each kernel of one step, and
# compute-sanitizer.  Usage: bash tools/round_profile.sh r02
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
K='regex:f1_hist|tf_kernel|f2_gather|b1_bucket|tgamma_kernel|tb_kernel|tb_split|b2_dw'
EDKM_PARITY_REPORT=$O/${TAG}_parity_errors.json python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/${TAG}_pytest_gpu.txt
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
for wl in cfg2 cfg4 cfg4_b2 cfg5; do
  python bench.py --workload $wl --no-e2e --no-cpu-baseline --steps 10 > $O/${TAG}_phases_$wl.json 2>/dev/null
done
EDKM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 5 > $O/${TAG}_bench_gloo_n2.json 2> $O/${TAG}_bench_gloo_n2.err
EDKM_SHARD=slice EDKM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 5 --no-e2e > $O/${TAG}_bench_gloo_n2_slice.json \
    2> $O/${TAG}_bench_gloo_n2_slice.err
python tools/rank_sim.py --workload cfg3 > $O/${TAG}_rank_sim_cfg3.jsonl 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    -k "$K" --log-file $O/${TAG}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "$K" \
    --launch-skip 7 --launch-count 7 -o $O/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-graph > $O/${TAG}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tf_kernel|tgamma|tb_kernel" --launch-count 3 \
    -o $O/${TAG}_cfg4_table -f python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-graph > $O/${TAG}_ncu_cfg4_table.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  echo "$tool: $(compute-sanitizer --tool $tool python tools/sanitize_step.py 2>&1 | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' | tail -1)"
done > $O/${TAG}_sanitizer.txt
cat $O/${TAG}_pytest_gpu.txt; cat $O/${TAG}_bench.json; cat $O/${TAG}_bench_ref.json; tail -3 $O/${TAG}_ncu_full.log; cat $O/${TAG}_sanitizer.txt
