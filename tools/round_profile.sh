# Round-end evidence on one B200 (run under gpurun): GPU tests, the bench line (with e2e and
# cpu_baseline), the reference arm, the ncu launch list of the bench command and one
# `--set full` capture of each kernel of one step.  Usage: bash tools/round_profile.sh r01
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/${TAG}_pytest_gpu.txt
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    -k regex:"f1_hist|tf_kernel|f2_gather|b1_bucket|tgamma_kernel|tb_kernel|b2_dw|nccl" \
    --log-file $O/${TAG}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"f1_hist|tf_kernel|f2_gather|b1_bucket|tgamma_kernel|tb_kernel|b2_dw" \
    --launch-skip 7 --launch-count 7 -o $O/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/${TAG}_ncu_full.log 2>&1
cat $O/${TAG}_pytest_gpu.txt; cat $O/${TAG}_bench.json; cat $O/${TAG}_bench_ref.json; tail -3 $O/${TAG}_ncu_full.log
