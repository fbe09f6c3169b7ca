# Round-2 measurements + profile captures (one gpurun call; each ncu run only after the same command exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in c4 c3 c2 c1; do
  python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/r02_bench_$cfg.jsonl 2> gpurun_out/r02_bench_$cfg.err
done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 8000 --csv \
    --log-file gpurun_out/r02_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu3.log 2>&1
python scripts/prof_hvp.py --m 3 > gpurun_out/plain_hvp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:gemm3_tc2|gs_pass|split_pair|ritz_tc" -s 60 -c 16 \
    -o gpurun_out/r02_hvp_kernels python scripts/prof_hvp.py --m 3 > gpurun_out/ncu1.log 2>&1
ls -la gpurun_out
