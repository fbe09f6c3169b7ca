# Round-end profile captures (one gpurun call; ncu runs only after the same command exited 0).
set -x
cd $GRAFT_REPO_ROOT
python scripts/prof_hvp.py --m 3 > gpurun_out/plain_hvp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:gemm3_tc2|gs_pass" -s 60 -c 12 -o gpurun_out/r01_hvp_kernels python scripts/prof_hvp.py --m 3 > gpurun_out/ncu1.log 2>&1
python scripts/upd_bench.py 30000000 32 > gpurun_out/plain_upd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:upd_p" -s 3 -c 3 -o gpurun_out/r01_upd python scripts/upd_bench.py 30000000 32 > gpurun_out/ncu2.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r01_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
