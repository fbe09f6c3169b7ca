set -x
cd $GRAFT_REPO_ROOT
python scripts/prof_hvp.py --m 3 > gpurun_out/plain_hvp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm3_tc2 -s 18 -c 1 -o gpurun_out/r01_gemm_fwdR python scripts/prof_hvp.py --m 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:gemm3_tc2_kernel<1" -s 2 -c 1 -o gpurun_out/r01_gemm_weight python scripts/prof_hvp.py --m 3 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:gemm3_tc2_kernel<0, 1>" -s 10 -c 1 -o gpurun_out/r01_gemm_bwdR python scripts/prof_hvp.py --m 3 > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:gs_pass" -s 2 -c 2 -o gpurun_out/r01_gs python scripts/prof_hvp.py --m 3 > gpurun_out/ncu4.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:upd_p2_tma|ritz_kernel|colsum_pairs" -s 8 -c 3 -o gpurun_out/r01_upd python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu5.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r01_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu6.log 2>&1
ls -la gpurun_out
