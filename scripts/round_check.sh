# Round verification: the full -m gpu suite, smoke, and bench lines for C1-C4 (C4 = the default line).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_gputest.log 2>&1; tail -3 gpurun_out/r02_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -2 gpurun_out/r02_smoke.log
for c in c1 c2 c3; do python bench.py --config $c > gpurun_out/r02_bench_$c.jsonl 2> gpurun_out/r02_bench_$c.err; python scripts/bench_summary.py < gpurun_out/r02_bench_$c.jsonl | head -1; done
python bench.py > gpurun_out/r02_bench_c4.jsonl 2> gpurun_out/r02_bench_c4.err; python scripts/bench_summary.py < gpurun_out/r02_bench_c4.jsonl | head -1
