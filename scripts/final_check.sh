# Round-end verification: the full -m gpu suite, smoke, and the default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r02_gputest.log 2>&1; tail -3 gpurun_out/r02_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -2 gpurun_out/r02_smoke.log
python bench.py > gpurun_out/r02_bench_default.jsonl 2> gpurun_out/r02_bench_default.err; tail -c 400 gpurun_out/r02_bench_default.jsonl
