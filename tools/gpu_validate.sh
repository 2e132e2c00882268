# Full GPU validation: the -m gpu suite, smoke(), the default bench line and the reference arm.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/val
python -m pytest tests -m gpu -x -q > gpurun_out/val/gputests.log 2>&1; echo "tests exit $?" >> gpurun_out/val/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/val/smoke.log
python bench.py > gpurun_out/val/bench.log 2> gpurun_out/val/bench.err; echo "bench exit $?" >> gpurun_out/val/bench.err
tail -3 gpurun_out/val/gputests.log; tail -2 gpurun_out/val/smoke.log; cat gpurun_out/val/bench.log
