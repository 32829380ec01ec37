# A/B helper for gpurun: parity subset, then C2 bench lines for each library in $LIBS
# (default: the in-tree librrg.so twice).
LIBS=${LIBS:-"librrg.so librrg.so"}
python -m pytest tests -m gpu -x -q -k "${PYK:-sweep or c2 or golden}" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for lib in $LIBS; do RRG_LIB=$PWD/paper_2410_18926_b200/$lib python bench.py --workload ${WL:-c2} --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['stage_ms'])"; done
