# New line-per-thread k_cg3: operator parity tests, then C5 operator timing via the bench line.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coeff.py tests/test_gpu_dist.py -x -q -m gpu > gpurun_out/r02c_op_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02c_op_tests.log
timeout 600 python bench.py --ordering rcm --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_op_bench_C5.json 2> gpurun_out/r02c_op_bench_C5.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02c_op_bench_C5.json')); print(d['value'], d['roofline_operator'])"
timeout 300 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_op_bench_C3.json 2> gpurun_out/r02c_op_bench_C3.err; echo "bench C3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02c_op_bench_C3.json')); print(d['value'], d['roofline_operator'])"
