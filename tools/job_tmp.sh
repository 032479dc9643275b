bash tools/run_checked.sh gpurun_out/r02_checked
timeout 900 python -m pytest tests/test_gpu_output_layer.py tests/test_gpu_trace.py -x -q 2>&1 | tail -5 > gpurun_out/r02_pytest_new.log
timeout 600 python tools/trace_bench.py --out gpurun_out/r02_trace_cfg4_full.jsonl > gpurun_out/r02_trace_cfg4.jsonl 2>&1
