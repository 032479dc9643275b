for pp in 0 1 2 3 13; do AMUN_PREPASS=$pp VT_VARIANTS=full timeout 300 python tools/variant_times.py beam 2>&1 | sed "s/^{/{\"pp\": $pp, /" >> gpurun_out/r02pp.jsonl; done
AMUN_PREPASS=3 timeout 600 python -m pytest tests/test_gpu_output_layer.py -x -q -k "not slow" 2>&1 | tail -2 > gpurun_out/r02pp_pytest.log
