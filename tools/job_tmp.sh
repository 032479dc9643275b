AMUN_MTFAST=1 timeout 600 python -m pytest tests/test_gpu_output_layer.py -x -q -k "not slow" 2>&1 | tail -2 > gpurun_out/r02mf_pytest.log
for m in 0 1; do AMUN_MTFAST=$m VT_VARIANTS=full,2,5 timeout 300 python tools/variant_times.py beam 2>&1 | grep '"round": 1' | sed "s/^{/{\"mf\": $m, /" >> gpurun_out/r02mf.jsonl; done
for m in 0 1; do AMUN_MTFAST=$m VT_S=96 VT_B=4 VT_VARIANTS=2,5 timeout 300 python tools/variant_times.py beam 2>&1 | grep '"round": 1' | sed "s/^{/{\"mf\": $m, /" >> gpurun_out/r02mf.jsonl; done
