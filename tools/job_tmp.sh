AB_SLEEP=1 AB_K=30 AB_VARIANTS=tail_pdl0,tail_pdl1,scores_pdl0,scores_pdl1 timeout 900 python tools/ab_path.py beam greedy > gpurun_out/r02pdl2_ab.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02pdl2_pytest.log
