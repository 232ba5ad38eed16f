L=paper_1512_08017_b200/lib/liblsqfit_cuda.so
python tools/ab.py build/lib_prev3.so $L 1e9 5,6,7,8,9,10,11,12 12 > gpurun_out/ab_final_split.log 2>&1
python tools/ab.py build/lib_prev3.so $L 1e6 6,8,12 40 >> gpurun_out/ab_final_split.log 2>&1
LSQ_PARITY_OUT=gpurun_out/parity_final2.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_final2.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final2.json 2> gpurun_out/sweep_final2.err
