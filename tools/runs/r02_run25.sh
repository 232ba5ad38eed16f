LSQ_PARITY_OUT=gpurun_out/parity_final.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
{ echo "== lazy init"; oracle/_ref/acceptance_on_b200; echo "rc=$?"; ./tools/cudart_init_probe; echo "== LSQFIT_CUDA_EAGER_INIT=1"; LSQFIT_CUDA_EAGER_INIT=1 oracle/_ref/acceptance_on_b200; echo "rc=$?"; echo "== reference order"; LSQFIT_CUDA_REFERENCE_ORDER=1 oracle/_ref/acceptance_on_b200; echo "rc=$?"; } > gpurun_out/acceptance_final.log 2>&1
python tools/sweep.py > gpurun_out/sweep_final.json 2> gpurun_out/sweep_final.err
