# run a pytest selection on the GPU box (arg: -k expression), full output tail to gpurun_out/pytest_sel.log
timeout 2400 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -40 > gpurun_out/pytest_sel.log; cat gpurun_out/pytest_sel.log
