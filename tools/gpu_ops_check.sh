mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q > gpurun_out/pytest_ops.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.txt
timeout 900 tests/refsuite/_bin/refsuite > gpurun_out/refsuite.txt 2> gpurun_out/refsuite_err.txt; echo "rc=$?" >> gpurun_out/refsuite.txt
