mkdir -p gpurun_out
(time timeout 1500 ./tests/refsuite/_bin/refsuite) > gpurun_out/refsuite.txt 2>&1; echo "rc=$?" >> gpurun_out/refsuite.txt
