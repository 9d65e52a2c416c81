mkdir -p gpurun_out/g5
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g5/tests.log 2>&1; echo rc=$? >> gpurun_out/g5/tests.log
timeout 300 python profiles/probe.py bfs24 > gpurun_out/g5/probe_bfs.txt 2>&1
timeout 600 python profiles/probe.py c4 > gpurun_out/g5/probe_c4.txt 2>&1
timeout 600 python profiles/probe.py c2 > gpurun_out/g5/probe_c2.txt 2>&1
tail -3 gpurun_out/g5/tests.log; grep -E "^==|it +[1-6] " gpurun_out/g5/probe_bfs.txt; grep "^==" gpurun_out/g5/probe_c4.txt gpurun_out/g5/probe_c2.txt
