python tools/loop_bench.py cgr:1:48:0:dmma:off cgr:1:48:0:dmma:on cg:1:48:0:dmma:off cgr:2:48:0:dmma:off cgr:2:48:0:dmma:on cgr:2:48:0:dfma:off cgr:3:48:0:dmma:off cgr:4:48:0:dmma:off > gpurun_out/loop1.jsonl 2> gpurun_out/loop1.err
echo rc=$?
