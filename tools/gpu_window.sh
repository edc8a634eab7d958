# (1) face-window tuning experiment (experimental build), (2) p-MG parameter sweep
set -x
timeout 1200 python tools/mg_sweep.py 128 321:3:30 321:3:15 321:3:60 321:2:30 321:4:30 31:3:30 321:3:8 > gpurun_out/mg_sweep.jsonl 2> gpurun_out/mg_sweep.err; echo "sweep rc=$?"
rm -rf /tmp/exp && mkdir /tmp/exp && cp -r paper_2509_10226_b200 include tools oracle /tmp/exp/
cd /tmp/exp && rm -rf paper_2509_10226_b200/csrc/_obj paper_2509_10226_b200/libtetmf_b200.so
timeout 600 python -c "import paper_2509_10226_b200._build as b; b.FLAGS.append('-DTMF_EXP_FACE_WINDOW_ENV'); b.build()" > $GRAFT_REPO_ROOT/gpurun_out/win_build.log 2>&1
for w in 8192 2048 512 32768 131072; do
  TMF_FACE_WINDOW=$w timeout 600 python tools/quick_bench.py dgv:3:64 hhv:2:96 > $GRAFT_REPO_ROOT/gpurun_out/win_$w.jsonl 2>> $GRAFT_REPO_ROOT/gpurun_out/win.err
done
echo done
