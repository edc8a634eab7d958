# timing experiment: CG cell kernels with the fp64 RED scatter replaced by plain stores
# NOTE: needs the TMF_EXP_SCATTER switch that was removed from the kernels after this experiment (see profiles/r01/red_scatter_experiments.json "how")
set -x
Q="cg:1:48 cgv:1:48 cg:2:48 cgv:2:48 cg:3:48 cgv:3:48 cg:4:48 cgv:4:48"
timeout 600 python tools/quick_bench.py $Q > gpurun_out/redexp_base.jsonl 2> gpurun_out/redexp_base.err
rm -rf /tmp/exp && mkdir /tmp/exp && cp -r paper_2509_10226_b200 include tools oracle /tmp/exp/
cd /tmp/exp && rm -rf paper_2509_10226_b200/csrc/_obj paper_2509_10226_b200/libtetmf_b200.so
timeout 600 python -c "import paper_2509_10226_b200._build as b; b.FLAGS.append('-DTMF_EXP_SCATTER=1'); b.build()" > $GRAFT_REPO_ROOT/gpurun_out/redexp_build.log 2>&1
timeout 600 python tools/quick_bench.py $Q > $GRAFT_REPO_ROOT/gpurun_out/redexp_store.jsonl 2> $GRAFT_REPO_ROOT/gpurun_out/redexp_store.err
echo done
