cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_VISIBLE_DEVICES=0
NOFLUSH=1 timeout 300 scripts/_bin/read_probe 536.9 1073.7 4295.0 > gpurun_out/read_probe_noflush.log 2>&1
