cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
for s in 1 0; do QG_PSD_SPLIT=$s QG_PSD_PROF=1 timeout 300 python tools/psd_probe.py 50 2>&1 | grep -v Warn | tail -4; done
timeout 600 ncu --set full --import-source on -k regex:k_step_psd -c 1 -o gpurun_out/prof/r02_c4_psd python tools/traffic_probe.py --config c4 --which ft > gpurun_out/prof/r02_c4_psd.log 2>&1; echo "ncu psd $?"
timeout 600 ncu --set full --import-source on --kernel-name-base mangled -k regex:k_stepILi1 -c 1 -o gpurun_out/prof/r02_c4_FT_main python tools/traffic_probe.py --config c4 --which ft > gpurun_out/prof/r02_c4_FT_main.log 2>&1; echo "ncu main $?"
