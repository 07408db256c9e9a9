# ncu --set full of the forward / back transform kernels on a 4096-cell c3 step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kf1|kf2|kb1|kb2|kb3" -s 5 -c 5 -o gpurun_out/r2x_xf python tools/profile_hot.py c3 4096 > gpurun_out/r2x_ncu.log 2>&1
tail -2 gpurun_out/r2x_ncu.log
