# ncu --set full of the term-loop kernel from the final build (one c3 launch of 10923 cells)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hot_kernel_v4 -s 1 -c 1 -o gpurun_out/r2nc_hot python tools/profile_hot.py c3 10923 > gpurun_out/r2nc_ncu_hot.log 2>&1
tail -2 gpurun_out/r2nc_ncu_hot.log
ls -la gpurun_out/r2nc_hot.ncu-rep
