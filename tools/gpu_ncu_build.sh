cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:symcheck_kernelIhLi8E -s 40 -c 1 -f -o gpurun_out/sym_full python tools/build_identity.py 300000 > gpurun_out/ncu_sym.log 2>&1; echo "ncu sym rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:descent_kernelIhhLi8E -s 40 -c 1 -f -o gpurun_out/desc_full python tools/build_identity.py 300000 > gpurun_out/ncu_desc.log 2>&1; echo "ncu desc rc=$?"
