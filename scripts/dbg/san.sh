cd $GRAFT_REPO_ROOT
ISDC_FAST3D_MASK=1 ISDC_NO_GRAPHS=1 timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --show-backtrace device python scripts/dbg3d.py child 31 > gpurun_out/san.log 2>&1
echo "rc=$?" >> gpurun_out/san.log
