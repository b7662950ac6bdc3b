# L2 vector-reduction probe (push instead of pull for hub rows' cold columns)
timeout 600 ./tools/probe/l2_red > gpurun_out/r2zc_l2_red.log 2>&1; echo "rc=$?" >> gpurun_out/r2zc_l2_red.log
