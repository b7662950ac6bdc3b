# PCIe copy rate of the e2e block: 1 / 2 / 4 streams; full GPU suite with the new tests
timeout 300 python tools/probe_pcie.py > gpurun_out/r2zr_pcie.log 2>&1
timeout 1800 python -m pytest -q tests -m gpu -x -p no:cacheprovider > gpurun_out/r2zr_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2zr_gpu_tests.log
