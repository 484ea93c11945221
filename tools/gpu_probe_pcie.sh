timeout 600 python tools/pcie_probe.py > gpurun_out/pcie_probe.json 2>&1; cat gpurun_out/pcie_probe.json
timeout 600 python -m pytest tests/test_gpu_edge.py -q -p no:cacheprovider 2>&1 | tail -3
