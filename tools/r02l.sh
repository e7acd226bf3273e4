# r02l: host-link ceiling (pcie_probe) and the config-5 portability sweep with the round-2 wisdom as anchors
timeout 600 python tools/pcie_probe.py > gpurun_out/r02l_pcie.json 2>&1
echo pcie rc $?
timeout 3300 python -m paper_2303_12374_b200.portability --anchor-wisdom wisdom --out gpurun_out/r02l_portability.json > gpurun_out/r02l_portability.log 2>&1
echo portability rc $?
