python tools/pcie_probe.py
nvidia-smi -q | grep -i -A3 "Link Width\|PCIe Generation" | head -20
