#!/bin/bash
# Box facts the engine tier choice depends on.
mkdir -p gpurun_out
{
echo "== cpu/mem"; nproc; free -g | head -2
echo "== disks"; lsblk -d -o NAME,SIZE,MODEL,ROTA 2>/dev/null | head -20; df -hT /tmp /root 2>/dev/null
echo "== nvidia-fs"; lsmod 2>/dev/null | grep -i nvidia; ls /proc/driver/nvidia-fs 2>/dev/null && cat /proc/driver/nvidia-fs/stats 2>/dev/null | head
echo "== cufile"; ls /usr/local/cuda/gds/tools 2>/dev/null; ls /usr/local/cuda/lib64/libcufile* 2>/dev/null; cat /etc/cufile.json 2>/dev/null | head -5
/usr/local/cuda/gds/tools/gdscheck -p 2>&1 | head -40
echo "== topo"; nvidia-smi topo -m 2>/dev/null | head -12
echo "== pcie"; nvidia-smi -q 2>/dev/null | grep -iA6 "PCI$\|GPU Link Info" | head -30
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt
