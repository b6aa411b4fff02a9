nvidia-smi > gpurun_out/probe_smi.txt 2>&1
lscpu > gpurun_out/probe_lscpu.txt 2>&1
nproc >> gpurun_out/probe_lscpu.txt
grep -o 'avx512[a-z_]*' /proc/cpuinfo | sort -u >> gpurun_out/probe_lscpu.txt
free -g >> gpurun_out/probe_lscpu.txt
echo done
