mkdir -p gpurun_out/probe2; cd tools/probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -DPLOG2N=12 -DPIPE phase_probe.cu -o probe_a > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -DPLOG2N=12 -DPIPE -DQFT_PIPE_TMA_WARP=7 phase_probe.cu -o probe_b > /dev/null 2>&1
./probe_a > ../../gpurun_out/probe2/a.log 2>&1; ./probe_b > ../../gpurun_out/probe2/b.log 2>&1
cd ../..
bash tools/ab.sh -c 2 -r 2 paper_1301_0763_b200/libqftb200.so variants/tma7.so variants/tmaearly.so > gpurun_out/probe2/ab.log 2>&1
