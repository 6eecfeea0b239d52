export PYTHONUNBUFFERED=1
out=gpurun_out/ab8; mkdir -p $out
QFT_LIB=$(realpath variants/l2pf.so) timeout 300 python tools/vcheck.py 4096 3 > $out/vcheck.log 2>&1
bash tools/ab.sh -c 2 -r 2 paper_1301_0763_b200/libqftb200.so variants/l2pf.so variants/l2pf7.so variants/tw7.so > $out/ab.log 2>&1
cd tools/probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -DPLOG2N=12 -DPIPE phase_probe.cu -o probe_a > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -DPLOG2N=12 -DPIPE -DQFT_PIPE_L2PF=1 phase_probe.cu -o probe_b > /dev/null 2>&1
./probe_a > ../../$out/pa.log 2>&1; ./probe_b > ../../$out/pb.log 2>&1
