# tcgen05 GEMM bottleneck probes on the standalone micro-benchmark (probes give wrong results).
# Needs a probe build: (cd paper_2603_20622_b200/csrc && make clean && make EXTRA=-DRTEC_GEMM_PROBES)
mkdir -p gpurun_out; out=gpurun_out/gemm_probe.txt; rm -f $out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> $out
for shape in "2000000 256 256 0" "1200000 100 256 1" "2000000 128 128 0"; do
for p in 0 1 2 4 7 8 16 15 23; do
  echo -n "probe=$p " >> $out
  RTEC_GEMM_PROBE=$p timeout 60 ./tools/gemm_micro $shape 20 >> $out 2>&1
done
for v in "RTEC_GEMM_NWIDE=1" "RTEC_GEMM_SA=2" "RTEC_GEMM_SA=4"; do
  echo -n "$v " >> $out; env $v timeout 60 ./tools/gemm_micro $shape 20 >> $out 2>&1
  echo -n "$v probe=7 " >> $out; env $v RTEC_GEMM_PROBE=7 timeout 60 ./tools/gemm_micro $shape 20 >> $out 2>&1
done
done
cat $out
