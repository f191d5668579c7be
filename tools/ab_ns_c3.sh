# c3-gat baselines (UER / Full / NS) with the four-row GAT recompute (new) vs two rows (old build)
mkdir -p gpurun_out; out=gpurun_out/ab_ns.txt; rm -f $out
L=paper_2603_20622_b200/librtec.so
cp $L /tmp/librtec_new.so
for v in new old new old; do
  if [ $v = old ]; then cp paper_2603_20622_b200/librtec_old.so.ab $L; else cp /tmp/librtec_new.so $L; fi
  timeout 900 python bench.py --workload c3-gat --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 3 > gpurun_out/ab_ns_$v.json 2>gpurun_out/ab_ns_$v.err
  python -c "import json;r=json.load(open('gpurun_out/ab_ns_$v.json'));b=r['gpu_baselines'];print('$v', r['p50_batch_ms'], {k:b[k]['p50_batch_ms'] for k in b})" >> $out 2>&1
done
cp /tmp/librtec_new.so $L
cat $out
