# GAT recompute windows: four Z rows in the two-pair registers (new) vs two rows (old build)
mkdir -p gpurun_out; out=gpurun_out/ab_g4.txt; rm -f $out
L=paper_2603_20622_b200/librtec.so
cp $L /tmp/librtec_new.so
timeout 900 python -m pytest tests -m gpu -x -q -k "gat or golden or parity" > gpurun_out/ab_g4_pytest.txt 2>&1; tail -1 gpurun_out/ab_g4_pytest.txt >> $out
for w in c3-gat c3-gat c3-gat; do
for v in new old; do
  if [ $v = old ]; then cp paper_2603_20622_b200/librtec_old.so.ab $L; else cp /tmp/librtec_new.so $L; fi
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/ab_g4_${w}_$v.json 2>gpurun_out/ab_g4_${w}_$v.err
  python -c "import json;r=json.load(open('gpurun_out/ab_g4_${w}_$v.json'));k=r['kernels'];print('$w $v', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'], 'gat', k['k_gat_layer']['ms_per_launch'])" >> $out 2>&1
done; done
cp /tmp/librtec_new.so $L
cat $out
