# A/B: PDL with early trigger (default build) vs PDL triggered at CTA exit vs no PDL
mkdir -p gpurun_out; out=gpurun_out/ab_pdl2.txt; rm -f $out
L=paper_2603_20622_b200/librtec.so
cp $L /tmp/librtec_trig.so
for w in c1-gcn c2-sage c3-gat c2-gcn c1-gcn c2-sage c3-gat; do
for v in trig exit off; do
  if [ $v = exit ]; then cp paper_2603_20622_b200/librtec_notrig.so.ab $L; else cp /tmp/librtec_trig.so $L; fi
  P=1; [ $v = off ] && P=0
  RTEC_PDL=$P timeout 400 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --no-baselines --no-parity --e2e-steps 5 > gpurun_out/ab_pdl2_${w}_$v.json 2>gpurun_out/ab_pdl2_${w}_$v.err
  python -c "import json;r=json.load(open('gpurun_out/ab_pdl2_${w}_$v.json'));print('$w $v', r['p50_batch_ms'], 'e2e', r['e2e']['p50_batch_ms'])" >> $out 2>&1
done; done
cp /tmp/librtec_trig.so $L
cat $out
