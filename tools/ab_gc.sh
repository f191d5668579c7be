mkdir -p gpurun_out
for w in c3-gat c1-gcn; do for f in 0 1; do
RTEC_BENCH_GC_FREEZE=$f timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline --no-parity --no-baselines > gpurun_out/gc_${w}_$f.json 2>/dev/null
python -c "import json;r=json.load(open('gpurun_out/gc_${w}_$f.json'));print('$w freeze=$f', r['e2e']['value'], r['e2e']['batch_ms'])"
done; done
