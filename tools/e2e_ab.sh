for t in off on off2 on2; do
  case $t in off*) E="HALO_K1_SM_FRAC=0";; *) E="X=0";; esac
  env $E python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-migration --other-configs "" > gpurun_out/e2e_$t.json 2> gpurun_out/e2e_$t.err
  python -c "import json; d=json.load(open('gpurun_out/e2e_$t.json')); print('$t', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'cont', json.dumps(d.get('continuous_batching', d.get('continuous')))[:200])"
done
