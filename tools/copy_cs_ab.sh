# A/B: copy kernels (K4 pack/unpack, K5, relocation) with st.global.cs stores (default) vs plain (libhalo_attn_nocs.so)
for rep in 1 2; do
for v in cs nocs; do
  if [ $v = nocs ]; then export HALO_LIB=$PWD/paper_2509_02121_b200/libhalo_attn_nocs.so; else unset HALO_LIB; fi
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --other-configs "" > gpurun_out/cs_${v}_$rep.json 2> gpurun_out/cs_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/cs_${v}_$rep.json')); m=d['migration']
sw=[round(x.get('relocate_hbm_frac', x.get('relocate_frac', 0)) or 0,3) for x in m.get('relocation',{}).get('sweep', m.get('sweep',[]))]
print('$v$rep', round(d['value']/1e6,3), 'pack', round(m['pack']['hbm_roofline']['frac'],3), 'unpack', round(m['unpack']['hbm_roofline']['frac'],3), json.dumps({k: (v.get('hbm_roofline',{}).get('frac') if isinstance(v, dict) else None) for k,v in m.items()})[:300], json.dumps(m.get('sweep', m.get('relocation',{}).get('sweep')))[:900])" || tail -3 gpurun_out/cs_${v}_$rep.err
done
done
