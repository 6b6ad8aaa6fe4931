import json, sys
rows=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
tot={}
for r in rows:
    if 'scale' not in r: print(r); continue
    for k in ('total_ms','traverse_ms','moments_ms','local_ms','base_ms','farfield_ms','final_ms'): tot[k]=tot.get(k,0)+r[k]
    print(f"{r['scale']:8.3g} h={r['h']:.3g} tot={r['total_ms']:.3f} trav={r['traverse_ms']:.3f} mom={r['moments_ms']:.3f} loc={r['local_ms']:.3f} base={r['base_ms']:.3f} ff={r['farfield_ms']:.3f} fin={r['final_ms']:.3f} lv={r['levels']} pairs={r['pairs_visited']} bc={r['base_cases']} kev={r['kernel_evaluations']:.3g} fd={r['prunes_finite_diff']} F={r['prunes_farfield']} D={r['prunes_direct_local']} T={r['prunes_far_to_local']} err={r.get('max_rel_err',0):.2e}")
print({k:round(v,3) for k,v in tot.items()})
