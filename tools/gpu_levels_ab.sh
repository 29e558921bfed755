cd "${GRAFT_REPO_ROOT:-.}"; O=gpurun_out/lv; mkdir -p $O
for m in 0 1 2; do
  echo "== QTNG_LEVELS=$m" >> $O/out.txt
  QTNG_LEVELS=$m timeout 200 python -c "
import json, numpy as np, paper_2204_06045_b200 as q
gold=json.load(open('tests/golden/energies.json'))['configs']
for name in ('C2','C4'):
    c=gold[name]; g=q.random_regular(c['n'],3,c['seed']); pl=q.Plan(g,len(c['gammas']))
    t=pl.execute(q.Angles(c['gammas'],c['betas'])); ref=np.array([complex(x,y) for x,y in c['terms_naive']])
    print(name,'parity', np.array_equal(t,ref))
" >> $O/out.txt 2>&1
  QTNG_LEVELS=$m timeout 300 python tools/shard_sim.py C2 C4:9 >> $O/out.txt 2>&1
  QTNG_LEVELS=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c3 --no-sub > $O/bench_$m.json 2>> $O/out.txt
  python -c "import json; d=json.loads(open('$O/bench_$m.json').read().strip().splitlines()[-1]); print('BENCH', $m, d['ms_per_step'], d['e2e']['ms_per_step'])" >> $O/out.txt
done
