# experiment: larger segments per CTA (S = 2^19) and 1024-thread CTAs, c3s count
for i in 1 2; do
echo "== base 512thr S=2^18"; python tools/prof_run.py c3s 3 2>&1 | tail -1
echo "== exp 1024thr S=2^18"; (cd scratch/exp && python tools/prof_run.py c3s 3 2>&1 | tail -1)
echo "== exp 1024thr S=2^19"; (cd scratch/exp && SEG=524288 python tools/prof_run.py c3s 3 2>&1 | tail -1)
echo "== exp512 512thr S=2^19"; (cd scratch/exp512 && SEG=524288 python tools/prof_run.py c3s 3 2>&1 | tail -1)
done
(cd scratch/exp && SEG=524288 python -c "
import sys; sys.path.insert(0,'.')
import paper_2310_17746_b200 as ws
sv=ws.Sieve(device=0, segment_slots=524288)
c=sv.count_range(0,10**12+1); print('pi(1e12) S=2^19 1024thr', c.count, c.count==37607912018)
c=sv.count_range(10**12, 10**12+10**9, checks=True); print(c)
")
