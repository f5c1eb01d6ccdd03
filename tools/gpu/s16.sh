for c in c2 c4 c5 c3s; do
echo "== $c base"; python tools/prof_run.py $c 3 2>&1 | tail -1
echo "== $c exp 1024thr S=2^19"; (cd scratch/exp && SEG=524288 python tools/prof_run.py $c 3 2>&1 | tail -1)
done
(cd scratch/exp && python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17746_b200 as ws
sv=ws.Sieve(device=0, segment_slots=524288)
out=torch.empty(455052511+1024, dtype=torch.int64, device='cuda')
_,n,c=sv.enumerate_range(0,10**10,out=out); print('c2', n, c.sum, c.xor, c.largest, n==455052511 and c.sum==2220822432581729238 and c.xor==16212951392)
c=sv.count_range(10**15,10**15+10**11,checks=True); print('c4', c.count==2895317534 and c.sum==6009025740971448886 and c.xor==996783733192)
")
