(cd scratch/ft512 && timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import paper_2310_17746_b200 as ws
sv=ws.Sieve(device=0)
c=sv.count_range(10**15,10**15+10**11,checks=True); print('c4 ok', c.count==2895317534 and c.sum==6009025740971448886 and c.xor==996783733192)
")
for i in 1 2; do
for c in c4 c5; do
echo "== $c 256"; python tools/prof_run.py $c 3 | tail -1
echo "== $c 512"; (cd scratch/ft512 && python tools/prof_run.py $c 3 | tail -1)
echo "== $c 128"; (cd scratch/ft128 && python tools/prof_run.py $c 3 | tail -1)
done; done
