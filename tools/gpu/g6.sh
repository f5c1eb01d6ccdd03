python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k window_goldens_per_segment 2>&1 | grep -E "^E " | head -8
WHEELSIEVE_HUGE_LOOP=1 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k window_goldens_per_segment 2>&1 | tail -2
python - <<'PY'
import json, paper_2310_17746_b200 as ws
g=json.load(open("tests/golden/reference_goldens.json"))
for S in (1<<18, 1<<12):
    sv=ws.Sieve(segment_slots=S)
    for rec in g["windows"]:
        c=sv.count_range(rec["L"],rec["R"],checks=True)
        if (c.count,c.sum,c.xor,c.largest)!=(rec["count"],rec["sum"],rec["xor"],rec["largest"]):
            print("MISMATCH S=",S, rec["L"], rec["R"], c.count, rec["count"])
    sv.close()
print("done")
PY
