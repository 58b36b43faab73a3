cd /root/repo
for S in 1 2 4; do
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --interp-images 0 --pretrain-batch 0 --tiny-batch 0 --e2e-steps 0 --no-parity --streams $S 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read()); print($S, d['value'], d['ms_per_step'], d['phase_ms'])"
done
