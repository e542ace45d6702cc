# A/B of M-step graph knobs on the cfg2 bench (10 timed runs each): ms per run, log ML, M steps
for V in "SPS_LOOP_BODY=4" "SPS_LOOP_BODY=4 SPS_K1_LATE_TRIGGER=1" "SPS_LOOP_BODY=2 SPS_K1_LATE_TRIGGER=1" "SPS_LOOP_BODY=4" "SPS_LOOP_BODY=4 SPS_K1_LATE_TRIGGER=1"; do
  echo "$V $(env $V python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["run"]["logml"], d["run"]["m_steps"])')"
done
