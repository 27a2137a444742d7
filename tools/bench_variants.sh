for cfg in "FMMBEM_P2P_NCT=384" "FMMBEM_P2P_NCT=256" "FMMBEM_P2P_NCT=512" "FMMBEM_P2P_NCT=384 FMMBEM_NEAR_PRIO_HIGH=1" "FMMBEM_P2P_NCT=256 FMMBEM_NEAR_PRIO_HIGH=1"; do
  echo "$cfg: $(env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["roofline"]["stage_ms_per_apply"])')"
done
