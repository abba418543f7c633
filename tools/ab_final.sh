# A/B of library variants (_ab/lib_<name>.so): parity of the config-3 tests, then phase times (frames 7..16 mean)
for v in "$@"; do
  RIANN_LIB=$PWD/_ab/lib_$v.so timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -q -p no:cacheprovider -k "cfg3_d192_golden or cfg3_full_scale" > gpurun_out/ab_${v}_pytest.log 2>&1; echo "$v pytest rc=$?"; tail -1 gpurun_out/ab_${v}_pytest.log
done
for rep in 1 2; do for v in "$@"; do
  RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/frame_phases.py 16 > gpurun_out/ab_${v}_ph$rep.jsonl 2>gpurun_out/ab_${v}_ph$rep.err
  python - $v gpurun_out/ab_${v}_ph$rep.jsonl <<'PY'
import json,sys
rows=[json.loads(l) for l in open(sys.argv[2]) if l.startswith('{')]
rows=[r for r in rows if 7<=r['t']<=16]
keys=['total','p0a','p0b','draw','group','window','filter','final','units']
print(sys.argv[1], {k: round(sum(r.get(k,0) for r in rows)/max(len(rows),1),2) for k in keys}, 'frame1', None)
PY
done; done
