# phase times of library variants (_ab/lib_<name>.so): config 3 frames 7..16 mean, config 2 frame 8, config 3 frame 1
for v in "$@"; do
  RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/frame_phases.py 16 > gpurun_out/ab_${v}.jsonl 2>/dev/null
  python - $v gpurun_out/ab_${v}.jsonl <<'PY'
import json,sys
rows=[json.loads(l) for l in open(sys.argv[2]) if l.startswith('{')]
f1=rows[0]['total'] if rows else None
rows=[r for r in rows if 7<=r['t']<=16]
keys=['total','group','filter','final']
print(sys.argv[1], {k: round(sum(r.get(k,0) for r in rows)/max(len(rows),1),2) for k in keys}, 'frame1', f1)
PY
  CFG=2 RIANN_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/frame_phases.py 8 2>/dev/null | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('   cfg2', r['total'], 'group', r['group'])"
done
