cd $GRAFT_REPO_ROOT
for t in ${TUNES:-"" host_chunks=8 host_chunks=12 host_chunks=16}; do
  timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-solve ${t:+--tune $t} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tune=$t', round(d['ms_per_step'],1), round(d['value']), round(d['e2e']['value']), d['e2e']['check_vs_device_entry_max_rel_diff'])"
done
