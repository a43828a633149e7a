cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --screen-ligands 10000 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['screening']['value'])"
