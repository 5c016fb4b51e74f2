import json,os,sys,subprocess,statistics
libs=sys.argv[1:]
res={l:[] for l in libs}
for rep in range(4):
    for l in libs:
        env=dict(os.environ,SPARROW_LIB_PATH=os.path.abspath(l))
        out=subprocess.run([sys.executable,'bench.py','--envs','4096','--steps','30','--warmup','5','--no-cpu-baseline','--no-lidar','--no-replay','--e2e-steps','3'],env=env,capture_output=True,text=True).stdout
        j=json.loads(out.strip().splitlines()[-1]); res[l].append(j['ms_per_step'])
for l,v in res.items(): print('cfg2',l,round(statistics.median(v),5),[round(x,5) for x in v])
