import json,glob,sys
for f in sorted(glob.glob(sys.argv[1])):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, "ERR", e); continue
    if 'value' not in d: print(f, d); continue
    ks={f"{k['kernel']}{k['layer']}":k['total_ms']/d['profiled_steps'] for k in d['kernels']}
    top=sorted(ks.items(), key=lambda kv:-kv[1])[:5]
    print(f"{f.split('/')[-1]:24s} {d['value']:9.1f} sps {d['ms_per_step']:8.3f} ms  CB={d['config']['chunk_batch']}/{d['config']['fwd_chunk_batch']}  frac={d['step_roofline']['frac']:.3f} | "+" ".join(f"{k}={v:.2f}" for k,v in top))
