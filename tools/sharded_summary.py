import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line)
        for l in d['sharded']['rows']:
            if l['batch']==1: print(sys.argv[1], l['layer'], {k:round(v,1) for k,v in l.items() if k in ('us_partial_engine','us_nccl_path_engine','us_fused_engine','us_fused')})
