import json,sys
for f in sys.argv[1:]:
    d=json.load(open(f))
    L=d['log']
    prev=0; out=[]
    for e in L[1:]:
        out.append(round(e['train_s']-prev,3)); prev=e['train_s']
    print(f, d['reached_s'], out)
