import json,sys
for f in sys.argv[1:]:
    try:
        l=[x for x in open(f) if x.startswith('{')][-1]; d=json.loads(l); e=d.get("e2e",{})
        print(f, round(d["value"]), round(d["ms_per_step"]*1e3,1), round(d["ms_per_step_p50"]*1e3,1), round(e.get("value",0)), round(e.get("sync_value",0)), [round(x) for x in e.get("pipelined_passes",[])], e.get("pipelined_recaptures"), d["loss_first_last"])
    except Exception as ex: print(f, "ERR", ex, open(f).read()[-1500:])
