import csv, sys, subprocess, collections
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","details","--csv"],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
hdr=r[0]
want = ["Duration","Executed Ipc Active","Issue Slots Busy","Registers Per Thread","Achieved Active Warps Per SM","Theoretical Active Warps per SM","Dynamic Shared Memory Per Block","Warp Cycles Per Issued Instruction","Executed Instructions","Avg. Active Threads Per Warp","Branch Efficiency","Block Limit Registers","Block Limit Shared Mem","No Eligible","DRAM Throughput","Compute (SM) Throughput","L1/TEX Hit Rate"]
for row in r[1:]:
    d=dict(zip(hdr,row))
    if d.get('Metric Name') in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
