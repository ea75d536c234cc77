"""Print kernel name + duration (us) from an ncu --csv launch list:
    python tools/launch_times.py launches.csv"""
import csv
import sys

for r in csv.reader(open(sys.argv[1])):
    if len(r) > 10 and r[0].isdigit() and r[-3] == "gpu__time_duration.sum":
        print(f"{r[4].split('(')[0][:48]:48s} {float(r[-1]) / 1e3:10.1f}")
