"""Print the ncu 'details' page (section / metric / value) of the first N kernels."""
import csv
import io
import subprocess
import sys


def main(path, n=1, grep=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    iid, isec, iname, iunit, ival = (hdr.index(k) for k in
                                     ("ID", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for r in rows[1:]:
        if int(r[iid]) >= n:
            break
        line = f"{r[isec][:28]:28s} {r[iname][:48]:48s} {r[ival]:>16s} {r[iunit]}"
        if grep is None or grep.lower() in line.lower():
            print(line)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1,
         sys.argv[3] if len(sys.argv) > 3 else None)
