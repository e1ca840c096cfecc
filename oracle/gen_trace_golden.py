"""Golden vectors for trace ingestion from the UNMODIFIED reference.

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference):
    python -m oracle.gen_trace_golden
Every case is a CSV or JSON-lines text fed to the reference's load_trace
(workload.py:422-431); the fixture stores the text and either the parsed records
(id, arrival, input, output (-1 = None), class) or the TraceFormatError line and
message.  Cases: the reference's own test inputs (test_workload.py:118-191),
gen_synthetic traces written by its save_trace, and the parser edge cases
(quotes, whitespace, underscores, inf / nan, headers, CRLF, field counts, types,
JSON syntax errors, unknown / missing keys, duplicate keys)."""

from __future__ import annotations

import gzip
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden", "traces.json.gz")
REF_SRC = os.environ.get("BUCKETSIM_REF_SRC", "/root/reference/pkg/src")


def cases(wl):
    out = []

    def add(name, fmt, text):
        out.append((name, fmt, text))

    # reference test inputs
    add("ref_single_line", "csv", "0.5,128,32,online\n")
    add("ref_sorts_by_arrival", "csv", "2.0,10,5,online\n1.0,20,5,offline\n")
    add("ref_parse_error_line1", "csv", "x,128,32,online\n")
    add("ref_error_past_header", "csv",
        "arrival_s,input_tokens,output_tokens,class\n1.0,10,5,online\n2.0,bad,5,online\n")
    add("ref_empty", "csv", "")
    add("ref_missing_output", "csv", "0.0,128,,offline\n")
    add("ref_bad_class", "csv", "0.0,128,32,urgent\n")
    add("ref_jsonl_fields", "jsonl",
        '{"arrival_s": 1.25, "input_tokens": 64, "output_tokens": 8, "class": "offline"}\n')
    add("ref_jsonl_unknown", "jsonl",
        '{"arrival_s": 1.0, "input_tokens": 64, "class": "online", "oops": 1}\n')
    add("ref_jsonl_invalid_line2", "jsonl",
        '{"arrival_s": 1.0, "input_tokens": 2, "class": "online"}\n{oops\n')
    # synthetic traces through the reference's own writer
    specs = [
        wl.WorkloadSpec(arrival=wl.PoissonArrivals(50.0),
                        length_dist=wl.LongTailLogNormal(5.5, 1.1, 4095),
                        output_dist=wl.ShortNormal(128, 40, 512),
                        horizon=wl.Horizon(requests=3000), online_fraction=0.4, seed=11),
        wl.WorkloadSpec(arrival=wl.FixedIntervalArrivals(0.01),
                        length_dist=wl.Mixture((wl.ShortNormal(83, 40), wl.LongTailLogNormal(10.6, 1.0, 131071)),
                                               (0.7, 0.3)),
                        output_dist=wl.ShortNormal(64, 0), horizon=wl.Horizon(requests=1500),
                        online_fraction=0.5, seed=12),
    ]
    for k, spec in enumerate(specs):
        tr = wl.gen_synthetic(spec)
        for fmt, tf in (("csv", wl.TraceFormat.CSV), ("jsonl", wl.TraceFormat.JSONL)):
            buf = io.StringIO()
            wl.save_trace(tr, buf, tf)
            add(f"synthetic{k}_{fmt}", fmt, buf.getvalue())
    # shuffled arrivals with ties (stable sort, ids in file order)
    add("ties_unsorted", "csv", "3,5,1,online\n1,6,,offline\n3,7,2,offline\n1,8,3,online\n0.5,9,4,ONLINE\n")
    # CSV edge cases
    add("csv_crlf_blank_lines", "csv", "1.0,10,5,online\r\n\r\n\n2.0,11,,offline\r\n   ,  ,\n")
    add("csv_whitespace_fields", "csv", " 1.5 , 12 , 3 , Offline \n")
    add("csv_underscores_sign", "csv", "1_0.5,+1_024,0_7,online\n")
    add("csv_inf_nan_exp", "csv", "1e3,5,5,online\ninf,6,6,offline\n-1.5E-2,7,7,online\n")
    add("csv_header_midfile", "csv", "1,2,3,online\narrival_s,x,y,z\n0,4,5,offline\n")
    add("csv_quoted", "csv", '"1.0","12","3","online"\n"2.0",13,"",offline\n')
    add("csv_quoted_comma", "csv", '"1,0",12,3,online\n')
    add("csv_quoted_newline", "csv", '1.0,12,3,online\n"2.0\n",13,4,online\n3,x,1,online\n')
    add("csv_three_fields", "csv", "1.0,12,online\n")
    add("csv_five_fields", "csv", "1.0,12,3,online,extra\n")
    add("csv_zero_input", "csv", "1.0,0,3,online\n")
    add("csv_negative_output", "csv", "1.0,10,-3,online\n")
    add("csv_float_input", "csv", "1.0,10.0,3,online\n")
    add("csv_bad_output", "csv", "1.0,10,x,online\n")
    add("csv_bad_arrival_quote", "csv", "it's,10,3,online\n")
    add("csv_double_underscore", "csv", "1.0,1__0,3,online\n")
    add("csv_no_trailing_newline", "csv", "1.0,10,3,online\n2.0,11,4,offline")
    add("csv_class_empty", "csv", "1.0,10,3,\n")
    add("csv_tab_in_field", "csv", "1.0,\t10\t,3,online\n2.0,1\t0,3,online\n")
    # JSON lines edge cases
    j = json.dumps
    add("jsonl_missing_output", "jsonl", j({"arrival_s": 1, "input_tokens": 5, "class": "online"}) + "\n")
    add("jsonl_null_output", "jsonl", '{"arrival_s": 1, "input_tokens": 5, "output_tokens": null, "class": "online"}\n')
    add("jsonl_blank_lines", "jsonl", "\n  \n" + j({"arrival_s": 2.5, "input_tokens": 5, "class": "offline"}) + "\n\n")
    add("jsonl_bool_arrival", "jsonl", '{"arrival_s": true, "input_tokens": 5, "class": "online"}\n')
    add("jsonl_float_input", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5.0, "class": "online"}\n')
    add("jsonl_string_input", "jsonl", '{"arrival_s": 1.0, "input_tokens": "5", "class": "online"}\n')
    add("jsonl_bool_output", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "output_tokens": false, "class": "online"}\n')
    add("jsonl_class_number", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "class": 1}\n')
    add("jsonl_class_bad", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "class": "Batch"}\n')
    add("jsonl_missing_class", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5}\n')
    add("jsonl_missing_arrival", "jsonl", '{"input_tokens": 5, "class": "online"}\n')
    add("jsonl_not_object", "jsonl", '[1, 2]\n')
    add("jsonl_extra_data", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "class": "online"} x\n')
    add("jsonl_trailing_comma", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5,}\n')
    add("jsonl_missing_colon", "jsonl", '{"arrival_s" 1.0}\n')
    add("jsonl_missing_comma", "jsonl", '{"arrival_s": 1.0 "input_tokens": 5}\n')
    add("jsonl_unterminated", "jsonl", '{"arrival_s": 1.0, "class": "onl\n')
    add("jsonl_bad_value", "jsonl", '{"arrival_s": tru}\n')
    add("jsonl_leading_zero", "jsonl", '{"arrival_s": 01}\n')
    add("jsonl_nan_inf", "jsonl", '{"arrival_s": NaN, "input_tokens": 5, "class": "online"}\n'
                                  '{"arrival_s": Infinity, "input_tokens": 5, "class": "online"}\n')
    add("jsonl_exp_int_arrival", "jsonl", '{"arrival_s": 2e1, "input_tokens": 5, "class": "online"}\n'
                                          '{"arrival_s": 7, "input_tokens": 6, "class": "offline"}\n')
    add("jsonl_duplicate_key", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "input_tokens": 9, "class": "online"}\n')
    add("jsonl_nested_unknown", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "class": "online", "meta": {"a": [1, {"b": null}]}}\n')
    add("jsonl_unknown_sorted", "jsonl", '{"zz": 1, "arrival_s": 1.0, "input_tokens": 5, "class": "online", "aa": 2}\n')
    add("jsonl_escapes", "jsonl", '{"arrival_s": 1.0, "input_tokens": 5, "class": "on\\u006cine"}\n')
    add("jsonl_zero_input", "jsonl", '{"arrival_s": 1.0, "input_tokens": 0, "class": "online"}\n')
    add("jsonl_negative_output", "jsonl", '{"arrival_s": 1.0, "input_tokens": 3, "output_tokens": -2, "class": "online"}\n')
    add("jsonl_empty_object", "jsonl", '{}\n')
    add("jsonl_error_line3", "jsonl", j({"arrival_s": 1, "input_tokens": 5, "class": "online"}) + "\n\n" + '{"arrival_s": }\n')
    return out


def main():
    if not os.path.isdir(os.path.join(REF_SRC, "bucketsim")):
        raise SystemExit("reference not available")
    sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    from bucketsim import workload as wl
    from bucketsim.errors import TraceFormatError
    fixtures = []
    for name, fmt, text in cases(wl):
        tf = wl.TraceFormat.CSV if fmt == "csv" else wl.TraceFormat.JSONL
        rec = {"name": name, "fmt": fmt, "text": text}
        try:
            tr = wl.load_trace(io.StringIO(text, newline=""), tf)
            rec["ok"] = True
            rec["id"] = [r.id for r in tr]
            rec["arrival"] = [repr(r.arrival_time) for r in tr]
            rec["input"] = [r.input_len for r in tr]
            rec["output"] = [-1 if r.output_len is None else r.output_len for r in tr]
            rec["cls"] = [0 if r.task_class is wl.TaskClass.ONLINE else 1 for r in tr]
        except TraceFormatError as e:
            rec["ok"] = False
            rec["err_line"] = e.line
            rec["err_msg"] = str(e)
        fixtures.append(rec)
        print(f"{name:28s} {fmt:5s} {'ok ' + str(len(rec.get('id', []))) if rec['ok'] else rec['err_msg']}")
    with gzip.open(OUT, "wt") as fh:
        json.dump(fixtures, fh)


if __name__ == "__main__":
    main()
