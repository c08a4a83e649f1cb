// Host-side macro-instance scheduler of include/ecoserve.h (SURVEY 8(a) rows
// a1-a4) and its virtual-clock discrete-event mode.
//
//  * Alg. 1 InterSchedule: probe instances cyclically from
//    the previously routed one, at most one cycle (prose P:556-559, reading A9);
//    the printed variant (route to next without re-checking) behind a flag.
//  * Alg. 2 CheckConstraints, integer nanoseconds:
//      C1 TTFT: sum of predicted prefill ns of Pending (arrived at/after
//         t_switch or still without first token, A11) plus the new request
//         must not exceed SLO_TTFT;
//      C2 TPOT: over Existed (arrived before t_switch, first token out,
//         unfinished) sum(n_gen*SLO_TPOT - (now - t_first)) >= |Existed|*t_total
//         (the exact integer form of "mean saved TPOT >= t_total", A10);
//      C3 KV: ceil((S+R)/64) <= total - sum(max(ceil((S_r+R)/64), ceil((S_r+n_r)/64))) (A14).
//  * Intra-instance policy (temporal disaggregation P:423-434) in the
//    DES: prefill windows drain the routed queue FIFO in <= token_budget
//    batches; decode steps are non-preemptive (A15); new decodes join at
//    window end (A16); completions before arrivals at equal time.
//    KV pressure (A14, only when R is below true outputs): a decode step preempts
//    the latest-arrived batch members until every member can hold
//    ceil((S + n_gen)/64) blocks after the step; they go to the front of the queue
//    and are recomputed by a prefill of prompt + generated tokens; a
//    prefill batch is the FIFO prefix that fits the budget and the free blocks.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <deque>
#include <map>
#include <queue>
#include <tuple>
#include <vector>

#include "../../include/ecoserve.h"

namespace {

enum { OK_ = 0, F_TTFT = 1, F_TPOT = 2, F_KV = 3 };

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// floor division toward -infinity
int64_t fdiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

struct SReq {
  int64_t arrival;
  int32_t S;
  int64_t t_first;
  int32_t n_gen;
};

struct SInst {
  int32_t phase = 0;
  int64_t t_switch = 0;
  int64_t total_blocks = 0;
  bool alive = true;
  std::map<int64_t, SReq> reqs;  // req_id -> view (ordered: deterministic iteration)
};

}  // namespace

struct ecoserve_macro {
  int32_t n = 0;
  int64_t slo_ttft = 0, slo_tpot = 0;
  int32_t R = 0, block = 64;
  bool printed = false;
  int64_t ca = 0, cb = 0, cc = 0;
  std::vector<int64_t> tlen, tns;
  std::vector<SInst> inst;
  int32_t prev = 0;
  std::deque<ecoserve_route_req> deferred;

  int64_t pred(int64_t S) const {
    if (tlen.empty()) return ca + (cb * S + cc * S * S) / 1000;
    if (tlen.size() == 1) return tns[0];
    size_t i = 0;
    while (i + 2 < tlen.size() && S > tlen[i + 1]) ++i;
    return tns[i] + fdiv((tns[i + 1] - tns[i]) * (S - tlen[i]), tlen[i + 1] - tlen[i]);
  }

  int32_t check(int32_t i, int32_t S, int64_t now) const {
    const SInst& st = inst[i];
    if (!st.alive) return F_KV;
    int64_t t_total = pred(S);
    for (auto& kv : st.reqs) {
      const SReq& r = kv.second;
      if (r.arrival >= st.t_switch || r.t_first < 0) t_total += pred(r.S);
    }
    if (t_total > slo_ttft) return F_TTFT;
    int64_t n_ex = 0, saved = 0;
    for (auto& kv : st.reqs) {
      const SReq& r = kv.second;
      if (r.arrival < st.t_switch && r.t_first >= 0) {
        ++n_ex;
        saved += (int64_t)r.n_gen * slo_tpot - (now - r.t_first);
      }
    }
    if (n_ex > 0 && saved < n_ex * t_total) return F_TPOT;
    int64_t committed = 0;
    for (auto& kv : st.reqs) {
      const SReq& r = kv.second;
      committed += std::max(cdiv(r.S + R, block), cdiv((int64_t)r.S + r.n_gen, block));
    }
    if (cdiv((int64_t)S + R, block) > st.total_blocks - committed) return F_KV;
    return OK_;
  }

  int32_t route(const ecoserve_route_req& q, int64_t now, int32_t* outcomes, int32_t* n_probed) {
    int32_t chosen = -1, k = 0;
    if (printed) {
      const int32_t res = check(prev, q.prompt_len, now);
      if (outcomes) outcomes[0] = res;
      k = 1;
      chosen = res == OK_ ? prev : (prev + 1) % n;
    } else {
      for (; k < n; ++k) {
        const int32_t i = (prev + k) % n;
        const int32_t res = check(i, q.prompt_len, now);
        if (outcomes) outcomes[k] = res;
        if (res == OK_) {
          chosen = i;
          ++k;
          break;
        }
      }
    }
    if (n_probed) *n_probed = k;
    if (chosen >= 0) {
      prev = chosen;
      inst[chosen].reqs[q.req_id] = SReq{q.arrival_ns, q.prompt_len, -1, 0};
    }
    return chosen;
  }
};

extern "C" {

ecoserve_status ecoserve_macro_create(const ecoserve_macro_config* c, ecoserve_macro** out) {
  if (!c || !out || c->n_instances < 1 || c->slo_ttft_ns < 0 || c->slo_tpot_ns < 0 || c->reserve_tokens < 0 ||
      c->block_tokens < 1 || !c->total_blocks || c->n_table < 0 || (c->n_table > 0 && (!c->table_len || !c->table_ns)))
    return ECOSERVE_ERR_INVALID_ARG;
  for (int i = 1; i < c->n_table; ++i)
    if (c->table_len[i] <= c->table_len[i - 1]) return ECOSERVE_ERR_INVALID_ARG;
  ecoserve_macro* m = new ecoserve_macro();
  m->n = c->n_instances;
  m->slo_ttft = c->slo_ttft_ns;
  m->slo_tpot = c->slo_tpot_ns;
  m->R = c->reserve_tokens;
  m->block = c->block_tokens;
  m->printed = c->probe_printed != 0;
  m->ca = c->cost_a_ns;
  m->cb = c->cost_b_ps;
  m->cc = c->cost_c_ps;
  m->tlen.assign(c->table_len, c->table_len + c->n_table);
  m->tns.assign(c->table_ns, c->table_ns + c->n_table);
  m->inst.resize(m->n);
  for (int i = 0; i < m->n; ++i) m->inst[i].total_blocks = c->total_blocks[i];
  *out = m;
  return ECOSERVE_OK;
}

void ecoserve_macro_destroy(ecoserve_macro* m) { delete m; }

int32_t ecoserve_macro_prev_idx(const ecoserve_macro* m) { return m ? m->prev : -1; }

int64_t ecoserve_macro_predict_prefill_ns(const ecoserve_macro* m, int32_t S) { return m ? m->pred(S) : -1; }

ecoserve_status ecoserve_macro_route(ecoserve_macro* m, const ecoserve_route_req* req, int64_t now_ns, int32_t* inst,
                                     int32_t* outcomes, int32_t* n_probed) {
  if (!m || !req || !inst || req->prompt_len < 1) return ECOSERVE_ERR_INVALID_ARG;
  *inst = m->route(*req, now_ns, outcomes, n_probed);
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_macro_check(const ecoserve_macro* m, int32_t i, const ecoserve_route_req* req, int64_t now_ns,
                                     int32_t* result) {
  if (!m || !req || !result || i < 0 || i >= m->n) return ECOSERVE_ERR_INVALID_ARG;
  *result = m->check(i, req->prompt_len, now_ns);
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_macro_defer(ecoserve_macro* m, const ecoserve_route_req* req) {
  if (!m || !req) return ECOSERVE_ERR_INVALID_ARG;
  m->deferred.push_back(*req);
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_macro_update_status(ecoserve_macro* m, int32_t i, const ecoserve_sched_status* st,
                                             const ecoserve_sched_req* reqs, int32_t n) {
  if (!m || !st || i < 0 || i >= m->n || n < 0 || (n > 0 && !reqs)) return ECOSERVE_ERR_INVALID_ARG;
  SInst& s = m->inst[i];
  s.phase = st->phase;
  s.t_switch = st->t_switch_ns;
  s.total_blocks = st->total_blocks;
  s.alive = st->alive != 0;
  for (int k = 0; k < n; ++k) {
    const ecoserve_sched_req& r = reqs[k];
    if (r.finished)
      s.reqs.erase(r.req_id);
    else
      s.reqs[r.req_id] = SReq{r.arrival_ns, r.prompt_len, r.t_first_ns, r.n_generated};
  }
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_macro_drain_deferred(ecoserve_macro* m, int64_t now_ns, ecoserve_routed* out, int32_t cap,
                                              int32_t* n) {
  if (!m || !n || cap < 0 || (cap > 0 && !out)) return ECOSERVE_ERR_INVALID_ARG;
  int32_t k = 0;
  while (!m->deferred.empty() && k < cap) {
    const ecoserve_route_req q = m->deferred.front();
    const int32_t i = m->route(q, now_ns, nullptr, nullptr);
    if (i < 0) break;
    m->deferred.pop_front();
    out[k].req_id = q.req_id;
    out[k].instance = i;
    ++k;
  }
  *n = k;
  return ECOSERVE_OK;
}

// ------------------------------------------------------------------ mitosis (N1)
// PAPER.md Sec. 3.5.1 (Fig. 7). Expansion: add to the first macro below N_u
// (creation order); if all are full the last one takes N_u + 1 and splits off a new
// macro of N_l. Contraction: shrink the smallest macro (last on ties) down to N_l;
// then shrink its partner (the other partial macro, else the last full one) until
// the pair totals N_u; the next removal merges the pair into one macro of N_u - 1.
ecoserve_status ecoserve_mitosis_step(int32_t* sizes, int32_t* n_macros, int32_t cap, int32_t n_l, int32_t n_u,
                                      int32_t expand, int32_t* action) {
  if (!sizes || !n_macros || !action || n_l < 1 || n_u < n_l || *n_macros < 0 || *n_macros > cap)
    return ECOSERVE_ERR_INVALID_ARG;
  int n = *n_macros;
  action[0] = action[1] = action[2] = -1;
  if (expand) {
    if (n == 0) {
      if (cap < 1) return ECOSERVE_ERR_INVALID_ARG;
      sizes[0] = 1;
      *n_macros = 1;
      action[0] = ECOSERVE_MITOSIS_CREATE;
      action[1] = 0;
      return ECOSERVE_OK;
    }
    for (int i = 0; i < n; ++i)
      if (sizes[i] < n_u) {
        ++sizes[i];
        action[0] = ECOSERVE_MITOSIS_ADD;
        action[1] = i;
        return ECOSERVE_OK;
      }
    if (n + 1 > cap) return ECOSERVE_ERR_INVALID_ARG;
    sizes[n - 1] = n_u + 1 - n_l;
    sizes[n] = n_l;
    *n_macros = n + 1;
    action[0] = ECOSERVE_MITOSIS_ADD_SPLIT;
    action[1] = n - 1;
    action[2] = n;
    return ECOSERVE_OK;
  }
  if (n == 0) return ECOSERVE_ERR_STATE;
  if (n == 1) {
    if (sizes[0] == 1) {
      *n_macros = 0;
      action[0] = ECOSERVE_MITOSIS_REMOVE_MACRO;
      action[1] = 0;
    } else {
      --sizes[0];
      action[0] = ECOSERVE_MITOSIS_REMOVE;
      action[1] = 0;
    }
    return ECOSERVE_OK;
  }
  int small = 0;
  for (int i = 1; i < n; ++i)
    if (sizes[i] <= sizes[small]) small = i;  // smallest, last on ties
  if (sizes[small] > n_l) {
    --sizes[small];
    action[0] = ECOSERVE_MITOSIS_REMOVE;
    action[1] = small;
    return ECOSERVE_OK;
  }
  int p = -1;
  for (int i = 0; i < n; ++i)
    if (i != small && sizes[i] < n_u) p = i;  // last partial macro
  if (p < 0)
    for (int i = 0; i < n; ++i)
      if (i != small) p = i;  // last full macro
  const int total = sizes[small] + sizes[p];
  if (total > n_u) {
    --sizes[p];
    action[0] = ECOSERVE_MITOSIS_REMOVE;
    action[1] = p;
    return ECOSERVE_OK;
  }
  const int keep = small < p ? small : p, gone = small < p ? p : small;
  sizes[keep] = total - 1;
  for (int i = gone; i + 1 < n; ++i) sizes[i] = sizes[i + 1];
  *n_macros = n - 1;
  action[0] = ECOSERVE_MITOSIS_REMOVE_MERGE;
  action[1] = p;
  action[2] = small;
  return ECOSERVE_OK;
}

// InstanceHandler: the serializable proxy moved between macro schedulers.
// Wire format v1, little-endian: u8 version | i64 actor_id | i32 device | i32 tp_size |
// i32 tp_rank | i64 kv_blocks | u16 address length | address bytes.
int32_t ecoserve_handler_serialize(const ecoserve_instance_handler* h, uint8_t* out, int32_t cap) {
  if (!h) return -1;
  int32_t alen = 0;
  while (alen < (int32_t)sizeof(h->address) && h->address[alen]) ++alen;
  const int32_t need = 1 + 8 + 4 + 4 + 4 + 8 + 2 + alen;
  if (!out || cap < need) return need <= cap ? -1 : -need;
  uint8_t* p = out;
  auto put = [&](const void* src, int nb) {
    memcpy(p, src, nb);  // the supported hosts are little-endian (x86-64, aarch64)
    p += nb;
  };
  const uint8_t ver = 1;
  const uint16_t al = (uint16_t)alen;
  put(&ver, 1);
  put(&h->actor_id, 8);
  put(&h->device, 4);
  put(&h->tp_size, 4);
  put(&h->tp_rank, 4);
  put(&h->kv_blocks, 8);
  put(&al, 2);
  put(h->address, alen);
  return need;
}

ecoserve_status ecoserve_handler_deserialize(const uint8_t* in, int32_t n, ecoserve_instance_handler* h) {
  if (!in || !h || n < 31) return ECOSERVE_ERR_INVALID_ARG;
  if (in[0] != 1) return ECOSERVE_ERR_UNSUPPORTED;  // unknown version
  const uint8_t* p = in + 1;
  memset(h, 0, sizeof(*h));
  memcpy(&h->actor_id, p, 8);
  memcpy(&h->device, p + 8, 4);
  memcpy(&h->tp_size, p + 12, 4);
  memcpy(&h->tp_rank, p + 16, 4);
  memcpy(&h->kv_blocks, p + 20, 8);
  uint16_t al;
  memcpy(&al, p + 28, 2);
  if (n != 31 + al || al >= sizeof(h->address)) return ECOSERVE_ERR_INVALID_ARG;
  memcpy(h->address, p + 30, al);
  return ECOSERVE_OK;
}

// ------------------------------------------------------------------ DES
ecoserve_status ecoserve_des_run(const ecoserve_macro_config* mcfg, const ecoserve_des_config* dcfg,
                                 const int64_t* arrival_ns, const int32_t* prompt_len, const int32_t* output_len,
                                 int32_t n_req, int32_t* out_inst, int64_t* out_first, int64_t* out_dbeg,
                                 int64_t* out_done, int64_t* route_log, int32_t route_log_cap, int32_t* n_route_log,
                                 int32_t* out_n_preempt) {
  if (!mcfg || !dcfg || n_req < 0 || (n_req > 0 && (!arrival_ns || !prompt_len || !output_len || !out_inst ||
                                                     !out_first || !out_dbeg || !out_done)))
    return ECOSERVE_ERR_INVALID_ARG;
  ecoserve_macro* m = nullptr;
  ecoserve_status s = ecoserve_macro_create(mcfg, &m);
  if (s != ECOSERVE_OK) return s;
  const int N = m->n;
  struct R {
    int64_t arr;
    int32_t S, G, inst = -1, n_gen = 0, n_pre = 0;
    int64_t first = -1, dbeg = -1, done = -1;
  };
  std::vector<R> rq(n_req);
  for (int i = 0; i < n_req; ++i) {
    rq[i].arr = arrival_ns[i];
    rq[i].S = prompt_len[i];
    rq[i].G = output_len[i];
  }
  struct I {
    int32_t phase = 0;
    int64_t t_switch = 0;
    bool busy = false;
    bool op_prefill = false;
    std::vector<int> op;
    std::deque<int> queue;
    std::vector<int> waiting, running, fin;
  };
  std::vector<I> in(N);
  int32_t nlog = 0;
  auto log = [&](int64_t t, int rid, int i) {
    if (route_log && nlog < route_log_cap) {
      route_log[3 * nlog] = t;
      route_log[3 * nlog + 1] = rid;
      route_log[3 * nlog + 2] = i;
    }
    ++nlog;
  };
  // exact status push of every instance (A17)
  auto push = [&]() {
    for (int i = 0; i < N; ++i) {
      I& x = in[i];
      SInst& v = m->inst[i];
      v.phase = x.phase;
      v.t_switch = x.t_switch;
      auto put = [&](int k) { v.reqs[k] = SReq{rq[k].arr, rq[k].S, rq[k].first, rq[k].n_gen}; };
      for (int k : x.queue) put(k);
      for (int k : x.waiting) put(k);
      for (int k : x.running) put(k);
      for (int k : x.op) put(k);
      for (int k : x.fin) v.reqs.erase(k);
      x.fin.clear();
    }
  };
  // events: (time, kind 0 completion / 1 arrival, index)
  typedef std::tuple<int64_t, int, int> Ev;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> ev;
  for (int k = 0; k < n_req; ++k) ev.push(Ev(rq[k].arr, 1, k));
  const int64_t BT = m->block;
  // tokens a prefill of k processes: the prompt, plus the generated tokens of a recompute (A14)
  auto plen = [&](int k) -> int64_t { return (int64_t)rq[k].S + rq[k].n_gen; };
  bool pool_error = false;
  auto start = [&](int i, int64_t t) {
    I& x = in[i];
    if (x.busy) return;
    const int64_t total = m->inst[i].total_blocks;
    int64_t held = 0;  // prompt + fed tokens of the prefilled requests
    for (int k : x.waiting) held += cdiv((int64_t)rq[k].S + rq[k].n_gen - 1, BT);
    for (int k : x.running) held += cdiv((int64_t)rq[k].S + rq[k].n_gen - 1, BT);
    int64_t free_b = total - held;
    if (!x.queue.empty() && cdiv(plen(x.queue.front()), BT) <= free_b) {
      if (x.phase != 1) { x.phase = 1; x.t_switch = t; }
      x.op.clear();
      int64_t tok = 0, dur = 0;
      while (!x.queue.empty()) {
        const int k = x.queue.front();
        if (!x.op.empty() && tok + plen(k) > dcfg->token_budget) break;
        if (cdiv(plen(k), BT) > free_b) break;
        x.queue.pop_front();
        x.op.push_back(k);
        tok += plen(k);
        free_b -= cdiv(plen(k), BT);
        dur += m->pred(plen(k));
      }
      x.busy = true;
      x.op_prefill = true;
      ev.push(Ev(t + dur, 0, i));
    } else if (!x.waiting.empty() || !x.running.empty()) {
      if (x.phase != 2) {
        x.phase = 2;
        x.t_switch = t;
        for (int k : x.waiting)
          if (rq[k].dbeg < 0) rq[k].dbeg = t;
        x.running.insert(x.running.end(), x.waiting.begin(), x.waiting.end());
        x.waiting.clear();
      }
      x.op = x.running;
      x.running.clear();
      for (;;) {  // A14: preempt latest arrivals until the grown batch fits the pool
        int64_t after = 0;
        for (int k : x.op) after += cdiv((int64_t)rq[k].S + rq[k].n_gen, BT);
        if (x.op.empty() || after <= total) break;
        size_t v = 0;
        for (size_t j = 1; j < x.op.size(); ++j)
          if (std::make_pair(rq[x.op[j]].arr, x.op[j]) > std::make_pair(rq[x.op[v]].arr, x.op[v])) v = j;
        const int k = x.op[v];
        x.op.erase(x.op.begin() + v);
        x.queue.push_front(k);
        ++rq[k].n_pre;
      }
      if (x.op.empty()) {
        pool_error = true;  // one request outgrew the whole pool
        return;
      }
      int64_t sum_ctx = 0;
      for (int k : x.op) sum_ctx += rq[k].S + rq[k].n_gen;
      const int64_t dur = dcfg->cost_d_ns + dcfg->cost_e_ns * (int64_t)x.op.size() + (dcfg->cost_f_ps * sum_ctx) / 1000;
      x.busy = true;
      x.op_prefill = false;
      ev.push(Ev(t + dur, 0, i));
    } else if (!x.queue.empty()) {
      pool_error = true;  // the queue head needs more blocks than the empty pool holds
    }
  };
  while (!ev.empty()) {
    const Ev e = ev.top();
    ev.pop();
    const int64_t t = std::get<0>(e);
    const int idx = std::get<2>(e);
    if (std::get<1>(e) == 0) {
      I& x = in[idx];
      for (int k : x.op) {
        if (x.op_prefill && rq[k].n_gen == 0) {
          rq[k].first = t;
          rq[k].n_gen = 1;
        } else {  // decode step, or a recompute prefill (A14): the next token
          rq[k].n_gen += 1;
        }
        if (rq[k].n_gen >= rq[k].G) {
          rq[k].done = t;
          if (x.op_prefill && rq[k].dbeg < 0) rq[k].dbeg = t;
          x.fin.push_back(k);
        } else if (x.op_prefill) {
          x.waiting.push_back(k);
        } else {
          x.running.push_back(k);
        }
      }
      x.op.clear();
      x.busy = false;
      push();
      while (!m->deferred.empty()) {
        const ecoserve_route_req q = m->deferred.front();
        const int32_t i = m->route(q, t, nullptr, nullptr);
        if (i < 0) break;
        m->deferred.pop_front();
        rq[q.req_id].inst = i;
        in[i].queue.push_back((int)q.req_id);
        log(t, (int)q.req_id, i);
      }
    } else {
      push();
      ecoserve_route_req q{idx, rq[idx].arr, rq[idx].S};
      const int32_t i = m->route(q, t, nullptr, nullptr);
      log(t, idx, i);
      if (i < 0) {
        m->deferred.push_back(q);
      } else {
        rq[idx].inst = i;
        in[i].queue.push_back(idx);
      }
    }
    for (int i = 0; i < N; ++i) start(i, t);
    if (pool_error) break;
  }
  for (int k = 0; k < n_req; ++k) {
    out_inst[k] = rq[k].inst;
    out_first[k] = rq[k].first;
    out_dbeg[k] = rq[k].dbeg;
    out_done[k] = rq[k].done;
    if (out_n_preempt) out_n_preempt[k] = rq[k].n_pre;
  }
  if (n_route_log) *n_route_log = nlog;
  ecoserve_macro_destroy(m);
  return pool_error ? ECOSERVE_ERR_KV_EXHAUSTED : ECOSERVE_OK;
}

}  // extern "C"
